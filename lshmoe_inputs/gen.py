"""Synthetic LSH-MoE layer inputs (DESIGN.md §4 "Input recipe").

Token similarity (§3.1) is modelled as a Zipf-weighted ("Zipf's Law") mixture
of C shared unit directions U_c:  x = sqrt(d) * U_c + rho * z,  z ~ N(0, I), rounded (RNE) to the
token dtype, so entries are O(1) like LayerNorm outputs.  Gate (the input zeta of Alg. 1 L2,
P:L519): linear scorer W_g ~ N(0, 1/d), top-k by fp64 score, ties to the smaller expert id, slot
order ascending expert id.  Experts: W1 ~ N(0, 1/d), W2 ~ N(0, 1/d_ffn), biases
N(0, 0.02^2), stored in the token dtype.  Seeds: numpy PCG64 streams from
SeedSequence([master_seed, label]) with SPEC's labels: centres=1, gate=2, experts=3
(+ expert id), lsh=4 (the rotation seed), tokens of rank i = 100+i.

Nothing here implements a step of the method; it draws inputs only.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, Optional

import numpy as np
import torch

__all__ = ["LayerConfig", "CONFIGS", "make_centers", "make_tokens", "make_gate", "make_experts",
           "rotation_seed", "make_rank_inputs", "torch_dtype", "make_codes", "make_zipf_gate", "gate_matrix"]


@dataclass(frozen=True)
class LayerConfig:
    name: str
    n: int            # tokens per rank
    d: int            # d_model
    E: int            # experts
    k: int            # top-k
    q: int            # hash functions
    dtype: str        # 'f32' | 'bf16'
    d_ffn: int
    C: int            # mixture components
    rho: float        # relative noise
    note: str = ""

    def with_(self, **kw) -> "LayerConfig":
        d = dict(self.__dict__)
        d.update(kw)
        return LayerConfig(**d)


# BASELINE.json configs[0..4]; d_ffn from Table 1; q = 6 is the paper default
# (P:L346); tokens/GPU from BASELINE.json (C5's 25,088 = 128 images x 14x14 window tokens is our
# choice); C / rho calibrated so q=6 gives r ~ 0.2 / ~0.117.
CONFIGS: Dict[str, LayerConfig] = {
    "C1": LayerConfig("C1", 256, 64, 4, 1, 2, "f32", 256, 16, 0.3,
                      "single MoE layer, 256 tokens, d=64, 4 experts top-1, 2 CP hashes, fp32"),
    "C2": LayerConfig("C2", 16384, 768, 16, 1, 6, "bf16", 3072, 512, 0.07,
                      "RoBERTa-MoE-shaped: d=768, 16 experts top-1, 16K tokens/GPU, bf16"),
    "C3": LayerConfig("C3", 32768, 1024, 32, 2, 6, "bf16", 4096, 512, 0.085,
                      "GPT-MoE-shaped: d=1024, 32 experts top-2, 32K tokens/GPU, bf16"),
    "C4": LayerConfig("C4", 65536, 1024, 64, 1, 6, "bf16", 16384, 1024, 0.09,
                      "T5-MoE-shaped encoder: d=1024, 64 experts top-1, 64K tokens/GPU, bf16"),
    "C5": LayerConfig("C5", 25088, 768, 32, 1, 6, "bf16", 3072, 512, 0.053,
                      "Swin-MoE-shaped: d=768 window tokens, 32 experts top-1, high similarity"),
}


def torch_dtype(dtype: str):
    return {"f32": torch.float32, "bf16": torch.bfloat16}[dtype]


def _rng(master_seed: int, *labels: int) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence([int(master_seed), *[int(x) for x in labels]]))


def rotation_seed(master_seed: int) -> int:
    """The u64 rotation seed of label 4 (lsh)."""
    return int(_rng(master_seed, 4).integers(0, 2 ** 63 - 1, dtype=np.int64)) * 2 + 1


def make_centers(cfg: LayerConfig, master_seed: int) -> np.ndarray:
    U = _rng(master_seed, 1).standard_normal((cfg.C, cfg.d))
    return U / np.linalg.norm(U, axis=1, keepdims=True)


def make_tokens(cfg: LayerConfig, master_seed: int, rank: int = 0, n: Optional[int] = None,
                rho: Optional[float] = None, iid: bool = False) -> torch.Tensor:
    """Tokens of one rank as a CPU tensor in the config dtype."""
    n = cfg.n if n is None else n
    rho = cfg.rho if rho is None else rho
    rng = _rng(master_seed, 100 + rank)
    if iid:
        X = rng.standard_normal((n, cfg.d))
    else:
        U = make_centers(cfg, master_seed)
        w = 1.0 / np.arange(1, cfg.C + 1, dtype=np.float64)
        comp = rng.choice(cfg.C, size=n, p=w / w.sum())
        X = np.sqrt(cfg.d) * U[comp]
        if rho > 0:
            X = X + rho * rng.standard_normal((n, cfg.d))
    return torch.from_numpy(X).to(torch.float32).to(torch_dtype(cfg.dtype)).contiguous()


def gate_matrix(cfg: LayerConfig, master_seed: int) -> np.ndarray:
    """The linear gate scorer W_g [E, d] ~ N(0, 1/d) (fp64) that make_gate draws."""
    return _rng(master_seed, 2).standard_normal((cfg.E, cfg.d)) / np.sqrt(cfg.d)


def make_gate(cfg: LayerConfig, master_seed: int, X: torch.Tensor, with_weights: bool = False):
    """zeta int32 [n, k] (ascending expert ids per row) and optional softmax weights fp32."""
    Wg = gate_matrix(cfg, master_seed)
    S = X.to(torch.float64).numpy() @ Wg.T
    order = np.argsort(-S, axis=1, kind="stable")          # ties keep the smaller expert id first
    top = np.sort(order[:, :cfg.k], axis=1).astype(np.int32)
    if not with_weights:
        return torch.from_numpy(top), None
    sel = np.take_along_axis(S, top, axis=1)
    ex = np.exp(sel - sel.max(axis=1, keepdims=True))
    g = (ex / ex.sum(axis=1, keepdims=True)).astype(np.float32)
    return torch.from_numpy(top), torch.from_numpy(g)


def make_experts(cfg: LayerConfig, master_seed: int, experts=None):
    """Dict e -> (W1 [d_ffn, d], b1 [d_ffn], W2 [d, d_ffn], b2 [d]) CPU tensors in the dtype."""
    ids = range(cfg.E) if experts is None else experts
    out = {}
    dt = torch_dtype(cfg.dtype)
    for e in ids:
        r = _rng(master_seed, 3, e)
        W1 = r.standard_normal((cfg.d_ffn, cfg.d)) / np.sqrt(cfg.d)
        b1 = 0.02 * r.standard_normal(cfg.d_ffn)
        W2 = r.standard_normal((cfg.d, cfg.d_ffn)) / np.sqrt(cfg.d_ffn)
        b2 = 0.02 * r.standard_normal(cfg.d)
        out[e] = tuple(torch.from_numpy(a).to(torch.float32).to(dt).contiguous() for a in (W1, b1, W2, b2))
    return out


def make_rank_inputs(cfg: LayerConfig, master_seed: int, rank: int = 0, with_weights: bool = False):
    X = make_tokens(cfg, master_seed, rank)
    zeta, g = make_gate(cfg, master_seed, X, with_weights)
    return X, zeta, g


def make_codes(n: int, q: int, d: int, master_seed: int, C: int = 512, p_noise: float = 0.1,
               iid: bool = False) -> np.ndarray:
    """Synthetic hash codes int16 [n, q] with the bucket structure of the paper's workloads, for
    stage-isolated tests of compress at sizes where hashing in the oracle would be slow: token t
    belongs to a Zipf(1.0) component; each (component, j) has a fixed code, replaced by a
    uniformly random one with probability p_noise (tokens near a cross-polytope cell border).
    iid=True draws every code uniformly.  Codes are in {+-1..+-d}; nothing here hashes."""
    rng = _rng(master_seed, 5)
    def rand_codes(shape):
        mag = rng.integers(1, d + 1, size=shape)
        return np.where(rng.random(shape) < 0.5, -mag, mag)
    if iid:
        return rand_codes((n, q)).astype(np.int16)
    w = 1.0 / np.arange(1, C + 1, dtype=np.float64)
    comp = rng.choice(C, size=n, p=w / w.sum())
    base = rand_codes((C, q))
    codes = base[comp]
    noise = rng.random((n, q)) < p_noise
    codes = np.where(noise, rand_codes((n, q)), codes)
    return codes.astype(np.int16)


def make_zipf_gate(n: int, k: int, E: int, master_seed: int, hot: float = 0.0) -> torch.Tensor:
    """zeta int32 [n, k]: k distinct experts per token (ascending), drawn Zipf(1.0)-skewed over
    experts; with hot > 0 that fraction of tokens always routes to expert E-1 (skew stress)."""
    rng = _rng(master_seed, 6)
    w = 1.0 / np.arange(1, E + 1, dtype=np.float64)
    p = w / w.sum()
    out = np.empty((n, k), np.int32)
    for t in range(n):
        out[t] = np.sort(rng.choice(E, size=k, replace=False, p=p))
    if hot > 0:
        idx = np.nonzero(rng.random(n) < hot)[0]
        for t in idx:
            if (out[t] == E - 1).any():
                continue
            out[t, 0] = E - 1
            out[t] = np.sort(out[t])
    return torch.from_numpy(out)
