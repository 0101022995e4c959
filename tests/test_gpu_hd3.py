"""GPU parity of NEXT-4, lshmoe_hash_hd3 (Eq. 3's cross-polytope hash under the structured rotation
H D3 H D2 H D1 of x zero-padded to 1024, reading R30), against the oracle's dense materialisation
of the same rotation + cp_hash (fp64).

Tier 1: codes bit-exact except (token, hash) pairs whose oracle top-two margin over the 1024
outputs is below 1e-5 (reported).  Then the codes drive lshmoe_compress exactly like CP codes."""
import functools

import numpy as np
import pytest
import torch

import oracle as O
from helpers import CONFIGS, NEAR_TIE, f64, small_cfg
from lshmoe_inputs import make_gate, make_tokens, rotation_seed

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    import paper_2411_08446_b200 as L
    return L


@functools.lru_cache(maxsize=None)
def _R(d, q, seed):
    return O.hd3_rotation(d, q, seed)


def _check(L, X, q, seed, label):
    signs = L.hd3_signs(q, seed).cuda()
    got = L.hash_hd3(X.cuda(), signs).cpu().numpy()
    want, margins = O.cp_hash(f64(X), _R(X.shape[1], q, seed))
    mism = got != want
    near = margins < NEAR_TIE
    bad = mism & ~near
    print(f"[hd3 {label}] n={X.shape[0]} d={X.shape[1]} q={q} mismatches={int(mism.sum())} "
          f"near-ties={int(near.sum())} outside band={int(bad.sum())}")
    assert not bad.any(), np.argwhere(bad)[:10]
    assert np.all(got != 0) and np.abs(got).max() <= O.HD3_DIM
    return got, want, near


@pytest.mark.parametrize("n,d,q,dtype", [(256, 64, 2, "f32"), (129, 100, 3, "f32"), (1000, 128, 3, "bf16"),
                                         (777, 1024, 16, "bf16"), (1, 8, 1, "bf16"), (4100, 768, 6, "bf16"),
                                         (3000, 1024, 6, "bf16")])
def test_hd3_hash_shapes(L, n, d, q, dtype):
    cfg = small_cfg(n=n, d=d, q=q, dtype=dtype)
    X = make_tokens(cfg, 3)
    _check(L, X, q, rotation_seed(3), f"{dtype} n={n} d={d}")


def test_hd3_hash_c2_full_size(L):
    cfg = CONFIGS["C2"]
    _check(L, make_tokens(cfg, 0), cfg.q, rotation_seed(0), "C2")


def test_hd3_zero_token_and_ties(L):
    """A zero token: every output is 0 -> the smallest index with '+' (code +1, reading R2); a token
    that is a multiple of a single padded output direction hashes to that coordinate."""
    X = torch.zeros((3, 64), dtype=torch.float32)
    X[1, 5] = 2.0
    X[2, 5] = -2.0
    got, want, _ = _check(L, X, 2, 11, "special")
    assert list(got[0]) == [1, 1]
    assert np.array_equal(got[1], -got[2])


def test_hd3_codes_drive_compress(L):
    """Structured-rotation codes key lshmoe_compress like CP codes: bucket ids bit-exact against the
    oracle's bucketize on the oracle's codes (near-tie tokens replaced by their predecessor)."""
    cfg = CONFIGS["C2"]
    X = make_tokens(cfg, 0)
    seed = rotation_seed(0)
    want, margins = O.cp_hash(f64(X), _R(cfg.d, cfg.q, seed))
    bad = np.nonzero(margins.min(axis=1) < NEAR_TIE)[0]
    for t in bad:
        X[t] = X[t - 1 if t > 0 else 1]
    want, margins = O.cp_hash(f64(X), _R(cfg.d, cfg.q, seed))
    assert margins.min() >= NEAR_TIE
    zeta, _ = make_gate(cfg, 0, X)
    codes = L.hash_hd3(X.cuda(), L.hd3_signs(cfg.q, seed).cuda())
    assert np.array_equal(codes.cpu().numpy(), want)
    out = L.compress(X.cuda(), codes, zeta.cuda(), cfg.E)
    b = O.bucketize(want, zeta.numpy(), cfg.E)
    assert int(out.num_rows.item()) == b.m
    assert np.array_equal(out.bucket.cpu().numpy(), b.bucket)
    print(f"[hd3 compress C2] m={b.m} ratio={b.m / cfg.n:.3f}")
