"""LSH-MoE oracle: a plain, slow, obviously-correct CPU implementation of the compressed
expert-parallel MoE layer of arXiv 2411.08446 ("LSH-MoE"), in fp64.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module.  It shares no code with the CUDA path
(``paper_2411_08446_b200``) and imports nothing from it.

Citation keys: ``P:Lnnn`` = /root/reference/PAPER.md line nnn (the paper; section / equation /
algorithm named beside each cite).  ``S:Lnnn`` = SPEC.md line nnn (used for interfaces and tie
rules only).  Readings of silent / ambiguous passages are numbered R1..R23 and listed in DESIGN.md
§3 ("Readings").

The functions follow Algorithm 1 (App. A "Framework of LSH-MoE") step by step:

  O1  rotation(d, q, seed)            random rotation R_j of Eq. 3            [pinned]
  O2  cp_hash(X, R)                   Eq. 3 cross-polytope hash           [pinned]
  O2" e4m3 quantisation + cp_hash     NEXT-2's fp8 rotation option: codes of the
                                      e4m3-rounded, power-of-two-scaled x and R_j (reading R28) [pinned]
  O0  gate_topk(X, Wg, k)             the gate of Eq. 1-2 as a linear scorer + top-k
                                      + softmax; NEXT-2 fuses it into the hash pass     [pinned]
  O2* hd3_rotation(d, q, seed)        NEXT-4 structured pseudo-random rotation of Eq. 3's R
                                      (P:L228): R_j = H D3 H D2 H D1 on x zero-padded to
                                      d' = 1024 (reading R30), materialised dense; cp_hash then
                                      takes its argmax over the d' outputs                [pinned]
  O2' sp_hash(X, N, q, b)             §4.5 spherical-plane hashing, SPEC's
                                      sign-bit construction (reading R26)   [pinned]
  O3  group_by_expert(zeta, E)        Alg. 1 L3 "Dispatch X into {X_i}"        [pinned]
  O4  bucketize(codes, zeta, E)       Alg. 1 L5-6 LSH buckets, §2.3 [pinned]
  O5  centroids(X, ...)               Alg. 1 L8 Mean; §2.3        [pinned]
  O6  round_to_dtype(c, dtype)        wire precision of C (reading R10/R23)             [pinned]
  O7  dispatch_sim / O9 combine_sim   Alg. 1 L14/L16 all-to-all        [pinned]
  O8  expert_ffn                      §2.1 "each FFN function works as an expert" [pinned]
  O10 restore                         Eq. 4-5 residual compensation, Alg. 1 L17-19
                                      (P:L536-538), composed with Eq. 2's k-sum [pinned]
  O11 stats                           compression rate (Table 3)
  O12 moe_dense                       Eq. 2 uncompressed MoE output          [pinned]
  B1  grad_compress(dY, b, k, g)      NEXT-1 backward: dL/dE(c~)_b = sum_{(t,s) in b} g dY_t [pinned]
  B3  expert_ffn_vjp(c, W1.., G)      expert backward J_E(c)^T G (the expert's own rule) [pinned]
  B5  grad_restore(...)               dL/dx_t and dL/dg_ts of Eq. 4-5 + Eq. 2 with the
                                      centroid mean, straight-through rounding (R27)    [pinned]

Every function above is pinned by a ``-m "not gpu"`` test in tests/test_oracle_*.py against
something other than itself (worked examples, closed forms, invariants, brute force, textbook
library routines).  The compression ratios the paper prints (11.7 %, ~20 %) come from real
activations and are NOT pinned (parity unpinned: calibration context only).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

__all__ = [
    "GAMMA", "splitmix64_stream", "irwin_hall_gaussian", "rotation_fp64", "rotation",
    "round_to_dtype", "f32_to_bf16_bits", "bf16_bits_to_f64", "to_stored",
    "cp_hash", "sp_hash", "sp_normals", "gate_topk", "HD3_DIM", "HD3_GAMMA", "hadamard", "hd3_signs", "hd3_rotation", "e4m3_values", "round_e4m3", "pow2_scale_e4m3",
    "quantize_tokens_e4m3", "quantize_rotation_e4m3", "group_by_expert", "bucketize", "Buckets", "centroids", "expert_ffn",
    "dispatch_sim", "combine_sim", "restore", "moe_dense", "lsh_layer", "lsh_layer_ranks",
    "LayerResult", "ulp_bf16", "grad_compress", "expert_ffn_vjp", "grad_restore", "lsh_layer_backward",
]

# ---------------------------------------------------------------------------------------------
# O1. Random rotation (Eq. 3: "R is a random rotation matrix").  The paper fixes no
# distribution or recipe (reading R3), so we fix one that two independent implementations can
# reproduce bit-for-bit: SplitMix64 counter stream -> Irwin-Hall(12) approximately-Gaussian
# matrix G -> modified Gram-Schmidt (SPEC S:L72 design decision) with every sum evaluated
# strictly left-to-right and no fused multiply-add -> R_j = Q^T -> RNE to the stored dtype.
# The C++ library (csrc/abi/rotation.cpp) implements the same recipe independently.
# ---------------------------------------------------------------------------------------------
GAMMA = 0x9E3779B97F4A7C15
_MASK64 = (1 << 64) - 1


def splitmix64_stream(state0: int, count: int, start: int = 0) -> np.ndarray:
    """Outputs number start+1 .. start+count of the SplitMix64 generator seeded with ``state0``.

    SplitMix64 is counter-based: output i (1-based) is mix(state0 + i*GAMMA mod 2^64), so it
    vectorises.  mix is the standard finaliser (Steele, Lea, Flood 2014)."""
    i = np.arange(start + 1, start + count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(state0 & _MASK64) + i * np.uint64(GAMMA)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def irwin_hall_gaussian(state0: int, count: int) -> np.ndarray:
    """count approximately-N(0,1) doubles: g = ((u0+u1)+...+u11) - 6, u = (z>>11)*2^-53.

    Only exact conversions and IEEE additions in a fixed order: bit-reproducible anywhere."""
    z = splitmix64_stream(state0, 12 * count).reshape(count, 12)
    u = (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    g = u[:, 0].copy()
    for i in range(1, 12):
        g = g + u[:, i]
    return g - 6.0


def _hash_state(rotation_seed: int, j: int) -> int:
    return (rotation_seed ^ ((GAMMA * (j + 1)) & _MASK64)) & _MASK64


def rotation_fp64(d: int, j: int, rotation_seed: int) -> np.ndarray:
    """fp64 rotation R_j (row-major, y = R_j x) of hash function j.  Reading R3.

    G[r, c] = irwin_hall_gaussian entry r*d + c.  Modified Gram-Schmidt over the columns of G,
    right-looking: q_i = a_i / ||a_i||; for every later column a_j: r = sum_k q_i[k]*a_j[k]
    (sequential in k), a_j[k] <- a_j[k] - q_i[k]*r.  R_j = Q^T.  np.cumsum (= add.accumulate) is
    strictly sequential, so every sum has the same left-to-right order as the C++ loop."""
    if d < 1:
        raise ValueError("d must be >= 1 (S:L51)")
    A = irwin_hall_gaussian(_hash_state(rotation_seed, j), d * d).reshape(d, d)
    Q = np.empty((d, d), dtype=np.float64)
    for i in range(d):
        v = A[:, i]
        ss = np.cumsum(v * v)[-1]
        nrm = math.sqrt(float(ss))
        qi = v / nrm
        Q[:, i] = qi
        if i + 1 < d:
            B = A[:, i + 1:]
            r = np.cumsum(qi[:, None] * B, axis=0)[-1]
            A[:, i + 1:] = B - qi[:, None] * r[None, :]
    return np.ascontiguousarray(Q.T)


def f32_to_bf16_bits(a32: np.ndarray) -> np.ndarray:
    """Round fp32 -> bf16, round-to-nearest-even, on the bit pattern (finite inputs)."""
    u = np.ascontiguousarray(a32, dtype=np.float32).view(np.uint32).astype(np.uint64)
    bias = np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))
    return ((u + bias) >> np.uint64(16)).astype(np.uint16)


def bf16_bits_to_f64(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)


def rotation(d: int, q: int, rotation_seed: int, dtype: str = "bf16") -> np.ndarray:
    """Stored rotations [q, d, d]: fp64 -> fp32 (RNE) -> bf16 (RNE) when dtype == 'bf16'.

    Returns float32 array for 'f32' and uint16 bf16 bit patterns for 'bf16' (the stored bytes)."""
    out = []
    for j in range(q):
        R32 = rotation_fp64(d, j, rotation_seed).astype(np.float32)
        out.append(R32 if dtype == "f32" else f32_to_bf16_bits(R32))
    return np.stack(out)


def to_stored(a, dtype: str) -> np.ndarray:
    """fp64 view of stored values (float32 array or uint16 bf16 bits)."""
    a = np.asarray(a)
    if dtype == "bf16" and a.dtype == np.uint16:
        return bf16_bits_to_f64(a)
    return a.astype(np.float64)


def ulp_bf16(x: np.ndarray) -> np.ndarray:
    """Spacing of bf16 numbers at |x| (8 significant bits)."""
    _, ex = np.frexp(np.asarray(x, dtype=np.float64))
    return np.ldexp(1.0, ex - 8)


def round_to_dtype(x: np.ndarray, dtype: str) -> np.ndarray:
    """O6: correctly rounded (RNE) fp64 -> dtype, returned as fp64 values.  Reading R23."""
    x = np.asarray(x, dtype=np.float64)
    if dtype == "f32":
        return x.astype(np.float32).astype(np.float64)
    if dtype == "f64":
        return x.copy()
    m, ex = np.frexp(x)                # |x| in [2^(ex-1), 2^ex)
    ulp = np.ldexp(1.0, ex - 8)        # bf16 keeps 8 significant bits
    return np.round(x / ulp) * ulp     # np.round is round-half-to-even; x/ulp is exact


# ---------------------------------------------------------------------------------------------
# O2. Cross-polytope hash, Eq. 3: LSH(x) = argmax_{i in {+-1..+-d}} |Rx|_i.
# Reading R1: i* = argmax_i |(Rx)_i|, code = sign((Rx)_{i*}) * (i*+1) (nearest vertex +-e_i,
# P:L230).  Reading R2: ties -> smallest index, zero winner -> '+'.  One R_j per hash
# function and the q codes are combined into the bucket key (reading R4).
# ---------------------------------------------------------------------------------------------
def cp_hash(X: np.ndarray, R: np.ndarray):
    """X [n, d] (stored values as fp64), R [q, d_out, d] (stored values as fp64; d_out = d for the
    dense rotations of O1, d_out = 1024 for NEXT-4's padded structured rotations, reading R30).

    Returns codes int16 [n, q] in {+-1..+-d_out} and margins fp64 [n, q]:
    margin = (max|y| - second max|y|) / max|y| (0 if max|y| = 0; 1 if d_out = 1).
    y = R_j x is evaluated in fp64: bf16/fp32 products are exact in fp64 and the sum's rounding
    (~1e-16 relative) is far below the 1e-5 near-tie band of BASELINE.json tier 1."""
    X = np.asarray(X, dtype=np.float64)
    R = np.asarray(R, dtype=np.float64)
    n = X.shape[0]
    q, dout = R.shape[0], R.shape[1]
    codes = np.empty((n, q), dtype=np.int16)
    margins = np.empty((n, q), dtype=np.float64)
    rows = np.arange(n)
    for j in range(q):
        Y = X @ R[j].T                       # y_i = sum_k R[i,k] x_k
        A = np.abs(Y)
        istar = np.argmax(A, axis=1)         # first occurrence of the maximum = smallest index
        amax = A[rows, istar]
        neg = Y[rows, istar] < 0             # zero winner (+0 or -0) counts as positive
        codes[:, j] = np.where(neg, -(istar + 1), istar + 1).astype(np.int16)
        if dout == 1:
            margins[:, j] = 1.0
        else:
            second = np.partition(A, dout - 2, axis=1)[:, dout - 2]
            with np.errstate(invalid="ignore", divide="ignore"):
                margins[:, j] = np.where(amax > 0, (amax - second) / np.where(amax > 0, amax, 1.0), 0.0)
    return codes, margins


# ---------------------------------------------------------------------------------------------
# O2*. NEXT-4: a structured pseudo-random rotation in place of Eq. 3's dense random
# rotation R ("R is a random rotation matrix"; the paper fixes no construction), "three
# rounds of Hadamard x random +-1 diagonal".  Reading R30: x is zero-padded to d' = 1024 (d <= 1024;
# d = 768 is not a power of two), R_j = H D3_j H D2_j H D1_j with H the unnormalised Sylvester
# Hadamard matrix of order d' (H[a, b] = (-1)^popcount(a & b)) and D_r,j diagonal +-1: entry i is
# -1 iff bit 63 of SplitMix64 output number r*d' + i + 1 of the stream seeded with
# rotation_seed ^ (0xD1B54A32D192ED03 * (j + 1) mod 2^64) is set.  R_j (d' x d after the padding
# columns are dropped) has exact integer entries (|R| <= d'^2) and orthogonal columns of norm
# d'^(3/2); Eq. 3's argmax is scale invariant, so no normalisation.  Codes index the d' outputs:
# code = sign(y_i*) (i* + 1), i* in [0, d').  The oracle materialises R_j densely and reuses
# cp_hash (the GPU applies it as three fast Walsh-Hadamard transforms).
# ---------------------------------------------------------------------------------------------
HD3_DIM = 1024
HD3_GAMMA = 0xD1B54A32D192ED03


def hadamard(order: int) -> np.ndarray:
    """Unnormalised Sylvester Hadamard matrix by the doubling recursion H_2m = [[H, H], [H, -H]]."""
    if order < 1 or order & (order - 1):
        raise ValueError("order must be a power of two")
    H = np.ones((1, 1))
    while H.shape[0] < order:
        H = np.block([[H, H], [H, -H]])
    return H


def hd3_signs(q: int, rotation_seed: int) -> np.ndarray:
    """D [q, 3, d'] in {+1, -1} (reading R30)."""
    out = np.empty((q, 3, HD3_DIM))
    for j in range(q):
        state = (rotation_seed ^ ((HD3_GAMMA * (j + 1)) & _MASK64)) & _MASK64
        z = splitmix64_stream(state, 3 * HD3_DIM).reshape(3, HD3_DIM)
        out[j] = np.where((z >> np.uint64(63)) == 1, -1.0, 1.0)
    return out


def hd3_rotation(d: int, q: int, rotation_seed: int) -> np.ndarray:
    """Dense R [q, d', d] = (H D3 H D2 H D1)[:, :d] per hash (reading R30), exact in fp64."""
    if not 1 <= d <= HD3_DIM:
        raise ValueError("NEXT-4 structured rotation needs 1 <= d <= 1024")
    H = hadamard(HD3_DIM)
    D = hd3_signs(q, rotation_seed)
    out = np.empty((q, HD3_DIM, d))
    for j in range(q):
        M = H @ np.diag(D[j, 2]) @ H @ np.diag(D[j, 1]) @ H @ np.diag(D[j, 0])
        out[j] = M[:, :d]
    return out


# ---------------------------------------------------------------------------------------------
# O0. The gate (Eq. 1-2: G(x) = TopK(softmax(x W_g)) selects k of the N experts and
# weights them).  Reading R29 (NEXT-2 "gate + hash in one projection"): scores s = W_g x in exact
# arithmetic on the stored values; the k largest, ties to the smaller expert id; slots in ascending
# expert id; weights = softmax over the k selected scores (S:L260 order).  margin = the
# gap between the k-th and (k+1)-th largest score over max |s| (near-tie if < 1e-5).
# ---------------------------------------------------------------------------------------------
def gate_topk(X: np.ndarray, Wg: np.ndarray, k: int):
    """-> zeta int32 [n, k] (ascending ids), g fp64 [n, k], margin fp64 [n]."""
    S = np.asarray(X, np.float64) @ np.asarray(Wg, np.float64).T
    n, E = S.shape
    order = np.argsort(-S, axis=1, kind="stable")        # equal scores keep the smaller id first
    top = np.sort(order[:, :k], axis=1)
    sel = np.take_along_axis(S, top, axis=1)
    ex = np.exp(sel - sel.max(axis=1, keepdims=True))
    g = ex / ex.sum(axis=1, keepdims=True)
    srt = -np.sort(-S, axis=1)
    scale = np.maximum(np.abs(S).max(axis=1), 1e-300)
    margin = (srt[:, k - 1] - srt[:, k]) / scale if k < E else np.ones(n)
    return top.astype(np.int32), g, margin


# ---------------------------------------------------------------------------------------------
# O2". NEXT-2's fp8 option ("optionally fp8 (kind::f8f6f4) rotation to halve
# the hash cost (codes then defined on fp8-rounded values)").  Reading R28: Eq. 3's argmax is
# invariant to a positive scale of x and, per hash function, of R_j, so each token and each R_j
# is scaled by the largest power of two 2^k with max|v| * 2^k <= 448 (e4m3's largest finite value)
# and rounded to e4m3 (round to nearest, ties to even); the codes are Eq. 3 evaluated exactly on
# those values.  R_j's source is the fp32-stored rotation (O1).
# ---------------------------------------------------------------------------------------------
def e4m3_values() -> np.ndarray:
    """The 127 non-negative finite e4m3 (e4m3fn) values in code order 0x00..0x7E."""
    vals = []
    for code in range(0x7F):
        e, m = code >> 3, code & 7
        vals.append(m * 2.0 ** -9 if e == 0 else (1 + m / 8.0) * 2.0 ** (e - 7))
    return np.array(vals)


def round_e4m3(a: np.ndarray) -> np.ndarray:
    """Nearest e4m3 value (ties to the even code), |a| <= 448; by search in the value table."""
    a = np.asarray(a, dtype=np.float64)
    if np.any(np.abs(a) > 448):
        raise ValueError("|a| > 448")
    tab = e4m3_values()
    mag = np.abs(a)
    hi = np.searchsorted(tab, mag, side="left").clip(0, len(tab) - 1)   # first value >= mag
    lo = np.maximum(hi - 1, 0)
    dlo, dhi = mag - tab[lo], tab[hi] - mag
    pick_hi = (dhi < dlo) | ((dhi == dlo) & (hi % 2 == 0) & (hi != lo))
    out = np.where(pick_hi, tab[hi], tab[lo])
    out = np.where(mag == tab[hi], tab[hi], out)
    return np.where(a < 0, -out, out)


def pow2_scale_e4m3(vmax: float) -> float:
    """Largest 2^k with vmax * 2^k <= 448 (1 for vmax == 0)."""
    if vmax == 0:
        return 1.0
    f, e = math.frexp(vmax)                 # vmax = f * 2^e, f in [0.5, 1)
    k = (9 - e) if f <= 0.875 else (8 - e)   # 448 = 0.875 * 2^9
    return math.ldexp(1.0, k)


def quantize_tokens_e4m3(X: np.ndarray) -> np.ndarray:
    """Per-token power-of-two scale, then e4m3 (values as fp64)."""
    X = np.asarray(X, np.float64)
    sc = np.array([pow2_scale_e4m3(float(np.abs(r).max())) for r in X])
    return round_e4m3(X * sc[:, None])


def quantize_rotation_e4m3(R32: np.ndarray) -> np.ndarray:
    """Per-hash power-of-two scale of the fp32-stored R_j, then e4m3 (values as fp64)."""
    R32 = np.asarray(R32, np.float64)
    return np.stack([round_e4m3(Rj * pow2_scale_e4m3(float(np.abs(Rj).max()))) for Rj in R32])


# ---------------------------------------------------------------------------------------------
# O2'. Spherical-plane (SP) hashing, the paper's other evaluated family (§4.5 "Impact of the Types
# of Hash Functions").  The paper never defines its construction; SPEC
# reads it as random-hyperplane sign bits: bit i = 1 iff n_i . x >= 0 (zero dots count as 1).
# Reading R26: hash function j uses b unit normals (rows j*b .. j*b+b-1 of N [q*b, d]) and its
# code is the integer sum_i bit_i * 2^i (0 .. 2^b - 1, b <= 15 so it fits an int16); the q codes
# form the composite key exactly like the CP codes (reading R4).  The recommended normals are the
# first b rows of the rotations R_j of O1 (orthonormal, hence unit), see sp_normals.
# ---------------------------------------------------------------------------------------------
def sp_normals(R: np.ndarray, b: int) -> np.ndarray:
    """N [q*b, d]: the first b rows of each rotation R_j (reading R26)."""
    R = np.asarray(R, dtype=np.float64)
    q = R.shape[0]
    return np.concatenate([R[j, :b, :] for j in range(q)], axis=0)


def sp_hash(X: np.ndarray, N: np.ndarray, q: int, b: int):
    """X [n, d], N [q*b, d] (stored values as fp64) -> codes int16 [n, q] in [0, 2^b), and
    margins fp64 [n, q] = min_i |n_i . x| / (||n_i|| ||x||) over the hash's b normals (0 for a
    zero token): a sign decision with margin < 1e-5 is a near-tie (BASELINE tier 1)."""
    X = np.asarray(X, dtype=np.float64)
    N = np.asarray(N, dtype=np.float64)
    n, d = X.shape
    if N.shape != (q * b, d):
        raise ValueError("N must be [q*b, d]")
    if not 1 <= b <= 15:
        raise ValueError("1 <= b <= 15")
    Y = X @ N.T                                          # [n, q*b] dots in fp64
    bits = (Y >= 0).astype(np.int64)                     # -0.0 >= 0: a zero dot is bit 1
    codes = np.zeros((n, q), dtype=np.int16)
    margins = np.empty((n, q), dtype=np.float64)
    xn = np.linalg.norm(X, axis=1)
    nn = np.linalg.norm(N, axis=1)
    for j in range(q):
        cols = slice(j * b, (j + 1) * b)
        codes[:, j] = (bits[:, cols] << np.arange(b)).sum(axis=1).astype(np.int16)
        with np.errstate(invalid="ignore", divide="ignore"):
            rel = np.abs(Y[:, cols]) / (xn[:, None] * nn[None, cols])
        margins[:, j] = np.where(xn > 0, rel.min(axis=1), 0.0)
    return codes, margins


# ---------------------------------------------------------------------------------------------
# O3. Alg. 1 L3: "Dispatch X into {X_i} based on zeta" -- the routed copies (t, s) of
# expert e in ascending (t, s) order (reading R5: clustering happens after gating duplication).
# ---------------------------------------------------------------------------------------------
def group_by_expert(zeta: np.ndarray, E: int) -> List[List[int]]:
    n, k = zeta.shape
    groups: List[List[int]] = [[] for _ in range(E)]
    for t in range(n):
        for s in range(k):
            e = int(zeta[t, s])
            if not (0 <= e < E):
                raise ValueError("expert id out of range (S:L312)")
            groups[e].append(t * k + s)
    return groups


@dataclass
class Buckets:
    bucket: np.ndarray        # int32 [n, k]   global centroid row of routed copy (t, s)
    perm: np.ndarray          # int32 [n*k]    copy ids t*k+s grouped by row, ascending within
    row_start: np.ndarray     # int32 [m+1]
    expert_rows: np.ndarray   # int32 [E]      m_e
    m: int


def bucketize(codes: np.ndarray, zeta: np.ndarray, E: int) -> Buckets:
    """O4. Alg. 1 L5-6: IDX_i <- LSH(X_i); divide X_i into clusters by IDX.

    The bucket of a routed copy is its q-tuple of codes (AND-composite key, reading
    R4).  Within each expert group, bucket ids are assigned in first-appearance order of the
    group's (t, s) order (reading R7); global row = sum_{e'<e} m_e' + local id; members
    of a row are listed in ascending (t, s) (reading R8).  A token's codes are computed once and
    shared by its k routed copies (reading R6: LSH(X_i) applies the same function to every X_i)."""
    n, k = zeta.shape
    groups = group_by_expert(zeta, E)
    bucket = np.empty((n, k), dtype=np.int32)
    members: List[List[int]] = []
    expert_rows = np.zeros(E, dtype=np.int32)
    off = 0
    for e in range(E):
        ids = {}
        for c in groups[e]:
            key = tuple(int(v) for v in codes[c // k])
            b = ids.get(key)
            if b is None:
                b = len(ids)
                ids[key] = b
                members.append([])
            members[off + b].append(c)
            bucket[c // k, c % k] = off + b
        expert_rows[e] = len(ids)
        off += len(ids)
    perm = np.array([c for mem in members for c in mem], dtype=np.int32)
    row_start = np.zeros(off + 1, dtype=np.int32)
    row_start[1:] = np.cumsum([len(mem) for mem in members]) if members else []
    return Buckets(bucket, perm, row_start, expert_rows, off)


def centroids(X: np.ndarray, b: Buckets, k: int) -> np.ndarray:
    """O5. Alg. 1 L8: centroid = Mean(cluster_j), i.e. C_j = (1/n_j) sum x (§2.3,
    P:L169, whose "1/n" is read as 1/n_j -- reading R9).  fp64."""
    X = np.asarray(X, dtype=np.float64)
    if b.m == 0:
        return np.zeros((0, X.shape[1]))
    rows = X[b.perm // k]
    sums = np.add.reduceat(rows, b.row_start[:-1], axis=0)
    counts = np.diff(b.row_start).astype(np.float64)
    return sums / counts[:, None]


# ---------------------------------------------------------------------------------------------
# O8. Expert network: "each FFN function works as an individual expert" (§2.1);
# E(x) = W2 act(W1 x + b1) + b2 with ReLU.  fp64 from the stored weights.
# ---------------------------------------------------------------------------------------------
def expert_ffn(Xin: np.ndarray, W1: np.ndarray, b1: np.ndarray, W2: np.ndarray, b2: np.ndarray) -> np.ndarray:
    H = np.maximum(np.asarray(Xin, np.float64) @ np.asarray(W1, np.float64).T + np.asarray(b1, np.float64), 0.0)
    return H @ np.asarray(W2, np.float64).T + np.asarray(b2, np.float64)


# ---------------------------------------------------------------------------------------------
# O7 / O9. All-to-all of the centroids (Alg. 1 L14) and of the expert outputs (L16,
# P:L535).  Expert placement: rank p owns the contiguous block [p*E/w, (p+1)*E/w).
# Receive layout on rank p (reading R24 in DESIGN.md): ordered by (local expert, source rank,
# local bucket), so every local expert's rows are contiguous for its FFN; rows of one
# (src, dst) pair are never reordered.
# ---------------------------------------------------------------------------------------------
def dispatch_sim(C_by_rank: Sequence[np.ndarray], expert_rows_by_rank: Sequence[np.ndarray], E: int):
    """Returns (recv per rank, recv_rows per rank [E/w, w])."""
    w = len(C_by_rank)
    epr = E // w
    offs = [np.concatenate([[0], np.cumsum(er)]) for er in expert_rows_by_rank]
    recv, recv_rows = [], []
    for p in range(w):
        parts = []
        rr = np.zeros((epr, w), dtype=np.int32)
        for el in range(epr):
            e = p * epr + el
            for src in range(w):
                a, bnd = offs[src][e], offs[src][e + 1]
                parts.append(C_by_rank[src][a:bnd])
                rr[el, src] = bnd - a
        d = C_by_rank[0].shape[1]
        recv.append(np.concatenate(parts, axis=0) if parts else np.zeros((0, d)))
        recv_rows.append(rr)
    return recv, recv_rows


def combine_sim(out_by_rank: Sequence[np.ndarray], expert_rows_by_rank: Sequence[np.ndarray], E: int):
    """Exact reverse of dispatch_sim: every source gets its rows back in its own C layout."""
    w = len(out_by_rank)
    epr = E // w
    d = out_by_rank[0].shape[1]
    offs = [np.concatenate([[0], np.cumsum(er)]) for er in expert_rows_by_rank]
    ret = [np.zeros((int(offs[src][-1]), d)) for src in range(w)]
    for p in range(w):
        pos = 0
        for el in range(epr):
            e = p * epr + el
            for src in range(w):
                a, bnd = offs[src][e], offs[src][e + 1]
                ret[src][a:bnd] = out_by_rank[p][pos:pos + (bnd - a)]
                pos += bnd - a
    return ret


# ---------------------------------------------------------------------------------------------
# O10. Residual-based error compensation.  Eq. 4: Delta = x - centroid; Eq. 5
# (P:L245-248): Y = E(centroid) + Delta; Alg. 1 L17-19.  The k outputs of a token
# are summed as in Eq. 2, optionally weighted by g (reading R13).  Reading R11: the
# residual is taken against the centroid as transmitted (c~), so identity experts restore x.
# ---------------------------------------------------------------------------------------------
def restore(X: np.ndarray, Ct: np.ndarray, ret: np.ndarray, bucket: np.ndarray,
            g: Optional[np.ndarray] = None) -> np.ndarray:
    X = np.asarray(X, np.float64)
    n, k = bucket.shape
    y = np.zeros_like(X)
    for s in range(k):
        b = bucket[:, s]
        term = np.asarray(ret, np.float64)[b] + (X - np.asarray(Ct, np.float64)[b])
        y += term if g is None else np.asarray(g, np.float64)[:, s:s + 1] * term
    return y


def moe_dense(X: np.ndarray, zeta: np.ndarray, experts, g: Optional[np.ndarray] = None) -> np.ndarray:
    """O12. Eq. 2: f(x) = sum_{i in G(x)} E_i(x), uncompressed.  experts[e] =
    (W1, b1, W2, b2)."""
    X = np.asarray(X, np.float64)
    n, k = zeta.shape
    y = np.zeros_like(X)
    for s in range(k):
        for e in np.unique(zeta[:, s]):
            idx = np.nonzero(zeta[:, s] == e)[0]
            out = expert_ffn(X[idx], *experts[int(e)])
            y[idx] += out if g is None else np.asarray(g, np.float64)[idx, s:s + 1] * out
    return y


# ---------------------------------------------------------------------------------------------
# The whole layer (Alg. 1), per simulated rank r = 0..w-1; ranks are independent until O7.
# ---------------------------------------------------------------------------------------------
@dataclass
class LayerResult:
    codes: list
    margins: list
    buckets: list
    C: list            # fp64 centroids per rank
    Ct: list           # centroids rounded to the wire dtype (fp64 values)
    recv: list
    recv_rows: list
    expert_out: list   # E(C~) per rank in recv layout, rounded to dtype
    ret: list          # combined E(C~) per rank in C layout
    y: list            # restored outputs per rank (fp64, before rounding)
    y_rounded: list
    ratio: float
    stats: dict = field(default_factory=dict)


def lsh_layer_ranks(X_by_rank, zeta_by_rank, R, experts, E: int, dtype: str,
                    g_by_rank=None, round_expert_out: bool = True) -> LayerResult:
    """Alg. 1 end to end on w simulated ranks (w = len(X_by_rank)).  X, R are stored values
    (fp64 arrays); experts[e] = (W1, b1, W2, b2) stored values (fp64)."""
    w = len(X_by_rank)
    if E % w != 0:
        raise ValueError("E % w != 0 (S:L285)")
    codes, margins, bks, Cs, Cts = [], [], [], [], []
    for r in range(w):
        X = np.asarray(X_by_rank[r], np.float64)
        zeta = np.asarray(zeta_by_rank[r])
        k = zeta.shape[1]
        c, mg = cp_hash(X, R)                                 # Alg. 1 L5
        b = bucketize(c, zeta, E)                             # Alg. 1 L3, L5-6
        C = centroids(X, b, k)                                # Alg. 1 L8
        codes.append(c); margins.append(mg); bks.append(b); Cs.append(C)
        Cts.append(round_to_dtype(C, dtype))                  # wire precision (R10/R23)
    recv, recv_rows = dispatch_sim(Cts, [b.expert_rows for b in bks], E)   # Alg. 1 L14
    epr = E // w
    outs = []
    for p in range(w):                                        # Alg. 1 L15: Expert(Input)
        o = np.zeros_like(recv[p])
        pos = 0
        for el in range(epr):
            cnt = int(recv_rows[p][el].sum())
            if cnt:
                o[pos:pos + cnt] = expert_ffn(recv[p][pos:pos + cnt], *experts[p * epr + el])
            pos += cnt
        outs.append(round_to_dtype(o, dtype) if round_expert_out else o)
    rets = combine_sim(outs, [b.expert_rows for b in bks], E)  # Alg. 1 L16
    ys, yrs = [], []
    for r in range(w):                                        # Alg. 1 L17-19
        g = None if g_by_rank is None else g_by_rank[r]
        y = restore(X_by_rank[r], Cts[r], rets[r], bks[r].bucket, g)
        ys.append(y); yrs.append(round_to_dtype(y, dtype))
    tot_m = sum(b.m for b in bks)
    tot_nk = sum(np.asarray(z).size for z in zeta_by_rank)
    return LayerResult(codes, margins, bks, Cs, Cts, recv, recv_rows, outs, rets, ys, yrs,
                       tot_m / tot_nk if tot_nk else 0.0)


def lsh_layer(X, zeta, R, experts, E: int, dtype: str, g=None, round_expert_out: bool = True) -> LayerResult:
    """Single-rank (w = 1) Alg. 1."""
    return lsh_layer_ranks([X], [zeta], R, experts, E, dtype, None if g is None else [g], round_expert_out)


# ---------------------------------------------------------------------------------------------
# NEXT-1. Backward of the compressed layer (the paper trains with LSH-MoE, App. B
# P:L577, but never writes the gradient; "residual-based gradient compensation", is read
# as compensating activations -- reading R14).  Reading R27: the codes and buckets are constants
# (piecewise-constant hash), the rounding c~ = RNE(c) is straight-through, and the forward is
#   c_b = (1/n_b) sum_{(t,s) in b} x_t        (O5, Alg. 1 L8)
#   o_b = E_{e(b)}(c~_b)                      (O8, Alg. 1 L15)
#   y_t = sum_s g_ts (o_{b_ts} + x_t - c~_{b_ts})   (O10, Eq. 4-5 inside Eq. 2)
# so, for an upstream gradient dY:
#   B1 G_b   = sum_{(t,s) in b} g_ts dY_t               dL/do_b; the c~ term contributes -G_b
#   B2/B4    G travels to the expert's rank and back like c~ / o (Alg. 1 L14/L16 in reverse)
#   B3 H_b   = J_E(c~_b)^T G_b                          the expert's backward
#   B5 dX_t  = sum_s [ g_ts dY_t + (H_b - G_b) / n_b ]  with b = b_ts (chain rule through c_b)
#      dg_ts = dY_t . (o_b + x_t - c~_b)
# ---------------------------------------------------------------------------------------------
def grad_compress(dY: np.ndarray, b: Buckets, k: int, g: Optional[np.ndarray] = None) -> np.ndarray:
    """B1: G [m, d] = per-row sums of g_ts dY_t over the row's routed copies (fp64), in the
    centroid (send) layout."""
    dY = np.asarray(dY, np.float64)
    if b.m == 0:
        return np.zeros((0, dY.shape[1]))
    w = np.ones(b.perm.shape[0]) if g is None else np.asarray(g, np.float64).reshape(-1)[b.perm]
    rows = dY[b.perm // k] * w[:, None]
    return np.add.reduceat(rows, b.row_start[:-1], axis=0)


def expert_ffn_vjp(Cin: np.ndarray, W1: np.ndarray, b1: np.ndarray, W2: np.ndarray, G: np.ndarray) -> np.ndarray:
    """B3: J_E(c)^T G for E(c) = W2 relu(W1 c + b1) + b2, row by row: W1^T (relu'(W1 c + b1) * (W2^T G)),
    relu'(0) = 0.  fp64."""
    pre = np.asarray(Cin, np.float64) @ np.asarray(W1, np.float64).T + np.asarray(b1, np.float64)
    dh = (np.asarray(G, np.float64) @ np.asarray(W2, np.float64)) * (pre > 0)
    return dh @ np.asarray(W1, np.float64)


def grad_restore(dY: np.ndarray, X: np.ndarray, Ct: np.ndarray, ret: np.ndarray, G: np.ndarray, H: np.ndarray,
                 b: Buckets, g: Optional[np.ndarray] = None):
    """B5: (dX [n, d], dg [n, k]) of y_t = sum_s g_ts (o_b + x_t - c~_b) with c_b the bucket mean
    (reading R27).  ret = o (combined expert outputs, C layout); G from B1, H from B3 (C layout)."""
    dY = np.asarray(dY, np.float64)
    X = np.asarray(X, np.float64)
    n, k = b.bucket.shape
    cnt = np.diff(b.row_start).astype(np.float64)
    Gm, Hm = np.asarray(G, np.float64), np.asarray(H, np.float64)
    dX = np.zeros_like(dY)
    dg = np.zeros((n, k))
    for s in range(k):
        bs = b.bucket[:, s]
        gw = np.ones(n) if g is None else np.asarray(g, np.float64)[:, s]
        dX += gw[:, None] * dY + (Hm[bs] - Gm[bs]) / cnt[bs][:, None]
        dg[:, s] = (dY * (np.asarray(ret, np.float64)[bs] + X - np.asarray(Ct, np.float64)[bs])).sum(axis=1)
    return dX, dg


def lsh_layer_backward(X, zeta, b: Buckets, Ct, ret, experts, dY, g=None):
    """Single-rank composition B1 -> B3 (per expert) -> B5 in fp64 (the exchanges B2/B4 are the
    identity at one rank; dispatch_sim/combine_sim move G and H like c~ and o)."""
    k = b.bucket.shape[1]
    G = grad_compress(dY, b, k, g)
    H = np.zeros_like(G)
    off = 0
    for e, me in enumerate(b.expert_rows):
        if me:
            W1, b1, W2, _ = experts[e]
            H[off:off + me] = expert_ffn_vjp(np.asarray(Ct, np.float64)[off:off + me], W1, b1, W2, G[off:off + me])
        off += me
    dX, dg = grad_restore(dY, X, Ct, ret, G, H, b, g)
    return G, H, dX, dg

