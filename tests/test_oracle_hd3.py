"""Pins of the oracle's NEXT-4 structured rotation (O2*, reading R30): the Hadamard matrix against a
library routine and its closed form, the sign stream against the published SplitMix64 outputs,
the dense R_j against textbook fast-Walsh-Hadamard butterfly loops, orthogonality, and Eq. 3's
argmax over the d' = 1024 padded outputs against the brute-force hash."""
import numpy as np
import pytest
import scipy.linalg

import oracle as O
from oracle import brute as B


@pytest.mark.parametrize("order", [1, 2, 4, 32, 256, 1024])
def test_hadamard_matches_library_and_closed_form(order):
    H = O.hadamard(order)
    assert np.array_equal(H, scipy.linalg.hadamard(order))
    assert np.array_equal(H @ H.T, order * np.eye(order))
    a, b = np.meshgrid(np.arange(order), np.arange(order), indexing="ij")
    pc = np.vectorize(lambda v: bin(v).count("1"))(a & b)
    assert np.array_equal(H, np.where(pc % 2 == 1, -1.0, 1.0))        # H[a, b] = (-1)^popcount(a & b)


def test_hd3_signs_from_splitmix64(golden):
    """With rotation_seed = 0xD1B54A32D192ED03 the stream of hash 0 is seeded with state 0, whose
    first outputs are the published SplitMix64 values: D[0, 0, i] = -1 iff bit 63 of output i+1."""
    D = O.hd3_signs(2, O.HD3_GAMMA)
    outs = [int(h, 16) for h in golden["splitmix64_seed0"]["outputs_hex"]]
    assert [float(v) for v in D[0, 0, :3]] == [-1.0 if z >> 63 else 1.0 for z in outs]
    assert set(np.unique(D)) == {-1.0, 1.0}
    assert abs(D.mean()) < 0.05                                         # balanced
    assert not np.array_equal(D[0], D[1]) and not np.array_equal(D[0, 0], D[0, 1])
    assert np.array_equal(D, O.hd3_signs(2, O.HD3_GAMMA))               # deterministic


def test_hd3_rotation_equals_three_fwht_rounds():
    """R_j x = FWHT(D3 * FWHT(D2 * FWHT(D1 * pad(x)))) by butterfly loops, exactly (integer x)."""
    rng = np.random.default_rng(0)
    d, q, seed = 100, 2, 77
    R = O.hd3_rotation(d, q, seed)
    D = O.hd3_signs(q, seed)
    for j in range(q):
        for _ in range(2):
            x = rng.integers(-50, 50, d).astype(float)
            v = list(np.concatenate([x, np.zeros(O.HD3_DIM - d)]))
            for r in range(3):
                v = B.fwht_loops([s * a for s, a in zip(D[j, r], v)])
            assert np.array_equal(np.array(v), R[j] @ x)


def test_hd3_rotation_orthogonal_columns():
    for d in (1, 64, 768, 1024):
        R = O.hd3_rotation(d, 1, 5)[0]
        assert R.shape == (O.HD3_DIM, d)
        assert np.array_equal(R.T @ R, O.HD3_DIM ** 3 * np.eye(d))     # exact: integer entries
    with pytest.raises(ValueError):
        O.hd3_rotation(1025, 1, 5)


def test_cp_hash_on_padded_outputs_matches_brute():
    """Eq. 3 with the rectangular R_j: argmax over the d' = 1024 outputs, codes in +-1..+-1024, ties
    to the smallest index, margins over the d' outputs."""
    rng = np.random.default_rng(3)
    d = 24
    R = O.hd3_rotation(d, 2, 9)
    X = rng.standard_normal((12, d))
    X[3] = 0.0                                                          # zero winner -> +1
    codes, margins = O.cp_hash(X, R)
    for t in range(12):
        for j in range(2):
            assert codes[t, j] == B.cp_hash_one(R[j].tolist(), X[t].tolist())
    assert codes[3, 0] == 1 and codes[3, 1] == 1
    assert np.abs(codes).max() <= O.HD3_DIM and np.all(codes != 0)
    Y = np.abs(X[0] @ R[0].T)
    srt = np.sort(Y)
    assert margins[0, 0] == pytest.approx((srt[-1] - srt[-2]) / srt[-1], rel=1e-12)
    assert np.array_equal(O.cp_hash(2.5 * X, R)[0], codes)              # positive-scale invariant
