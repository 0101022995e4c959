"""Pins for oracle O2: cross-polytope hash, Eq. 3."""
import numpy as np
import pytest

import oracle as O
from oracle import brute


def test_identity_rotation_examples(golden):
    for case in golden["cp_hash_identity_rotation"]["cases"]:
        x = np.array([case["x"]])
        codes, _ = O.cp_hash(x, np.eye(3)[None])
        assert codes[0, 0] == case["code"]


def _rand(n, d, q, seed):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, d))
    R = np.stack([np.linalg.qr(rng.standard_normal((d, d)))[0] for _ in range(q)])
    return X, R


def test_codes_range_never_zero():
    X, R = _rand(500, 16, 4, 0)
    codes, _ = O.cp_hash(X, R)
    assert codes.dtype == np.int16
    assert np.all(codes != 0) and np.all(np.abs(codes) <= 16)


@pytest.mark.parametrize("alpha", [3.0, 0.5, 1e-3])
def test_positive_scale_invariance(alpha):
    X, R = _rand(300, 12, 3, 1)
    assert np.array_equal(O.cp_hash(X, R)[0], O.cp_hash(alpha * X, R)[0])


def test_negation_flips_sign():
    X, R = _rand(300, 12, 3, 2)
    c1, m = O.cp_hash(X, R)
    c2, _ = O.cp_hash(-X, R)
    ok = m > 1e-12
    assert np.array_equal(c2[ok], -c1[ok])


def test_signed_permutation_rotation_closed_form():
    """R = P D (signed permutation): (Rx)_i = D_pi(i) x_pi(i); the argmax is the textbook argmax
    of |x| mapped through the permutation."""
    rng = np.random.default_rng(3)
    d = 10
    perm = rng.permutation(d)
    sgn = rng.choice([-1.0, 1.0], d)
    R = np.zeros((d, d))
    R[np.arange(d), perm] = sgn
    X = rng.standard_normal((200, d))
    codes, _ = O.cp_hash(X, R[None])
    for t in range(200):
        y = sgn * X[t, perm]
        i = int(np.argmax(np.abs(y)))
        assert codes[t, 0] == (i + 1 if y[i] >= 0 else -(i + 1))


def test_matches_bruteforce_loops():
    X, R = _rand(60, 8, 3, 4)
    codes, _ = O.cp_hash(X, R)
    for t in range(60):
        for j in range(3):
            assert codes[t, j] == brute.cp_hash_one(R[j].tolist(), X[t].tolist())


def test_ties_go_to_smallest_index_and_margin_zero():
    X = np.array([[3.0, -3.0, 1.0], [-2.0, 2.0, 2.0], [0.0, 0.0, 0.0]])
    codes, margins = O.cp_hash(X, np.eye(3)[None])
    assert list(codes[:, 0]) == [1, -1, 1]
    assert np.all(margins[:, 0] == 0.0)


def test_margin_definition():
    X = np.array([[4.0, -1.0, 3.0]])
    _, m = O.cp_hash(X, np.eye(3)[None])
    assert m[0, 0] == pytest.approx(0.25)


def test_d1():
    codes, m = O.cp_hash(np.array([[2.0], [-0.5], [0.0]]), np.ones((1, 1, 1)))
    assert list(codes[:, 0]) == [1, -1, 1] and np.all(m == 1.0)


def test_collision_similarity_trend():
    """S:L176 restating §2.3: closer pairs collide at least as often."""
    rng = np.random.default_rng(5)
    d, q = 16, 1
    R = np.stack([np.linalg.qr(rng.standard_normal((d, d)))[0] for _ in range(200)])
    rates = []
    for eps in (0.05, 0.3, 1.0):
        X = rng.standard_normal((400, d))
        Y = X + eps * rng.standard_normal((400, d))
        cx, _ = O.cp_hash(X, R)
        cy, _ = O.cp_hash(Y, R)
        rates.append(float((cx == cy).mean()))
    assert rates[0] >= rates[1] >= rates[2]
