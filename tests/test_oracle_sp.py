"""Pins of the oracle's spherical-plane (SP) hash, O2' (§4.5; SPEC's
sign-bit construction S:L124-132, reading R26) against what SPEC and the mathematics fix."""
import math

import numpy as np

import oracle as O
from oracle import brute


def test_sp_identity_normals_spec_example(golden):
    """normals = I (dim 3), x = (1, -1, 0) -> bits (1, 0, 1) (zero dot counts as 1)."""
    g = golden["sp_hash_identity_normals"]
    x = np.array([g["x"]])
    codes, margins = O.sp_hash(x, np.eye(3), q=1, b=3)
    want = sum(bit << i for i, bit in enumerate(g["bits"]))
    assert int(codes[0, 0]) == want == 5
    assert margins[0, 0] == 0.0                     # the zero dot is an exact tie


def test_sp_negation_complements_bits():
    """x and -x with no zero dots give complementary bit patterns."""
    rng = np.random.default_rng(0)
    X = rng.standard_normal((200, 16))
    N = rng.standard_normal((3 * 5, 16))
    a, ma = O.sp_hash(X, N, 3, 5)
    b, _ = O.sp_hash(-X, N, 3, 5)
    assert np.all(ma > 0)
    assert np.array_equal(a.astype(np.int64) ^ b.astype(np.int64), np.full(a.shape, (1 << 5) - 1))


def test_sp_positive_scale_invariant_and_range():
    rng = np.random.default_rng(1)
    X = rng.standard_normal((100, 8))
    N = rng.standard_normal((2 * 7, 8))
    a, _ = O.sp_hash(X, N, 2, 7)
    b, _ = O.sp_hash(3.5 * X, N, 2, 7)
    assert np.array_equal(a, b)
    assert a.min() >= 0 and a.max() < (1 << 7)


def test_sp_matches_brute_force_loops():
    rng = np.random.default_rng(2)
    X = rng.standard_normal((40, 6))
    N = rng.standard_normal((3 * 4, 6))
    codes, _ = O.sp_hash(X, N, 3, 4)
    for t in range(40):
        for j in range(3):
            assert codes[t, j] == brute.sp_hash_one(N[j * 4:(j + 1) * 4].tolist(), X[t].tolist())


def test_sp_hyperplane_collision_probability():
    """S:L131 [DERIVED]: one random hyperplane separates two unit vectors at angle theta with
    probability theta/pi (Goemans-Williamson), so the collision rate is 1 - theta/pi."""
    rng = np.random.default_rng(3)
    d, trials = 16, 4000
    for theta in (0.3, 1.0, 2.0):
        u = rng.standard_normal((trials, d))
        u /= np.linalg.norm(u, axis=1, keepdims=True)
        w = rng.standard_normal((trials, d))
        w -= (w * u).sum(1, keepdims=True) * u
        w /= np.linalg.norm(w, axis=1, keepdims=True)
        v = math.cos(theta) * u + math.sin(theta) * w
        same = 0
        for t in range(trials):
            nrm = rng.standard_normal((1, d))
            a, _ = O.sp_hash(u[t:t + 1], nrm, 1, 1)
            b, _ = O.sp_hash(v[t:t + 1], nrm, 1, 1)
            same += int(a[0, 0] == b[0, 0])
        assert abs(same / trials - (1 - theta / math.pi)) < 0.04


def test_sp_normals_are_rotation_rows_and_unit():
    R = O.rotation(32, 3, 12345, "f32")
    N = O.sp_normals(O.to_stored(R, "f32"), 5)
    assert N.shape == (15, 32)
    assert np.allclose(np.linalg.norm(N, axis=1), 1.0, atol=1e-6)
    assert np.array_equal(N[5:10], O.to_stored(R, "f32")[1, :5])
