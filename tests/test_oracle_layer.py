"""Pins for oracle O5-O12: centroid, expert, dispatch/combine, restore and the whole Alg. 1."""
import numpy as np
import pytest

import oracle as O
from oracle import brute


def _experts_random(E, d, dff, seed):
    rng = np.random.default_rng(seed)
    return {e: (rng.standard_normal((dff, d)) / np.sqrt(d), 0.1 * rng.standard_normal(dff),
                rng.standard_normal((d, dff)) / np.sqrt(dff), 0.1 * rng.standard_normal(d)) for e in range(E)}


def _experts_linear(E, d, scales):
    """E_e(x) = a_e x built from ReLU: W1 = [I; -I], W2 = a [I, -I]."""
    I = np.eye(d)
    return {e: (np.vstack([I, -I]), np.zeros(2 * d), scales[e] * np.hstack([I, -I]), np.zeros(d)) for e in range(E)}


def _experts_affine(E, d, seed):
    rng = np.random.default_rng(seed)
    out, Ws = {}, {}
    for e in range(E):
        W = rng.standard_normal((d, d)) / np.sqrt(d)
        b = rng.standard_normal(d)
        # W x + b = [W, -W] relu([I; -I] x) + b
        out[e] = (np.vstack([np.eye(d), -np.eye(d)]), np.zeros(2 * d), np.hstack([W, -W]), b)
        Ws[e] = (W, b)
    return out, Ws


def _clustered(n, d, comps, rho, seed):
    rng = np.random.default_rng(seed)
    U = rng.standard_normal((comps, d))
    return U[rng.integers(0, comps, n)] + rho * rng.standard_normal((n, d))


def _zeta(n, k, E, seed):
    rng = np.random.default_rng(seed)
    return np.sort(np.stack([rng.choice(E, k, replace=False) for _ in range(n)]), axis=1).astype(np.int32)


def _R(d, q, seed=1):
    return np.stack([O.rotation_fp64(d, j, seed) for j in range(q)])


def test_centroid_equals_fsum_mean_and_residuals_vanish():
    X = _clustered(120, 6, 4, 0.2, 0)
    zeta = _zeta(120, 2, 3, 0)
    codes, _ = O.cp_hash(X, _R(6, 2))
    b = O.bucketize(codes, zeta, 3)
    C = O.centroids(X, b, 2)
    for r in range(b.m):
        mem = b.perm[b.row_start[r]:b.row_start[r + 1]]
        rows = X[mem // 2]
        assert np.allclose(C[r], brute.mean_fsum(rows.tolist()), rtol=0, atol=1e-14)
        assert np.abs((rows - C[r]).sum(axis=0)).max() <= 1e-9 * np.abs(X).mean()
        if len(mem) == 1:
            assert np.array_equal(C[r], rows[0])                    # singleton: c = x exactly


def test_expert_ffn_closed_forms_and_loops(golden):
    d = 5
    I = np.eye(d)
    x = np.abs(np.random.default_rng(0).standard_normal((3, d)))
    assert np.array_equal(O.expert_ffn(x, I, np.zeros(d), I, np.zeros(d)), x)
    assert np.array_equal(O.expert_ffn(np.zeros((1, d)), I, np.zeros(d), I, np.zeros(d)), np.zeros((1, d)))
    W1, b1, W2, b2 = _experts_random(1, 8, 12, 1)[0]
    xr = np.random.default_rng(2).standard_normal(8)
    assert np.allclose(O.expert_ffn(xr[None], W1, b1, W2, b2)[0], brute.ffn_loops(xr, W1, b1, W2, b2), atol=1e-12)


def test_moe_dense_linear_example(golden):
    g = golden["moe_dense_linear"]
    d = 4
    X = np.random.default_rng(3).standard_normal((10, d))
    ex = _experts_linear(2, d, [g["scale_e1"], g["scale_e2"]])
    y = O.moe_dense(X, np.tile(np.array([[0, 1]], np.int32), (10, 1)), ex)
    assert np.allclose(y, X, atol=1e-15)


@pytest.mark.parametrize("k", [1, 2])
def test_identity_experts_restore_kx_exactly(k):
    """Eq. 4-5 algebra: identity experts give y = k x (to 1e-12 in fp64,
    where x - c rounds; exactly on the bf16 wire, below)."""
    d, E = 8, 4
    X = _clustered(200, d, 5, 0.1, 4)
    zeta = _zeta(200, k, E, 4)
    ident = {e: (np.vstack([np.eye(d), -np.eye(d)]), np.zeros(2 * d), np.hstack([np.eye(d), -np.eye(d)]), np.zeros(d))
             for e in range(E)}
    res = O.lsh_layer(X, zeta, _R(d, 2), ident, E, "f64")
    assert res.ratio < 1.0
    assert np.abs(res.y[0] - k * X).max() <= 1e-12


def test_identity_experts_bf16_wire():
    """Same with bf16 wire rounding of the centroids: x - c~ and c~ + (x - c~) are exact."""
    d, E = 8, 2
    X = O.round_to_dtype(_clustered(150, d, 4, 0.2, 5), "bf16")
    zeta = _zeta(150, 1, E, 5)
    ident = {e: (np.vstack([np.eye(d), -np.eye(d)]), np.zeros(2 * d), np.hstack([np.eye(d), -np.eye(d)]), np.zeros(d))
             for e in range(E)}
    res = O.lsh_layer(X, zeta, _R(d, 3), ident, E, "bf16")
    assert np.array_equal(res.y[0], X)


def test_affine_experts_error_closed_form():
    """E(x)=Wx+b: y - y_base = sum_s (I - W_s)(x - c~_s)  (S:L167 up to the sign convention)."""
    d, E, k = 6, 3, 2
    X = _clustered(120, d, 4, 0.3, 6)
    zeta = _zeta(120, k, E, 6)
    ex, Ws = _experts_affine(E, d, 6)
    res = O.lsh_layer(X, zeta, _R(d, 2), ex, E, "f64", round_expert_out=False)
    ybase = O.moe_dense(X, zeta, ex)
    b = res.buckets[0]
    pred = np.zeros_like(X)
    for s in range(k):
        for t in range(120):
            W, _ = Ws[int(zeta[t, s])]
            pred[t] += (np.eye(d) - W) @ (X[t] - res.Ct[0][b.bucket[t, s]])
    assert np.abs((res.y[0] - ybase) - pred).max() <= 1e-9


def test_singleton_buckets_recover_uncompressed():
    """Every token its own bucket => y = Eq. 2's dense output."""
    d, E = 16, 4
    X = np.random.default_rng(7).standard_normal((100, d))        # iid -> distinct keys at q=6
    zeta = _zeta(100, 2, E, 7)
    ex = _experts_random(E, d, 24, 7)
    res = O.lsh_layer(X, zeta, _R(d, 6), ex, E, "f64", round_expert_out=False)
    assert res.ratio == 1.0
    assert np.abs(res.y[0] - O.moe_dense(X, zeta, ex)).max() <= 1e-12


def test_zero_residuals_recover_uncompressed():
    """All tokens of a group identical => y = sum_s E(x) for any experts."""
    d, E = 8, 2
    x = np.random.default_rng(8).standard_normal(d)
    X = np.tile(x, (30, 1))
    zeta = np.tile(np.array([[0, 1]], np.int32), (30, 1))
    ex = _experts_random(E, d, 10, 8)
    res = O.lsh_layer(X, zeta, _R(d, 2), ex, E, "f64", round_expert_out=False)
    assert res.buckets[0].m == 2
    assert np.abs(res.y[0] - O.moe_dense(X, zeta, ex)).max() <= 1e-12


@pytest.mark.parametrize("w", [2, 4])
def test_w_invariance_and_conservation(w):
    """Clustering is per source rank and an expert's output does not depend on where it runs, so
    rank r's result in a w-rank run equals running rank r's tokens alone (w = 1)."""
    d, E, k, n = 8, 8, 2, 80
    R = _R(d, 3)
    ex = _experts_random(E, d, 12, 9)
    Xs = [_clustered(n, d, 6, 0.15, 100 + r) for r in range(w)]
    zs = [_zeta(n, k, E, 200 + r) for r in range(w)]
    res = O.lsh_layer_ranks(Xs, zs, R, ex, E, "f64", round_expert_out=False)
    sent = sum(b.m for b in res.buckets)
    assert sum(len(r) for r in res.recv) == sent
    for p in range(w):
        assert res.recv_rows[p].sum() == len(res.recv[p])
    for r in range(w):
        solo = O.lsh_layer(Xs[r], zs[r], R, ex, E, "f64", round_expert_out=False)
        assert np.array_equal(solo.y[0], res.y[r])


def test_roundtrip_identity_returns_centroids_exactly():
    d, E, w = 4, 4, 2
    Cs = [np.random.default_rng(r).standard_normal((m, d)) for r, m in enumerate([7, 5])]
    er = [np.array([2, 1, 3, 1]), np.array([0, 2, 2, 1])]
    recv, rr = O.dispatch_sim(Cs, er, E)
    assert [len(x) for x in recv] == [2 + 1 + 0 + 2, 3 + 1 + 2 + 1]
    back = O.combine_sim(recv, er, E)
    assert all(np.array_equal(a, b) for a, b in zip(back, Cs))
    # rank 1 owns experts 2, 3: rows ordered (expert 2: src0, src1; expert 3: src0, src1)
    assert np.array_equal(recv[1], np.vstack([Cs[0][3:6], Cs[1][2:4], Cs[0][6:7], Cs[1][4:5]]))


def test_byte_proportionality():
    """Dispatch rows = compression ratio x routed copies (AC8 S:L531)."""
    d, E = 8, 4
    X = _clustered(400, d, 8, 0.05, 11)
    zeta = _zeta(400, 1, E, 11)
    res = O.lsh_layer(X, zeta, _R(d, 4), _experts_random(E, d, 8, 11), E, "f64")
    assert len(res.recv[0]) == res.buckets[0].m and res.ratio == res.buckets[0].m / 400


def test_weighted_restore():
    d, E, k = 6, 3, 2
    X = _clustered(50, d, 3, 0.2, 12)
    zeta = _zeta(50, k, E, 12)
    g = np.random.default_rng(12).random((50, k))
    ex = _experts_random(E, d, 10, 12)
    res = O.lsh_layer(X, zeta, _R(d, 2), ex, E, "f64", g=g, round_expert_out=False)
    b = res.buckets[0]
    manual = sum(g[:, s:s + 1] * (res.ret[0][b.bucket[:, s]] + X - res.Ct[0][b.bucket[:, s]]) for s in range(k))
    assert np.abs(res.y[0] - manual).max() <= 1e-13
