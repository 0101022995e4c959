"""Pins of the oracle's backward (NEXT-1, reading R27: buckets constant, straight-through rounding)
against what the mathematics fixes: torch.autograd (fp64) of the forward written independently in
torch, central finite differences of the oracle's forward, and two closed forms (identity experts;
singleton buckets = the dense Eq. 2 MoE backward)."""
import numpy as np
import pytest
import torch

import oracle as O


def _setup(seed, n=60, d=8, E=3, k=2, q=2, d_ffn=12, dup=True):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, d))
    if dup:                                   # plenty of shared buckets
        X[n // 2:] = X[: n - n // 2] * (1 + 1e-3 * rng.standard_normal((n - n // 2, 1)))
    R = np.stack([np.linalg.qr(rng.standard_normal((d, d)))[0] for _ in range(q)])
    codes, _ = O.cp_hash(X, R)
    zeta = np.stack([np.sort(rng.choice(E, size=k, replace=False)) for _ in range(n)]).astype(np.int32)
    g = rng.random((n, k)) + 0.1
    experts = {e: (rng.standard_normal((d_ffn, d)) / np.sqrt(d), 0.3 * rng.standard_normal(d_ffn),
                   rng.standard_normal((d, d_ffn)) / np.sqrt(d_ffn), 0.1 * rng.standard_normal(d)) for e in range(E)}
    b = O.bucketize(codes, zeta, E)
    dY = rng.standard_normal((n, d))
    return X, zeta, g, experts, b, dY


def _forward_np(X, g, experts, b, k):
    """The oracle's own forward with identity rounding (fp64 wire)."""
    C = O.centroids(X, b, k)
    ret = np.zeros_like(C)
    off = 0
    for e, me in enumerate(b.expert_rows):
        if me:
            ret[off:off + me] = O.expert_ffn(C[off:off + me], *experts[e])
        off += me
    return C, ret, O.restore(X, C, ret, b.bucket, g)


def _forward_torch(Xt, gt, experts, b, k):
    """Independent torch forward: scatter-add centroids, per-expert FFN, Eq. 4-5 + Eq. 2."""
    n, d = Xt.shape
    copies = torch.arange(n * k)
    rows = torch.from_numpy(b.bucket.reshape(-1).astype(np.int64))
    cnt = torch.zeros(b.m, dtype=torch.float64).index_add_(0, rows, torch.ones(n * k, dtype=torch.float64))
    C = torch.zeros(b.m, d, dtype=torch.float64).index_add_(0, rows, Xt[copies // k]) / cnt[:, None]
    C.retain_grad()
    outs, off = [], 0
    for e, me in enumerate(b.expert_rows):
        if me:
            W1, b1, W2, b2 = (torch.from_numpy(a) for a in experts[e])
            outs.append(torch.relu(C[off:off + me] @ W1.T + b1) @ W2.T + b2)
        off += me
    Ov = torch.cat(outs)
    Ov.retain_grad()
    Y = torch.zeros_like(Xt)
    for s in range(k):
        bs = torch.from_numpy(b.bucket[:, s].astype(np.int64))
        Y = Y + gt[:, s:s + 1] * (Ov[bs] + Xt - C[bs])
    return C, Ov, Y


@pytest.mark.parametrize("seed,with_g", [(0, True), (1, False), (2, True)])
def test_backward_matches_autograd(seed, with_g):
    X, zeta, g, experts, b, dY = _setup(seed)
    k = zeta.shape[1]
    g = g if with_g else None
    Xt = torch.tensor(X, requires_grad=True)
    gt = torch.tensor(g if g is not None else np.ones_like(zeta, dtype=np.float64), requires_grad=True)
    C, Ov, Y = _forward_torch(Xt, gt, experts, b, k)
    (Y * torch.from_numpy(dY)).sum().backward()
    Cn, ret, _ = _forward_np(X, g, experts, b, k)
    G, H, dX, dg = O.lsh_layer_backward(X, zeta, b, Cn, ret, experts, dY, g)
    assert b.m < X.shape[0] * k                               # some buckets are shared
    np.testing.assert_allclose(G, Ov.grad.numpy(), rtol=1e-11, atol=1e-11)          # dL/do
    np.testing.assert_allclose(H - G, C.grad.numpy(), rtol=1e-10, atol=1e-10)       # dL/dc
    np.testing.assert_allclose(dX, Xt.grad.numpy(), rtol=1e-10, atol=1e-10)
    if with_g:
        np.testing.assert_allclose(dg, gt.grad.numpy(), rtol=1e-10, atol=1e-10)


def test_backward_finite_differences():
    X, zeta, g, experts, b, dY = _setup(3, n=30)
    k = zeta.shape[1]
    Cn, ret, _ = _forward_np(X, g, experts, b, k)
    _, _, dX, dg = O.lsh_layer_backward(X, zeta, b, Cn, ret, experts, dY, g)
    rng = np.random.default_rng(9)
    h = 1e-6
    for _ in range(12):
        t, i = rng.integers(X.shape[0]), rng.integers(X.shape[1])
        Xp, Xm = X.copy(), X.copy()
        Xp[t, i] += h
        Xm[t, i] -= h
        fd = ((_forward_np(Xp, g, experts, b, k)[2] - _forward_np(Xm, g, experts, b, k)[2]) * dY).sum() / (2 * h)
        assert abs(fd - dX[t, i]) <= 1e-6 * max(1.0, abs(fd))
    for _ in range(6):
        t, s = rng.integers(X.shape[0]), rng.integers(k)
        gp, gm = g.copy(), g.copy()
        gp[t, s] += h
        gm[t, s] -= h
        fd = ((_forward_np(X, gp, experts, b, k)[2] - _forward_np(X, gm, experts, b, k)[2]) * dY).sum() / (2 * h)
        assert abs(fd - dg[t, s]) <= 1e-6 * max(1.0, abs(fd))


def test_backward_identity_experts_closed_form():
    """E(c) = c: H = G, so dX_t = sum_s g_ts dY_t exactly (the residual path cancels the mean)."""
    X, zeta, g, experts, b, dY = _setup(4)
    k = zeta.shape[1]
    d = X.shape[1]
    C = O.centroids(X, b, k)
    G = O.grad_compress(dY, b, k, g)
    dX, _ = O.grad_restore(dY, X, C, C, G, G.copy(), b, g)
    np.testing.assert_allclose(dX, (g.sum(axis=1)[:, None]) * dY, rtol=0, atol=1e-13)
    assert d == 8


def test_backward_singletons_equal_dense_moe_backward():
    """Every copy its own bucket (iid tokens, many hashes): dX equals the dense Eq. 2 MoE's
    dX_t = sum_s g_ts J_E(x_t)^T dY_t (autograd of the independent dense form)."""
    X, zeta, g, experts, b, dY = _setup(5, dup=False, q=6)
    k = zeta.shape[1]
    assert b.m == X.shape[0] * k
    Cn, ret, _ = _forward_np(X, g, experts, b, k)
    _, _, dX, _ = O.lsh_layer_backward(X, zeta, b, Cn, ret, experts, dY, g)
    Xt = torch.tensor(X, requires_grad=True)
    Y = torch.zeros_like(Xt)
    for s in range(k):
        for e in range(len(experts)):
            W1, b1, W2, b2 = (torch.from_numpy(a) for a in experts[e])
            mask = torch.from_numpy((zeta[:, s] == e).astype(np.float64))[:, None]
            Y = Y + mask * torch.from_numpy(g[:, s:s + 1]) * (torch.relu(Xt @ W1.T + b1) @ W2.T + b2)
    (Y * torch.from_numpy(dY)).sum().backward()
    np.testing.assert_allclose(dX, Xt.grad.numpy(), rtol=1e-10, atol=1e-10)


def test_backward_multi_rank_exchange_is_w_invariant():
    """NEXT-1 across ranks: G travels to the expert owners with dispatch_sim, H = J_E^T G is
    computed there, combine_sim brings H back; each rank's dX equals its single-rank backward
    (clustering is per source rank, so the exchanges only move rows) — for w = 2 and 4."""
    rng = np.random.default_rng(11)
    E, k, d, d_ffn, q = 4, 2, 8, 12, 2
    experts = {e: (rng.standard_normal((d_ffn, d)) / np.sqrt(d), 0.3 * rng.standard_normal(d_ffn),
                   rng.standard_normal((d, d_ffn)) / np.sqrt(d_ffn), 0.1 * rng.standard_normal(d)) for e in range(E)}
    R = np.stack([np.linalg.qr(rng.standard_normal((d, d)))[0] for _ in range(q)])
    for w in (2, 4):
        per = []
        for r in range(w):
            X = rng.standard_normal((40, d))
            X[20:] = X[:20] * (1 + 1e-3 * rng.standard_normal((20, 1)))
            zeta = np.stack([np.sort(rng.choice(E, size=k, replace=False)) for _ in range(40)]).astype(np.int32)
            g = rng.random((40, k)) + 0.1
            b = O.bucketize(O.cp_hash(X, R)[0], zeta, E)
            C = O.centroids(X, b, k)
            dY = rng.standard_normal((40, d))
            per.append((X, zeta, g, b, C, dY))
        # forward outputs o per rank via the simulated exchange, then the backward chain
        recv, rr = O.dispatch_sim([p[4] for p in per], [p[3].expert_rows for p in per], E)
        epr = E // w
        outs, Hs = [], []
        G_by_rank = [O.grad_compress(p[5], p[3], k, p[2]) for p in per]
        Grecv, _ = O.dispatch_sim(G_by_rank, [p[3].expert_rows for p in per], E)
        for p_ in range(w):
            o = np.zeros_like(recv[p_])
            h = np.zeros_like(recv[p_])
            pos = 0
            for el in range(epr):
                e = p_ * epr + el
                n_e = int(rr[p_][el].sum())
                W1, b1, W2, b2 = experts[e]
                o[pos:pos + n_e] = O.expert_ffn(recv[p_][pos:pos + n_e], W1, b1, W2, b2)
                h[pos:pos + n_e] = O.expert_ffn_vjp(recv[p_][pos:pos + n_e], W1, b1, W2, Grecv[p_][pos:pos + n_e])
                pos += n_e
            outs.append(o)
            Hs.append(h)
        ret = O.combine_sim(outs, [p[3].expert_rows for p in per], E)
        Hback = O.combine_sim(Hs, [p[3].expert_rows for p in per], E)
        for r, (X, zeta, g, b, C, dY) in enumerate(per):
            dX, dg = O.grad_restore(dY, X, C, ret[r], G_by_rank[r], Hback[r], b, g)
            _, _, dX1, dg1 = O.lsh_layer_backward(X, zeta, b, C, ret[r], experts, dY, g)
            np.testing.assert_allclose(dX, dX1, rtol=0, atol=1e-12)
            np.testing.assert_allclose(dg, dg1, rtol=0, atol=1e-12)
