"""Phase-1 exchange (lshmoe_dispatch / lshmoe_combine over NCCL, Alg. 1 L14 / L16: P:L533)
executed on one GPU: a one-rank NCCL communicator (lshmoe_comm_init at world 1 WITH an id) takes the
phase-1 code path — the count all-gather, the host plan (lshmoe_exchange_plan), the self segments
and the grouped send/recv — instead of the aliased local exchange.  Checked byte-exactly against the
oracle's dispatch_sim / combine_sim (reading R24), then a whole bf16 layer through it against the
default (aliased) world-1 exchange.  NCCL refuses two ranks on one GPU, so the cross-rank sends are
covered by the gloo plan test and the phase-2 tests instead."""
import numpy as np
import pytest
import torch

import oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(300)]


@pytest.fixture(scope="module")
def L():
    import paper_2411_08446_b200 as L
    return L


@pytest.fixture(scope="module")
def comm(L):
    return L.Comm(1, 0, L.Comm.unique_id())


@pytest.mark.parametrize("E,d,dtype", [(16, 768, torch.bfloat16), (4, 64, torch.float32), (32, 1024, torch.bfloat16)])
def test_phase1_dispatch_combine_one_rank(L, comm, E, d, dtype):
    rng = np.random.default_rng(E + d)
    for it in range(3):
        counts = rng.integers(0, 300, size=E).astype(np.int32)
        counts[rng.random(E) < 0.25] = 0                  # empty experts
        if it == 2:
            counts[:] = 0                                 # nothing to send at all
        m = int(counts.sum())
        C = rng.standard_normal((m + 1, d))                 # one spare row: a non-null pointer at m = 0
        Cfull = torch.from_numpy(C).to(dtype).cuda()
        Cd = Cfull[:m]
        er = torch.from_numpy(counts).cuda()
        want_recv, want_rr = O.dispatch_sim([Cd.to(torch.float64).cpu().numpy()], [counts], E)
        recv = torch.full((m + 7, d), float("nan"), dtype=dtype, device="cuda")
        rr = torch.full((E, 1), -1, dtype=torch.int32, device="cuda")
        tot = L.dispatch(comm, Cfull, er, E, recv, rr)   # rows past the counts are never read
        torch.cuda.synchronize()
        assert tot == m
        assert np.array_equal(rr.cpu().numpy(), want_rr[0])
        assert np.array_equal(recv[:m].to(torch.float64).cpu().numpy(), want_recv[0])
        assert np.array_equal(comm.last_counts(E).numpy(), counts[None, :])
        outf = (recv[:m + 1].to(torch.float32) * 3 - 1).to(dtype)   # stand-in expert output (+ a spare row)
        out = outf[:m]
        want_ret = O.combine_sim([out.to(torch.float64).cpu().numpy()], [counts], E)
        ret = torch.full((m + 3, d), float("nan"), dtype=dtype, device="cuda")
        L.combine(comm, outf, er, E, ret)
        torch.cuda.synchronize()
        assert np.array_equal(ret[:m].to(torch.float64).cpu().numpy(), want_ret[0])


def test_phase1_layer_matches_aliased_exchange(L, comm):
    """A whole C2-shaped bf16 layer (hash -> compress -> dispatch -> FFN -> combine -> restore) through
    the one-rank NCCL exchange is bit-identical to the aliased world-1 exchange."""
    from lshmoe_inputs import CONFIGS, make_experts, make_rank_inputs, rotation_seed
    cfg = CONFIGS["C2"]
    X, zeta, _ = make_rank_inputs(cfg, 0, 0)
    X, zeta = X.cuda(), zeta.cuda()
    R = L.rotation(cfg.d, cfg.q, rotation_seed(0), X.dtype).cuda()
    ex = make_experts(cfg, 0)
    W = [torch.stack([ex[e][i] for e in range(cfg.E)]).cuda() for i in range(4)]
    comp = L.compress(X, L.hash(X, R), zeta, cfg.E)
    m = int(comp.num_rows.item())
    ys = []
    for c in (None, comm):
        recv = torch.empty_like(comp.centroids)
        rr = torch.empty((cfg.E, 1), dtype=torch.int32, device="cuda")
        L.dispatch(c, comp.centroids, comp.expert_rows, cfg.E, recv, rr)
        out = L.expert_ffn(recv, rr, *W)
        ret = torch.empty_like(comp.centroids)
        L.combine(c, out, comp.expert_rows, cfg.E, ret)
        ys.append(L.restore(X, comp.centroids, ret, comp.bucket))
    torch.cuda.synchronize()
    assert m > 0 and torch.equal(ys[0], ys[1])
