"""Phase-2 exchange: device-initiated dispatch / combine over peer memory, Alg. 1 L14
and L16, checked byte-exactly against the oracle's dispatch_sim / combine_sim
(reading R24 layouts).  A local group of virtual ranks shares the one GPU: each rank's kernels run
on its own stream, so every rank's flags and mailboxes go through the same code as on NVLink."""
import numpy as np
import pytest
import torch

import oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(300)]


def _counts(rng, world, E, m_max, zero_rank=None):
    out = []
    for r in range(world):
        if r == zero_rank:
            out.append(np.zeros(E, dtype=np.int32))
            continue
        c = rng.integers(0, m_max // E * 2 + 1, size=E).astype(np.int32)
        c[rng.random(E) < 0.2] = 0                       # empty experts
        out.append(c)
    return out


def _run_group(world, E, d, dtype, rounds, grid, seed):
    import paper_2411_08446_b200 as L
    rng = np.random.default_rng(seed)
    m_max = 3000                                          # counts below sum to < 2 m_max per rank
    cap = 2 * world * m_max
    comms = L.Comm.local_group(world, cap, 2 * m_max, d, dtype, E)
    streams = [torch.cuda.Stream() for _ in range(world)]
    try:
        for it in range(rounds):
            counts = _counts(rng, world, E, m_max, zero_rank=(1 if it == 1 and world > 1 else None))
            C = [rng.standard_normal((int(c.sum()), d)) for c in counts]
            Cd = [torch.from_numpy(c).to(dtype).cuda() for c in C]
            er = [torch.from_numpy(c).cuda() for c in counts]
            want_recv, want_rr = O.dispatch_sim([c.to(torch.float64).cpu().numpy() for c in Cd], counts, E)
            cur = torch.cuda.current_stream()
            for s in streams:
                s.wait_stream(cur)
            for r in range(world):
                with torch.cuda.stream(streams[r]):
                    L.dispatch_p2p(comms[r], Cd[r], er[r], grid=grid, stream=streams[r])
            for s in streams:
                cur.wait_stream(s)
            torch.cuda.synchronize()
            outs = []
            for r in range(world):
                recv, _, rr = comms[r].p2p_buffers()
                n = int(want_rr[r].sum())
                assert np.array_equal(rr.cpu().numpy(), want_rr[r]), f"round {it} rank {r}: recv_rows"
                got = recv[:n].to(torch.float64).cpu().numpy()
                assert np.array_equal(got, want_recv[r]), f"round {it} rank {r}: recv rows differ"
                outs.append((recv[:n].to(torch.float32) * 3 - 1).to(dtype))   # stand-in expert output
            want_ret = O.combine_sim([o.to(torch.float64).cpu().numpy() for o in outs], counts, E)
            for s in streams:
                s.wait_stream(cur)
            for r in range(world):
                with torch.cuda.stream(streams[r]):
                    L.combine_p2p(comms[r], outs[r], grid=grid, stream=streams[r])
            for s in streams:
                cur.wait_stream(s)
            torch.cuda.synchronize()
            for r in range(world):
                comms[r].p2p_check()
                _, ret, _ = comms[r].p2p_buffers()
                m = int(counts[r].sum())
                assert np.array_equal(ret[:m].to(torch.float64).cpu().numpy(), want_ret[r]), \
                    f"round {it} rank {r}: returned rows differ"
    finally:
        torch.cuda.synchronize()
        for c in comms:
            c.close()


@pytest.mark.parametrize("world,E,d,dtype,grid", [
    (1, 8, 128, torch.bfloat16, 0),
    (2, 8, 128, torch.bfloat16, 16),
    (2, 16, 64, torch.float32, 3),
    (4, 32, 256, torch.bfloat16, 32),
    (8, 64, 512, torch.bfloat16, 16),
    (8, 256, 8, torch.bfloat16, 8),          # 16-byte rows, 256 experts: the mailbox / segment limits
])
def test_p2p_exchange_matches_oracle(world, E, d, dtype, grid):
    _run_group(world, E, d, dtype, rounds=3, grid=grid, seed=world * 100 + E)


def test_p2p_overflow_is_flagged():
    """Rows past the owner's receive capacity are dropped (no out-of-window store) and reported."""
    import paper_2411_08446_b200 as L
    E, d = 4, 64
    comms = L.Comm.local_group(2, 100, 100, d, torch.bfloat16, E)
    streams = [torch.cuda.Stream() for _ in range(2)]
    try:
        er = [torch.tensor([60, 60, 0, 0], dtype=torch.int32, device="cuda"),   # 120 rows for rank 0's experts
              torch.tensor([0, 0, 5, 5], dtype=torch.int32, device="cuda")]
        C = [torch.ones((int(e.sum()), d), dtype=torch.bfloat16, device="cuda") for e in er]
        torch.cuda.synchronize()
        for r in range(2):
            with torch.cuda.stream(streams[r]):
                L.dispatch_p2p(comms[r], C[r], er[r], grid=4, stream=streams[r])
        torch.cuda.synchronize()
        with pytest.raises(L.LshmoeError):
            comms[0].p2p_check()
        comms[1].p2p_check()
        comms[0].p2p_check()                                 # cleared by the first read
    finally:
        torch.cuda.synchronize()
        for c in comms:
            c.close()


def test_p2p_matches_phase1_world1():
    """At world 1 phase 2 and phase 1 (lshmoe_dispatch / lshmoe_combine) produce the same bytes."""
    import paper_2411_08446_b200 as L
    E, d = 16, 256
    rng = np.random.default_rng(7)
    counts = rng.integers(0, 200, size=E).astype(np.int32)
    C = torch.from_numpy(rng.standard_normal((int(counts.sum()), d))).to(torch.bfloat16).cuda()
    er = torch.from_numpy(counts).cuda()
    comm = L.Comm(1, 0).p2p_init(C.shape[0], C.shape[0], d, torch.bfloat16, E)
    try:
        L.dispatch_p2p(comm, C, er)
        recv1 = torch.empty_like(C)
        rr1 = torch.empty((E, 1), dtype=torch.int32, device="cuda")
        L.dispatch(None, C, er, E, recv1, rr1)
        torch.cuda.synchronize()
        recv, ret, rr = comm.p2p_buffers()
        assert torch.equal(recv[:C.shape[0]], recv1) and torch.equal(rr, rr1)
        L.combine_p2p(comm, recv1 * 2)
        torch.cuda.synchronize()
        assert torch.equal(ret[:C.shape[0]], recv1 * 2)
    finally:
        comm.close()


def test_p2p_graph_replay():
    """The epoch lives on the device, so a captured dispatch + combine replays correctly with new
    counts and rows copied into the captured buffers before every replay."""
    import paper_2411_08446_b200 as L
    world, E, d, m_max = 2, 8, 128, 2000
    rng = np.random.default_rng(11)
    comms = L.Comm.local_group(world, 2 * world * m_max, m_max, d, torch.bfloat16, E)
    streams = [torch.cuda.Stream() for _ in range(world)]
    Cbuf = [torch.zeros((m_max, d), dtype=torch.bfloat16, device="cuda") for _ in range(world)]
    erbuf = [torch.zeros(E, dtype=torch.int32, device="cuda") for _ in range(world)]
    obuf = [torch.zeros((2 * world * m_max, d), dtype=torch.bfloat16, device="cuda") for _ in range(world)]
    graphs = [torch.cuda.CUDAGraph() for _ in range(world)]
    try:
        torch.cuda.synchronize()
        for r in range(world):
            with torch.cuda.graph(graphs[r], stream=streams[r]):
                L.dispatch_p2p(comms[r], Cbuf[r], erbuf[r], grid=8, stream=streams[r])
                recv, _, _ = comms[r].p2p_buffers()
                torch.mul(recv, 2, out=obuf[r])
                L.combine_p2p(comms[r], obuf[r], grid=8, stream=streams[r])
        torch.cuda.synchronize()
        for it in range(4):
            counts = [rng.integers(0, 2 * m_max // E // 2 + 1, size=E).astype(np.int32) for _ in range(world)]
            C = [torch.from_numpy(rng.standard_normal((int(c.sum()), d))).to(torch.bfloat16) for c in counts]
            for r in range(world):
                erbuf[r].copy_(torch.from_numpy(counts[r]))
                Cbuf[r][:C[r].shape[0]].copy_(C[r])
            torch.cuda.synchronize()
            for r in range(world):
                with torch.cuda.stream(streams[r]):
                    graphs[r].replay()
            torch.cuda.synchronize()
            want_recv, want_rr = O.dispatch_sim([c.to(torch.float64).numpy() for c in C], counts, E)
            want_ret = O.combine_sim([w * 2 for w in want_recv], counts, E)
            for r in range(world):
                recv, ret, rr = comms[r].p2p_buffers()
                n = int(want_rr[r].sum())
                assert np.array_equal(rr.cpu().numpy(), want_rr[r]), f"replay {it} rank {r}: recv_rows"
                assert np.array_equal(recv[:n].to(torch.float64).cpu().numpy(), want_recv[r]), f"replay {it}"
                m = int(counts[r].sum())
                assert np.array_equal(ret[:m].to(torch.float64).cpu().numpy(), want_ret[r]), f"replay {it}"
    finally:
        torch.cuda.synchronize()
        for c in comms:
            c.close()


def test_p2p_peer_timeout_is_flagged_not_trapped():
    """A peer that never joins (rank 1 of a local group skips the call): rank 0's dispatch gives up
    after the comm's spin limit, flags error bit 2 and returns — no trap, so the CUDA context
    survives and the next calls on a fresh group work (a straggler must not kill the job)."""
    import paper_2411_08446_b200 as L
    E, d = 4, 64
    comms = L.Comm.local_group(2, 100, 100, d, torch.bfloat16, E)
    try:
        comms[0].p2p_set_timeout(0.05)
        er = torch.tensor([3, 3, 3, 3], dtype=torch.int32, device="cuda")
        C = torch.ones((12, d), dtype=torch.bfloat16, device="cuda")
        L.dispatch_p2p(comms[0], C, er)
        torch.cuda.synchronize()                             # completes (no hang, no sticky error)
        with pytest.raises(L.LshmoeError, match="spin limit"):
            comms[0].p2p_check()
        comms[0].p2p_check()                                  # the flag was read and cleared
    finally:
        torch.cuda.synchronize()
        for c in comms:
            c.close()
    _run_group(2, 8, 128, torch.bfloat16, rounds=1, grid=8, seed=5)   # the context is healthy


def test_compress_p2p_refuses_local_group():
    """The fused compress + dispatch needs every rank on its own GPU: a local group at world > 1 is
    refused before any launch, and the comm is not marked as dispatched."""
    import paper_2411_08446_b200 as L
    E, d, n = 4, 64, 256
    comms = L.Comm.local_group(2, 2 * n, n, d, torch.bfloat16, E)
    try:
        x = torch.ones((n, d), dtype=torch.bfloat16, device="cuda")
        codes = torch.ones((n, 2), dtype=torch.int16, device="cuda")
        zeta = (torch.arange(n, dtype=torch.int32, device="cuda") % E).view(n, 1)
        with pytest.raises(L.LshmoeError, match="EUNSUPPORTED"):
            L.compress_p2p(comms[0], x, codes, zeta, E)
        with pytest.raises(L.LshmoeError, match="no matching dispatch"):
            L.combine_p2p(comms[0], x)
    finally:
        torch.cuda.synchronize()
        for c in comms:
            c.close()


def test_duplicate_expert_in_row_is_flagged():
    """The k experts of a token must be distinct: a repeated id sets the device error word
    and lshmoe_check_device_error returns LSHMOE_EDEVICE."""
    import paper_2411_08446_b200 as L
    n, d, E = 300, 64, 4
    x = torch.randn((n, d), device="cuda").to(torch.bfloat16)
    codes = torch.ones((n, 1), dtype=torch.int16, device="cuda")
    zeta = torch.stack([torch.arange(n) % E, (torch.arange(n) + 1) % E], 1).to(torch.int32)
    zeta[17, 1] = zeta[17, 0]
    L.compress(x, codes, zeta.cuda(), E)
    with pytest.raises(L.LshmoeError, match="twice"):
        L.check_device_error()
    L.check_device_error()                                    # cleared
