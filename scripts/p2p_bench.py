"""Phase-2 exchange timing on one GPU: dispatch_p2p / combine_p2p at world 1 (a window copy) and in
local groups of w virtual ranks (concurrent streams), CUDA-graph replays, C2-shaped rows."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_08446_b200 as L  # noqa: E402


FLUSH = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device="cuda")


def timed(fn, reps=20, flush=True):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    fn(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn(s)
    ts = []
    for _ in range(reps):
        if flush:
            with torch.cuda.stream(s):
                FLUSH.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):              # replay on the stream the events are recorded on
            a.record(s)
            g.replay()
            b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return statistics.median(ts)


def world1(m, d, E, grid):
    comm = L.Comm(1, 0).p2p_init(m, m, d, torch.bfloat16, E)
    er = torch.full((E,), m // E, dtype=torch.int32, device="cuda")
    C = torch.randn((m // E * E, d), device="cuda").to(torch.bfloat16)
    recv, ret, rr = comm.p2p_buffers()
    t_d = timed(lambda s: L.dispatch_p2p(comm, C, er, grid=grid, stream=s))
    t_c = timed(lambda s: (L.dispatch_p2p(comm, C, er, grid=grid, stream=s),
                           L.combine_p2p(comm, recv, grid=grid, stream=s)))
    t_copy = timed(lambda s: recv[:C.shape[0]].copy_(C))
    eag = []
    for _ in range(10):
        FLUSH.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        L.dispatch_p2p(comm, C, er, grid=grid)
        b.record()
        torch.cuda.synchronize()
        eag.append(a.elapsed_time(b) * 1e3)
    print(f"   eager dispatch (flushed): median {statistics.median(eag):.1f} us, all {[round(x, 1) for x in eag]}")
    if int(os.environ.get("LSHMOE_P2P_EXP", "0")) & 16:
        import ctypes
        buf = (ctypes.c_ulonglong * (4 * grid))()
        L._lib.lshmoe_debug_p2p_stamps(buf, grid)
        st = [[buf[4 * i + j] for j in range(4)] for i in range(grid)]
        t0 = min(x[0] for x in st)
        rel = lambda j, f: (f(x[j] for x in st) - t0) / 1e3   # noqa: E731
        print(f"   stamps (us from first CTA start): start max {rel(0, max):.1f}; counts seen min {rel(1, min):.1f} "
              f"max {rel(1, max):.1f}; copies done max {rel(2, max):.1f}; end max {rel(3, max):.1f}")
    eag = []
    for _ in range(10):
        FLUSH.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        recv[:C.shape[0]].copy_(C)
        b.record()
        torch.cuda.synchronize()
        eag.append(a.elapsed_time(b) * 1e3)
    print(f"   eager torch copy (flushed): median {statistics.median(eag):.1f} us")
    nbytes = 2 * C.numel() * 2
    print(f"world1 m={m} d={d} E={E} grid={grid}: dispatch {t_d:.1f} us ({nbytes / t_d / 1e3:.0f} GB/s r+w), "
          f"dispatch+combine {t_c:.1f} us; torch copy {t_copy:.1f} us", flush=True)
    torch.cuda.synchronize()
    comm.close()


if __name__ == "__main__":
    os.environ["LSHMOE_EXPERIMENTS"] = "1"
    for exp in [int(a) for a in sys.argv[1:]] or [0]:
        os.environ["LSHMOE_P2P_EXP"] = str(exp)
        print(f"-- LSHMOE_P2P_EXP={exp} (L2 flushed before each replay)")
        for grid in (64, 296):
            world1(3128, 768, 16, grid)
