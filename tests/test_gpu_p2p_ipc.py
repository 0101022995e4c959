"""Phase-2 exchange through real CUDA IPC: two processes (ranks) on the one GPU, each mapping the other's
window with cudaIpcOpenMemHandle (the handles travel over a gloo process group), checked against the
oracle's dispatch_sim / combine_sim (Alg. 1 L14 / L16, P:L533 / P:L535, reading R24).  Without MPS the
two contexts time-slice the device, so this exercises the protocol's cross-context visibility and
progress, not its speed."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(300)]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, E, d, q):
    try:
        sys.path.insert(0, ROOT)
        import torch.distributed as dist
        import oracle as O
        import paper_2411_08446_b200 as L
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        rng = np.random.default_rng(5)                      # every rank draws every rank's inputs
        comm = L.Comm(world, rank, None).p2p_init(4000 * world, 4000, d, torch.bfloat16, E,
                                                  group=dist.group.WORLD)
        for it in range(3):
            counts = [rng.integers(0, 2 * 1500 // E + 1, size=E).astype(np.int32) for _ in range(world)]
            C = [rng.standard_normal((int(c.sum()), d)) for c in counts]
            Cb = [torch.from_numpy(c).to(torch.bfloat16) for c in C]
            want_recv, want_rr = O.dispatch_sim([c.to(torch.float64).numpy() for c in Cb], counts, E)
            dist.barrier()
            L.dispatch_p2p(comm, Cb[rank].cuda(), torch.from_numpy(counts[rank]).cuda(), grid=8)
            torch.cuda.synchronize()
            comm.p2p_check()
            recv, ret, rr = comm.p2p_buffers()
            n = int(want_rr[rank].sum())
            assert np.array_equal(rr.cpu().numpy(), want_rr[rank]), "recv_rows"
            assert np.array_equal(recv[:n].to(torch.float64).cpu().numpy(), want_recv[rank]), "recv rows"
            outs = [torch.from_numpy(w) * 2 + 1 for w in want_recv]            # stand-in expert output
            outs = [o.to(torch.bfloat16) for o in outs]
            want_ret = O.combine_sim([o.to(torch.float64).numpy() for o in outs], counts, E)
            L.combine_p2p(comm, outs[rank].cuda(), grid=8)
            torch.cuda.synchronize()
            comm.p2p_check()
            m = int(counts[rank].sum())
            assert np.array_equal(ret[:m].to(torch.float64).cpu().numpy(), want_ret[rank]), "returned rows"
        dist.barrier()
        comm.close()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as exc:  # noqa: BLE001
        q.put((rank, repr(exc)))


def test_p2p_ipc_two_processes():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, 8, 256, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
