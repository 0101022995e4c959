"""The whole N = 2 layer through the phase-2 exchange, against the oracle's multi-rank Alg. 1
(lsh_layer_ranks: hash, bucket, centroids, simulated all-to-all, expert FFN, reverse all-to-all,
restore): two processes (ranks) share the one GPU, map each other's windows with CUDA
IPC (handles over a gloo group) and run hash -> compress -> dispatch_p2p -> expert FFN -> combine_p2p
-> restore through the C ABI.  Codes and buckets must match bit-exactly (near-tie tokens replaced as
in smoke()), the restored outputs within the bf16 layer tolerance (tier 3)."""
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


def _inputs(cfg, world):
    """Every rank's tokens and gate (near-tie tokens replaced, as smoke() does), rotation, experts."""
    import oracle as O
    from lshmoe_inputs import make_experts, make_gate, make_tokens, rotation_seed
    R64 = O.to_stored(O.rotation(cfg.d, cfg.q, rotation_seed(0), cfg.dtype), cfg.dtype)
    Xs, zs = [], []
    for r in range(world):
        X = make_tokens(cfg, 0, r)
        _, margins = O.cp_hash(X.to(torch.float64).numpy(), R64)
        for t in np.nonzero(margins.min(axis=1) < 1e-5)[0]:
            X[t] = X[t - 1 if t > 0 else 1]
        zeta, _ = make_gate(cfg, 0, X)
        Xs.append(X)
        zs.append(zeta)
    return R64, Xs, zs, make_experts(cfg, 0)


def _worker(rank, world, port, q, fused=False):
    try:
        sys.path.insert(0, ROOT)
        import torch.distributed as dist
        import oracle as O
        import paper_2411_08446_b200 as L
        from lshmoe_inputs import LayerConfig, rotation_seed
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        cfg = LayerConfig("p2p-layer", 600, 128, 4, 2, 3, "bf16", 256, 24, 0.1)
        R64, Xs, zs, ex = _inputs(cfg, world)
        want = O.lsh_layer_ranks([X.to(torch.float64).numpy() for X in Xs], [z.numpy() for z in zs], R64,
                                 {e: tuple(t.to(torch.float64).numpy() for t in ex[e]) for e in range(cfg.E)},
                                 cfg.E, cfg.dtype)
        epr = cfg.E // world
        W = [torch.stack([ex[e][i] for e in range(rank * epr, (rank + 1) * epr)]).cuda() for i in range(4)]
        X, zeta = Xs[rank].cuda(), zs[rank].cuda()
        R = L.rotation(cfg.d, cfg.q, rotation_seed(0), X.dtype).cuda()
        nk = cfg.n * cfg.k
        comm = L.Comm(world, rank, None).p2p_init(world * nk, nk, cfg.d, X.dtype, cfg.E, group=dist.group.WORLD)
        for it in range(2):                                   # twice: the second call reuses the windows
            codes = L.hash(X, R)
            if fused:                                         # the centroid kernel stores to the owners
                out = L.compress_p2p(comm, X, codes, zeta, cfg.E)
            else:
                out = L.compress(X, codes, zeta, cfg.E)
                L.dispatch_p2p(comm, out.centroids, out.expert_rows)
            recv, ret, rr = comm.p2p_buffers()
            eo = L.expert_ffn(recv, rr, *W)
            L.combine_p2p(comm, eo)
            y = L.restore(X, out.centroids, ret, out.bucket)
            torch.cuda.synchronize()
            comm.p2p_check()
            L.check_device_error()
            assert np.array_equal(codes.cpu().numpy(), want.codes[rank]), "codes"
            assert np.array_equal(out.bucket.cpu().numpy(), want.buckets[rank].bucket), "buckets"
            assert np.array_equal(rr.cpu().numpy(), want.recv_rows[rank]), "recv_rows"
            yg = y.to(torch.float64).cpu().numpy()
            err = float((np.abs(yg - want.y[rank]).max(1) / np.abs(want.y[rank]).max(1)).max())
            assert err <= 2e-2, f"rank {rank} iteration {it}: restored output error {err:.3e}"
            dist.barrier()
        comm.close()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as exc:  # noqa: BLE001
        q.put((rank, repr(exc)))


@pytest.mark.parametrize("fused", [False, True], ids=["dispatch_p2p", "compress_p2p"])
def test_layer_two_ranks_p2p_matches_oracle(fused):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, fused)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=280) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
