"""World-size-2 CPU test (gloo) of the multi-rank exchange: each rank plans dispatch/combine with the
library's host plan (lshmoe_exchange_plan, the same code lshmoe_dispatch/combine run before their NCCL
calls), moves the oracle's centroids with gloo point-to-point in that layout, and the result must
equal the oracle's simulated all-to-all (Alg. 1 L14/L16) and, after restore, the
single-rank result (w-invariance).  No GPU is needed."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O

W, E, K, D, N, Q = 2, 4, 2, 16, 120, 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_inputs(r):
    rng = np.random.default_rng(100 + r)
    U = np.random.default_rng(7).standard_normal((6, D))
    X = U[rng.integers(0, 6, N)] + 0.05 * rng.standard_normal((N, D))
    zeta = np.sort(np.stack([rng.choice(E, K, replace=False) for _ in range(N)]), axis=1).astype(np.int32)
    return X, zeta


def _experts():
    rng = np.random.default_rng(3)
    return {e: (rng.standard_normal((24, D)) / 4, 0.1 * rng.standard_normal(24),
                rng.standard_normal((D, 24)) / 5, 0.1 * rng.standard_normal(D)) for e in range(E)}


def _worker(rank, port, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=W)
    import paper_2411_08446_b200 as L
    R = np.stack([O.rotation_fp64(D, j, 11) for j in range(Q)])
    ex = _experts()
    # this rank's compress (oracle stands in for the GPU stage on a CPU-only box)
    X, zeta = _rank_inputs(rank)
    codes, _ = O.cp_hash(X, R)
    b = O.bucketize(codes, zeta, E)
    C = O.centroids(X, b, K)
    counts_me = torch.from_numpy(b.expert_rows.astype(np.int32))
    gathered = [torch.empty_like(counts_me) for _ in range(W)]
    dist.all_gather(gathered, counts_me)
    counts = torch.stack(gathered)
    send_off, recv_off, recv_rows = L.exchange_plan(W, rank, counts)
    epr = E // W
    assert int(send_off[-1]) == b.m
    # dispatch: to peer p the rows of p's experts (contiguous in the expert-major layout)
    recv = np.zeros((int(recv_off[-1]), D))
    Ct = torch.from_numpy(C)
    reqs = []
    for p in range(W):
        seg = Ct[int(send_off[p * epr]):int(send_off[(p + 1) * epr])].contiguous()
        if p == rank:
            parts = [seg]
        else:
            reqs.append(dist.isend(seg, dst=p))
    incoming = {}
    for s in range(W):
        rows = int(recv_rows[:, s].sum())
        buf = torch.empty((rows, D), dtype=torch.float64)
        if s == rank:
            buf = parts[0]
        else:
            dist.recv(buf, src=s)
        incoming[s] = buf
    for r_ in reqs:
        r_.wait()
    for s in range(W):                         # place (local expert, src) segments
        pos = 0
        for el in range(epr):
            n_ = int(recv_rows[el, s])
            dst = int(recv_off[el * W + s])
            recv[dst:dst + n_] = incoming[s][pos:pos + n_].numpy()
            pos += n_
    # expert FFN on the received centroids (per local expert segment)
    out = np.zeros_like(recv)
    for el in range(epr):
        a, z = int(recv_off[el * W]), int(recv_off[(el + 1) * W])
        out[a:z] = O.expert_ffn(recv[a:z], *ex[rank * epr + el])
    # combine: the exact reverse, results go back to their source ranks
    ret = np.zeros((b.m, D))
    Out = torch.from_numpy(out)
    reqs = []
    for s in range(W):
        segs = [Out[int(recv_off[el * W + s]):int(recv_off[el * W + s]) + int(recv_rows[el, s])] for el in range(epr)]
        payload = torch.cat(segs).contiguous()
        if s == rank:
            mine = payload
        else:
            reqs.append(dist.isend(payload, dst=s))
    for p in range(W):
        lo, hi = int(send_off[p * epr]), int(send_off[(p + 1) * epr])
        if p == rank:
            ret[lo:hi] = mine.numpy()
        else:
            buf = torch.empty((hi - lo, D), dtype=torch.float64)
            dist.recv(buf, src=p)
            ret[lo:hi] = buf.numpy()
    for r_ in reqs:
        r_.wait()
    y = O.restore(X, C, ret, b.bucket)
    results[rank] = (recv, recv_rows.numpy(), ret, y)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_exchange_matches_oracle_simulation():
    port = _free_port()
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(port, results), nprocs=W, join=True)
    R = np.stack([O.rotation_fp64(D, j, 11) for j in range(Q)])
    ex = _experts()
    Xs, zs = zip(*[_rank_inputs(r) for r in range(W)])
    sim = O.lsh_layer_ranks(list(Xs), list(zs), R, ex, E, "f64", round_expert_out=False)
    for r in range(W):
        recv, rr, ret, y = results[r]
        assert np.array_equal(recv, sim.recv[r])                 # dispatch layout (bit-exact)
        assert np.array_equal(rr, sim.recv_rows[r])
        assert np.array_equal(ret, sim.ret[r])                   # combine returns to the C layout
        assert np.array_equal(y, sim.y[r])
        solo = O.lsh_layer(Xs[r], zs[r], R, ex, E, "f64", round_expert_out=False)
        assert np.array_equal(y, solo.y[0])                      # w-invariance


def test_exchange_plan_edge_cases():
    import paper_2411_08446_b200 as L
    counts = torch.tensor([[2, 0, 3, 1], [0, 4, 1, 0]], dtype=torch.int32)
    so, ro, rr = L.exchange_plan(2, 1, counts)
    assert so.tolist() == [0, 0, 4, 5, 5]
    # rank 1 owns experts 2, 3: segments (e2, src0)=3, (e2, src1)=1, (e3, src0)=1, (e3, src1)=0
    assert rr.tolist() == [[3, 1], [1, 0]]
    assert ro.tolist() == [0, 3, 4, 5, 5]
    with pytest.raises(L.LshmoeError):
        L.exchange_plan(3, 0, torch.zeros((3, 4), dtype=torch.int32))    # E % w != 0
