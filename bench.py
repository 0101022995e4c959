#!/usr/bin/env python
"""Benchmark of the LSH-MoE compressed expert-parallel layer (Alg. 1) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl lsh|reference]

A step = one pass of the whole hot path over one batch per rank: hash (tcgen05) -> compress
(bucket + centroid) -> dispatch (all-to-all of centroids) -> expert FFN -> combine -> restore.
Workload per rank = BASELINE.json configs[1] (C2, RoBERTa-MoE-shaped, 16K tokens/GPU, bf16);
weak scaling over N ranks (one process per GPU, experts partitioned across ranks).  Inputs are
seeded synthetic (lshmoe_inputs).  Timed loops run K steps back to back in one CUDA graph over
S >= 4 copies of the inputs at distinct addresses (S x (x + y bytes) > 2 x the 126 MB L2), so no step
finds its tokens in L2; timed events.  Rank 0 prints one JSON line.

--impl reference times the CPU oracle (the tier's reference arm) on the same workload/metric.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MoE-layer dispatch+combine tokens/s (LSH-compressed EP layer: hash, compress, all-to-all, expert FFN, all-to-all, restore)"
UNIT = "tokens/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--config", default="C2")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--q", type=int, default=None, help="override the number of hash functions")
    p.add_argument("--impl", default="lsh", choices=["lsh", "reference"])
    p.add_argument("--hash", default="cp", choices=["cp", "sp", "cp8", "hd3"],
                   help="hash family: cross-polytope (paper default, Eq. 3), spherical-plane (NEXT-3), "
                        "cross-polytope on e4m3 operands (NEXT-2 fp8 option), or cross-polytope under the "
                        "structured rotation H D3 H D2 H D1 (NEXT-4, reading R30)")
    p.add_argument("--sp-bits", type=int, default=12, help="sign bits per SP hash function")
    p.add_argument("--exchange", default="auto", choices=["auto", "nccl", "p2p", "p2p-fused"],
                   help="a6/a8 at N>1: phase 1 (NCCL, one host count sync), phase 2 (device-initiated stores "
                        "into the peers' windows, no host sync, CUDA-graph captured), or phase 2 with the dispatch "
                        "fused into the centroid kernel (lshmoe_compress_p2p).  auto = p2p (the parity-tested "
                        "exchange; phase 1 has not run on several GPUs)")
    p.add_argument("--share-gpu", action="store_true",
                   help="testing only: every rank on cuda:0 with a gloo group (p2p exchange); the line is "
                        "marked and is not a measurement")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-uncompressed", action="store_true")
    p.add_argument("--no-graph", action="store_true")
    p.add_argument("--no-backward", action="store_true", help="skip the NEXT-1 backward timing")
    p.add_argument("--profile", action="store_true", help="minimal run for ncu: warmup + steps eager, no extras")
    return p.parse_args()


def spawn_ranks(args) -> int:
    """`python bench.py --gpus N` without a launcher: start N ranks (one process per GPU) through
    torch.distributed.run on 127.0.0.1, exactly as the driver would, and return their exit code."""
    import socket
    import subprocess
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained"), "source": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "source": "fallback (B200_PROFILING.md)"}


def pk_clock_ghz():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)["sm_max_mhz"] / 1e3
    except Exception:
        return 1.965


def ncu_traffic():
    """Per-launch DRAM bytes of the hash kernel from the committed ncu --set full summary."""
    path = os.path.join(ROOT, "profiles", "ncu_hash_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get("dram_bytes_per_launch")
    except Exception:
        return None


class L2Flush:
    """Evicts L2 between timed steps: a 256 MiB write (> the 126 MB L2), then a 256 MiB read, so that
    L2 holds only clean, unrelated lines when the timed region starts (the write's dirty lines are
    written back here, not inside the next timed kernel)."""

    def __init__(self, dev):
        import torch
        self.w = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=dev)
        self.r = torch.ones(64 * 1024 * 1024, dtype=torch.int32, device=dev)

    def __call__(self):
        self.w.zero_()
        self.r.max()


class ClockSampler:
    """Polls SM clock and throttle reasons via NVML during the timed region."""

    def __init__(self, dev_index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._ok = False
        try:
            import pynvml as N
            N.nvmlInit()
            self.N = N
            self.h = N.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
            self._ok = True
        except Exception:
            pass

    def _run(self):
        N = self.N
        names = {getattr(N, k): k for k in dir(N) if k.startswith("nvmlClocksEventReason") or k.startswith("nvmlClocksThrottleReason")}
        bits = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40, "sw_power_cap": 0x4,
                "hw_power_brake_slowdown": 0x80}
        while not self._stop.is_set():
            try:
                self.samples.append(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM))
                r = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, b in bits.items():
                    if r & b:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.0002)   # a timed region of a few ms still gets several samples

    def __enter__(self):
        if self._ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._ok:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------------------------
def run_reference(args, cfg):
    """The oracle (CPU, fp64, NumPy) as it stands, timed on the host cores: each step = Alg. 1 on a
    bounded sample of rank 0's tokens of the same workload."""
    import numpy as np
    import torch

    import oracle as O
    from lshmoe_inputs import make_experts, make_rank_inputs, rotation_seed
    X, zeta, _ = make_rank_inputs(cfg, args.seed, 0)
    ex = make_experts(cfg, args.seed)
    oex = {e: tuple(t.to(torch.float64).numpy() for t in v) for e, v in ex.items()}
    R64 = O.to_stored(O.rotation(cfg.d, cfg.q, rotation_seed(args.seed), cfg.dtype), cfg.dtype)
    X64 = X.to(torch.float64).numpy()
    z = zeta.numpy()
    sample = min(cfg.n, 2048)
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        O.lsh_layer(X64[:sample], z[:sample], R64, oex, cfg.E, cfg.dtype)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
    ms = 1e3 * sum(times) / len(times)
    value = sample / (ms / 1e3)
    cores = len(os.sched_getaffinity(0))
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(cfg, args.gpus),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"Alg. 1 on the first {sample} of rank 0's {cfg.n} tokens per step (fp64 NumPy oracle, "
                                       f"rotation generation excluded); one process on rank 0's host whatever "
                                       f"n_gpus is (the other ranks exit without work)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def workload_config(cfg, world, args=None):
    hashing = "cross-polytope (Eq. 3)"
    if args is not None and args.hash == "sp":
        hashing = f"spherical-plane sign bits, {args.sp_bits} per hash (NEXT-3)"
    if args is not None and args.hash == "cp8":
        hashing = "cross-polytope on e4m3-quantised x and R (NEXT-2 fp8 option, reading R28)"
    if args is not None and args.hash == "hd3":
        hashing = "cross-polytope under H D3 H D2 H D1 on x padded to 1024 (NEXT-4 structured rotation, reading R30)"
    return {"workload": f"{cfg.name}: {cfg.note}", "hash": hashing, "tokens_per_gpu": cfg.n, "d_model": cfg.d,
            "experts": cfg.E,
            "experts_per_gpu": cfg.E // world, "top_k": cfg.k, "hash_functions": cfg.q, "d_ffn": cfg.d_ffn,
            "parallelism": f"ep{world}", "l2": "inputs larger than L2: K steps back to back cycle S >= 4 copies of x / zeta / y at "
                    "distinct addresses, S x (x + y bytes) > 2 x 126 MB L2"}


def cpu_baseline(cfg, seed, X, zeta, ex, codes_gpu=None):
    """The oracle (Alg. 1 in fp64 NumPy) timed on this host's cores on full steps of rank 0, and, from
    the same oracle run, the in-run parity record of the bench's own inputs: BASELINE.json tier 1's
    near-ties (oracle top-two margin < 1e-5 relative) for the hash and for the gate (reading R29),
    and how many GPU codes differ from the oracle's (outside near-ties this must be 0)."""
    import numpy as np
    import torch

    import oracle as O
    from lshmoe_inputs import gate_matrix, rotation_seed
    R64 = O.to_stored(O.rotation(cfg.d, cfg.q, rotation_seed(seed), cfg.dtype), cfg.dtype)
    oex = {e: tuple(t.to(torch.float64).numpy() for t in v) for e, v in ex.items()}
    X64 = X.to(torch.float64).numpy()
    z = zeta.numpy()
    reps, t0 = 0, time.perf_counter()
    while True:
        res = O.lsh_layer(X64, z, R64, oex, cfg.E, cfg.dtype)
        reps += 1
        if time.perf_counter() - t0 > 10.0 or reps >= 5:
            break
    dt = (time.perf_counter() - t0) / reps
    cpu = {"value": cfg.n / dt, "unit": UNIT, "cores": len(os.sched_getaffinity(0)), "kind": "oracle",
           "sample": f"{reps} full step(s) of rank 0 (all {cfg.n} tokens, Alg. 1 incl. expert FFN) in fp64 NumPy; "
                     f"rotation generation excluded"}
    margins = res.margins[0]
    near = margins < 1e-5
    _, _, gmargin = O.gate_topk(X64, gate_matrix(cfg, seed), cfg.k)
    parity = {"hash_near_ties": int(near.sum()), "hash_codes": int(near.size),
              "gate_near_ties": int((gmargin < 1e-5).sum()),
              "near_tie_band": "oracle top-two margin < 1e-5 relative (BASELINE.json tier 1; gate: reading R29)"}
    if codes_gpu is not None:
        diff = codes_gpu != res.codes[0]
        parity["hash_code_mismatches"] = int(diff.sum())
        parity["hash_code_mismatches_outside_near_ties"] = int((diff & ~near).sum())
        parity["compression_ratio_oracle"] = res.ratio
    return cpu, parity


# ---------------------------------------------------------------------------------------------
def main():
    args = parse()
    from lshmoe_inputs import CONFIGS
    cfg = CONFIGS[args.config]
    if args.q:
        cfg = cfg.with_(q=args.q)
    launched = "WORLD_SIZE" in os.environ
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":       # the oracle runs once, on rank 0's host cores, whatever N is
        if rank == 0:
            run_reference(args, cfg)
        return
    if args.gpus > 1 and not launched:
        sys.exit(spawn_ranks(args))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} ranks were launched")
    if args.exchange == "auto":        # world 1: the exchange is an alias (no copy, no kernel)
        args.exchange = "p2p" if world > 1 else "nccl"
    if world > 1:      # NCCL's init lines (rank / nranks per communicator) on stderr, for the record
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2411_08446_b200 as L
    from lshmoe_inputs import make_experts, make_rank_inputs, rotation_seed

    if args.share_gpu:
        assert args.exchange != "nccl", "--share-gpu needs a phase-2 exchange (NCCL refuses two ranks on one GPU)"
        local_rank = 0
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        if args.share_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    assert cfg.E % world == 0, "experts must split evenly over ranks"
    E_local = cfg.E // world
    p2p = args.exchange in ("p2p", "p2p-fused")
    comm = None
    if p2p:     # phase 2: a window per rank (receive + returned buffers), peers mapped over CUDA IPC
        ok = 1
        try:
            comm = L.Comm(world, rank, None).p2p_init(cfg.n * cfg.k * world, cfg.n * cfg.k, cfg.d, X_dtype(cfg),
                                                      cfg.E, group=dist.group.WORLD if world > 1 else None)
        except Exception as ex:   # noqa: BLE001  (e.g. no peer access between these GPUs)
            ok = 0
            print(f"bench.py rank {rank}: phase-2 window setup failed ({str(ex)[:200]})", file=sys.stderr)
        if world > 1:             # every rank takes the same exchange
            flag = torch.tensor([ok], dtype=torch.int32, device="cpu" if args.share_gpu else dev)
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            ok = int(flag.item())
        if not ok:
            if world == 1 or args.share_gpu:
                raise SystemExit("bench.py: the phase-2 exchange could not be set up")
            print("bench.py: falling back to the phase-1 (NCCL) exchange", file=sys.stderr)
            args.exchange, p2p = "nccl", False
    if not p2p:
        comm = L.Comm.from_process_group() if world > 1 else None

    # ---- inputs (seeded synthetic, per rank) and buffers ----
    X_cpu, zeta_cpu, _ = make_rank_inputs(cfg, args.seed, rank)
    ex = make_experts(cfg, args.seed, range(rank * E_local, (rank + 1) * E_local))
    W1, b1, W2, b2 = (torch.stack([ex[e][i] for e in sorted(ex)]).to(dev).contiguous() for i in range(4))
    R = L.rotation(cfg.d, cfg.q, rotation_seed(args.seed), X_cpu.dtype).to(dev)
    X = X_cpu.to(dev)
    zeta = zeta_cpu.to(dev)
    n, k, d = cfg.n, cfg.k, cfg.d
    nk = n * k
    codes = torch.empty((n, cfg.q), dtype=torch.int16, device=dev)
    comp = L.alloc_compressed(n, k, cfg.E, d, X.dtype, dev)
    ws = torch.full((L.compress_workspace_bytes(n, k, cfg.E, cfg.q, d, X.dtype),), 255, dtype=torch.uint8, device=dev)
    cap = nk * world
    recv = comp.centroids if world == 1 else torch.empty((cap, d), dtype=X.dtype, device=dev)
    # world 1: recv aliases the centroids and recv_rows [E, 1] aliases expert_rows (no copies)
    rr = comp.expert_rows.view(cfg.E, 1) if world == 1 else torch.empty((E_local, world), dtype=torch.int32, device=dev)
    hid = torch.empty((cap, cfg.d_ffn), dtype=X.dtype, device=dev)
    eo = torch.empty((cap, d), dtype=X.dtype, device=dev)
    ret = eo if world == 1 else torch.empty((nk, d), dtype=X.dtype, device=dev)
    if p2p:     # the exchange lands in the window
        recv, ret, rr = comm.p2p_buffers()
    y = torch.empty_like(X)
    flush = L2Flush(dev)                            # 256 MiB write + 256 MiB read > 126 MB L2
    stream = torch.cuda.Stream(device=dev)          # non-default stream (graph capture needs one)
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        run_bench(args, cfg, L, world, rank, local_rank, dev, comm, E_local, X_cpu, zeta_cpu, X, zeta, R, codes, comp,
                  ws, cap, recv, rr, hid, eo, ret, y, flush, stream, W1, b1, W2, b2, dist)
    if world > 1:
        torch.cuda.synchronize()
        dist.barrier()
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()


def run_bench(args, cfg, L, world, rank, local_rank, dev, comm, E_local, X_cpu, zeta_cpu, X, zeta, R, codes, comp, ws,
              cap, recv, rr, hid, eo, ret, y, flush, stream, W1, b1, W2, b2, dist):
    import torch
    from lshmoe_inputs import make_experts, rotation_seed
    n, k, d = cfg.n, cfg.k, cfg.d
    nk = n * k
    p2p = args.exchange in ("p2p", "p2p-fused")
    fused = args.exchange == "p2p-fused"

    Nrm = L.sp_normals(R, args.sp_bits) if args.hash == "sp" else None
    R8 = L.rotation_e4m3(cfg.d, cfg.q, rotation_seed(args.seed)).to(dev) if args.hash == "cp8" else None
    x8 = torch.empty((n, d), dtype=torch.uint8, device=dev) if args.hash == "cp8" else None
    S3 = L.hd3_signs(cfg.q, rotation_seed(args.seed)).to(dev) if args.hash == "hd3" else None

    def make_stages(Xb, zb, yb):
        """The six calls of one step on token / gate / output buffers (Xb, zb, yb); the
        intermediates (codes, compressed rows, exchange and FFN buffers) are shared."""
        if args.hash == "sp":
            h = lambda: L.sp_hash(Xb, Nrm, cfg.q, args.sp_bits, codes)   # noqa: E731
        elif args.hash == "cp8":
            h = lambda: (L.quantize_e4m3(Xb, out=x8), L.hash_e4m3(x8, R8, codes))   # noqa: E731
        elif args.hash == "hd3":
            h = lambda: L.hash_hd3(Xb, S3, codes)   # noqa: E731
        else:
            h = lambda: L.hash(Xb, R, codes)   # noqa: E731
        return [
            h,
            (lambda: L.compress_p2p(comm, Xb, codes, zb, cfg.E, out=comp, workspace=ws)) if fused else
            (lambda: L.compress(Xb, codes, zb, cfg.E, out=comp, workspace=ws)),
            (lambda: None) if fused else
            (lambda: L.dispatch_p2p(comm, comp.centroids, comp.expert_rows)) if p2p else
            (lambda: L.dispatch(comm, comp.centroids, comp.expert_rows, cfg.E, recv, rr)),
            lambda: L.expert_ffn(recv, rr, W1, b1, W2, b2, out=eo, hidden=hid),
            (lambda: L.combine_p2p(comm, eo)) if p2p else (lambda: L.combine(comm, eo, comp.expert_rows, cfg.E, ret)),
            lambda: L.restore(Xb, comp.centroids, ret, comp.bucket, y=yb),
        ]

    stages = make_stages(X, zeta, y)
    hash_call = stages[0]
    # Input sets cycled by every timed loop: S copies of x / zeta / y at distinct addresses with
    # S * (x + y bytes) > 2 x the 126 MB L2, so no step finds its tokens in L2 from an earlier step
    # (SURVEY §8d.2's "cycle >= 4 input sets whose total exceeds L2") -- K steps then run back to
    # back in one CUDA graph, timed by two events, with no flush inside the timed region.
    set_bytes = 2 * X.numel() * X.element_size()
    S = max(4, -(-2 * 126 * 1000 * 1000 // set_bytes))
    sets = [(X, zeta, y)] + [(X.clone(), zeta.clone(), torch.empty_like(y)) for _ in range(S - 1)]
    set_stages = [stages] + [make_stages(*st) for st in sets[1:]]
    stage_names = ["hash", "compress", "dispatch", "expert_ffn", "combine", "restore"]

    def step():
        for f in stages:
            f()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cpu" if args.share_gpu else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(max(3, args.warmup)):
        step()
    barrier()
    L.check_device_error()

    if args.profile:
        for _ in range(args.steps):
            flush()
            step()
        barrier()
        return

    # ---- per-stage breakdown (eager, CUDA events on the launching stream) ----
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(len(stages) + 1)] for _ in range(args.steps)]
    barrier()
    for s in range(args.steps):
        flush()
        ev[s][0].record(stream)
        for i, f in enumerate(stages):
            f()
            ev[s][i + 1].record(stream)
    barrier()
    stage_ms = {nm: statistics.mean(ev[s][i].elapsed_time(ev[s][i + 1]) for s in range(args.steps))
                for i, nm in enumerate(stage_names)}
    eager_ms = statistics.mean(ev[s][0].elapsed_time(ev[s][-1]) for s in range(args.steps))
    hash_ms = stage_ms["hash"]
    # one extra compress with per-CTA stamps on (outside every timed region): kernel spans (us)
    L.set_diagnostics(True)
    L.compress(X, codes, zeta, cfg.E, out=comp, workspace=ws)
    torch.cuda.synchronize()
    L.set_diagnostics(False)
    compress_phases = L.compress_phase_times(ws)
    compress_cta = L.compress_cta_times(ws)

    # ---- headline: K whole steps back to back over the cycled input sets, one CUDA graph replay
    # between two events on `stream` at world 1 / phase 2 (no host sync inside a step); phase 1 at
    # N>1 syncs the host once per exchange, so there the K steps run eagerly between the events ----
    use_graph = (world == 1 or p2p) and not args.no_graph

    def k_steps():
        for i in range(args.steps):
            for f in set_stages[i % S]:
                f()
    run = k_steps
    if use_graph:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            k_steps()
        run = g.replay
        run()
    barrier()
    l0 = L.kernel_launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        barrier()
        e0.record(stream)
        run()
        e1.record(stream)
        barrier()
    launches = L.kernel_launches() - l0
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    if use_graph:   # kernels inside a replayed graph are not re-counted on the host
        l1 = L.kernel_launches()
        step()
        torch.cuda.synchronize()
        launches_per_step = L.kernel_launches() - l1
    else:
        launches_per_step = launches // args.steps

    # ---- e2e: every step copies its inputs host->device (pinned) and its output device->host, all
    # inside the timed region.  The copies run on their own streams, double-buffered, so step i's
    # H2D and step i-1's D2H overlap step i-1 / i's kernels (PCIe is full duplex); the value is the
    # K-step wall time on the device clock / K.  Inputs are re-copied from the host every step. ----
    X_h = X_cpu.pin_memory()
    z_h = zeta_cpu.pin_memory()
    Xs, zs, ys = [X, torch.empty_like(X)], [zeta, torch.empty_like(zeta)], [y, torch.empty_like(y)]
    y_hs = [torch.empty(y.shape, dtype=y.dtype).pin_memory() for _ in range(2)]
    bsteps = [make_stages(Xs[bb], zs[bb], ys[bb]) for bb in range(2)]
    runs = []
    for bb in range(2):
        Xs[bb].copy_(X_h)
        zs[bb].copy_(z_h)
        for f in bsteps[bb]:
            f()
        if use_graph:
            gb = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gb, stream=stream):
                for f in bsteps[bb]:
                    f()
            runs.append(gb.replay)
        else:
            runs.append(lambda fs=bsteps[bb]: [f() for f in fs])
    s_h2d = torch.cuda.Stream(device=dev)
    s_d2h = torch.cuda.Stream(device=dev)

    def e2e_pipeline(K):
        ev = lambda: torch.cuda.Event(enable_timing=False)   # noqa: E731
        e_h2d, e_cmp, e_d2h = [ev() for _ in range(K)], [ev() for _ in range(K)], [ev() for _ in range(K)]
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        s_h2d.wait_event(t0)
        for i in range(K):
            bb = i % 2
            with torch.cuda.stream(s_h2d):
                if i >= 2:
                    s_h2d.wait_event(e_cmp[i - 2])        # buffer bb no longer read by step i-2
                Xs[bb].copy_(X_h, non_blocking=True)
                zs[bb].copy_(z_h, non_blocking=True)
                e_h2d[i].record(s_h2d)
            stream.wait_event(e_h2d[i])
            if i >= 2:
                stream.wait_event(e_d2h[i - 2])           # ys[bb] drained to the host
            runs[bb]()
            e_cmp[i].record(stream)
            with torch.cuda.stream(s_d2h):
                s_d2h.wait_event(e_cmp[i])
                y_hs[bb].copy_(ys[bb], non_blocking=True)
                e_d2h[i].record(s_d2h)
        stream.wait_event(e_d2h[K - 1])
        t1.record(stream)
        return t0, t1

    e2e_pipeline(2)
    barrier()
    t0, t1 = e2e_pipeline(args.steps)
    barrier()
    e2e_ms = max_over_ranks(t0.elapsed_time(t1) / args.steps)
    assert torch.equal(y_hs[(args.steps - 1) % 2], y.cpu()), "e2e output differs from the device step"
    h2d = X_h.numel() * X_h.element_size() + z_h.numel() * z_h.element_size()
    d2h = y_hs[0].numel() * y_hs[0].element_size()

    # ---- generic device timing of a sequence of calls, the same way as the headline: K repetitions
    # cycling the input sets (fns_of(s) = the calls on set s), back to back in one CUDA graph (when the
    # exchange allows it, else eagerly) between two events on `stream`; us per repetition, max over
    # ranks ----
    def graph_time(fns_of, graph=None):
        graph = use_graph if graph is None else graph
        K = max(args.steps, 2 * S)

        def reps():
            for i in range(K):
                for fn in fns_of(i % S):
                    fn()
        for s_ in range(S):
            for fn in fns_of(s_):
                fn()
        run_ = reps
        if graph:
            gph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gph, stream=stream):
                reps()
            run_ = gph.replay
            run_()
        barrier()
        a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a_.record(stream)
        run_()
        b_.record(stream)
        barrier()
        return max_over_ranks(a_.elapsed_time(b_) * 1e3 / K)

    sb = 2 if X.dtype == torch.bfloat16 else 4
    row_bytes = d * sb
    m = int(comp.num_rows.item())
    ratio = m / nk
    lo_e, hi_e = rank * E_local, (rank + 1) * E_local

    def off_gpu_rows(counts):            # rows this rank sends to experts owned by other ranks
        c = counts.cpu().to(torch.int64)
        return int(c.sum()) - int(c[lo_e:hi_e].sum())

    # ---- context: uncompressed expert-parallel baseline on the same machinery ----
    unc = None
    send = torch.empty((nk, d), dtype=X.dtype, device=dev)
    slot = torch.empty((n, k), dtype=torch.int32, device=dev)
    er = torch.empty(cfg.E, dtype=torch.int32, device=dev)
    brr = er.view(cfg.E, 1) if world == 1 else torch.empty((E_local, world), dtype=torch.int32, device=dev)
    urecv = send if world == 1 else torch.empty((cap, d), dtype=X.dtype, device=dev)
    uret = eo if world == 1 else torch.empty((nk, d), dtype=X.dtype, device=dev)
    if p2p:
        urecv, uret, brr = recv, ret, rr

    def base_parts(s_):
        Xs_, zs_, ys_ = sets[s_]
        return {
            "permute": lambda: L.permute(Xs_, zs_, cfg.E, send, slot, er, ws),
            "dispatch": (lambda: L.dispatch_p2p(comm, send, er)) if p2p else
                        (lambda: L.dispatch(comm, send, er, cfg.E, urecv, brr)),
            "expert_ffn": lambda: L.expert_ffn(urecv, brr, W1, b1, W2, b2, out=eo, hidden=hid),
            "combine": (lambda: L.combine_p2p(comm, eo)) if p2p else (lambda: L.combine(comm, eo, er, cfg.E, uret)),
            "unpermute": lambda: L.unpermute(uret, slot, ys_),
        }
    base_sets = [base_parts(s_) for s_ in range(S)]
    if not args.no_uncompressed:
        bus = graph_time(lambda s_: list(base_sets[s_].values()))
        unc = {"ms_per_step": bus / 1e3, "tokens_per_s": world * n / (bus / 1e6),
               "what": "permute -> all-to-all of every routed token -> expert FFN on n*k rows -> all-to-all -> unpermute",
               "speedup_of_lsh": (bus / 1e3) / ms}

    # ---- T_dc: hash + compress + dispatch + combine + restore, the expert FFN excluded;
    # the same for both uncompressed baselines (this library's exchange; torch.distributed's NCCL
    # all_to_all_single on the permuted tokens) ----
    t_dc = graph_time(lambda s_: [set_stages[s_][i] for i in (0, 1, 2, 4, 5)])
    t_base_dc = graph_time(lambda s_: [base_sets[s_][k_] for k_ in ("permute", "dispatch", "combine", "unpermute")])
    t_exch = graph_time(lambda s_: [stages[2], stages[4]]) if world > 1 else 0.0
    off_rows = off_gpu_rows(comp.expert_rows)
    base_off_rows = off_gpu_rows(er)
    nccl_base = None
    if world > 1 and not args.share_gpu:
        try:
            nrecv = torch.empty((cap, d), dtype=X.dtype, device=dev)
            nret = torch.empty((nk, d), dtype=X.dtype, device=dev)
            rcnt = torch.empty(world, dtype=torch.int64, device=dev)

            def nccl_step(s_):
                Xs_, zs_, ys_ = sets[s_]
                L.permute(Xs_, zs_, cfg.E, send, slot, er, ws)          # rows grouped by destination rank
                cnt = er.view(world, E_local).sum(1).to(torch.int64)
                dist.all_to_all_single(rcnt, cnt)
                ins, outs = cnt.tolist(), rcnt.tolist()                   # one host sync, like phase 1
                dist.all_to_all_single(nrecv[:sum(outs)], send[:nk], outs, ins)
                dist.all_to_all_single(nret, nrecv[:sum(outs)], ins, outs)   # the reverse (FFN excluded)
                L.unpermute(nret, slot, ys_)
            t_nccl = graph_time(lambda s_: [lambda: nccl_step(s_)], graph=False)
            # the in-run NCCL all-to-all peak: 256 MiB per rank, equal splits
            big = torch.empty(128 << 20, dtype=torch.bfloat16, device=dev)
            bigo = torch.empty_like(big)
            t_peak = graph_time(lambda s_: [lambda: dist.all_to_all_single(bigo, big)], graph=False)
            peak_gbs = big.numel() * 2 * (world - 1) / world / (t_peak / 1e6) / 1e9
            del big, bigo
            nccl_base = {"t_dc_us": t_nccl, "tokens_per_s": world * n / (t_nccl / 1e6),
                         "what": "permute -> torch.distributed.all_to_all_single (NCCL) of every routed token -> "
                                 "the reverse -> unpermute (FFN excluded; splits learned by one count all-to-all + "
                                 "host sync)",
                         "nccl_alltoall_peak_gbs": peak_gbs,
                         "nccl_alltoall_peak_how": "all_to_all_single of 256 MiB per rank, off-GPU bytes per direction / time"}
        except Exception as ex:   # noqa: BLE001  (a context baseline must not cost the measured line)
            nccl_base = {"error": f"{type(ex).__name__}: {str(ex)[:300]}"}
    pk = peaks()
    nvlink_gbs = 770.0                       # B200_PROFILING.md: measured peer copy per direction
    t_dc_block = {
        "definition": "SURVEY §8d.2: wall time from x, zeta in HBM to y in HBM for hash + compress + dispatch + "
                      "combine + restore, expert FFN excluded; K repetitions over the cycled input sets in one "
                      "CUDA graph, us per repetition, max over ranks",
        "lsh_us": t_dc, "lsh_tokens_per_s": world * n / (t_dc / 1e6),
        "uncompressed_same_exchange_us": t_base_dc,
        "uncompressed_same_exchange_tokens_per_s": world * n / (t_base_dc / 1e6),
        "speedup_vs_same_exchange": t_base_dc / t_dc,
        "uncompressed_nccl_all_to_all_single": nccl_base,
        "speedup_vs_nccl": (nccl_base["t_dc_us"] / t_dc) if nccl_base and "t_dc_us" in nccl_base else None,
        "exchange_pair_us": t_exch if world > 1 else None,
        "off_gpu_bytes_per_direction": off_rows * row_bytes,
        "uncompressed_off_gpu_bytes_per_direction": base_off_rows * row_bytes,
        "nvlink_gbs_achieved": (2 * off_rows * row_bytes / (t_exch / 1e6) / 1e9) if world > 1 and t_exch else None,
        "nvlink_peak_gbs": nvlink_gbs,
        "nvlink_peak_source": "B200_PROFILING.md measured peer copy per direction (900 nominal)",
    }

    # ---- per-kernel roofline fractions: each stage alone, K launches over the cycled sets ----
    hbm = pk["hbm_gbs"]
    tc_peak = pk["bf16_tflops"] * (1 if cfg.dtype == "bf16" else 0.5)   # f32 SIMT path: no tensor peak, context only
    q_ = cfg.q
    hash_bytes = n * d * sb + q_ * d * d * sb + 2 * n * q_
    hash_flops = 2.0 * n * q_ * d * d
    comp_bytes = nk * row_bytes + m * row_bytes + 4 * nk + 2 * n * q_ + 4 * nk + 4 * nk + 4 * (m + 1)
    cent_bytes = nk * row_bytes + m * row_bytes + 4 * nk + 4 * nk
    rest_bytes = 2 * n * row_bytes + 4 * nk + 2 * m * row_bytes
    ffn_flops = 4.0 * m * d * cfg.d_ffn
    t_comp = graph_time(lambda s_: [set_stages[s_][1]])
    t_ffn = graph_time(lambda s_: [set_stages[s_][3]])
    t_rest = graph_time(lambda s_: [set_stages[s_][5]])
    t_hash = graph_time(lambda s_: [set_stages[s_][0]])
    span = {k_: v for k_, v in (compress_phases or {}).items() if not k_.startswith("gap")}

    def kern(name, bound, work, us):
        if bound == "tensor":
            ach = work / (us / 1e6) / 1e12
            return {"kernel": name, "bound": bound, "flops": work, "us": us, "achieved": ach, "unit": "TFLOP/s",
                    "peak": tc_peak, "frac": ach / tc_peak}
        ach = work / (us / 1e6) / 1e9
        return {"kernel": name, "bound": bound, "bytes": work, "us": us, "achieved": ach, "unit": "GB/s",
                "peak": hbm, "frac": ach / hbm}
    kernels = [kern("hash: tc_gemm_kernel<ArgmaxEpi>", "tensor", hash_flops, t_hash)] if args.hash == "cp" else \
        [{"kernel": f"hash ({args.hash})", "us": t_hash, "note": "see roofline"}]
    group_path = bool(span) and not span.get("tiles")   # the group path has no tile kernel (compress.cu)
    kernels.append(kern("compress: group + centroid (2 launches)" if group_path else
                        "compress: tile + bucket + centroid (3 launches)", "hbm", comp_bytes, t_comp))
    if span.get("centroid"):
        kc = kern("centroid_kernel (span, diagnostics stamps)", "hbm", cent_bytes, span["centroid"])
        kc["note"] = ("the gathered token rows are L2-resident (read by the hash just before; application-replay "
                      "ncu: ~1.4 MB of DRAM reads per launch at C2, profiles/l2_residency_r2g.md): the fraction "
                      "of HBM is a latency figure (ring rounds of L2 latency per warp, index and cut-row phases)")
        kernels.append(kc)
    for nm_ in ("tiles", "bucket"):
        if span.get(nm_):
            label = "group_kernel" if group_path and nm_ == "bucket" else f"{nm_} kernel"
            kk = kern(f"{label} (span, diagnostics stamps)", "hbm", 4 * nk * (3 if nm_ == "tiles" else 4), span[nm_])
            kk["bound"] = "latency"
            kk["note"] = "integer index work of < 1 MB: dependent global round trips and barriers, not bytes"
            kernels.append(kk)
    # the expert FFN on the m centroid rows: both rooflines; the binding one (more time) is its bound.
    # Bytes: the local experts' W1 / W2 (read once), the received rows, the hidden activation written
    # by GEMM 1 and read by GEMM 2, and the output rows.
    ffn_bytes = E_local * 2 * d * cfg.d_ffn * sb + m * row_bytes + 2 * m * cfg.d_ffn * sb + m * row_bytes
    kf = kern("expert FFN: tc_gemm_kernel<BiasActEpi> x2 (on the m centroid rows)", "tensor", ffn_flops, t_ffn)
    kh = kern("expert FFN: tc_gemm_kernel<BiasActEpi> x2 (on the m centroid rows)", "hbm", ffn_bytes, t_ffn)
    if ffn_bytes / (hbm * 1e9) > ffn_flops / (tc_peak * 1e12):
        kh["tensor_frac"] = kf["frac"]
        kernels.append(kh)
    else:
        kf["hbm_frac"] = kh["frac"]
        kernels.append(kf)
    kernels.append(kern("restore (restore_stage_kernel: rows staged by cp.async.bulk, k <= 4, rows <= 2 KB)", "hbm",
                        rest_bytes, t_rest))
    t_lower = max(hash_flops / (tc_peak * 1e12), hash_bytes / (hbm * 1e9)) * 1e6 + comp_bytes / (hbm * 1e9) * 1e6 \
        + rest_bytes / (hbm * 1e9) * 1e6 + 2 * off_rows * row_bytes / (nvlink_gbs * 1e9) * 1e6
    layer_roofline = {"t_lower_us": t_lower, "t_dc_us": t_dc, "frac": t_lower / t_dc,
                      "how": "T_lower = sum over the T_dc steps of max(flops / bf16 peak, algorithmic bytes / HBM, "
                             "off-GPU bytes / 770 GB/s); frac = T_lower / T_dc (SURVEY §8d.2)"}

    # ---- NEXT-1 backward (reading R27): grad_compress -> dispatch(G) -> expert backward (dX path)
    # -> combine(H) -> grad_restore, graph-timed as one chain and per part over cycled dY / x / dX
    # sets.  At world 1 the exchanges are aliases (no kernel) and are left out. ----
    bwd = None
    if not args.no_backward and world == 1:
        gen = torch.Generator(device=dev).manual_seed(11)
        dY = torch.randn(X.shape, generator=gen, device=dev).to(X.dtype)
        dYs = [dY] + [dY.clone() for _ in range(S - 1)]
        dXs = [torch.empty_like(X) for _ in range(S)]
        Gb = torch.empty((nk, d), dtype=X.dtype, device=dev)
        Hb = torch.empty((cap, d), dtype=X.dtype, device=dev)
        dhid = torch.empty((cap, cfg.d_ffn), dtype=X.dtype, device=dev)
        gws = torch.full((1 << 22,), 255, dtype=torch.uint8, device=dev)
        W2T = W2.transpose(1, 2).contiguous()
        W1T = W1.transpose(1, 2).contiguous()
        def parts(s_):
            return {"grad_compress": lambda: L.grad_compress(dYs[s_], comp, out=Gb, workspace=gws),
                    "expert_backward": lambda: L.expert_ffn_backward(Gb, rr, W2T, W1T, hid, out=Hb, dhidden=dhid),
                    "grad_restore": lambda: L.grad_restore(dYs[s_], sets[s_][0], comp.centroids, ret, Gb, Hb, comp,
                                                           dx=dXs[s_])}
        part_sets = [parts(s_) for s_ in range(S)]
        bwd = {nm + "_us": graph_time(lambda s_, nm=nm: [part_sets[s_][nm]]) for nm in part_sets[0]}
        bwd["chain_us"] = graph_time(lambda s_: list(part_sets[s_].values()))
        bwd["tokens_per_s"] = n / (bwd["chain_us"] / 1e6)
        bwd["grad_compress_hbm_bytes"] = (nk + m) * d * sb
        bwd["grad_compress_gbs"] = bwd["grad_compress_hbm_bytes"] / bwd["grad_compress_us"] / 1e3
        bwd["what"] = ("NEXT-1 (reading R27) dX path: G = per-bucket sums of dY -> H = J_E(c~)^T G "
                       "(expert backward, transposed weights, relu' from the forward's hidden) -> "
                       "dX = sum_s g dY + (H - G)/n_b; world 1: the two exchanges are aliases (no kernel); "
                       "weight gradients not computed; K repetitions over cycled input sets in one CUDA graph")

    L.check_device_error()
    # ---- the dominant kernel (the hash launch): its device time per launch from graph_time above (K
    # launches over the cycled token sets back to back in one CUDA graph, events on `stream`) ----
    hash_dev_ms = t_hash / 1e3
    if args.hash == "cp8":
        flops = 2.0 * n * cfg.q * d * d
        achieved = flops / (hash_dev_ms / 1e3) / 1e12
        roof = {"bound": "tensor", "kernel": "quantize_e4m3 + tc_gemm_kernel<ArgmaxEpi, e4m3> (lshmoe_hash_e4m3)",
                "achieved": achieved, "peak": 2 * pk["bf16_tflops"], "unit": "TFLOP/s",
                "frac": achieved / (2 * pk["bf16_tflops"]), "traffic": None,
                "per_launch": {"flops": flops, "avg_ms": hash_dev_ms, "eager_stage_ms": hash_ms},
                "peak_source": pk["source"] + " bf16 dense (burst) x 2 (the guide's fp8:bf16 nominal ratio)"}
    elif args.hash == "hd3":
        adds = 3.0 * 1024 * 10 * n * cfg.q                 # three 1024-point FWHTs per (token, hash)
        alu_peak = 148 * 128 * pk_clock_ghz() * 1e9 / 1e12   # fp32 add lanes per SM x SMs x max clock
        achieved = adds / (hash_dev_ms / 1e3) / 1e12
        roof = {"bound": "alu", "kernel": "hd3_hash_kernel (lshmoe_hash_hd3)", "achieved": achieved,
                "peak": alu_peak, "unit": "Tadd/s", "frac": achieved / alu_peak, "traffic": None,
                "per_launch": {"fp32_adds": adds, "avg_ms": hash_dev_ms, "eager_stage_ms": hash_ms,
                               "dense_equivalent_tflops": 2.0 * n * cfg.q * d * d / (hash_dev_ms / 1e3) / 1e12},
                "peak_source": "148 SMs x 128 fp32 lanes x sm_max_mhz (B200_PROFILING.md / MEASURED_PEAKS.json): "
                               "the CUDA-core fp32 add rate; the algorithmic work is 3 x 1024 x log2(1024) "
                               "add/sub per (token, hash)"}
    elif args.hash == "sp":
        nbytes = n * d * 2 + L.sp_rows(cfg.q, args.sp_bits) * d * 2 + n * cfg.q * 2
        achieved = nbytes / (hash_dev_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "kernel": "tc_gemm_kernel<SignBitsEpi> (lshmoe_sp_hash)", "achieved": achieved,
                "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": achieved / pk["hbm_gbs"], "traffic": None,
                "per_launch": {"algorithmic_bytes": nbytes, "avg_ms": hash_dev_ms, "eager_stage_ms": hash_ms},
                "peak_source": pk["source"] + " HBM copy bandwidth"}
    else:
        flops = 2.0 * n * cfg.q * d * d
        achieved = flops / (hash_dev_ms / 1e3) / 1e12
        roof = {"bound": "tensor", "kernel": "tc_gemm_kernel<ArgmaxEpi> (lshmoe_hash)", "achieved": achieved,
                "peak": pk["bf16_tflops"], "unit": "TFLOP/s", "frac": achieved / pk["bf16_tflops"],
                "traffic": ncu_traffic(),
                "per_launch": {"flops": flops, "algorithmic_bytes": n * d * 2 + cfg.q * d * d * 2 + n * cfg.q * 2,
                               "avg_ms": hash_dev_ms, "eager_stage_ms": hash_ms,
                               "timing": "K launches over the cycled token sets (tokens never L2-resident) back to "
                                         "back in one CUDA graph, events on its stream; us per launch"},
                "peak_source": pk["source"] + " bf16 dense (burst) — cuBLAS bf16 GEMM",
                "frac_of_sustained": achieved / pk["bf16_tflops_sustained"] if pk.get("bf16_tflops_sustained") else None,
                # the measured cuBLAS figure is not the hardware ceiling: the kernel can exceed it (frac > 1);
                # against NVIDIA's nominal dense bf16 figure it stays below 1
                "frac_of_nominal": achieved / 2250.0, "nominal_tflops": 2250.0}
        # the binding resource: TMA ingest from L2.  Each CTA-pair chunk (256 tokens x hash j x 256-column
        # slice) stages its CTAs' 128 x d token rows and 128 x d rotation rows: 4 * 128 * d bytes per CTA
        # chunk, d / 256 slices x q hashes per 256-token pair tile.  The chip's TMA / L2 (LTS) throughput
        # cap is ~6300 B/cycle (B300_MICROARCH.md, measured on B300; the same per-SM figure the FFN's TMA
        # streams reach here), times the SM clock of the run.
        if d % 256 == 0:
            chunks = 2 * ((n + 255) // 256) * cfg.q * (d // 256)
            ingest = chunks * 4.0 * 128 * d
            clk_ghz = pk_clock_ghz()
            l2_peak = 6300.0 * clk_ghz * 1e9 / 1e12
            roof["l2_ingest"] = {"bytes": ingest, "achieved_tbs": ingest / (hash_dev_ms / 1e3) / 1e12,
                                 "peak_tbs": l2_peak, "frac": ingest / (hash_dev_ms / 1e3) / 1e12 / l2_peak,
                                 "peak_source": "B300_MICROARCH.md TMA chip throughput ~6300 B/cycle (LTS cap) x "
                                                "sm_max_mhz: the hash's binding roof (it re-stages each token "
                                                "tile once per (hash, slice))"}

    cpu = None
    parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu, parity = cpu_baseline(cfg, args.seed, X_cpu, zeta_cpu, make_experts(cfg, args.seed),
                                   codes.cpu().numpy() if args.hash == "cp" else None)
        if args.hash != "cp":
            parity["note"] = "hash near-ties / mismatches above refer to the Eq. 3 dense-rotation hash (the oracle's cp_hash)"

    if rank == 0:
        line = {"metric": METRIC, "value": world * n / (ms / 1e3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "bf16" if cfg.dtype == "bf16" else "f32",
                "data": "synthetic (seeded Zipf mixture tokens, linear top-k gate, random experts)",
                "config": workload_config(cfg, world, args),
                "compression_ratio": ratio, "centroids": m, "routed_copies": nk,
                "gpu_launches": launches_per_step * args.steps, "gpu_launches_per_step": launches_per_step,
                "cuda_graph": use_graph, "input_sets": S,
                "exchange": ("phase 2 fused: the centroid kernel stores every centroid row into its owner's "
                             "window (CUDA IPC), no host sync" if fused else
                             "phase 2: device-initiated stores into the peers' windows (CUDA IPC), no host sync"
                             if p2p else "phase 1: NCCL all-gather of counts + grouped send/recv"
                             if world > 1 else "world 1: aliased (no copy)"),
                "stages_ms": stage_ms, "eager_ms_per_step": eager_ms,
                "compress_kernels_us": compress_phases,
                "compress_centroid_cta_us": compress_cta,
                "roofline": roof,
                "kernels": kernels,
                "t_dc": t_dc_block,
                "layer_roofline": layer_roofline,
                "e2e": {"value": world * n / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                        "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms,
                        "how": "K steps, each: pinned H2D of x and zeta, the step, D2H of y; copies on two side "
                               "streams, double-buffered (H2D of step i / D2H of step i-1 overlap the kernels)"},
                "clocks": clk.summary(),
                "uncompressed_baseline": unc,
                "backward_lsh": bwd,
                "parity_in_run": parity,
                "cpu_baseline": cpu}
        if args.share_gpu:
            line["share_gpu"] = "all ranks time-slice cuda:0: a correctness run of the N>1 path, not a measurement"
        print(json.dumps(line), flush=True)


def X_dtype(cfg):
    import torch
    return torch.bfloat16 if cfg.dtype == "bf16" else torch.float32


if __name__ == "__main__":
    main()
