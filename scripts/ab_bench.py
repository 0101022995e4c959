"""A/B timing of kernel variants (env-selected) on the C2 workload, one process, CUDA events,
L2 flushed before every timed launch.  Usage: python scripts/ab_bench.py [hash|ffn|all]"""
import os
import statistics

os.environ.setdefault("LSHMOE_EXPERIMENTS", "1")   # honour the work-skipping experiment switches
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_08446_b200 as L  # noqa: E402
from lshmoe_inputs import CONFIGS, make_experts, make_rank_inputs, rotation_seed  # noqa: E402


_RB = {}


def _settle(flush):
    """Read a second buffer larger than L2: evicts the flush's dirty lines (their write-back happens
    here, outside the timed region) and leaves L2 holding clean, unrelated lines."""
    rb = _RB.get(flush.device)
    if rb is None:
        rb = _RB[flush.device] = torch.ones(64 * 1024 * 1024, dtype=torch.int32, device=flush.device)
    rb.max()


def timeit(fn, iters=30, flush=None):
    """Device time of fn: captured once into a CUDA graph (no host launch overhead in the timed
    region), replayed between CUDA events; L2 flushed before each replay when flush is given."""
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    ts = []
    mode = os.environ.get("AB_FLUSH", "write")
    for _ in range(iters):
        if flush is not None:
            if mode in ("write", "writeread"):
                flush.zero_()
            if mode in ("read", "writeread"):
                _settle(flush)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return statistics.median(ts), min(ts)


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    cfgname = sys.argv[2] if len(sys.argv) > 2 else "C2"
    cfg = CONFIGS[cfgname]
    X, zeta, _ = make_rank_inputs(cfg, 0, 0)
    X, zeta = X.cuda(), zeta.cuda()
    R = L.rotation(cfg.d, cfg.q, rotation_seed(0), X.dtype).cuda()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device="cuda")
    codes = torch.empty((cfg.n, cfg.q), dtype=torch.int16, device="cuda")
    flops = 2.0 * cfg.n * cfg.q * cfg.d * cfg.d
    if what in ("hash8",):
        R8 = L.rotation_e4m3(cfg.d, cfg.q, rotation_seed(0)).cuda()
        x8 = L.quantize_e4m3(X)
        for ex in ("0", "1", "2"):
            os.environ["LSHMOE_HASH_EXP"] = ex
            med, mn = timeit(lambda: L.hash_e4m3(x8, R8, codes), flush=flush)
            print(f"hash_e4m3 exp={ex}: median {med:.1f} us  min {mn:.1f} us  {flops / med / 1e6:.0f} TFLOP/s", flush=True)
        os.environ.pop("LSHMOE_HASH_EXP")
    if what in ("hash", "all"):
        for cta in ("1", "2") if not os.environ.get("AB_QUICK") else ():
            for ex in ("1", "2"):
                os.environ["LSHMOE_HASH_EXP"] = ex
                os.environ["LSHMOE_HASH_CTA"] = cta
                med, mn = timeit(lambda: L.hash(X, R, codes), flush=flush)
                print(f"hash cta={cta} exp={ex} (1: no argmax scan, 2: no MMA): median {med:.1f} us", flush=True)
        os.environ.pop("LSHMOE_HASH_EXP", None)
        os.environ.pop("LSHMOE_HASH_CTA", None)
        for contig in ("1", "0"):
            for cta in ("1", "2"):
                os.environ["LSHMOE_HASH_CONTIG"] = contig
                os.environ["LSHMOE_HASH_CTA"] = cta
                med, mn = timeit(lambda: L.hash(X, R, codes), flush=flush)
                print(f"hash contig={contig} cta={cta}: median {med:.1f} us  min {mn:.1f} us  "
                      f"{flops / med / 1e6:.0f} TFLOP/s", flush=True)
        os.environ.pop("LSHMOE_HASH_CONTIG")
        if os.environ.get("AB_QUICK"):
            return
        for split in ("1", "2"):
            for cta in ("1", "2"):
                os.environ["LSHMOE_HASH_SPLIT"] = split
                os.environ["LSHMOE_HASH_CTA"] = cta
                med, mn = timeit(lambda: L.hash(X, R, codes), flush=flush)
                print(f"hash split={split == '1'} cta={cta}: median {med:.1f} us  min {mn:.1f} us  "
                      f"{flops / med / 1e6:.0f} TFLOP/s", flush=True)
        os.environ.pop("LSHMOE_HASH_SPLIT")
        os.environ.pop("LSHMOE_HASH_CTA")
        # library reference for the same contraction (Y = X R^T, Y materialised, no argmax)
        Rt = R.reshape(cfg.q * cfg.d, cfg.d)
        med, mn = timeit(lambda: torch.matmul(X, Rt.t()), flush=flush)
        print(f"cuBLAS X @ R^T [{cfg.n}x{cfg.d}]x[{cfg.d}x{cfg.q * cfg.d}]: median {med:.1f} us  "
              f"{flops / med / 1e6:.0f} TFLOP/s", flush=True)
        A = torch.randn(8192, 8192, device="cuda").to(torch.bfloat16)
        med, mn = timeit(lambda: torch.matmul(A, A), flush=flush)
        print(f"cuBLAS 8192^3: median {med:.1f} us  {2 * 8192 ** 3 / med / 1e6:.0f} TFLOP/s", flush=True)
    if what in ("compress", "all"):
        ws = torch.full((L.compress_workspace_bytes(cfg.n, cfg.k, cfg.E, cfg.q, cfg.d, X.dtype),), 255, dtype=torch.uint8,
                         device="cuda")
        L.hash(X, R, codes)
        comp = L.alloc_compressed(cfg.n, cfg.k, cfg.E, cfg.d, X.dtype, "cuda")
        med, mn = timeit(lambda: L.compress(X, codes, zeta, cfg.E, out=comp, workspace=ws), flush=flush)
        print(f"compress: median {med:.1f} us  min {mn:.1f}", flush=True)
        pass
        print("  centroid CTAs", L.compress_cta_times(ws))
        raw = ws[:128].cpu().view(torch.int32).numpy().astype("int64") & 0xFFFFFFFF
        if int(os.environ.get("LSHMOE_CDBG", "0")) & 8:
            import numpy as np
            hdr = ws[:4 * 1000].cpu().view(torch.int32).numpy().astype("int64") & 0xFFFFFFFF
            st = hdr[64:64 + 2 * 148:2]; en = hdr[65:65 + 2 * 148:2]
            q = hdr[400:400 + 4 * 148].reshape(148, 4)
            idx = (q[:, 0] - st) / 1e3; loop = q[:, 1] / 1e3; sync = (q[:, 2] - q[:, 0]) / 1e3 - loop
            comb = (q[:, 3] - q[:, 2]) / 1e3; tail = (en - q[:, 3]) / 1e3
            for nm, v in (("idx", idx), ("loop", loop), ("sync", sync), ("combine", comb), ("tail", tail)):
                print(f"  {nm}: min {v.min():.2f} med {np.median(v):.2f} max {v.max():.2f}")
        print(f"  row_lo scatter sub-steps: offsets {(raw[20] - raw[6]) / 1e3:.2f} us, scatter "
              f"{(raw[21] - raw[20]) / 1e3:.2f} us, barrier {(raw[7] - raw[21]) / 1e3:.2f} us", flush=True)
    if what in ("restore", "all"):
        comp = L.compress(X, L.hash(X, R, codes), zeta, cfg.E)
        ret = comp.centroids.clone()
        y = torch.empty_like(X)
        nb = 2 * X.numel() * X.element_size()
        for fl in (flush, None):
            med, mn = timeit(lambda: L.restore(X, comp.centroids, ret, comp.bucket, y=y), flush=fl)
            print(f"restore V={'v1'} flush={fl is not None}: median {med:.1f} us "
                  f"min {mn:.1f}  x+y streams {nb / med / 1e3:.0f} GB/s", flush=True)
        med, mn = timeit(lambda: y.copy_(X), flush=flush)
        print(f"torch copy x->y (same bytes, no gathers): median {med:.1f} us  {nb / med / 1e3:.0f} GB/s", flush=True)
    if what in ("ffn", "all"):
        comp = L.compress(X, L.hash(X, R, codes), zeta, cfg.E)
        ex = make_experts(cfg, 0)
        W = [torch.stack([ex[e][i] for e in range(cfg.E)]).cuda() for i in range(4)]
        rr = comp.expert_rows.view(cfg.E, 1)
        out = torch.empty_like(comp.centroids)
        hid = torch.empty((comp.centroids.shape[0], cfg.d_ffn), dtype=X.dtype, device="cuda")
        m = int(comp.num_rows.item())
        fl = 4.0 * m * cfg.d * cfg.d_ffn
        for only in ("1", "2"):
            for cta, bn, od, ex in (("2", "256", "0", "0"), ("2", "256", "1", "0"), ("1", "256", "0", "0"),
                                    ("1", "256", "1", "0"), ("2", "128", "1", "0")):
                    os.environ.update(LSHMOE_FFN_CTA=cta, LSHMOE_FFN_BN1=bn, LSHMOE_FFN_BN2=bn, LSHMOE_FFN_ONLY=only,
                                      LSHMOE_FFN_ORDER=od, LSHMOE_FFN_EXP=ex)
                    for fl_ in ((flush, None) if ex == "0" else (flush,)):
                        med, mn = timeit(lambda: L.expert_ffn(comp.centroids, rr, *W, out=out, hidden=hid), flush=fl_)
                        print(f"ffn GEMM{only} cta={cta} bn={bn} order={od} flush={fl_ is not None}: median {med:.1f} us  "
                              f"min {mn:.1f} us  {fl / 2 / med / 1e6:.0f} TFLOP/s  (m={m})", flush=True)
        for k in ("LSHMOE_FFN_CTA", "LSHMOE_FFN_BN1", "LSHMOE_FFN_BN2", "LSHMOE_FFN_ONLY", "LSHMOE_FFN_ORDER", "LSHMOE_FFN_EXP"):
            os.environ.pop(k)
        med, mn = timeit(lambda: L.expert_ffn(comp.centroids, rr, *W, out=out, hidden=hid), flush=None)
        print(f"ffn default, NO L2 flush (weights L2-resident): median {med:.1f} us  {fl / med / 1e6:.0f} TFLOP/s",
              flush=True)
        er = comp.expert_rows.cpu().tolist()
        offs = [0]
        for r in er:
            offs.append(offs[-1] + r)

        def torch_ffn():
            for e in range(cfg.E):
                a = comp.centroids[offs[e]:offs[e + 1]]
                h = torch.relu(torch.addmm(W[1][e], a, W[0][e].t()))
                torch.addmm(W[3][e], h, W[2][e].t(), out=out[offs[e]:offs[e + 1]])
        med, mn = timeit(torch_ffn, flush=flush)
        print(f"cuBLAS per-expert FFN (torch.addmm x{2 * cfg.E}): median {med:.1f} us  {fl / med / 1e6:.0f} TFLOP/s",
              flush=True)
        if hasattr(torch, "_grouped_mm"):   # library grouped GEMM (the FFN's two layers, no bias/act)
            offs_t = torch.tensor(offs[1:], dtype=torch.int32, device="cuda")
            W1t = W[0].transpose(1, 2)          # [E, d, d_ffn] views: out = A @ W1^T per group
            W2t = W[2].transpose(1, 2)
            a = comp.centroids[:m]
            try:
                def grouped():
                    h = torch._grouped_mm(a, W1t, offs=offs_t)
                    torch._grouped_mm(h, W2t, offs=offs_t)
                med, mn = timeit(grouped, flush=flush)
                print(f"torch._grouped_mm x2 (no bias/ReLU): median {med:.1f} us  {fl / med / 1e6:.0f} TFLOP/s", flush=True)
            except Exception as ex:   # noqa: BLE001
                print("torch._grouped_mm unavailable:", str(ex)[:200])


if __name__ == "__main__":
    main()
