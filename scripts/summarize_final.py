"""Collect the evidence of scripts/gpu_final.sh (gpurun_out/) into profiles/ (committed):
bench lines (default, reference arm, SP / fp8 variants, C3-C5), the C5 hash-count sweep table, and
the ncu summaries (via scripts/ncu_summary.py).  Usage: python scripts/summarize_final.py <tag>"""
import glob
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT, SRC = os.path.join(ROOT, "profiles"), os.path.join(ROOT, "gpurun_out")


def load(path):
    try:
        with open(path) as f:
            return json.loads(f.read().strip().splitlines()[-1])
    except Exception:
        return None


def main():
    tag = sys.argv[1]
    lines = {}
    for nm, f in [("default", f"bench_{tag}.json"), ("reference", f"bench_ref_{tag}.json"),
                  ("sp", f"bench_{tag}_sp.json"), ("cp8", f"bench_{tag}_cp8.json"), ("hd3", f"bench_{tag}_hd3.json"),
                  ("C3", f"bench_{tag}_C3.json"), ("C4", f"bench_{tag}_C4.json"), ("C5", f"bench_{tag}_C5.json"),
                  ("p2p_n2_share_gpu", f"bench_{tag}_p2p_n2share.json")]:
        d = load(os.path.join(SRC, f))
        if d:
            lines[nm] = d
    with open(os.path.join(OUT, f"bench_{tag}_lines.json"), "w") as f:
        json.dump(lines, f, indent=1)
    rows = ["# C5 (Swin-MoE-shaped, 25,088 tokens, d=768, 32 experts top-1) hash-count sweep, one B200",
            "", "q | compression ratio | centroids | step ms | hash ms | compress ms | FFN ms | uncompressed ms | LSH/uncompressed"
            " | T_dc LSH us | T_dc uncompressed us | T_dc speedup",
            "---:|---:|---:|---:|---:|---:|---:|---:|---:|---:|---:|---:"]
    for q in range(1, 9):
        d = load(os.path.join(SRC, f"qsweep_{tag}_q{q}.json"))
        if not d:
            continue
        st = d["stages_ms"]
        unc = d.get("uncompressed_baseline") or {}
        rows.append(f"{q} | {d['compression_ratio']:.3f} | {d['centroids']} | {d['ms_per_step']:.3f} | {st['hash']:.3f} | "
                    f"{st['compress']:.3f} | {st['expert_ffn']:.3f} | {unc.get('ms_per_step', float('nan')):.3f} | "
                    f"{unc.get('speedup_of_lsh', float('nan')):.2f} | {d.get('t_dc', {}).get('lsh_us', float('nan')):.1f} | "
                    f"{d.get('t_dc', {}).get('uncompressed_same_exchange_us', float('nan')):.1f} | "
                    f"{d.get('t_dc', {}).get('speedup_vs_same_exchange', float('nan')):.2f}")
    with open(os.path.join(OUT, f"q_sweep_C5_{tag}.md"), "w") as f:
        f.write("\n".join(rows) + "\n")
    reps = sorted(glob.glob(os.path.join(SRC, f"prof_{tag}_*.ncu-rep")))
    launches = os.path.join(SRC, f"launches_{tag}.csv")
    if reps and os.path.exists(launches):
        subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_summary.py"), tag, launches, *reps], check=False)
    for nm, f in [("clocks", f"clocks_{tag}.csv"), ("tests", f"tests_{tag}.log"), ("smoke", f"smoke_{tag}.log"),
                  ("p2p_micro", f"p2p_micro_{tag}.log")]:
        p = os.path.join(SRC, f)
        if os.path.exists(p):
            with open(p) as a, open(os.path.join(OUT, f"{nm}_{tag}" + os.path.splitext(f)[1]), "w") as b:
                b.write(a.read())
    print("summarised", sorted(lines), "into profiles/")


if __name__ == "__main__":
    main()
