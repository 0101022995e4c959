"""Summarise ncu captures into profiles/ (committed evidence).

    python scripts/ncu_summary.py <tag> gpurun_out/launches_<tag>.csv gpurun_out/prof_<tag>_*.ncu-rep

Writes profiles/<tag>_launches.md (per-launch device times of one step: the kernel's SHARE of
the step), profiles/<tag>_<kernel>.md (key counters per captured kernel) and, for the hash kernel,
profiles/ncu_hash_summary.json (per-launch DRAM bytes, read by bench.py as roofline.traffic).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles")

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "launch__grid_size", "launch__block_size",
    "launch__cluster_dim_x", "launch__registers_per_thread", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__ops_path_tensor_src_bf16_dst_fp32.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
]


def launches(path, tag):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h, data = rows[hi], rows[hi + 1:]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    # the last step: from the last hash launch to the end
    last = max(i for i, r in enumerate(data) if "HashSched" in r[ki] or "hash_f32" in r[ki] or "tc_gemm_kernel" in r[ki]
               and data[i + 1:] and "tile_kernel" in data[i + 1][ki])
    step = data[last:]
    tot = sum(float(r[vi]) for r in step if "lshmoe" in r[ki])
    lines = [f"# {tag}: kernel launches of one bench step (ncu --metrics gpu__time_duration.sum "
             f"--clock-control none; cold-cache, serialised: compare shares, not absolutes)", "",
             "| kernel | ns | share of lshmoe kernels |", "|---|---:|---:|"]
    for r in step:
        name = r[ki].split("(")[0].replace("void ", "")
        v = float(r[vi])
        share = f"{100 * v / tot:.1f}%" if "lshmoe" in r[ki] else "(torch L2 flush / not ours)"
        lines.append(f"| `{name[:110]}` | {v:.0f} | {share} |")
    lines.append(f"| **total lshmoe** | {tot:.0f} | 100% |")
    with open(os.path.join(OUT, f"{tag}_launches.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    return tot


def report(rep, tag):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    name = os.path.basename(rep).replace(".ncu-rep", "")
    out = []
    for v in rows[2:]:
        d = {k: (v[h.index(k)], units[h.index(k)]) for k in KEYS if k in h}
        kn = v[h.index("Kernel Name")] if "Kernel Name" in h else name
        out.append((kn, d))
    lines = [f"# {name} (ncu --set full --clock-control none)", ""]
    for kn, d in out:
        lines += [f"kernel: `{kn[:160]}`", "", "| metric | value | unit |", "|---|---:|---|"]
        lines += [f"| {k} | {val} | {u} |" for k, (val, u) in d.items()]
        lines.append("")
    with open(os.path.join(OUT, f"{name}.md"), "w") as f:
        f.write("\n".join(lines))
    return out


def main():
    tag = sys.argv[1]
    os.makedirs(OUT, exist_ok=True)
    for p in sys.argv[2:]:
        if p.endswith(".csv"):
            print("launch total ns", launches(p, tag))
        elif p.endswith(".ncu-rep"):
            res = report(p, tag)
            for kn, d in res:
                if "HashSched" in kn and "dram__bytes_read.sum" in d:
                    def to_bytes(val, unit):
                        return float(val.replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
                    rd = to_bytes(*d["dram__bytes_read.sum"])
                    wr = to_bytes(*d["dram__bytes_write.sum"])
                    with open(os.path.join(OUT, "ncu_hash_summary.json"), "w") as f:
                        json.dump({"source": os.path.basename(p), "kernel": kn[:200], "dram_bytes_read": rd,
                                   "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
                                   "duration_us_under_ncu": d.get("gpu__time_duration.sum", ("", ""))[0]}, f, indent=1)
            print("summarised", p)


if __name__ == "__main__":
    main()
