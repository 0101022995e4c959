#!/bin/bash
# centroid kernel shape A/B: default build vs an LSHMOE_NVCC_EXTRA build (VARIANT), rebuilt on the box
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
summ() { python - "$1" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
k = {r["kernel"][:20]: round(r["us"], 1) for r in d.get("kernels", [])}
print("step_us", round(d["ms_per_step"] * 1e3, 1), "t_dc", round(d["t_dc"]["lsh_us"], 1), k)
PY
}
for round in 1 2; do
  python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
  timeout 300 python bench.py --no-cpu-baseline --no-backward ${BENCH_ARGS} > gpurun_out/cg_A$round.json 2>/dev/null; echo -n "A$round "; summ gpurun_out/cg_A$round.json
  LSHMOE_NVCC_EXTRA="$VARIANT" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
  timeout 300 python bench.py --no-cpu-baseline --no-backward ${BENCH_ARGS} > gpurun_out/cg_B$round.json 2>/dev/null; echo -n "B$round "; summ gpurun_out/cg_B$round.json
done
timeout 120 python scripts/compress_diag.py C2 2>&1 | sed -n 1,2p
timeout 120 python scripts/compress_diag.py C2 2>&1 | grep -A8 "^centroid"
if [ -n "$TESTS" ]; then timeout 900 python -m pytest $TESTS -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2; fi
