#!/bin/bash
# A/B of two builds: paper_2411_08446_b200/liblshmoe.so (B, the working tree) against
# paper_2411_08446_b200/liblshmoe_prev.so (A, built from the previous commit), alternating; then TESTS on B.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
PK=paper_2411_08446_b200
cp $PK/liblshmoe.so /tmp/lib_B.so
summ() { python - "$1" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    k = {r["kernel"][:20]: round(r["us"], 1) for r in d.get("kernels", [])}
    print("step_us", round(d["ms_per_step"] * 1e3, 1), "t_dc", round(d["t_dc"]["lsh_us"], 1), k)
except Exception as e:
    print("failed", e)
PY
}
for round in 1 2; do
  for v in A B; do
    if [ $v = A ]; then cp $PK/liblshmoe_prev.so $PK/liblshmoe.so; else cp /tmp/lib_B.so $PK/liblshmoe.so; fi
    timeout 300 python bench.py --no-cpu-baseline --no-backward ${BENCH_ARGS} > gpurun_out/so_$v$round.json 2>/dev/null; echo -n "$v$round "; summ gpurun_out/so_$v$round.json
  done
done
cp /tmp/lib_B.so $PK/liblshmoe.so
for c in ${DIAG:-C2}; do timeout 120 python scripts/compress_diag.py $c 2>&1 | sed -n 1,2p; done
if [ -n "$TESTS" ]; then timeout 1500 python -m pytest $TESTS -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3; fi
