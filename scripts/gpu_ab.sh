#!/bin/bash
# A/B of an env switch on the default bench line (alternating runs) + selected GPU tests.
# usage: TAG=x AB="LSHMOE_EARLY_GATE=0" TESTS="tests/test_gpu_compress.py" bash scripts/gpu_ab.sh
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-ab}
if [ -n "$TESTS" ]; then
  timeout 900 python -m pytest $TESTS -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_${TAG}.log 2>&1; echo "pytest rc=$?"
  tail -3 gpurun_out/pytest_${TAG}.log
fi
for i in 1 2; do
  for v in A B; do
    if [ $v = A ]; then E=""; else E="$AB"; fi
    env $E timeout 600 python bench.py --no-cpu-baseline --no-backward ${BENCH_ARGS} > gpurun_out/bench_${TAG}_$v$i.json 2> gpurun_out/bench_${TAG}_$v$i.err
    python - "$v$i" "gpurun_out/bench_${TAG}_$v$i.json" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    k = {r["kernel"].split(":")[0]: round(r["us"], 1) for r in d.get("kernels", [])}
    print(sys.argv[1], "step_us", round(d["ms_per_step"] * 1e3, 1), "t_dc", round(d["t_dc"]["lsh_us"], 1), k, d.get("compress_kernels_us"))
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
  done
done
