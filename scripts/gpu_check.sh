#!/bin/bash
# GPU session: parity tests (the files in $TESTS first, then the whole -m gpu suite unless
# QUICK is set), then one bench run without the CPU baseline.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-chk}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_${TAG}.log 2>&1 || { echo "build failed"; tail -20 gpurun_out/build_${TAG}.log; exit 1; }
if [ -n "$TESTS" ]; then
  timeout 900 python -m pytest $TESTS -m gpu -x -q -s 2>&1 | grep -v "^$" | tail -${TAIL:-25}
fi
if [ -z "$QUICK" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -8
fi
if [ -z "$SKIP_BENCH" ]; then
  timeout 600 python bench.py --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench rc=$?"
  python - <<PY
import json
d = json.load(open('gpurun_out/bench_${TAG}.json'))
print('ms', round(d['ms_per_step'] * 1e3, 1), 'stages', {k: round(v * 1e3, 1) for k, v in d['stages_ms'].items()})
print("kernels", d.get("compress_kernels_us"))
print('cta', d.get('compress_centroid_cta_us'))
print('hash_frac', round(d['roofline']['frac'], 3), 'unc', round(d['uncompressed_baseline']['ms_per_step'] * 1e3, 1),
      'launches', d['gpu_launches_per_step'], 'clocks', d.get('clocks'))
PY
  tail -3 gpurun_out/bench_${TAG}.err
fi
