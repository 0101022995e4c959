#!/bin/bash
# ncu --set full (with source) of the kernels in $KERNELS (mangled-name regexes), then a bench.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-n}
if [ -z "$SKIP_NCU" ]; then
for K in ${KERNELS:-compress_kernel}; do
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:$K -s ${SKIPK:-2} -c 1 \
     -o gpurun_out/prof_${TAG}_${K} python bench.py --profile --steps 1 --warmup 3 ${BENCH_ARGS} > gpurun_out/ncu_${TAG}_${K}.log 2>&1; echo "ncu $K rc=$?"
done
fi
if [ -z "$SKIP_BENCH" ]; then
timeout 600 python bench.py --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_${TAG}.json'))
print('ms', round(d['ms_per_step']*1e3,1), 'stages', {k: round(v*1e3,1) for k,v in d['stages_ms'].items()})
print('phases', d.get('compress_phases_us'))
print('cta', d.get('compress_centroid_cta_us'))
print('hash_frac', round(d['roofline']['frac'],3), 'unc', round(d['uncompressed_baseline']['ms_per_step']*1e3,1), 'launches', d['gpu_launches_per_step'])
"
tail -3 gpurun_out/bench_${TAG}.err
fi
