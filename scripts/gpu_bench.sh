#!/bin/bash
# GPU session: bench (N=1, default flags), reference arm, ncu launch list, ncu --set full of the
# kernels in $KERNELS (mangled-name regexes), clocks sampled by nvidia-smi during the bench.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-r1}
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/clocks_${TAG}.csv 2>&1 &
SMI=$!
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench rc=$?"
kill $SMI 2>/dev/null
if [ -z "$SKIP_REF" ]; then
  timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_${TAG}.json 2> gpurun_out/bench_ref_${TAG}.err; echo "ref rc=$?"
fi
if [ -z "$SKIP_NCU" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
     python bench.py --profile --steps 2 --warmup 3 > gpurun_out/ncu_launch_${TAG}.log 2>&1; echo "ncu launches rc=$?"
  for K in ${KERNELS:-HashSched compress_kernel restore_kernel FfnSched}; do
    timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:$K -s 2 -c 1 \
       -o gpurun_out/prof_${TAG}_${K} python bench.py --profile --steps 1 --warmup 3 > gpurun_out/ncu_${TAG}_${K}.log 2>&1; echo "ncu $K rc=$?"
  done
fi
cat gpurun_out/bench_${TAG}.json; tail -3 gpurun_out/bench_${TAG}.err; cat gpurun_out/bench_ref_${TAG}.json 2>/dev/null
