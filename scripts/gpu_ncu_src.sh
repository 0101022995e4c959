#!/bin/bash
# High-rate warp-sampling ncu capture (source page) of one kernel: KERNEL regex, TAG.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-s}
timeout 600 ncu --section WarpStateStats --section SourceCounters --section SpeedOfLight --section MemoryWorkloadAnalysis \
  --warp-sampling-interval 0 --clock-control none --import-source on --kernel-name-base mangled \
  -k regex:${KERNEL:-compress_kernel} -s ${SKIPK:-2} -c 1 -o gpurun_out/src_${TAG} \
  python bench.py --profile --steps 1 --warmup 3 ${BENCH_ARGS} > gpurun_out/ncu_src_${TAG}.log 2>&1; echo "ncu rc=$?"
