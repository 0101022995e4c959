#!/bin/bash
# tests + bench (no ncu)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-q}
timeout 900 python -m pytest tests -m gpu -q -s -p no:cacheprovider ${PYTEST_ARGS} > gpurun_out/pytest_${TAG}.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed" gpurun_out/pytest_${TAG}.log | tail -3
grep -E "^FAILED|Error" gpurun_out/pytest_${TAG}.log | head -20
timeout 600 python bench.py --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench rc=$?"
cat gpurun_out/bench_${TAG}.json; tail -5 gpurun_out/bench_${TAG}.err
