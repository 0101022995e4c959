#!/bin/bash
# pytest subset (PYK = -k expression) + bench summary
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-t}
timeout ${TT:-600} python -m pytest tests -m gpu -q -s -p no:cacheprovider -k "${PYK:-gpu}" > gpurun_out/pytest_${TAG}.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed" gpurun_out/pytest_${TAG}.log | tail -2
grep -E "^FAILED|^E  " gpurun_out/pytest_${TAG}.log | head -20
if [ -z "$SKIP_BENCH" ]; then SKIP_NCU=1 TAG=${TAG} bash scripts/gpu_ncu.sh; fi
