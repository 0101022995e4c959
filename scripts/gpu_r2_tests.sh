#!/bin/bash
# r2: build, then the given pytest selection (-m gpu), output under gpurun_out/r2/
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2
TAG=${TAG:-t}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2/build_${TAG}.log 2>&1 || { echo build failed; tail -30 gpurun_out/r2/build_${TAG}.log; exit 1; }
timeout ${TT:-1500} python -m pytest ${TESTS:-tests} -m gpu -q -s ${PYARGS} > gpurun_out/r2/tests_${TAG}.log 2>&1; echo "tests rc=$?"
grep -E "passed|failed|error" gpurun_out/r2/tests_${TAG}.log | tail -5
grep -E "^\[|FAIL|Error" gpurun_out/r2/tests_${TAG}.log | head -${HEADN:-60}
