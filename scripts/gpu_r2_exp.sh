#!/bin/bash
# r2 experiments: build then run the command in $EXP, log to gpurun_out/r2/exp_$TAG.log
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2
TAG=${TAG:-e}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2/build_${TAG}.log 2>&1 || { echo build failed; tail -30 gpurun_out/r2/build_${TAG}.log; exit 1; }
eval "$EXP" > gpurun_out/r2/exp_${TAG}.log 2>&1; echo "exp rc=$?"
tail -${TAILN:-40} gpurun_out/r2/exp_${TAG}.log
