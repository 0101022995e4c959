#!/bin/bash
# r2: build, default bench line (+ optional N=2 shared-GPU spawn run), outputs under gpurun_out/r2/
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2
TAG=${TAG:-b}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2/build_${TAG}.log 2>&1 || { echo build failed; tail -30 gpurun_out/r2/build_${TAG}.log; exit 1; }
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/r2/bench_${TAG}.json 2> gpurun_out/r2/bench_${TAG}.err; echo "bench rc=$?"
tail -3 gpurun_out/r2/bench_${TAG}.err
if [ -n "$N2" ]; then
  timeout 900 python bench.py --gpus 2 --share-gpu --steps 3 --warmup 3 --no-backward ${N2_ARGS} > gpurun_out/r2/bench_${TAG}_n2.json 2> gpurun_out/r2/bench_${TAG}_n2.err; echo "bench n2 rc=$?"
  tail -5 gpurun_out/r2/bench_${TAG}_n2.err
fi
