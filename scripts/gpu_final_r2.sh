#!/bin/bash
# Round-2 evidence in one GPU session (outputs in gpurun_out/, summarised by scripts/summarize_final.py):
# full -m gpu suite, smoke, the default bench line (with the oracle's CPU baseline and in-run parity),
# the reference arm, SP / fp8 / structured-rotation variants, C3-C5 lines, the N=2 line through the
# spawned phase-2 path on one shared GPU, the C5 hash-count sweep, the ncu launch list of one step and
# --set full captures of the step's kernels.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-r2final}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_${TAG}.log 2>&1 || { echo build failed; exit 1; }
if [ -z "$SKIP_TESTS" ]; then
  timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/tests_${TAG}.log; cat gpurun_out/tests_${TAG}.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke rc=$?"
fi
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 100 > gpurun_out/clocks_${TAG}.csv 2>&1 &
SMI=$!
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench rc=$?"
kill $SMI 2>/dev/null
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_${TAG}.json 2> gpurun_out/bench_ref_${TAG}.err; echo "ref rc=$?"
for h in sp cp8 hd3; do
  timeout 600 python bench.py --hash $h --no-cpu-baseline > gpurun_out/bench_${TAG}_$h.json 2> gpurun_out/bench_${TAG}_$h.err; echo "bench $h rc=$?"
done
for c in C3 C4 C5; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_${TAG}_$c.json 2> gpurun_out/bench_${TAG}_$c.err; echo "bench $c rc=$?"
done
# the N=2 path through the phase-2 exchange, spawned by bench.py itself, both ranks on this one GPU
timeout 900 python bench.py --gpus 2 --steps 4 --warmup 3 --share-gpu --no-backward \
   > gpurun_out/bench_${TAG}_p2p_n2share.json 2> gpurun_out/bench_${TAG}_p2p_n2share.err; echo "bench n2 share rc=$?"
timeout 300 python scripts/p2p_bench.py 0 16 > gpurun_out/p2p_micro_${TAG}.log 2>&1; echo "p2p micro rc=$?"
for q in 1 2 3 4 5 6 7 8; do
  timeout 600 python bench.py --config C5 --q $q --no-cpu-baseline --no-backward --steps 10 > gpurun_out/qsweep_${TAG}_q$q.json 2> gpurun_out/qsweep_${TAG}_q$q.err; echo "q=$q rc=$?"
done
if [ -z "$SKIP_NCU" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
     python bench.py --profile --steps 2 --warmup 3 > gpurun_out/ncu_launch_${TAG}.log 2>&1; echo "ncu launches rc=$?"
  for K in ${KERNELS:-HashSched group_kernel centroid_kernel FfnSched restore_stage_kernel}; do
    timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:$K -s 2 -c 1 \
       -o gpurun_out/prof_${TAG}_${K} python bench.py --profile --steps 1 --warmup 3 > gpurun_out/ncu_${TAG}_${K}.log 2>&1; echo "ncu $K rc=$?"
  done
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:hd3_hash -s 2 -c 1 \
     -o gpurun_out/prof_${TAG}_hd3_hash python bench.py --profile --hash hd3 --steps 1 --warmup 3 > gpurun_out/ncu_${TAG}_hd3.log 2>&1; echo "ncu hd3 rc=$?"
fi
