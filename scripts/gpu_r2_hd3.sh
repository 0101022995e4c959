#!/bin/bash
cd /root/repo
TAG=hd3a TESTS="tests/test_gpu_hd3.py" scripts/gpu_r2_tests.sh
timeout 600 python bench.py --hash hd3 --no-cpu-baseline --no-backward --no-uncompressed > gpurun_out/r2/bench_hd3a.json 2> gpurun_out/r2/bench_hd3a.err; echo "bench rc=$?"; tail -3 gpurun_out/r2/bench_hd3a.err
