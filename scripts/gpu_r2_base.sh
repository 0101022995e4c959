#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2/build.log 2>&1 || { echo build failed; tail gpurun_out/r2/build.log; exit 1; }
timeout 300 python scripts/compress_diag.py C2 > gpurun_out/r2/diag_C2.log 2>&1; echo diag rc=$?
timeout 300 python scripts/compress_diag.py C3 > gpurun_out/r2/diag_C3.log 2>&1; echo diag rc=$?
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2/bench_base.json 2> gpurun_out/r2/bench_base.err; echo bench rc=$?
nvidia-smi > gpurun_out/r2/smi.txt
