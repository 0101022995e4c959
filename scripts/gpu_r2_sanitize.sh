#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over scripts/sanitize_run.py; logs under gpurun_out/r2/
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2/build_san.log 2>&1 || { echo build failed; exit 1; }
timeout 300 python scripts/sanitize_run.py > gpurun_out/r2/san_plain.log 2>&1; echo "plain rc=$?"; tail -3 gpurun_out/r2/san_plain.log
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 python scripts/sanitize_run.py > gpurun_out/r2/san_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Error|ok" gpurun_out/r2/san_$tool.log | tail -8
done
