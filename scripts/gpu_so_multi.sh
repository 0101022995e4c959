#!/bin/bash
# A/B/C... of several library builds on one box: every paper_2411_08446_b200/so_*.so in turn, ROUNDS
# rounds, the default bench line each (step and T_dc); the working-tree build is restored at the end.
cd "$(dirname "$0")/.."
PK=paper_2411_08446_b200
cp $PK/liblshmoe.so /tmp/lib_cur.so
for round in $(seq 1 ${ROUNDS:-2}); do
  for f in $PK/so_*.so; do
    cp $f $PK/liblshmoe.so
    timeout 300 python bench.py --no-cpu-baseline --no-backward ${BENCH_ARGS} > /tmp/b.json 2>/dev/null
    python - "$(basename $f)" <<'PY'
import json, sys
try:
    d = json.loads(open("/tmp/b.json").read().strip().splitlines()[-1])
    k = {r["kernel"][:8]: round(r["us"], 1) for r in d.get("kernels", [])}
    print(sys.argv[1], "step", round(d["ms_per_step"] * 1e3, 1), "t_dc", round(d["t_dc"]["lsh_us"], 1), k)
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
  done
done
cp /tmp/lib_cur.so $PK/liblshmoe.so
