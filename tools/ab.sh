#!/bin/bash
# A/B of library variants on one box: tools/ab.sh REPS name1 name2 ...   ("base" = the in-tree build)
# prints each run's mean ms per outer iteration (bench.py --no-e2e --no-cpu, same window)
reps=$1; shift
mkdir -p gpurun_out
for i in $(seq $reps); do
  for v in "$@"; do
    if [ "$v" = base ]; then L=paper_1604_04026_b200/libklnmf.so; else L=_variants/$v/libklnmf.so; fi
    KLNMF_LIB=$L python bench.py --no-e2e --no-cpu --steps ${AB_STEPS:-10} --warmup ${AB_WARMUP:-8} ${AB_ARGS} > gpurun_out/ab_${v}_$i.log 2>&1
    python - "$v" $i <<'PY'
import json,sys
v,i=sys.argv[1:3]
for l in open(f"gpurun_out/ab_{v}_{i}.log"):
    if l.startswith("{"):
        d=json.loads(l); print(v,i,round(d["ms_per_step"],3),d["step_ms"],flush=True)
PY
  done
done
