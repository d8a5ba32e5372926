#!/bin/bash
# A/B/n: us per draft step of several library builds (lib_var/<name>/libdynaspec.so), alternating,
# in ONE process tree on one box (cross-box differences are larger than most effects measured here).
# usage: scripts/abn.sh "v0 v1 v2" [config] [reps] [extra bench flags]
cfg=${2:-llama3}; reps=${3:-3}; extra=${4:-}
for rep in $(seq $reps); do
  for v in $1; do
    DS_LIB_PATH=$PWD/lib_var/$v/libdynaspec.so timeout 300 python bench.py --config $cfg --profile --no-cpu-baseline \
      --steps 30 --warmup 5 $extra 2>/dev/null | tail -1 | \
      python -c "import json,sys; j=json.loads(sys.stdin.read()); print('$cfg $extra $v', round(j['config']['us_per_draft_step'],2))"
  done
done
