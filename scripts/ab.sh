#!/bin/bash
# A/B: us per draft step of the working-tree library vs lib_ab/ (another build), alternating.
for rep in 1 2 3; do
  for v in cur ab; do
    if [ $v = ab ]; then export DS_LIB_PATH=$PWD/lib_ab/libdynaspec.so; else unset DS_LIB_PATH; fi
    timeout 300 python bench.py --profile --no-cpu-baseline --steps 30 --warmup 5 2>/dev/null | tail -1 | \
      python -c "import json,sys; j=json.loads(sys.stdin.read()); print('$v', round(j['config']['us_per_draft_step'],2))"
  done
done
