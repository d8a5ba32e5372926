#!/bin/bash
# A/B of the working-tree library vs lib_ab/ on one bench config: $1 = config, $2 = extra args.
for rep in 1 2 3; do
  for v in cur ab; do
    if [ $v = ab ]; then export DS_LIB_PATH=$PWD/lib_ab/libdynaspec.so; else unset DS_LIB_PATH; fi
    timeout 300 python bench.py --config $1 $2 --profile --no-cpu-baseline --steps 10 --warmup 3 2>/dev/null | tail -1 | \
      python -c "import json,sys; j=json.loads(sys.stdin.read()); print('$1 $v', round(j['config']['us_per_draft_step'],2))"
  done
done
