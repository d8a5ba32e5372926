#!/bin/bash
# us per draft step for each environment setting given as an argument (e.g. DS_CSTEP_LOCAL=0),
# alternating, 3 reps.
for rep in 1 2 3; do
  for v in "$@"; do
    env $v timeout 300 python bench.py --profile --no-cpu-baseline --steps 30 --warmup 5 2>/dev/null | tail -1 | \
      python -c "import json,sys; j=json.loads(sys.stdin.read()); print('$v', round(j['config']['us_per_draft_step'],2))"
  done
done
