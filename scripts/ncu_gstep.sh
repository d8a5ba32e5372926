#!/bin/bash
# ncu on the grid step (the default B = 1 path): --set full of one k = 32 and one k = 8 launch of each of
# two cycles (-s skips the pool warm-up launches), and the launch list (gpu__time_duration, DRAM bytes)
# of a short bench run.  $1 = output tag.  With --no-graph every draft position is its own launch.
tag=${1:-r2}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gstep_kernel -s 8 -c 4 \
  -o gpurun_out/gstep_full_$tag python bench.py --steps 2 --warmup 1 --profile --no-graph > gpurun_out/ncu_gstep_full_$tag.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:gstep_kernel -s 8 -c 64 --csv --log-file gpurun_out/launches_gstep_$tag.csv \
  python bench.py --steps 8 --warmup 1 --profile --no-graph > gpurun_out/launch_gstep_$tag.log 2>&1
echo ncu-done
