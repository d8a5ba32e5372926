#!/bin/bash
# ncu on the cluster step: --set full for a k=32 (cycle positions 0,1) and a k=8 (positions 2,3)
# launch, and the launch list (gpu__time_duration) of a short bench run.  $1 = output tag.
tag=${1:-r1}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cstep_kernel -s 8 -c 4 \
  -o gpurun_out/cstep_full_$tag python bench.py --steps 2 --warmup 1 --profile > gpurun_out/ncu_cstep_full_$tag.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:cstep_kernel -s 128 -c 64 --csv \
  --log-file gpurun_out/launches_cstep_$tag.csv python bench.py --steps 4 --warmup 1 --profile > gpurun_out/launch_cstep_$tag.log 2>&1
echo ncu-done
