#!/bin/bash
# ncu on the cluster step: --set full for a k=32 (cycle positions 0,1) and a k=8 (positions 2,3)
# launch, and the launch list (gpu__time_duration) of a short bench run.
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cstep_kernel -s 8 -c 4 \
  -o gpurun_out/cstep_full_r1 python bench.py --steps 2 --warmup 1 --profile > gpurun_out/ncu_cstep_full.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:cstep_kernel -s 128 -c 64 --csv \
  --log-file gpurun_out/launches_cstep_r1.csv python bench.py --steps 4 --warmup 1 --profile > gpurun_out/launch_cstep.log 2>&1
echo ncu-done
