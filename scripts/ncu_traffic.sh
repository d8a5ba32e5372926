#!/bin/bash
# ncu --set full on the fused step for a k=32 (cycle positions 0,1) and a k=8 (positions 2,3) launch.
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 8 -c 4 \
  -o gpurun_out/step_full_r1 python bench.py --steps 2 --warmup 1 --profile > gpurun_out/ncu_r1.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"step_kernel|head_kernel|meta_l|tc_head|union" \
  -c 64 --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 4 --warmup 1 --profile > gpurun_out/launch_r1.log 2>&1
echo ncu-done
