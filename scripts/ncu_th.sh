#!/bin/bash
# ncu on the balanced tree head (th.cu, Qwen-2.5 tree): --set full of one k = 32 and one k = 8 depth of the
# second cycle (-s skips the first), and the launch list (gpu__time_duration, DRAM bytes) of the router
# and head kernels of a short bench run.  $1 = output tag.
tag=${1:-r2}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:th_kernel -s 6 -c 3 \
  -o gpurun_out/th_full_$tag python bench.py --config qwen25 --steps 2 --warmup 1 --profile --no-graph \
  > gpurun_out/ncu_th_full_$tag.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"th_kernel|meta_" --csv --log-file gpurun_out/launches_qwen_th_$tag.csv \
  python bench.py --config qwen25 --steps 2 --warmup 1 --profile --no-graph > gpurun_out/launch_th_$tag.log 2>&1
echo ncu-done
