#!/bin/bash
# Round-end evidence on one GPU: bench lines for every BASELINE config, ncu of the cluster step.
tag=${1:-r1}
timeout 500 python bench.py > gpurun_out/bench_llama3_$tag.json 2> gpurun_out/bench_llama3_$tag.err
for c in tiny llama2 qwen25; do
  timeout 400 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${c}_$tag.json 2> gpurun_out/bench_${c}_$tag.err
done
timeout 600 python bench.py --config gemma3 --batch 64 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_gemma3_b64_$tag.json 2> gpurun_out/bench_gemma3_b64_$tag.err
bash scripts/ncu_cstep.sh $tag
echo artifacts-done
