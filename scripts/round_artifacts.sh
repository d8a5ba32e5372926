#!/bin/bash
# Round-end bench lines on one GPU for every BASELINE config (+ the Llama-3 batch sweep) -> gpurun_out/.
tag=${1:-r2}
for c in tiny llama2 qwen25; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${c}_$tag.json 2> gpurun_out/bench_${c}_$tag.err
done
timeout 900 python bench.py --config gemma3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_gemma3_b512_$tag.json 2> gpurun_out/bench_gemma3_b512_$tag.err
for B in 2 4 8 16 32 64; do
  timeout 600 python bench.py --batch $B --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_llama3_b${B}_$tag.json 2> gpurun_out/bench_llama3_b${B}_$tag.err
done
echo artifacts-done
