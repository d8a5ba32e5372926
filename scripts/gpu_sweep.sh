#!/bin/bash
# GPU-box sweep: full gpu test suite + bench lines for the other BASELINE configs.
timeout 1500 python -m pytest tests -m gpu -q -rf --durations=5 2>&1 | tail -20 > gpurun_out/pytest_gpu.log
for c in tiny llama2 qwen25; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
timeout 900 python bench.py --config gemma3 --batch 64 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_gemma3_b64.json 2> gpurun_out/bench_gemma3_b64.err
echo sweep-done
