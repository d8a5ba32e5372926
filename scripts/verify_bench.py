"""Stand-alone timing of the verification kernels (NEXT-4) at the bench shape (for ncu / tuning)."""
import sys
import statistics
sys.path.insert(0, ".")
import torch
import bench
from synth import inputs as S
from paper_2510_13847_b200 import dynaspec as D

C = S.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "llama3"]
B = int(sys.argv[2]) if len(sys.argv) > 2 else 64
dev = torch.device("cuda:0")
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
r = bench.verify_run(D, C, dev, flush, 6988, B=B, reps=int(sys.argv[3]) if len(sys.argv) > 3 else 10)
print(r)
