"""Eager draft steps at one configuration (for ncu / compute-sanitizer): `n` steps cycling the
positions t = 0..gamma-1 of the config's k schedule.  Usage: run_steps.py [config] [n] [dtype]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_13847_b200 import dynaspec as D  # noqa: E402
from synth import inputs as S  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "llama3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 16
dt = sys.argv[3] if len(sys.argv) > 3 else "bf16"
C = S.CONFIGS[cfg]
dev = "cuda"
W = S.lm_head(C.V, C.d, 0, dt, device=dev)
tau = torch.as_tensor(S.random_partition(C.V, C.M, 2, zipf=0.0), dtype=torch.int32, device=dev)
c = D.Clusters.from_tau(W, tau, C.M)
del W
r = D.Router(*[None if x is None else x.to(dev) for x in S.router(C.d, C.h_r, C.M, 1, dt)])
B = int(os.environ.get("DS_RUN_B", C.B))
steps = [D.DraftStep(c, r, B, C.k_t, shared=C.shared) for _ in range(C.positions)]
inp = [[x.to(dev) for x in S.step_inputs(B, C.d, t, dt)] for t in range(C.positions)]
for i in range(n):
    t = i % C.positions
    steps[t](*inp[t], t, C.k_max, C.k_min)
torch.cuda.synchronize()
print("ok", cfg, n, "steps;", [st.ws.error() for st in steps[:1]])
