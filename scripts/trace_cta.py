"""Raw per-CTA phase marks of the cluster step over many draft cycles (flush L2, then t = 0..gamma-1
back to back, as in bench.py), saved as an .npz for offline analysis (scripts/trace_cta_report.py).

Array `ns[rep, t, cta, slot]` = %globaltimer, `cy[rep, t, cta, slot]` = clock64, `sm[rep, t, cta]` =
SM id (slot 31 of the trace, written at mark 0)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_13847_b200 import dynaspec as D  # noqa: E402
from synth import inputs as S  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "llama3"
out = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/trace_cta.npz"
reps = int(os.environ.get("REPS", "20"))
C = S.CONFIGS[cfg]
dev = "cuda"
W = S.lm_head(C.V, C.d, 0, "bf16", device=dev)
tau = torch.as_tensor(S.random_partition(C.V, C.M, 2, zipf=0.0), dtype=torch.int32, device=dev)
c = D.Clusters.from_tau(W, tau, C.M)
r = D.Router(*[x.to(dev) for x in S.router(C.d, C.h_r, C.M, 1, "bf16")])
steps = [D.DraftStep(c, r, 1, C.k_t) for _ in range(C.positions)]
G = torch.cuda.get_device_properties(0).multi_processor_count
bufs = [torch.zeros(G * 64, dtype=torch.int64, device=dev) for _ in range(C.positions)]
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
inp = [[x.to(dev) for x in S.step_inputs(1, C.d, t, "bf16")] for t in range(C.positions)]
ns = np.zeros((reps, C.positions, G, 32))
cy = np.zeros((reps, C.positions, G, 32))
sm = np.zeros((reps, C.positions, G), dtype=np.int64)
for rep in range(reps + 2):
    flush.zero_()
    for b in bufs:
        b.zero_()
    torch.cuda.synchronize()
    for t in range(C.positions):
        D.debug_set_trace(bufs[t])
        steps[t](*inp[t], t, C.k_max, C.k_min)
    D.debug_set_trace(None)
    torch.cuda.synchronize()
    if rep >= 2:
        for t in range(C.positions):
            a = bufs[t].view(G, 64).cpu().numpy()
            ns[rep - 2, t] = a[:, :32]
            cy[rep - 2, t] = a[:, 32:]
            sm[rep - 2, t] = a[:, 31] - 1
os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
np.savez_compressed(out, ns=ns, cy=cy, sm=sm, k=np.array([D.budget(t, C.k_max, C.k_min) for t in range(C.positions)]))
print("saved", out, ns.shape)
