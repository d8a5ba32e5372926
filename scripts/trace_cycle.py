"""Per-phase timeline of every step of one draft cycle (flush L2 once, then t = 0..gamma-1
back to back, as in bench.py)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_13847_b200 import dynaspec as D  # noqa: E402
from synth import inputs as S  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "llama3"
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
names = ["start", "pdl", "phaseA", "sel_vis", "segs", "streamed", "partials", "merged", "B:ctrA", "B:w2", "B:pub",
         "B:hid", "B:out", "B:rank", "ticket", "ticket+1", "M:load",
         "M:lse", "M:thr", "M:surv", "M:done"]
CSTEP = os.environ.get("DS_CLUSTER_Q", "16") != "0"
if CSTEP:  # cluster step (cstep.cu) mark slots
    names = ["start", "pdl", "L1done", "-", "stream0", "streamed", "-", "merged", "a1_bar", "cta_rec",
             "-", "-", "sc_bar", "mask", "recs_seen", "T2", "-", "-", "-", "-", "-"]
inp = [[x.to(dev) for x in S.step_inputs(1, C.d, t, "bf16")] for t in range(C.positions)]
for rep in range(3):
    flush.zero_()
    for b in bufs:
        b.zero_()
    torch.cuda.synchronize()
    for t in range(C.positions):
        D.debug_set_trace(bufs[t])
        steps[t](*inp[t], t, C.k_max, C.k_min)
    D.debug_set_trace(None)
    torch.cuda.synchronize()
t_prev_end = None
for t in range(C.positions):
    a = bufs[t].view(G, 64).cpu().numpy().astype(np.float64)[:, :32]
    t0 = a[:, 0][a[:, 0] > 0].min()
    print(f"t={t} k={D.budget(t, C.k_max, C.k_min)}" + (f"  gap since previous merge {1e-3*(t0-t_prev_end):.2f} us"
                                                       if t_prev_end else ""))
    for i, n in enumerate(names):
        col = a[:, i]
        col = col[col > 0]
        if col.size and n != "-":
            print(f"  {n:9s} n={col.size:3d} min={1e-3*(col.min()-t0):8.2f} med={1e-3*(np.median(col)-t0):8.2f} "
                  f"max={1e-3*(col.max()-t0):8.2f} us")
    cy = bufs[t].view(G, 64).cpu().numpy().astype(np.float64)[:, 32:]
    last = np.argmax(a[:, 7])
    if CSTEP:  # cluster step: per-CTA SM-cycle deltas from 'start' (median over CTAs)
        ok = cy[:, 0] > 0
        print("  median SM cycles since start:", {n: int(np.median(cy[ok & (cy[:, i] > 0), i] - cy[ok & (cy[:, i] > 0), 0]))
                                                  for i, n in enumerate(names) if n != "-" and (cy[ok, i] > 0).any()})
    if not CSTEP:
        print("  last-CTA cycles between marks:", {names[i]: int(cy[last, i] - cy[last, 14])
                                                   for i in (15, 16, 17, 19, 20, 7) if cy[last, i] > 0})
    t_prev_end = a[:, 7][a[:, 7] > 0].max()
