"""Per-CTA phase marks of the balanced tree head (th.cu) over the Qwen tree cycle (L2 flushed before
the cycle, depths back to back, as trace_tc.py).  Marks: 0 start (before the dependency wait),
1 plan done, 2 streamed + TMEM drained, 3 merge start (merging CTAs), 4 done."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_13847_b200 import dynaspec as D  # noqa: E402
from synth import inputs as S  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "qwen25"
reps = int(os.environ.get("REPS", "10"))
C = S.CONFIGS[cfg]
dev = "cuda"
W = S.lm_head(C.V, C.d, 0, "bf16", device=dev)
tau = torch.as_tensor(S.random_partition(C.V, C.M, 2, zipf=0.0), dtype=torch.int32, device=dev)
c = D.Clusters.from_tau(W, tau, C.M)
r = D.Router(*[x.to(dev) for x in S.router(C.d, C.h_r, C.M, 1, "bf16")])
steps = [D.DraftStep(c, r, C.B, C.k_t, shared=C.shared) for _ in range(C.positions)]
G = torch.cuda.get_device_properties(0).multi_processor_count
bufs = [torch.zeros(G * 64, dtype=torch.int64, device=dev) for _ in range(C.positions)]
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
inp = [[x.to(dev) for x in S.step_inputs(C.B, C.d, t, "bf16", sibling_eps=0.1)] for t in range(C.positions)]
ns = np.zeros((reps, C.positions, G, 64))
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
tot = []
for rep in range(reps + 2):
    if not os.environ.get("NOFLUSH"):
        flush.zero_()
    for bb in bufs:
        bb.zero_()
    torch.cuda.synchronize()
    ev[0].record()
    for t in range(C.positions):
        D.debug_set_trace(bufs[t])
        steps[t](*inp[t], t, C.k_max, C.k_min)
    ev[1].record()
    D.debug_set_trace(None)
    torch.cuda.synchronize()
    if rep >= 2:
        tot.append(ev[0].elapsed_time(ev[1]) * 1e3 / C.positions)
        for t in range(C.positions):
            ns[rep - 2, t] = bufs[t].view(G, 64).cpu().numpy()[:, :64]
print(f"us per step (traced, events): {np.median(tot):.1f}")
for t in range(C.positions):
    print(f"t={t} positions per CTA: max {int(ns[-1, t, :, 12].max())} median {int(np.median(ns[-1, t, :, 12]))}")
names = {0: "start", 13: "released", 14: "sel", 1: "plan", 5: "H", 6: "slot0", 7: "issued", 8: "mma_done", 2: "streamed", 10: "keys", 9: "records", 3: "merge0", 4: "done"}
for t in range(C.positions):
    a = ns[:, t]
    t0 = np.where(a[:, :, 0] > 0, a[:, :, 0], np.inf).min(1)
    line = []
    for sl, nm in names.items():
        x = a[:, :, sl]
        if (x > 0).any():
            mx = np.median([np.max(xx[xx > 0]) - tt for xx, tt in zip(x, t0) if (xx > 0).any()]) / 1e3
            md = np.median([np.median(xx[xx > 0]) - tt for xx, tt in zip(x, t0) if (xx > 0).any()]) / 1e3
            line.append(f"{nm}={mx:.2f}(med {md:.2f})")
    print(f"t={t} k={steps[t].k if hasattr(steps[t], 'k') else ''}: " + " ".join(line))

# router layer 2 (meta_l2_kernel, one CTA per row; slots 16-22), relative to the th kernel's first start
ln = {16: "l2start", 17: "l2wait", 18: "hidden", 19: "scores", 20: "topk", 21: "ticket", 22: "union"}
for t in range(C.positions):
    a = ns[:, t]
    t0 = np.where(a[:, :, 0] > 0, a[:, :, 0], np.inf).min(1)
    line = []
    for sl, nm in ln.items():
        x = a[:, :C.B, sl]
        if (x > 0).any():
            mx = np.median([np.max(xx[xx > 0]) - tt for xx, tt in zip(x, t0) if (xx > 0).any()]) / 1e3
            line.append(f"{nm}={mx:.2f}")
    print(f"t={t} router: " + " ".join(line))

# few-row router (meta_rows_kernel, all CTAs; slots 24-29), relative to the th kernel's first start
ln = {24: "mr_start", 25: "mr_wait", 26: "units", 27: "polled", 28: "topk", 29: "union"}
for t in range(C.positions):
    a = ns[:, t]
    t0 = np.where(a[:, :, 0] > 0, a[:, :, 0], np.inf).min(1)
    line = []
    for sl, nm in ln.items():
        x = a[:, :, sl]
        if (x > 0).any():
            mx = np.median([np.max(xx[xx > 0]) - tt for xx, tt in zip(x, t0) if (xx > 0).any()]) / 1e3
            mn = np.median([np.min(xx[xx > 0]) - tt for xx, tt in zip(x, t0) if (xx > 0).any()]) / 1e3
            line.append(f"{nm}={mn:.2f}..{mx:.2f}")
    print(f"t={t} few-row router: " + " ".join(line))

# SM-clock cycles between router marks in the row CTAs (CTA b < B): poll->topk, topk->end
for t in range(C.positions):
    a = ns[-1, t, :C.B]
    print(f"t={t} row CTAs cycles: wait->units {np.median(a[:, 58] - a[:, 57]):.0f} units->polled {np.median(a[:, 59] - a[:, 58]):.0f} "
          f"polled->topk {np.median(a[:, 60] - a[:, 59]):.0f}; union CTA topk?->union: {a[0, 61] - a[0, 60]:.0f}")
# effective SM clock in the merger CTAs (clock64 / globaltimer between marks 3 and 4), and cycles per phase
for t in range(C.positions):
    a = ns[-1, t]
    mc = np.where(a[:, 3] > 0)[0]
    if len(mc):
        dc = a[mc, 32 + 4] - a[mc, 32 + 3]
        dt = a[mc, 4] - a[mc, 3]
        print(f"t={t} mergers: cycles {np.median(dc):.0f} in {np.median(dt):.0f} ns -> {np.median(dc / np.maximum(dt, 1)):.2f} GHz;"
              f" keys->records cycles (all CTAs) {np.median(a[:, 32 + 9] - a[:, 32 + 10]):.0f}")
for t in range(C.positions):
    a = ns[-1, t]
    mc = np.where(a[:, 3] > 0)[0]
    if len(mc):
        c = lambda x, y: np.median(a[mc, 32 + y] - a[mc, 32 + x])
        print(f"t={t} merger cycles: start->staged {c(3, 5):.0f} staged->heads {c(5, 6):.0f} heads->cands {c(6, 7):.0f} cands->done {c(7, 4):.0f}")
