"""Per-CTA phase marks of the tcgen05 shared-shortlist head (tc_head.cu) over the Qwen tree cycle
(flush L2, then the gamma depths back to back), saved for offline analysis.  Marks: 0 start,
1 setup (segments + boxes), 2 producer issued all, 3 last MMA committed, 4 epilogue tiles done,
5 block sync, 6 per-CTA partials, 7 merge done; slot 29 = tiles of the CTA."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_13847_b200 import dynaspec as D  # noqa: E402
from synth import inputs as S  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "qwen25"
out = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/trace_tc.npz"
reps = int(os.environ.get("REPS", "10"))
C = S.CONFIGS[cfg]
B = int(os.environ.get("B", C.B))
dev = "cuda"
W = S.lm_head(C.V, C.d, 0, "bf16", device=dev)
tau = torch.as_tensor(S.random_partition(C.V, C.M, 2, zipf=0.0), dtype=torch.int32, device=dev)
c = D.Clusters.from_tau(W, tau, C.M)
r = D.Router(*[x.to(dev) for x in S.router(C.d, C.h_r, C.M, 1, "bf16")])
steps = [D.DraftStep(c, r, B, C.k_t, shared=C.shared) for _ in range(C.positions)]
G = torch.cuda.get_device_properties(0).multi_processor_count
bufs = [torch.zeros(G * 64, dtype=torch.int64, device=dev) for _ in range(C.positions)]
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
inp = [[x.to(dev) for x in S.step_inputs(B, C.d, t, "bf16", sibling_eps=0.1 if C.shared else None)]
       for t in range(C.positions)]
ns = np.zeros((reps, C.positions, G, 32))
for rep in range(reps + 2):
    flush.zero_()
    for b in bufs:
        b.zero_()
    torch.cuda.synchronize()
    for t in range(C.positions):
        D.debug_set_trace(bufs[t])
        kmax = int(os.environ.get("KMAX", C.k_max))
        steps[t](*inp[t], t, kmax, min(kmax, int(os.environ.get("KMIN", C.k_min))))
    D.debug_set_trace(None)
    torch.cuda.synchronize()
    if rep >= 2:
        for t in range(C.positions):
            ns[rep - 2, t] = bufs[t].view(G, 64).cpu().numpy()[:, :32]
np.savez_compressed(out, ns=ns)
names = {0: "start", 1: "setup", 2: "issued", 3: "mma_done", 4: "epi_done", 5: "sync", 6: "partials", 7: "merged"}
for t in range(C.positions):
    a = ns[:, t]
    t0 = np.where(a[:, :, 0] > 0, a[:, :, 0], np.inf).min(1)
    line = []
    for sl, n in names.items():
        x = a[:, :, sl]
        if (x > 0).any():
            line.append(f"{n}={np.median(np.where(x > 0, x, -np.inf).max(1) - t0) / 1e3:.1f}"
                        f"(med {np.median([np.median(xx[xx > 0]) - tt for xx, tt in zip(x, t0) if (xx > 0).any()]) / 1e3:.1f})")
    print(f"t={t} tiles/CTA max {int(a[0, :, 29].max())}: " + " ".join(line))
print("online epilogue cycles per CTA (median over CTAs, last rep): wait, stage, rows:",
      [np.median(ns[-1, t, :, 20:23], axis=0).astype(int).tolist() for t in range(C.positions)])
# merge phases of the merging CTAs (marks 6 partials, 16 staged, 17 lse, 19 top-k, 20 row done)
for t in range(C.positions):
    a = ns[-1, t]
    mcta = np.where(a[:, 16] > 0)[0]
    if len(mcta):
        d = lambda x, y: np.median(a[mcta, y] - a[mcta, x]) / 1e3
        print(f"t={t} merge CTAs {len(mcta)}: partials->staged {d(6,16):.2f} staged->lse {d(16,17):.2f} "
              f"lse->topk {d(17,19):.2f} topk->done {d(19,20):.2f} us; last partial -> first staged "
              f"{(a[mcta,16].min() - a[:,6].max())/1e3:.2f} us")
