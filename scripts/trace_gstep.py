"""Per-phase timeline of every step of one draft cycle of the grid step (gstep.cu), flushed L2 once
per cycle, t = 0..gamma-1 back to back (PDL-chained in one CUDA graph, as in bench.py).

Marks (gstep.cu trace_mark slots): 0 start, 1 after the PDL wait, 2 layer-1 unit published,
3 all units polled, 4 layer 2 done, 5 TopK mask ready (streaming starts), 6 consumers done,
7 record written, 8 merger: all records in, 9 outputs written (CTA 0)."""
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
del W
r = D.Router(*[x.to(dev) for x in S.router(C.d, C.h_r, C.M, 1, "bf16")])
steps = [D.DraftStep(c, r, 1, C.k_t) for _ in range(C.positions)]
G = torch.cuda.get_device_properties(0).multi_processor_count
bufs = [torch.zeros(G * 64, dtype=torch.int64, device=dev) for _ in range(C.positions)]
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import L2Flush  # noqa: E402
flush = L2Flush(dev)
names = ["start", "pdl", "L1pub", "a_in", "layer2", "mask", "streamed", "record", "recs_in", "out", "M:fields", "M:cands",
         "-", "tk:thr", "tk:surv", "M:issued"]
inp = [[x.to(dev) for x in S.step_inputs(1, C.d, t, "bf16")] for t in range(C.positions)]


def cycle():
    for t in range(C.positions):
        D.debug_set_trace(bufs[t])
        steps[t](*inp[t], t, C.k_max, C.k_min)
    D.debug_set_trace(None)


s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    cycle()
torch.cuda.current_stream().wait_stream(s)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    cycle()
tot = []
for rep in range(5):
    flush.zero_()
    for b in bufs:
        b.zero_()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    tot.append(e0.elapsed_time(e1) * 1e3 / C.positions)
print(f"{cfg}: us per step (events, traced) {np.round(tot, 2)}")
t_prev_end = None
ends = []
for t in range(C.positions):
    a = bufs[t].view(G, 64).cpu().numpy().astype(np.float64)[:, :32]
    p1 = a[:, 1][a[:, 1] > 0]
    mg = int(np.argmax(a[:, 9]))
    ends.append((p1.min(), p1.max(), a[:, 9].max(), a[:, 5][a[:, 5] > 0].min(), a[:, 6].max(), a[:, 7].max(),
                 a[mg, 15], a[mg, 8], a[mg, 10], a[mg, 11]))
print("per step (us): pdl release (first..last CTA) -> mask | -> streamed (last) | -> last record | -> outputs | -> next pdl")
for t in range(C.positions):
    p0, p1, out, mk, sd, rc, mi, mr, mf, mc = ends[t]
    nxt = ends[t + 1][0] if t + 1 < C.positions else float("nan")
    print(f"  t={t}: merger candidates {int(bufs[t].view(G, 64)[:, 29].max().item())} |"
          f" pdl spread {1e-3 * (p1 - p0):.2f} | mask {1e-3 * (mk - p0):.2f} | streamed {1e-3 * (sd - p0):.2f} | "
          f"record {1e-3 * (rc - p0):.2f} | merger: headers+issued {1e-3 * (mi - p0):.2f} staged {1e-3 * (mr - p0):.2f} "
          f"fields {1e-3 * (mf - p0):.2f} cands {1e-3 * (mc - p0):.2f} | out {1e-3 * (out - p0):.2f} | next pdl {1e-3 * (nxt - p0):.2f}")
for t in range(C.positions):
    a = bufs[t].view(G, 64).cpu().numpy().astype(np.float64)[:, :32]
    t0 = a[:, 0][a[:, 0] > 0].min()
    cnt = steps[t].sel_count[0].item()
    rows = steps[t].sl_offsets[0, cnt].item()
    print(f"t={t} k={D.budget(t, C.k_max, C.k_min)} |V_S|={rows} ({rows * C.d * 2 / 1e6:.1f} MB)" +
          (f"  prev outputs -> this start {1e-3 * (t0 - t_prev_end):.2f} us" if t_prev_end else ""))
    for i, n in enumerate(names):
        col = a[:, i]
        col = col[col > 0]
        if col.size and n != "-":
            print(f"  {n:9s} n={col.size:3d} min={1e-3 * (col.min() - t0):8.2f} med={1e-3 * (np.median(col) - t0):8.2f} "
                  f"max={1e-3 * (col.max() - t0):8.2f} us")
    cy = bufs[t].view(G, 64).cpu().numpy().astype(np.float64)[:, 32:]
    seq = [0, 1, 2, 3, 4, 13, 14, 5, 6, 7]
    ok = cy[:, 0] > 0
    print("  median SM cycles between marks:",
          {f"{names[i]}->{names[j]}": int(np.median(cy[ok, j] - cy[ok, i])) for i, j in zip(seq, seq[1:])})
    print("  one trace mark costs", int(np.median(cy[ok, 17] - cy[ok, 16])), "SM cycles")
    m0 = int(np.argmax(a[:, 9]))
    mseq = [7, 15, 8, 10, 11, 9]
    print("  merger CTA cycles:", {f"{names[i]}->{names[j]}": int(cy[m0, j] - cy[m0, i]) for i, j in zip(mseq, mseq[1:])})
    ok2 = (a[:, 5] > 0) & (a[:, 12] > 0) & (a[:, 18] > 0)
    if ok2.any():
        q = lambda v: np.round(1e-3 * np.percentile(v, [0, 50, 90, 100]), 2)
        print("  per CTA (us, p0/p50/p90/max): mask->1st landed", q(a[ok2, 12] - a[ok2, 5]),
              "| mask->last issued", q(a[ok2, 18] - a[ok2, 5]), "| mask->streamed", q(a[ok2, 6] - a[ok2, 5]),
              "| mask skew", q(a[ok2, 5] - a[ok2, 5].min()))
    st0, st1 = a[:, 5][a[:, 5] > 0].min(), a[:, 6][a[:, 6] > 0].max()
    print(f"  streaming: {rows * C.d * 2 / (st1 - st0):.0f} GB/s over [first mask, last streamed]")
    t_prev_end = a[:, 9][a[:, 9] > 0].max()
