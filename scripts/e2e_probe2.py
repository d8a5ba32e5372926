"""Qwen tree cycle: device time with separate input tensors vs slices of one [P, 3, B, d] tensor
(the e2e layout), and with outputs bound into one buffer."""
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2510_13847_b200 import dynaspec as D  # noqa: E402
from synth import inputs as S  # noqa: E402

C = S.CONFIGS["qwen25"]
dev = "cuda"
W = S.lm_head(C.V, C.d, 0, "bf16", device=dev)
tau = torch.as_tensor(S.random_partition(C.V, C.M, 2), dtype=torch.int32, device=dev)
c = D.Clusters.from_tau(W, tau, C.M)
r = D.Router(*[x.to(dev) for x in S.router(C.d, C.h_r, C.M, 1, "bf16")])
P, B = C.positions, C.B
st = [D.DraftStep(c, r, B, C.k_t, shared=True) for _ in range(P)]
sep = [[x.to(dev) for x in S.step_inputs(B, C.d, t, "bf16", sibling_eps=0.1)] for t in range(P)]
packed = torch.stack([torch.stack(sep[t]) for t in range(P)]).contiguous()  # [P, 3, B, d]
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)


def run(mode):
    for t in range(P):
        hp, e, hn = (sep[t] if mode == "sep" else (packed[t, 0], packed[t, 1], packed[t, 2]))
        st[t](hp, e, hn, t, C.k_max, C.k_min)


for mode in ("sep", "packed", "sep", "packed"):
    ts = []
    for i in range(8):
        flush.zero_()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        run(mode)
        b.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(a.elapsed_time(b))
    ts.sort()
    print(mode, f"{1e3 * ts[len(ts) // 2] / P:.1f} us per step (no graph)")

# graphs: cycle only / H2D + cycle / H2D + cycle + D2H (the e2e graph)
host_in = packed.cpu().pin_memory()
dev_out = torch.empty((P, 2, B, C.k_t), dtype=torch.int32, device=dev)
host_out = torch.empty((P, 2, B, C.k_t), dtype=torch.int32).pin_memory()
for t, s_ in enumerate(st):
    s_.bind_outputs(top_ids=dev_out[t, 0], top_logp=dev_out[t, 1].view(torch.float32))


def body(h2d, d2h):
    if h2d:
        packed.copy_(host_in, non_blocking=True)
    run("packed")
    if d2h:
        host_out.copy_(dev_out, non_blocking=True)


for h2d, d2h in ((False, False), (True, False), (True, True), (False, True)):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        body(h2d, d2h)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        body(h2d, d2h)
    ts = []
    for i in range(8):
        flush.zero_()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(a.elapsed_time(b))
    ts.sort()
    print(f"graph h2d={h2d} d2h={d2h}: {1e3 * ts[len(ts) // 2] / P:.1f} us per step")

# two e2e graphs replayed alternately (the bench's e2e loop) vs one graph
gs = []
for i in range(2):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        body(True, True)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        body(True, True)
    gs.append(g)
for alt in (False, True):
    ts = []
    for i in range(10):
        flush.zero_()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        (gs[i % 2] if alt else gs[0]).replay()
        b.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(a.elapsed_time(b))
    ts.sort()
    print(f"e2e graphs alternate={alt}: {1e3 * ts[len(ts) // 2] / P:.1f} us per step")
