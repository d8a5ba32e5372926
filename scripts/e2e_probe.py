"""Where the end-to-end time goes: pinned H2D copy of one cycle's inputs alone, and the e2e graph
(copy + cycle + D2H) vs the device-only cycle (Qwen tree shape)."""
import sys
import time

import torch

sys.path.insert(0, ".")
dev = "cuda"
for nbytes in (196608, 1290240, 16 << 20):
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    for _ in range(3):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        t0 = time.perf_counter()
        d.copy_(h, non_blocking=True)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    ts.sort()
    print(f"H2D {nbytes} B: median {1e6 * ts[10]:.1f} us ({nbytes / ts[10] / 1e9:.1f} GB/s)")
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        d.copy_(h, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s)
    with torch.cuda.graph(g):
        d.copy_(h, non_blocking=True)
    ts = []
    for _ in range(20):
        t0 = time.perf_counter()
        g.replay()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    ts.sort()
    print(f"  in a graph: median {1e6 * ts[10]:.1f} us")
