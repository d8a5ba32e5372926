"""Device time of the router + selection (dynaspec_step_route) and of the union for B rows at a
config's shape: CUDA events around 50 back-to-back calls (async launches; no host sync inside)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_13847_b200 import dynaspec as D  # noqa: E402
from synth import inputs as S  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "gemma3"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 64
C = S.CONFIGS[cfg]
dev = "cuda"
W = S.lm_head(C.V, C.d, 0, "bf16", device=dev)
tau = torch.as_tensor(S.random_partition(C.V, C.M, 2, zipf=0.0), dtype=torch.int32, device=dev)
c = D.Clusters.from_tau(W, tau, C.M)
r = D.Router(*[x.to(dev) for x in S.router(C.d, C.h_r, C.M, 1, "bf16")])
st = D.DraftStep(c, r, B, C.k_t, shared=C.shared, two_streams=True)
hp, e, hn = [x.to(dev) for x in S.step_inputs(B, C.d, 3, "bf16")]
s = torch.cuda.current_stream()
for t in (0, 2):
    for _ in range(5):
        st.route(hp, e, t, C.k_max, C.k_min, s)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(50):
        st.route(hp, e, t, C.k_max, C.k_min, s)
    b.record()
    torch.cuda.synchronize()
    print(f"{cfg} B={B} t={t}: router + select {a.elapsed_time(b) * 1e3 / 50:.1f} us per call")
