"""Debug: repeat the exceed-ring exact case and report mismatching top-k rows."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import dynaspec_oracle as O
from synth import inputs as S
from tests.parity import Rows, f64
from paper_2510_13847_b200 import dynaspec as D
DEV = "cuda"
V, d, M, h_r, k_t = int(os.environ.get("V", 9001)), int(os.environ.get("DD", 4096)), 32, 128, 8
W = S.lm_head(V, d, 0, "bf16", "exact")
rt = S.router(d, h_r, M, 1, "bf16", "exact")
tau = S.random_partition(V, M, 2)
perm, off = O.layout(tau, M)
part = {"perm": perm, "offsets": off}
c = D.Clusters.from_tau(W.to(DEV), torch.as_tensor(tau, dtype=torch.int32, device=DEV), M)
r = D.Router(*[None if x is None else x.to(DEV) for x in rt])
Wo, ro = Rows(W), tuple(f64(x) for x in rt)
st = D.DraftStep(c, r, 1, k_t, z_out=True)
bad = 0
for rep in range(int(os.environ.get("REPS", 20))):
    t = rep % 3
    hp, e, hn = S.step_inputs(1, d, t, "bf16", "exact", h_r=h_r)
    st(hp.to(DEV), e.to(DEV), hn.to(DEV), t=t, k_max=8, k_min=2)
    torch.cuda.synchronize()
    ref = O.draft_step(part, ro, Wo, f64(hp), f64(e), f64(hn), t, 8, 2, k_t)[0]
    res = O.epilogue(ref["z"], ref["V_S"], k_t)
    g = st.top_ids[0].cpu().tolist()
    if g != res["top_ids"].tolist():
        bad += 1
        print("rep", rep, "t", t, "gpu", g, "ref", res["top_ids"].tolist())
print("bad", bad)

