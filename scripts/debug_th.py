"""Debug: th.cu logits vs the oracle for one shared selection; prints the mismatching positions."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import dynaspec_oracle as O  # noqa: E402
from paper_2510_13847_b200 import dynaspec as Dy  # noqa: E402
from synth import inputs as S  # noqa: E402

R, d, V, M, k = [int(x) for x in (sys.argv[1:] + ["4", "256", "6007", "24", "24"])[:5]]
os.environ["DS_DISABLE_TC"] = "0"
q = max(1, min(127, int((2 ** 21 / d) ** 0.5)))
W = S.lm_head(V, d, 0, "bf16", "exact", q=q)
tau = S.random_partition(V, M, 2)
perm, off = O.layout(tau, M)
c = Dy.Clusters.from_tau(W.cuda(), torch.as_tensor(tau, dtype=torch.int32, device="cuda"), M)
hn = S.hidden(R, d, 11, "bf16", "exact", q=q)
sel = np.sort(np.random.default_rng(R).choice(M, k, replace=False)).astype(np.int32)
selt = torch.zeros((1, M), dtype=torch.int32)
selt[0, :k] = torch.as_tensor(sel)
offs = torch.zeros((1, M + 1), dtype=torch.int32)
offs[0, :k + 1] = torch.as_tensor(O.shortlist_offsets(sel, off), dtype=torch.int32)
cnt = torch.tensor([k], dtype=torch.int32)
out = Dy.head_forward(c, hn.cuda(), selt.cuda(), cnt.cuda(), offs.cuda(), 8, shared=True, z_out=True)
V_S = O.shortlist(sel, perm, off)
zref = O.head(hn.double().numpy(), W.double().numpy(), V_S)
n = len(V_S)
sizes = np.diff(off)[sel]
print("cluster sizes", sizes.tolist(), "n", n)
for r in range(R):
    z = out["z"][r, :n].cpu().numpy()
    bad = np.nonzero(z != zref[r].astype(np.float32))[0]
    print(f"row {r}: {len(bad)} bad; first {bad[:20].tolist()}")
    if len(bad):
        print("   gpu", z[bad[:5]].tolist(), "ref", zref[r][bad[:5]].tolist())
