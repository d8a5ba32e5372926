"""One small invocation of one kernel path, for compute-sanitizer (scripts/sanitize.sh runs every
case under memcheck, racecheck, synccheck and initcheck).  Usage: sanitize_cases.py CASE

Cases: gstep (B = 1 grid step), gstep_head (head-only grid step), cstep (B = 1 cluster step),
step (grid-wide fused step, B = 4), head (head_forward B = 3), tc_tree (few-row router + balanced tree
head, 10 rows; tc_tree_z with z_out; tc_tree_old: the general tcgen05 shared head + split-K router),
tc_batched (tcgen05 batched head, 16 rows), gh (grouped tcgen05 head, 16 rows), gh_wide (160 rows:
tcgen05 router layer 1 + grid-wide grouping + grouped head), verify (verify_chain), build (k-means build)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_13847_b200 import dynaspec as D  # noqa: E402
from synth import inputs as S  # noqa: E402

case = sys.argv[1]
dev = "cuda"
V, d, M, h_r = 4099, 256, 32, 16
W = S.lm_head(V, d, 0, "bf16").to(dev)
tau = torch.as_tensor(S.random_partition(V, M, 2), dtype=torch.int32, device=dev)
c = D.Clusters.from_tau(W, tau, M)
r = D.Router(*[x.to(dev) for x in S.router(d, h_r, M, 1, "bf16")])


def steps(B, shared=False, two=False, n=3, z_out=None):
    st = D.DraftStep(c, r, B, 4, shared=shared, two_streams=two, z_out=(not shared) if z_out is None else z_out)
    for t in range(n):
        hp, e, hn = [x.to(dev) for x in S.step_inputs(B, d, t, "bf16")]
        st(hp, e, hn, t, 8, 2)
    torch.cuda.synchronize()
    return st


if case == "gstep":
    st = steps(1)
elif case == "gstep_head":
    st = steps(1, two=True)
elif case == "cstep":
    os.environ["DS_GSTEP"] = "0"
    st = steps(1)
elif case == "step":
    os.environ["DS_GSTEP"] = "0"
    os.environ["DS_CLUSTER_Q"] = "0"
    st = steps(4)
elif case == "head":
    sel = torch.arange(M, dtype=torch.int32, device=dev).repeat(3, 1).contiguous()
    cnt = torch.full((3,), M, dtype=torch.int32, device=dev)
    off = c.offsets.repeat(3, 1).contiguous()
    hn = S.hidden(3, d, 5, "bf16").to(dev)
    D.head_forward(c, hn, sel, cnt, off, 8)
    torch.cuda.synchronize()
elif case == "tc_tree":
    st = steps(10, shared=True)          # few-row router (meta_rows.cu) + balanced tree head (th.cu)
    assert st.kernel.startswith("ds::th_kernel"), st.kernel
elif case == "tc_tree_z":
    st = steps(10, shared=True, z_out=True)   # tree head writing the caller's z_out
elif case == "tc_tree_old":
    os.environ["DS_TH"] = "0"
    os.environ["DS_META_ROWS"] = "0"
    st = steps(10, shared=True)          # general tcgen05 shared head + split-K router
elif case == "tc_batched":
    st = steps(16)
elif case == "gh":
    st = steps(16, z_out=False)          # grouped cluster-major tcgen05 head, one-CTA grouping
    assert st.kernel.startswith("ds::gh_head_kernel"), st.kernel
elif case == "gh_wide":
    st = steps(160, z_out=False, n=2)    # + router layer 1 on tcgen05 (B >= 32), grid-wide grouping
    assert st.kernel.startswith("ds::gh_head_kernel") and st.launches == 7, (st.kernel, st.launches)
elif case == "verify":
    B, gam, n_short = 4, 3, 64
    vi = S.verify_inputs(B, gam, 1024, n_short)
    ver = D.Verifier(1024, B, gam, dev)
    ids = vi["q_ids"].to(dev)
    ql = vi["q_logits"].to(dev)
    lse = torch.logsumexp(ql, -1).contiguous()
    x = ids[:, :, 0].contiguous()
    slot = torch.zeros((B, gam), dtype=torch.int32, device=dev)
    cnt = torch.full((B, gam), n_short, dtype=torch.int32, device=dev)
    ver(vi["p_logits"].to(dev), ids, ql, cnt, lse, x, slot, vi["u_acc"].to(dev), vi["u_res"].to(dev))
    torch.cuda.synchronize()
elif case == "build":
    D.Clusters.build(W, M, seed=2, max_iters=4)
    torch.cuda.synchronize()
else:
    raise SystemExit(f"unknown case {case}")
print("case", case, "ok")
