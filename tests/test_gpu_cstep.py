"""GPU parity of the cluster draft step (cstep.cu: B = 1, router per thread-block cluster, DSMEM
exchanges, online per-warp top-k / log-sum-exp, three-level list merge) against the CPU oracle.

The exact regime (integer-grid inputs) makes every fp32 dot product exact in any
summation order, so scores, selections, offsets, every shortlist logit and the top-k_t ids and
logits must be bit-identical to the oracle's, whatever the cluster size Q (DS_CLUSTER_Q; 0 = the
grid-wide step.cu kernel).  The random regime is checked at the Llama-3 head's full size.
"""
import numpy as np
import pytest
import torch

from oracle import dynaspec_oracle as O
from synth import inputs as S
from tests.parity import Rows, check_topk, f64, score_tol, selection_certified

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _cluster_step_only(monkeypatch):
    """These tests exercise cstep.cu: keep the grid step (gstep.cu) out of the dispatch."""
    monkeypatch.setenv("DS_GSTEP", "0")


DEV = "cuda"


def _dyn():
    from paper_2510_13847_b200 import dynaspec
    return dynaspec


def _setup(V, d, M, h_r, dtype, regime, seed_part=2):
    D = _dyn()
    W = S.lm_head(V, d, 0, dtype, regime)
    rt = S.router(d, h_r, M, 1, dtype, regime)
    tau = S.random_partition(V, M, seed_part)
    perm, off = O.layout(tau, M)
    c = D.Clusters.from_tau(W.to(DEV), torch.as_tensor(tau, dtype=torch.int32, device=DEV), M)
    r = D.Router(*[None if x is None else x.to(DEV) for x in rt])
    return W, rt, {"perm": perm, "offsets": off}, c, r


@pytest.mark.parametrize("Q", ["16", "8", "4", "2", "1", "0"])
@pytest.mark.parametrize("dtype,h_r,k_t", [("bf16", 16, 8), ("f32", 16, 1), ("bf16", 0, 32), ("f32", 8, 32)])
@pytest.mark.parametrize("k_max,k_min", [(16, 4), (40, 33)])  # k <= 32 and k > 32 up to k = M
def test_cluster_step_exact_bit_exact(Q, dtype, h_r, k_t, k_max, k_min, monkeypatch):
    monkeypatch.setenv("DS_CLUSTER_Q", Q)
    D = _dyn()
    V, d, M = 7919, 384, 40     # prime V, ragged clusters, M not a multiple of Q
    W, rt, part, c, r = _setup(V, d, M, h_r, dtype, "exact")
    Wo, ro = Rows(W), tuple(f64(x) for x in rt)
    st = D.DraftStep(c, r, 1, k_t, z_out=True)
    assert st.launches == 1
    for t in range(4):
        hp, e, hn = S.step_inputs(1, d, t, dtype, "exact", h_r=h_r)
        st(hp.to(DEV), e.to(DEV), hn.to(DEV), t=t, k_max=k_max, k_min=k_min)
        torch.cuda.synchronize()
        ref = O.draft_step(part, ro, Wo, f64(hp), f64(e), f64(hn), t, k_max, k_min, k_t)[0]
        assert np.array_equal(st.scores[0].cpu().numpy(), ref["scores"].astype(np.float32)), "scores"
        cnt = st.sel_count[0].item()
        assert st.sel[0, :cnt].cpu().tolist() == ref["sel"].tolist()
        assert st.sl_offsets[0, :cnt + 1].cpu().tolist() == ref["sl_offsets"].tolist()
        n = len(ref["V_S"])
        assert np.array_equal(st.z[0, :n].cpu().numpy(), ref["z"].astype(np.float32)), "logits"
        check_topk(st.top_ids[0].cpu().numpy(), st.top_logits[0].cpu().numpy(), st.top_logp[0].cpu().numpy(),
                   st.lse[0].item(), ref["z"], ref["V_S"], k_t, torch.float32, exact=True)


@pytest.mark.parametrize("Q", ["16", "2"])
def test_cluster_step_router_rows_exceed_ring(Q, monkeypatch):
    """Q = 2 with h_r = 128 at d = 4096: each CTA's W1 slice (64 rows, 1 MB) cycles the TMA ring
    several times before the head reuses it (producer/consumer phase bookkeeping)."""
    monkeypatch.setenv("DS_CLUSTER_Q", Q)
    D = _dyn()
    V, d, M, h_r, k_t = 9001, 4096, 32, 128, 8
    W, rt, part, c, r = _setup(V, d, M, h_r, "bf16", "exact")
    Wo, ro = Rows(W), tuple(f64(x) for x in rt)
    st = D.DraftStep(c, r, 1, k_t, z_out=True)
    for t in range(3):
        hp, e, hn = S.step_inputs(1, d, t, "bf16", "exact", h_r=h_r)
        st(hp.to(DEV), e.to(DEV), hn.to(DEV), t=t, k_max=8, k_min=2)
        torch.cuda.synchronize()
        ref = O.draft_step(part, ro, Wo, f64(hp), f64(e), f64(hn), t, 8, 2, k_t)[0]
        assert np.array_equal(st.scores[0].cpu().numpy(), ref["scores"].astype(np.float32))
        cnt = st.sel_count[0].item()
        assert st.sel[0, :cnt].cpu().tolist() == ref["sel"].tolist()
        n = len(ref["V_S"])
        assert np.array_equal(st.z[0, :n].cpu().numpy(), ref["z"].astype(np.float32))
        check_topk(st.top_ids[0].cpu().numpy(), st.top_logits[0].cpu().numpy(), st.top_logp[0].cpu().numpy(),
                   st.lse[0].item(), ref["z"], ref["V_S"], k_t, torch.float32, exact=True)


def test_cluster_step_llama3_random_full_size(monkeypatch):
    """Llama-3 head (V 128256, d 4096, M 256, h_r 128) at k = 32 and 8, random regime, bf16."""
    monkeypatch.setenv("DS_CLUSTER_Q", "16")
    D = _dyn()
    C = S.CONFIGS["llama3"]
    W, rt, part, c, r = _setup(C.V, C.d, C.M, C.h_r, "bf16", "random")
    Wo, ro = Rows(W), tuple(f64(x) for x in rt)
    st = D.DraftStep(c, r, 1, C.k_t, z_out=True)
    for t in (0, 2, 5):
        hp, e, hn = S.step_inputs(1, C.d, t, "bf16")
        st(hp.to(DEV), e.to(DEV), hn.to(DEV), t=t, k_max=C.k_max, k_min=C.k_min)
        torch.cuda.synchronize()
        ref = O.draft_step(part, ro, Wo, f64(hp), f64(e), f64(hn), t, C.k_max, C.k_min, C.k_t)[0]
        s_ref = ref["scores"]
        assert np.max(np.abs(st.scores[0].cpu().numpy() - s_ref)) <= score_tol(s_ref)
        cnt = st.sel_count[0].item()
        sel = np.array(st.sel[0, :cnt].cpu().tolist())
        if selection_certified(s_ref, ref["k"]):
            assert sel.tolist() == ref["sel"].tolist()
            rb = ref
        else:
            rb = O.draft_step(part, ro, Wo, f64(hp), f64(e), f64(hn), t, C.k_max, C.k_min, C.k_t,
                              sel_override=[sel])[0]
        assert st.sl_offsets[0, :cnt + 1].cpu().tolist() == rb["sl_offsets"].tolist()
        n = len(rb["V_S"])
        assert np.max(np.abs(st.z[0, :n].cpu().double().numpy() - rb["z"])) <= 2e-2
        check_topk(st.top_ids[0].cpu().numpy(), st.top_logits[0].cpu().numpy(), st.top_logp[0].cpu().numpy(),
                   st.lse[0].item(), rb["z"], rb["V_S"], C.k_t, torch.bfloat16)


def test_cluster_step_deterministic_and_matches_grid_step(monkeypatch):
    """Same launch configuration => identical output bytes (R19); the cluster step and the
    grid-wide step agree on ids, selections and every logit (same per-row dot code)."""
    D = _dyn()
    C = S.CONFIGS["tiny"]
    W, rt, part, c, r = _setup(C.V, C.d, C.M, C.h_r, "bf16", "random")
    hp, e, hn = [x.to(DEV) for x in S.step_inputs(1, C.d, 0, "bf16")]
    outs = {}
    for Q in ("16", "16", "0"):
        monkeypatch.setenv("DS_CLUSTER_Q", Q)
        st = D.DraftStep(c, r, 1, 16, z_out=True)
        st(hp, e, hn, t=0, k_max=8, k_min=8)
        torch.cuda.synchronize()
        o = {k: v.clone() for k, v in st.outputs().items() if v is not None}
        if Q in outs:
            for k in o:
                assert torch.equal(o[k].view(torch.uint8), outs[Q][k].view(torch.uint8)), k
        outs[Q] = o
    a, b = outs["16"], outs["0"]
    assert torch.equal(a["sel"], b["sel"]) and torch.equal(a["top_ids"], b["top_ids"])
    assert torch.equal(a["top_logits"], b["top_logits"])
    n = int(a["sl_offsets"][0, a["sel_count"][0]].item())
    assert torch.equal(a["z"][0, :n], b["z"][0, :n])
    assert abs(a["lse"][0].item() - b["lse"][0].item()) <= 1e-5
