"""Cluster-sharded head on one GPU (shard emulation): G shards computed one after another, each
holding only its W_perm slice, records stacked as the all-gather would, merged in rank order —
must equal the unsharded head (ids and logits identical, lse to fp32 rounding)."""
import numpy as np
import pytest
import torch

from oracle import dynaspec_oracle as O
from synth import inputs as S

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.mark.parametrize("cfg,B,shared,G", [("tiny", 3, False, 2), ("tiny", 4, True, 3), ("llama3", 1, False, 4),
                                            ("tiny", 2, False, 1)])
def test_shard_emulation_matches_unsharded(cfg, B, shared, G, monkeypatch):
    monkeypatch.setenv("DS_DISABLE_TC", "1")  # same (CUDA-core) head on both sides: bit-identical logits
    from paper_2510_13847_b200 import dynaspec as D
    from paper_2510_13847_b200 import parallel as P
    C = S.CONFIGS[cfg]
    W = S.lm_head(C.V, C.d, 0, "bf16", device=DEV)
    tau = torch.as_tensor(S.random_partition(C.V, C.M, 2), dtype=torch.int32, device=DEV)
    full = D.Clusters.from_tau(W, tau, C.M)
    r = D.Router(*[x.to(DEV) for x in S.router(C.d, C.h_r, C.M, 1, "bf16")])
    hp, e, hn = [x.to(DEV) for x in S.step_inputs(B, C.d, 0, "bf16")]
    scores = D.meta_score(r, hp, e)
    sel, cnt, off = D.select(scores, full, C.k_max, shared=shared)
    ref = D.head_forward(full, hn, sel, cnt, off, C.k_t, shared=shared)
    ranges = P.cluster_ranges(full.offsets.cpu().tolist(), G)
    recs = []
    for lo, hi in ranges:
        sh = full.shard(lo, hi)
        rs, rc, ro = D.restrict_selection(sel, cnt, off, sh, lo, hi)
        recs.append(D.head_partial(sh, hn, rs, rc, ro, C.k_t, shared=shared))
    out = D.merge_records(torch.stack(recs), C.k_t)
    torch.cuda.synchronize()
    assert torch.equal(out["top_ids"], ref["top_ids"])
    assert torch.equal(out["top_logits"], ref["top_logits"])
    assert torch.allclose(out["lse"], ref["lse"], rtol=2e-6, atol=1e-6)
    assert torch.allclose(out["top_logp"], ref["top_logp"], rtol=0, atol=1e-5)
    # restricted selections partition the full one
    tot = sum(int(D.restrict_selection(sel, cnt, off, full, lo, hi)[1].sum()) for lo, hi in ranges)
    assert tot == int(cnt.sum())


@pytest.mark.parametrize("G", [1, 2, 3])
def test_merge_records_on_oracle_records(G):
    """The library's dynaspec_merge_records on records built from ORACLE logits in the header's
    layout (tests/records.py, the same builder the gloo world-2 test all-gathers): lse, ids and
    logits equal the oracle's unsharded epilogue over the union shortlist."""
    from paper_2510_13847_b200 import dynaspec as D
    from paper_2510_13847_b200 import parallel as P
    from tests import records as RC
    V, d, M, k, kt, B = 3000, 32, 20, 6, 8, 3
    W = S.lm_head(V, d, 0, "f32").double().numpy()
    tau = S.random_partition(V, M, 2)
    perm, off = O.layout(tau, M)
    rt = [None if x is None else x.double().numpy() for x in S.router(d, 8, M, 1, "f32")]
    hp, e, hn = [x.double().numpy() for x in S.step_inputs(B, d, 0, "f32")]
    scores = O.meta_score(*rt, hp, e)
    recs = np.zeros((G, B, 2 + 2 * kt), dtype=np.float32)
    for g, (lo, hi) in enumerate(P.cluster_ranges(off.tolist(), G)):
        for b in range(B):
            sel = O.select(scores[b], k)
            own = sel[(sel >= lo) & (sel < hi)]
            VS = O.shortlist(own, perm, off) if len(own) else np.zeros(0, dtype=np.int64)
            z = O.head(hn[b], W, VS)[0] if len(VS) else np.zeros(0)
            recs[g, b] = RC.oracle_record(z, VS, kt)
    out = D.merge_records(torch.as_tensor(recs, device=DEV), kt)
    torch.cuda.synchronize()
    for b in range(B):
        VS = O.shortlist(O.select(scores[b], k), perm, off)
        ref = O.epilogue(O.head(hn[b], W, VS)[0], VS, kt)
        assert out["top_ids"][b].cpu().tolist() == ref["top_ids"].tolist()
        assert np.array_equal(out["top_logits"][b].cpu().numpy(), ref["top_logits"].astype(np.float32))
        assert abs(out["lse"][b].item() - ref["lse"]) <= 1e-5 * max(1.0, abs(ref["lse"]))
        assert np.allclose(out["top_logp"][b].cpu().numpy(), ref["top_logp"], atol=2e-5, rtol=0)


@pytest.mark.parametrize("cfg,B,G", [("tiny", 2, 1), ("tiny", 3, 3), ("llama3", 1, 2)])
def test_cluster_sharded_step_vs_oracle(cfg, B, G):
    """parallel.ClusterShardedStep (router + select replicated, head_partial over the owned
    clusters, record exchange, rank-order merge) against the ORACLE's unsharded draft step.  G = 1
    is the world-1 path as bench.py --shard clusters runs it; G > 1 emulates the ranks on one GPU
    and stacks their records as the all-gather would."""
    from paper_2510_13847_b200 import dynaspec as D
    from paper_2510_13847_b200 import parallel as P
    from tests.parity import Rows, check_topk, f64, selection_certified
    C = S.CONFIGS[cfg]
    W = S.lm_head(C.V, C.d, 0, "bf16")
    tau = S.random_partition(C.V, C.M, 2)
    perm, off = O.layout(tau, C.M)
    part = {"perm": perm, "offsets": off}
    full = D.Clusters.from_tau(W.to(DEV), torch.as_tensor(tau, dtype=torch.int32, device=DEV), C.M)
    rt = S.router(C.d, C.h_r, C.M, 1, "bf16")
    r = D.Router(*[x.to(DEV) for x in rt])
    ranges = P.cluster_ranges(full.offsets.cpu().tolist(), G)
    steps = [P.ClusterShardedStep(D, full.shard(lo, hi), r, B, C.k_t, G, g) for g, (lo, hi) in enumerate(ranges)]
    Wo, ro = Rows(W), tuple(f64(x) for x in rt)
    for t in (0, 2):
        hp, e, hn = S.step_inputs(B, C.d, t, "bf16")
        if G == 1:
            out = steps[0](hp.to(DEV), e.to(DEV), hn.to(DEV), t, C.k_max, C.k_min)
        else:
            recs = []
            for st in steps:   # each emulated rank: replicated router/select, its own partial head
                st.world = 1
                st(hp.to(DEV), e.to(DEV), hn.to(DEV), t, C.k_max, C.k_min)
                recs.append(st.records.clone())
            out = D.merge_records(torch.stack(recs), C.k_t)
        torch.cuda.synchronize()
        ref = O.draft_step(part, ro, Wo, f64(hp), f64(e), f64(hn), t, C.k_max, C.k_min, C.k_t)
        checked = 0
        for b in range(B):
            rb = ref[b]
            if not selection_certified(rb["scores"], rb["k"]):
                continue  # the GPU's selection is not recoverable from records alone: skip uncertified rows
            checked += 1
            check_topk(out["top_ids"][b].cpu().numpy(), out["top_logits"][b].cpu().numpy(),
                       out["top_logp"][b].cpu().numpy(), out["lse"][b].item(), rb["z"], rb["V_S"], C.k_t,
                       torch.bfloat16)
        assert checked > 0
