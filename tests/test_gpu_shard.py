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
