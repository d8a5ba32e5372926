"""NEXT-1: draft-tree bookkeeping on the device (Alg. 1 lines 12-18) vs the oracle."""
import numpy as np
import pytest
import torch

from oracle import dynaspec_oracle as O
from synth import inputs as S
from tests.parity import Rows, f64

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.mark.parametrize("R,K", [(1, 1), (1, 8), (4, 4), (10, 10), (64, 64)])
def test_tree_step_bit_exact(R, K):
    from paper_2510_13847_b200 import dynaspec as D
    rng = np.random.default_rng(R * 100 + K)
    tree = D.DraftTree(K, 3 * K * K + 16)
    ref_nodes, last_s, last_n, base = [], None, None, 0
    for j in range(3):
        RR = 1 if j == 0 else len(last_s)          # beams = valid expansions kept at j - 1
        # dyadic log-probs (exact in fp32 sums), with deliberate duplicates to exercise ties
        lp = -rng.integers(0, 6, size=(RR, K)).astype(np.float64) / 4.0
        lp = np.sort(lp, axis=1)[:, ::-1].copy()
        ids = rng.integers(0, 1000, size=(RR, K))
        if K > 2:
            ids[0, -1] = -1
            lp[0, -1] = -np.inf
        tree.step(torch.as_tensor(ids, dtype=torch.int32, device=DEV),
                  torch.as_tensor(lp, dtype=torch.float32, device=DEV), j)
        if R == 1 and j == 0:
            pass
        nodes, nxt = O.tree_step(ids, lp, last_s, last_n, j, base, K)
        ref_nodes += nodes
        base += RR * K
        last_s, last_n = nxt["score"], nxt["node"]
        torch.cuda.synchronize()
        nk = len(nxt["tok"])
        assert tree.next_tok[:nk].cpu().tolist() == nxt["tok"].tolist()
        assert tree.next_node[:nk].cpu().tolist() == nxt["node"].tolist()
        assert tree.next_beam[:nk].cpu().tolist() == nxt["beam"].tolist()
        assert np.array_equal(tree.next_score[:nk].cpu().numpy(), nxt["score"].astype(np.float32))
        assert (tree.next_tok[nk:].cpu() == -1).all()
    n = tree.n
    assert tree.tok[:n].cpu().tolist() == [t for t, _, _, _ in ref_nodes]
    assert tree.parent[:n].cpu().tolist() == [p for _, _, p, _ in ref_nodes]
    sc = tree.score[:n].cpu().numpy()
    ref_sc = np.array([s if t >= 0 else -np.inf for t, s, _, _ in ref_nodes], dtype=np.float32)
    assert np.array_equal(sc, ref_sc)
    for n_out in (1, 7, n):
        got = tree.rerank(n_out).cpu().numpy()
        ref = O.tree_rerank(ref_nodes, n_out)
        assert got[:len(ref)].tolist() == ref.tolist()
        assert (got[len(ref):] == -1).all()


def test_tree_draft_cycle_qwen_shape():
    """gamma = 4 tree-drafting cycle at the Qwen head shape: shared-shortlist head (tcgen05) for the
    k_t beam rows of each depth, tree_step on the device, next router inputs e = E[x_j]."""
    from paper_2510_13847_b200 import dynaspec as D
    C = S.CONFIGS["qwen25"]
    K = C.k_t
    W = S.lm_head(C.V, C.d, 0, "bf16")
    E = S.lm_head(C.V, C.d, 5, "bf16")                 # embedding table stand-in (same distribution)
    rt = S.router(C.d, C.h_r, C.M, 1, "bf16")
    tau = S.random_partition(C.V, C.M, 2)
    perm, off = O.layout(tau, C.M)
    c = D.Clusters.from_tau(W.to(DEV), torch.as_tensor(tau, dtype=torch.int32, device=DEV), C.M)
    r = D.Router(*[x.to(DEV) for x in rt])
    st1 = D.DraftStep(c, r, 1, K, shared=True)
    stK = D.DraftStep(c, r, K, K, shared=True)
    tree = D.DraftTree(K, 1 + 4 * K * K)
    h = S.hidden(1, C.d, 3, "bf16")
    x0 = 17
    h_prev, e, h_new = h, E[x0:x0 + 1], h
    Wo, ro = Rows(W), tuple(f64(x) for x in rt)
    for j in range(4):
        st = st1 if j == 0 else stK
        st(h_prev.to(DEV), e.to(DEV), h_new.to(DEV), t=j, k_max=C.k_max, k_min=C.k_min)
        tree.step(st.top_ids, st.top_logp, j)
        torch.cuda.synchronize()
        # invariants: score = parent score + logp; parents from the previous frontier
        R = h_new.shape[0]
        cnt = st.sel_count[0].item()
        ref = O.draft_step({"perm": perm, "offsets": off}, ro, Wo, f64(h_prev), f64(e), f64(h_new), j, C.k_max,
                           C.k_min, K, shared=True, sel_override=[st.sel[0, :cnt].cpu().numpy()] * R)
        for b in range(R):
            assert st.top_ids[b, 0].item() == ref[b]["top_ids"][0] or \
                abs(ref[b]["top_logits"][0] - ref[b]["top_logits"][1]) < 4e-2
        beam = tree.next_beam.cpu().numpy()
        tok = tree.next_tok.cpu().numpy()
        assert (beam >= 0).all() and (beam < R).all()
        # next inputs (Alg. 1 lines 15-16): parent hidden and the embedding of the chosen token
        h_prev = h_new[torch.as_tensor(beam, dtype=torch.long)]
        h_new = h_prev
        e = E[torch.as_tensor(tok, dtype=torch.long)]
    n = tree.n
    sc = tree.score[:n].cpu().numpy()
    par = tree.parent[:n].cpu().numpy()
    for i in range(n):
        if par[i] >= 0:
            assert sc[i] <= sc[par[i]] + 1e-6           # log-probs <= 0 accumulate
    top = set(tree.rerank(3 * K).cpu().tolist())
    for i in top:
        assert par[i] == -1 or par[i] in top            # re-ranked top-N is a tree
