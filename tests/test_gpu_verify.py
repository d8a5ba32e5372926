"""GPU parity of the lossless verification kernels (NEXT-4, Eq. 3, R25) and of
the shortlist-id materialisation (S4) against the oracle, through the C-ABI.

Accept / reject is a floating-point decision and the corrective token an inverse-CDF lookup, so the
comparison is conditional (tests/parity.py style): a chain is certified when every decision the oracle
takes has margin (|u - min(1, p/q)| > 1e-5 relative; u_res * Z more than 1e-5 Z away from the cumulative
weights bracketing the drawn token); certified chains must match exactly, and most chains must certify.
Independently of the oracle, the Monte-Carlo test checks the kernel's committed tokens follow the
target law."""
import math

import numpy as np
import pytest
import torch

from oracle import dynaspec_oracle as O
from synth import inputs as S

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _dyn():
    from paper_2510_13847_b200 import dynaspec as Dy
    return Dy


def _prepare(inp):
    """q_lse and the drafted tokens (drawn from q with u_draw by the oracle's inverse CDF)."""
    ql = inp["q_logits"].double().numpy()
    B, g, _ = ql.shape
    q_lse = np.zeros((B, g))
    x = np.zeros((B, g), dtype=np.int64)
    slot = np.zeros((B, g), dtype=np.int64)
    ids = inp["q_ids"].numpy()
    for b in range(B):
        for i in range(g):
            m = ql[b, i].max()
            q_lse[b, i] = float(np.float32(m + math.log(np.exp(ql[b, i] - m).sum())))
            slot[b, i] = O.sample_inverse_cdf(np.exp(ql[b, i] - q_lse[b, i]), float(inp["u_draw"][b, i]))
            x[b, i] = ids[b, i, slot[b, i]]
    return q_lse, x, slot


def _certified(pl, ids, ql, qs, x, u_acc, u_res, n, margin=1e-5):
    """True when every decision the oracle takes for this chain has margin."""
    V = pl.shape[1]
    for i in range(n + 1 if n < len(x) else n):
        p = O.softmax_full(pl[i])
        q = O.embed_q(V, ids[i], ql[i], qs[i])
        r = min(1.0, p[x[i]] / q[x[i]])
        if abs(u_acc[i] - r) <= margin * r + 1e-9:
            return False
    if n < len(x):
        p = O.softmax_full(pl[n])
        w = np.maximum(p - O.embed_q(V, ids[n], ql[n], qs[n]), 0.0)
    else:
        w = O.softmax_full(pl[n])
    c = np.cumsum(w)
    Z, t = c[-1], u_res * c[-1]
    k = O.sample_inverse_cdf(w, u_res)
    lo = c[k - 1] if k > 0 else 0.0
    return (t - lo) > margin * Z and (c[k] - t) > margin * Z


def _run(inp, dtype, q_lse, x, slot, ver=None):
    Dy = _dyn()
    p = inp["p_logits"].to(DEV)
    B, g1, V = p.shape
    g = g1 - 1
    ver = ver or Dy.Verifier(V, B, g, DEV)
    q_ids = inp["q_ids"].to(DEV).contiguous()
    acc, com = ver(p, q_ids, inp["q_logits"].to(DEV), torch.full((B, g), q_ids.shape[-1], dtype=torch.int32,
                                                                   device=DEV),
                   torch.tensor(q_lse, dtype=torch.float32, device=DEV), torch.tensor(x, dtype=torch.int32, device=DEV),
                   torch.tensor(slot, dtype=torch.int32, device=DEV), inp["u_acc"].to(DEV), inp["u_res"].to(DEV))
    torch.cuda.synchronize()
    return acc.cpu().numpy().copy(), com.cpu().numpy().copy()


@pytest.mark.parametrize("V,n_short,dtype,poly", [(32000, 4000, "bf16", "0"), (128256, 27000, "bf16", "0"),
                                                  (128256, 27000, "f32", "0"), (4104, 300, "f32", "0"),
                                                  (128256, 27000, "bf16", "8"), (32000, 4000, "bf16", "4"),
                                                  (128256, 27000, "bf16", "pf3"), (128256, 27000, "f32", "pdl"),
                                                  (32000, 4000, "bf16", "pdl")])
def test_verify_parity(V, n_short, dtype, poly, monkeypatch):
    if poly == "pdl":  # the residual pass as a programmatic dependent launch
        monkeypatch.setenv("DS_VERIFY_PDL", "1")
    elif poly.startswith("pf"):  # lse pass: L2 bulk-prefetch distance
        monkeypatch.setenv("DS_VERIFY_PF", poly[2:])
    else:  # lse pass: word pairs per lane on the FMA-pipe exp2
        monkeypatch.setenv("DS_VERIFY_POLY", poly)
    B, g = 12, 4
    inp = S.verify_inputs(B, g, V, n_short, seed=V % 97, dtype=dtype)
    q_lse, x, slot = _prepare(inp)
    acc, com = _run(inp, dtype, q_lse, x, slot)
    pl = inp["p_logits"].double().numpy()
    ql = inp["q_logits"].double().numpy()
    ids = inp["q_ids"].numpy()
    ua = inp["u_acc"].double().numpy()
    ur = inp["u_res"].double().numpy()
    cert = 0
    seen = set()
    for b in range(B):
        n, c = O.verify_chain(pl[b], ids[b], ql[b], q_lse[b], x[b], ua[b], ur[b])
        seen.add(n)
        if not _certified(pl[b], ids[b], ql[b], q_lse[b], x[b], ua[b], ur[b], n):
            continue
        cert += 1
        assert acc[b] == n, (b, acc[b], n)
        assert com[b, :n + 1].tolist() == c, (b, com[b, :n + 1], c)
    assert cert >= int(0.75 * B)
    assert len(seen) >= 2  # both rejections and full acceptance occur across the batch


def test_verify_gamma0_bonus_and_q_equals_p():
    Dy = _dyn()
    V, B = 8192, 6
    inp = S.verify_inputs(B, 0, V, 1, seed=3, dtype="f32")
    ver = Dy.Verifier(V, B, 0, DEV)
    acc, com = ver(inp["p_logits"].to(DEV), None, None, None, None, None, None, None, inp["u_res"].to(DEV))
    torch.cuda.synchronize()
    for b in range(B):
        n, c = O.verify_chain(inp["p_logits"][b].double().numpy(), [], [], [], [], [], float(inp["u_res"][b]))
        assert acc[b].item() == 0 and com[b, 0].item() == c[0]
    # q = p over the whole vocabulary -> every drafted token accepted, bonus from p_gamma
    g = 3
    inp = S.verify_inputs(B, g, V, 16, seed=4, dtype="f32")
    pl = inp["p_logits"]
    ids = torch.arange(V, dtype=torch.int32).expand(B, g, V).contiguous()
    ql = pl[:, :g].float().contiguous()
    q_lse = torch.logsumexp(ql.double(), dim=-1).float()
    x = torch.randint(0, V, (B, g), generator=torch.Generator().manual_seed(1), dtype=torch.int32)
    ver = Dy.Verifier(V, B, g, DEV)
    acc, com = ver(pl.to(DEV), ids.to(DEV), ql.to(DEV), torch.full((B, g), V, dtype=torch.int32, device=DEV),
                   q_lse.to(DEV), x.to(DEV), x.to(DEV), torch.full((B, g), 0.999, device=DEV), inp["u_res"].to(DEV))
    torch.cuda.synchronize()
    assert (acc.cpu() == g).all()  # p/q = 1 up to fp32 rounding: u = 0.999 accepts
    assert (com.cpu()[:, :g][acc.cpu() == g] == x[acc.cpu() == g]).all()


def test_verify_invalid_proposal_and_errors():
    Dy = _dyn()
    V, B, g = 8192, 2, 2
    inp = S.verify_inputs(B, g, V, 64, seed=5, dtype="bf16")
    q_lse, x, slot = _prepare(inp)
    slot[1, 0] = (slot[1, 0] + 1) % 64  # q_ids[slot] != x at the first position of chain 1
    acc, com = _run(inp, "bf16", q_lse, x, slot)
    assert acc[1] == -1 and com[1, 0] == -1
    assert acc[0] >= 0
    lib = Dy.lib()
    assert lib.dynaspec_verify_chain(None, 0, 8190, 1, 1, None, None, 1, None, None, None, None, None, None, None,
                                     None, None, 0, None) != 0
    assert lib.dynaspec_verify_ws(8192, 1, 33) == 0


def test_verify_workspace_reuse_stays_zero():
    """Two calls through one Verifier equal fresh-workspace calls (the q buffer is cleared)."""
    Dy = _dyn()
    V, B, g = 32000, 8, 3
    a = S.verify_inputs(B, g, V, 2000, seed=6, dtype="bf16")
    b = S.verify_inputs(B, g, V, 2000, seed=7, dtype="bf16")
    qa, xa, sa = _prepare(a)
    qb, xb, sb = _prepare(b)
    ver = Dy.Verifier(V, B, g, DEV)
    _run(a, "bf16", qa, xa, sa, ver)
    r1 = _run(b, "bf16", qb, xb, sb, ver)
    r2 = _run(b, "bf16", qb, xb, sb)
    assert (r1[0] == r2[0]).all()
    for b_ in range(B):  # committed[b][0..accepted] is defined; later entries are left untouched
        assert (r1[1][b_, :r1[0][b_] + 1] == r2[1][b_, :r2[0][b_] + 1]).all()
    # the counters and the dense q buffer (the first 3 x 256 + B V 4 bytes of the layout) are zero again
    assert int(ver.ws.buf[:256 * 3 + B * V * 4].count_nonzero()) == 0


def test_verify_monte_carlo_target_law():
    """the first committed token follows p_0 (TV < 0.02 over 200k chains), q zero off V_S."""
    Dy = _dyn()
    V, B, g = 64, 200_000, 2
    rng = np.random.default_rng(9)
    pl1 = (rng.standard_normal((g + 1, V)) * 1.5).astype(np.float32)
    Sids = [np.sort(rng.choice(V, 40, replace=False)) for _ in range(g)]
    ql1 = [rng.standard_normal(40).astype(np.float32) for _ in range(g)]
    qs1 = [float(np.float32(np.log(np.exp(z.astype(np.float64)).sum()))) for z in ql1]
    p0 = O.softmax_full(pl1[0])
    p1 = O.softmax_full(pl1[1])
    slots = np.stack([np.searchsorted(np.cumsum(np.exp(ql1[i] - qs1[i])), rng.random(B) * np.exp(
        ql1[i] - qs1[i]).sum(), side="right").clip(0, 39) for i in range(g)], 1)
    xs = np.stack([Sids[i][slots[:, i]] for i in range(g)], 1)
    dev = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device=DEV)
    ver = Dy.Verifier(V, B, g, DEV)
    acc, com = ver(dev(np.broadcast_to(pl1, (B, g + 1, V)), torch.float32),
                   dev(np.broadcast_to(np.stack(Sids), (B, g, 40)), torch.int32),
                   dev(np.broadcast_to(np.stack(ql1), (B, g, 40)), torch.float32),
                   dev(np.full((B, g), 40), torch.int32), dev(np.broadcast_to(qs1, (B, g)), torch.float32),
                   dev(xs, torch.int32), dev(slots, torch.int32), dev(rng.random((B, g)), torch.float32),
                   dev(rng.random(B), torch.float32))
    torch.cuda.synchronize()
    acc, com = acc.cpu().numpy(), com.cpu().numpy()
    assert (acc >= 0).all()
    first = np.bincount(com[:, 0], minlength=V) / B
    assert 0.5 * np.abs(first - p0).sum() < 0.02
    m = acc >= 1
    second = np.bincount(com[m, 1], minlength=V) / m.sum()
    assert 0.5 * np.abs(second - p1).sum() < 0.025


def test_shortlist_ids_match_oracle():
    """S4 materialisation: ids in shortlist order equal the oracle's V_S (bit-exact), per-row and shared."""
    Dy = _dyn()
    C = S.CONFIGS["llama3"]
    tau = S.random_partition(C.V, C.M, seed=2)
    perm, offsets = O.layout(tau, C.M)
    W = torch.zeros((C.V, 8), dtype=torch.bfloat16)
    cl = Dy.Clusters.from_tau(W.to(DEV), torch.as_tensor(tau).to(DEV), C.M)
    rng = np.random.default_rng(3)
    B, k = 5, 12
    sel = np.zeros((B, C.M), dtype=np.int32)
    cnt = np.full(B, k, dtype=np.int32)
    slo = np.zeros((B, C.M + 1), dtype=np.int32)
    for b in range(B):
        s = np.sort(rng.choice(C.M, k, replace=False))
        sel[b, :k] = s
        slo[b, :k + 1] = O.shortlist_offsets(s, offsets)
    stride = int(slo[:, k].max())
    ids = Dy.shortlist_ids(cl, torch.as_tensor(sel).to(DEV), torch.as_tensor(cnt).to(DEV),
                           torch.as_tensor(slo).to(DEV), stride).cpu().numpy()
    for b in range(B):
        VS = O.shortlist(sel[b, :k], perm, offsets)
        assert ids[b, :len(VS)].tolist() == list(VS)
        assert (ids[b, len(VS):] == -1).all()
