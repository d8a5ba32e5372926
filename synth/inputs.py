"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no normalisation, no k-means, no
routing, no selection, no head, no softmax).  It only draws random numbers with
fixed seeds and rounds them to the storage dtype, so that `oracle/` and the CUDA
path receive byte-identical inputs (task rule ③; recipe in DESIGN.md §3).

Distributions follow SURVEY.md §8(d) "Synthetic inputs":
  * random regime: W, E ~ N(0, 0.02^2); h ~ N(0, 1); router W1 ~ N(0, 2/(2d)),
    W2 ~ N(0, 1/h_r), b = 0 (optionally b2 = log Zipf(1.0) prior);
  * exact regime: every value an integer times a power of two, small enough that
    every dot product is exact in fp32 in any summation order (§8(c) "Exact regime");
  * seeded cluster partitions with every cluster non-empty (unbalanced).

Seeds: 0 = W/E, 1 = router, 2 = partition, 1000+t = per-step inputs.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

# ---------------------------------------------------------------------------
# Workload configurations (BASELINE.json "configs"; k schedule per SURVEY R1).
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class Config:
    name: str
    V: int
    d: int
    M: int
    h_r: int          # router hidden size (R5: M/2 by default; 0 = linear router)
    k_max: int
    k_min: int
    positions: int    # draft positions per verification cycle (gamma)
    B: int            # rows per draft step
    k_t: int = 8      # token budget (R15)
    shared: bool = False  # tree mode: rows of one depth share one shortlist (R9)
    extra: dict = field(default_factory=dict)


CONFIGS = {
    # configs[0]: DynaSpec-F, fixed k = 8 (k_max = k_min), 16 positions.
    "tiny": Config("tiny", V=32000, d=1024, M=64, h_r=32, k_max=8, k_min=8, positions=16, B=1),
    # configs[1]: k(pos) 16 -> 4, gamma = 8.
    "llama2": Config("llama2", V=32000, d=4096, M=128, h_r=64, k_max=16, k_min=4, positions=8, B=1),
    # configs[2]: the metric's configuration (V = 128k, d = 4096), k(pos) 32 -> 8.
    "llama3": Config("llama3", V=128256, d=4096, M=256, h_r=128, k_max=32, k_min=8, positions=8, B=1),
    # configs[3]: EAGLE-style tree, 6 depths x R = 10 rows sharing one shortlist per depth.
    "qwen25": Config("qwen25", V=151936, d=3584, M=256, h_r=128, k_max=32, k_min=8, positions=6, B=10,
                     k_t=10, shared=True),
    # configs[4]: 512 requests (sharded over GPUs).
    "gemma3": Config("gemma3", V=262144, d=5376, M=512, h_r=256, k_max=64, k_min=16, positions=8, B=512),
}

TORCH_DTYPES = {"bf16": torch.bfloat16, "f32": torch.float32}


def _gen(seed: int, device="cpu") -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def _normal(shape, std, seed, dtype, device="cpu"):
    """N(0, std^2) drawn in fp32 with a seeded generator, rounded to `dtype`."""
    g = _gen(seed, device)
    x = torch.randn(shape, generator=g, device=device, dtype=torch.float32)
    if std != 1.0:
        x.mul_(std)
    return x.to(TORCH_DTYPES[dtype])


def _grid(shape, q, scale_pow2, seed, dtype, device="cpu"):
    """Uniform integers in [-q, q] times 2**scale_pow2 (exactly representable in bf16 for q <= 256)."""
    g = _gen(seed, device)
    x = torch.randint(-q, q + 1, shape, generator=g, device=device, dtype=torch.int32).to(torch.float32)
    x.mul_(2.0 ** scale_pow2)
    return x.to(TORCH_DTYPES[dtype])


# ---------------------------------------------------------------------------
# LM head W (token rows, nn.Linear layout [V][d]) and embeddings.
# ---------------------------------------------------------------------------


def lm_head(V, d, seed=0, dtype="bf16", regime="random", q=None, device="cpu"):
    """W_LM^T stored as [V][d]: row v is token v's column of W_LM."""
    if regime == "random":
        return _normal((V, d), 0.02, seed, dtype, device)
    if regime == "exact":
        q = q if q is not None else exact_q(d)
        return _grid((V, d), q, -6, seed, dtype, device)
    raise ValueError(regime)


def exact_q(d: int) -> int:
    """Largest Q with d*Q^2 <= 2^24 (SURVEY §8(c) exact regime), capped at 127."""
    return min(127, int(math.isqrt((1 << 24) // d)))


def hidden(B, d, seed, dtype="bf16", regime="random", q=None, device="cpu"):
    """Drafter hidden states h (RMS-normed scale, N(0,1))."""
    if regime == "random":
        return _normal((B, d), 1.0, seed, dtype, device)
    q = q if q is not None else exact_q(d)
    return _grid((B, d), q, -4, seed, dtype, device)


def embedding_rows(B, d, seed, dtype="bf16", regime="random", q=None, device="cpu"):
    """e = E(x_t) rows, N(0, 0.02^2) like W (the caller gathers real embeddings)."""
    if regime == "random":
        return _normal((B, d), 0.02, seed, dtype, device)
    q = q if q is not None else exact_q(d)
    return _grid((B, d), q, -6, seed, dtype, device)


def router_q(d, h_r, qb=16):
    """Exact-regime grid bound for router inputs and W1: every partial sum of both layers
    stays within 2^24 units (SURVEY §8(c) 'The 2-layer router is much tighter')."""
    if h_r == 0:
        return max(1, min(127, int(math.isqrt((1 << 24) // (2 * d)))))
    return max(1, min(127, int(math.isqrt(((1 << 24) // h_r - qb) // (2 * d)))))


def step_inputs(B, d, t, dtype="bf16", regime="random", pool=64, q=None, device="cpu", base_seed=1000,
                sibling_eps=None, h_r=None):
    """(h_prev, e, h_new) for draft position t; seeds 1000+(t mod pool)*3+{0,1,2}.

    Exact regime: h_prev and e (router inputs) on the 2^-2 grid with |q| <= router_q(d, h_r);
    h_new (head input) on the 2^-4 grid with |q| <= exact_q(d).
    sibling_eps: tree rows (SURVEY §8(d) "Tree rows"): row i = parent + eps * g_i.
    """
    if regime == "exact":
        s = base_seed + (t % pool) * 3
        qr = router_q(d, h_r if h_r is not None else 0)
        return (_grid((B, d), qr, -2, s, dtype, device),
                _grid((B, d), qr, -2, s + 1, dtype, device),
                hidden(B, d, s + 2, dtype, "exact", q, device))
    s = base_seed + (t % pool) * 3
    if sibling_eps is not None and regime == "random":
        out = []
        for j, fn in enumerate((hidden, embedding_rows, hidden)):
            parent = fn(1, d, s + j, "f32", "random", device=device)
            noise = fn(B, d, s + j + 7919, "f32", "random", device=device)
            out.append((parent + sibling_eps * noise).to(TORCH_DTYPES[dtype]))
        return tuple(out)
    return (hidden(B, d, s, dtype, regime, q, device),
            embedding_rows(B, d, s + 1, dtype, regime, q, device),
            hidden(B, d, s + 2, dtype, regime, q, device))


# ---------------------------------------------------------------------------
# Router parameters theta (R5: one hidden layer, ReLU, f32 biases).
# ---------------------------------------------------------------------------


def router(d, h_r, M, seed=1, dtype="bf16", regime="random", zipf_b2=False, device="cpu", qx=None):
    """Returns (W1, b1, W2, b2).

    h_r > 0: W1 [h_r][2d], b1 [h_r] f32, W2 [M][h_r], b2 [M] f32.
    h_r == 0 (linear router): W1 [M][2d], b1 [M] f32, W2 = b2 = None.
    Exact regime: inputs and W1 on the 2^-2 grid with |q| <= router_q(d, h_r) (products on 2^-4),
    b1 on the 2^-4 grid, W2 in {-1,0,1}*2^-1, b2 on the 2^-5 grid (SURVEY §8(c) "The 2-layer router").
    """
    dr = 2 * d
    rows1 = h_r if h_r > 0 else M
    if regime == "random":
        W1 = _normal((rows1, dr), math.sqrt(2.0 / dr), seed, dtype, device)
        b1 = torch.zeros(rows1, dtype=torch.float32, device=device)
        if h_r == 0:
            if zipf_b2:
                b1 = zipf_log_prior(M, device)
            return W1, b1, None, None
        W2 = _normal((M, h_r), math.sqrt(1.0 / h_r), seed + 101, dtype, device)
        b2 = zipf_log_prior(M, device) if zipf_b2 else torch.zeros(M, dtype=torch.float32, device=device)
        return W1, b1, W2, b2
    if regime == "exact":
        qx = qx if qx is not None else router_q(d, h_r)
        W1 = _grid((rows1, dr), qx, -2, seed, dtype, device)
        b1 = _grid((rows1,), 16, -4, seed + 5, "f32", device)
        if h_r == 0:
            return W1, b1, None, None
        W2 = _grid((M, h_r), 1, -1, seed + 101, dtype, device)
        b2 = _grid((M,), 16, -5, seed + 105, "f32", device)
        return W1, b1, W2, b2
    raise ValueError(regime)


def zipf_log_prior(M, device="cpu"):
    """b2_m = log of a Zipf(1.0) prior over clusters (a trained router's cluster popularity)."""
    r = torch.arange(1, M + 1, dtype=torch.float64)
    p = (1.0 / r) / (1.0 / r).sum()
    return torch.log(p).to(torch.float32).to(device)


# ---------------------------------------------------------------------------
# Seeded partitions (head parity does not depend on how tau was built).
# ---------------------------------------------------------------------------


def random_partition(V, M, seed=2, zipf=1.0):
    """tau: V -> [M] with every cluster non-empty and Zipf(zipf)-skewed sizes (unbalanced)."""
    if not (1 <= M <= V):
        raise ValueError("need 1 <= M <= V")
    rng = np.random.default_rng(seed)
    tau = np.empty(V, dtype=np.int64)
    order = rng.permutation(V)
    tau[order[:M]] = rng.permutation(M)          # one guaranteed member per cluster
    w = 1.0 / np.arange(1, M + 1) ** zipf
    w = w / w.sum()
    tau[order[M:]] = rng.choice(M, size=V - M, p=w)
    return tau


def uniform_scores(B, M, seed):
    """Scores whose top-k is a uniformly random cluster set (SURVEY §8(d) 'uniform' control)."""
    g = _gen(seed)
    return torch.rand((B, M), generator=g, dtype=torch.float32)


def planted_lm_head(V, d, M, seed=0, dtype="bf16", zipf=1.0, device="cpu"):
    """W with M latent directions and Zipf cluster sizes (SURVEY §8(d) 'planted-cluster W')."""
    g = _gen(seed, device)
    mu = torch.randn((M, d), generator=g, device=device)
    mu = mu / mu.norm(dim=1, keepdim=True)
    tau = torch.as_tensor(random_partition(V, M, seed + 17, zipf), device=device)
    noise = torch.randn((V, d), generator=g, device=device)
    noise = noise / noise.norm(dim=1, keepdim=True)
    w = 0.6 * mu[tau] + 0.8 * noise
    w = 0.02 * math.sqrt(d) * w / w.norm(dim=1, keepdim=True)
    return w.to(TORCH_DTYPES[dtype]), tau.cpu().numpy()


def to_f64(x):
    """Exact widening of a bf16/f32 tensor to a numpy fp64 array (oracle input)."""
    if x is None:
        return None
    return x.detach().to("cpu", torch.float64).numpy()


def zipf_token_counts(V, seed=3, a=1.1, n_tokens=10_000_000):
    """Synthetic corpus token counts (Zipf(a) over a random permutation of the vocabulary) — the
    stand-in for the FR-Spec frequency statistics (the paper's corpora are out of scope)."""
    rng = np.random.default_rng(seed)
    ranks = rng.permutation(V)
    p = 1.0 / (np.arange(1, V + 1) ** a)
    p /= p.sum()
    counts = np.zeros(V, dtype=np.int64)
    counts[ranks] = rng.multinomial(n_tokens, p)
    return counts


def verify_inputs(B, gamma, V, n_short, seed=11, dtype="bf16", logit_std=3.0, q_noise=0.5):
    """Synthetic verification workload (NEXT-4): target logits [B][gamma+1][V] ~ N(0, logit_std^2)
    (peaked next-token distributions); for each drafted position a shortlist of the n_short tokens
    with the largest noisy target logit (random order) whose drafter logits are the target's logits
    there + N(0, q_noise^2) (a drafter that approximates the target); q_lse is left to the caller.  Uniforms u_acc [B][gamma], u_res [B] and
    u_draw [B][gamma] (for picking the drafted tokens) in [0, 1)."""
    g = _gen(seed)
    p = torch.randn((B, gamma + 1, V), generator=g) * logit_std
    p = p.to(TORCH_DTYPES[dtype])
    pf = p.float()
    # the shortlist holds the n_short tokens with the largest noisy target logit (a drafter shortlist
    # that captures most, not all, of the target mass), in random order
    ids = torch.empty((B, gamma, n_short), dtype=torch.int32)
    for b in range(B):
        for i in range(gamma):
            noisy = pf[b, i] + torch.randn(V, generator=g) * logit_std
            top = torch.topk(noisy, n_short).indices
            ids[b, i] = top[torch.randperm(n_short, generator=g)].to(torch.int32)
    ql = torch.empty((B, gamma, n_short), dtype=torch.float32)
    for b in range(B):
        for i in range(gamma):
            ql[b, i] = pf[b, i, ids[b, i].long()] + torch.randn(n_short, generator=g) * q_noise
    u = torch.rand((B, 2 * gamma + 1), generator=g, dtype=torch.float64)
    return dict(p_logits=p, q_ids=ids, q_logits=ql, u_acc=u[:, :gamma].float(), u_draw=u[:, gamma:2 * gamma],
                u_res=u[:, 2 * gamma].float())
