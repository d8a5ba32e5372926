"""GPU offline partition (S0, dynaspec_build_clusters) vs the oracle's integer-exact spherical
k-means (reading R12): tau, perm, offsets, W_perm and the iteration count must be
bit-identical."""
import itertools
import json
import os

import numpy as np
import pytest
import torch

from oracle import dynaspec_oracle as O
from synth import inputs as S

pytestmark = pytest.mark.gpu
DEV = "cuda"
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "e2e1.json")))


def _D():
    from paper_2510_13847_b200 import dynaspec
    return dynaspec


def _compare(W, M, seed=2, max_iters=20, init=None):
    D = _D()
    c = D.Clusters.build(W.to(DEV), M, seed=seed, max_iters=max_iters, init_ids=init)
    ref = O.build_clusters(W.to(torch.float64).numpy(), M, seed=seed, max_iters=max_iters, init_ids=init)
    assert c.iters == ref["iters"]
    assert np.array_equal(c.tau.cpu().numpy(), ref["tau"])
    assert np.array_equal(c.perm.cpu().numpy(), ref["perm"])
    assert np.array_equal(c.offsets.cpu().numpy(), ref["offsets"])
    assert torch.equal(c.W_perm.cpu(), W[torch.as_tensor(ref["perm"])])
    sizes = np.diff(ref["offsets"])
    assert c.min_size == sizes.min() and c.max_size == sizes.max()
    return c, ref


def test_e2e1_golden_inits_gpu():
    W = torch.zeros((6, 8), dtype=torch.float32)
    W[:, :2] = torch.tensor(GOLD["W_rows"], dtype=torch.float32)
    for key, exp in GOLD["golden_inits"].items():
        init = [int(x) for x in key.split(",")]
        c, ref = _compare(W, 3, init=init)
        assert c.tau.cpu().tolist() == GOLD["partition"]["tau"]
        assert c.iters == exp["iters"]


def test_four_angles_all_inits_gpu():
    ang = np.deg2rad([1, 3, 88, 91])
    W = torch.zeros((4, 8), dtype=torch.float32)
    W[:, 0] = torch.tensor(np.cos(ang), dtype=torch.float32)
    W[:, 1] = torch.tensor(np.sin(ang), dtype=torch.float32)
    for init in itertools.permutations(range(4), 2):
        c, _ = _compare(W, 2, init=list(init))
        assert c.tau.cpu().tolist() == [0, 0, 1, 1]


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("V,d,M,seed", [(3001, 64, 17, 5), (2000, 136, 40, 9), (500, 32, 1, 3)])
def test_random_heads_bit_exact(dtype, V, d, M, seed):
    W = S.lm_head(V, d, seed, dtype)
    _compare(W, M, seed=seed, max_iters=25)


def test_planted_unbalanced_clusters():
    W, _ = S.planted_lm_head(4000, 128, 32, seed=4, dtype="bf16")
    c, ref = _compare(W, 32, seed=4, max_iters=30)
    sizes = np.diff(ref["offsets"])
    assert sizes.max() > 2 * sizes.min()      # unbalanced, as the paper allows


def test_duplicates_force_reseeding():
    """Many identical token vectors and M close to V: empty clusters and reseeds every pass."""
    base = S.lm_head(6, 16, 1, "f32")
    W = base[torch.tensor([0, 0, 0, 1, 1, 2, 2, 2, 3, 4, 5, 5])]
    for seed in range(6):
        _compare(W, 9, seed=seed, max_iters=12)


def test_tiny_config_full_size():
    C = S.CONFIGS["tiny"]
    W = S.lm_head(C.V, C.d, 0, "bf16")
    _compare(W, C.M, seed=2, max_iters=4)


def test_llama3_full_size_two_iterations():
    """BASELINE configs[2] at full size: V=128256, d=4096, M=256 (2 Lloyd passes)."""
    C = S.CONFIGS["llama3"]
    W = S.lm_head(C.V, C.d, 0, "bf16")
    _compare(W, C.M, seed=2, max_iters=2)


def test_degenerate_column_error():
    D = _D()
    W = S.lm_head(100, 16, 0, "bf16")
    W[37] = 0
    with pytest.raises(D.DynaspecError) as ei:
        D.Clusters.build(W.to(DEV), 4)
    assert ei.value.name == "DS_ERR_DEGENERATE_COLUMN"
    with pytest.raises(D.DynaspecError) as ei:
        D.Clusters.build(S.lm_head(10, 16, 0, "bf16").to(DEV), 11)
    assert ei.value.name == "DS_ERR_INVALID_CLUSTER_COUNT"
