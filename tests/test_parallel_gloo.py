"""Multi-rank host logic on CPU with the gloo backend (world_size 2): request-row sharding,
token-balanced cluster ranges, and the cluster-sharded record protocol (per-rank records over the
owned clusters, in the float32 / bit-cast-id layout dynaspec.h fixes for dynaspec_head_partial ->
all-gather -> rank-order merge) against the unsharded oracle.  tests/test_gpu_shard.py feeds records
built by the same helper (tests/records.py) into the library's dynaspec_merge_records."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_13847_b200 import parallel as P
from tests import records as RC


def test_row_range_partitions():
    for B in (1, 7, 64, 512):
        for G in (1, 2, 3, 8):
            rs = [P.row_range(B, g, G) for g in range(G)]
            assert rs[0][0] == 0 and rs[-1][1] == B
            assert all(rs[g][1] == rs[g + 1][0] for g in range(G - 1))
            assert max(r1 - r0 for r0, r1 in rs) - min(r1 - r0 for r0, r1 in rs) <= 1


def test_cluster_ranges_balanced_and_covering():
    rng = np.random.default_rng(0)
    for M, G in [(256, 2), (512, 8), (64, 4), (5, 5)]:
        sizes = rng.integers(1, 1000, size=M)
        off = np.concatenate([[0], np.cumsum(sizes)])
        rs = P.cluster_ranges(off.tolist(), G)
        assert rs[0][0] == 0 and rs[-1][1] == M and all(lo < hi for lo, hi in rs)
        assert all(rs[g][1] == rs[g + 1][0] for g in range(G - 1))
        toks = [off[hi] - off[lo] for lo, hi in rs]
        if M >= 8 * G:
            assert max(toks) <= off[-1] / G + sizes.max() + 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import dynaspec_oracle as O
    from synth import inputs as S
    V, d, M, k, kt, B = 3000, 32, 20, 6, 8, 3
    W = S.lm_head(V, d, 0, "f32").double().numpy()
    tau = S.random_partition(V, M, 2)
    perm, off = O.layout(tau, M)
    rt = [None if x is None else x.double().numpy() for x in S.router(d, 8, M, 1, "f32")]
    hp, e, hn = [x.double().numpy() for x in S.step_inputs(B, d, 0, "f32")]
    lo, hi = P.cluster_ranges(off.tolist(), world)[rank]
    scores = O.meta_score(*rt, hp, e)                      # replicated
    recs = []
    for b in range(B):
        sel = O.select(scores[b], k)
        own = sel[(sel >= lo) & (sel < hi)]                # restricted selection
        VS = O.shortlist(own, perm, off) if len(own) else np.zeros(0, dtype=np.int64)
        z = O.head(hn[b], W, VS)[0] if len(VS) else np.zeros(0)
        recs.append(RC.oracle_record(z, VS, kt))   # the header's layout: float32, ids bit-cast
    mine = torch.tensor(np.stack(recs), dtype=torch.float32)
    out = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(out, mine)                            # the one exchange step
    gathered = torch.stack(out).numpy()                    # [G][B][rec]
    res = []
    for b in range(B):
        lse, ids, _ = RC.merge(gathered[:, b, :], kt)
        ref = O.epilogue(O.head(hn[b], W, O.shortlist(O.select(scores[b], k), perm, off))[0],
                         O.shortlist(O.select(scores[b], k), perm, off), kt)
        res.append((abs(lse - ref["lse"]), ids == ref["top_ids"].tolist()))
    # request sharding: max over ranks of a per-rank time
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    result_q.put((rank, res, float(t.item())))
    dist.destroy_process_group()


def test_cluster_sharded_protocol_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, res, tmax in results:
        assert tmax == 2.0
        for dlse, same in res:
            assert dlse < 1e-5 and same   # float32 record words


def _bench_worker(rank, world, port, q):
    os.environ.update({"MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port), "RANK": str(rank),
                       "WORLD_SIZE": str(world), "LOCAL_RANK": str(rank)})
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench", os.path.join(os.path.dirname(os.path.dirname(
        os.path.abspath(__file__))), "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    ws, r, local = bench.dist_setup(None)
    bench.barrier(ws)
    m = bench.max_over_ranks(float(10 * (rank + 1)), ws)
    q.put((r, ws, m))
    dist.destroy_process_group()


def test_bench_distributed_helpers_gloo_world2():
    """bench.py's launch plumbing (env rendezvous, barrier, max-over-ranks timing) at world size 2."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res == [(0, 2, 20.0), (1, 2, 20.0)]
