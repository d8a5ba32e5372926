"""Multi-GPU plumbing for the DynaSpec head; torch.distributed only moves bytes.

* Request sharding (primary, `scaling: weak`): rows are independent requests; rank g takes
  rows row_range(B, g, G) and runs the whole draft step locally — no data-path collective.
* Cluster sharding (optional): rank g stores only the W_perm rows of its cluster range
  (token-balanced); the router + selection run replicated, each rank emits per-row records
  over its clusters and ONE all-gather (NCCL over NVLink / NVSwitch) exchanges them before the
  rank-order merge (dynaspec_merge_records).
"""
from __future__ import annotations

import bisect


def row_range(B: int, rank: int, world: int):
    """Contiguous, balanced split of B request rows over `world` ranks: [r0, r1)."""
    return (B * rank) // world, (B * (rank + 1)) // world


def cluster_ranges(offsets, world: int):
    """Split clusters 0..M-1 into `world` contiguous ranges with ~equal token counts (the bytes a
    rank stores and, under uniform selection, streams).  offsets: host sequence of M+1 ints."""
    offsets = [int(x) for x in offsets]
    M, V = len(offsets) - 1, offsets[-1]
    if world > M:
        raise ValueError("more ranks than clusters")
    cuts = [0]
    for g in range(1, world):
        target = V * g / world
        m = bisect.bisect_left(offsets, target)          # offsets[m-1] < target <= offsets[m]
        if m > 0 and target - offsets[m - 1] <= offsets[min(m, M)] - target:
            m -= 1                                        # the closer cluster boundary
        m = min(max(m, cuts[-1] + 1), M - (world - g))   # every range non-empty
        cuts.append(m)
    cuts.append(M)
    return [(cuts[g], cuts[g + 1]) for g in range(world)]


class ClusterShardedStep:
    """One cluster-sharded draft step on this rank (router + select replicated; head over the
    owned clusters; all-gather of records; merge).  `group` is a torch.distributed group."""

    def __init__(self, D, clusters_full_or_shard, router, B, k_t, world, rank, group=None, shared=False):
        import torch
        self.D, self.router, self.B, self.k_t, self.shared = D, router, B, k_t, shared
        self.world, self.rank, self.group = world, rank, group
        self.c = clusters_full_or_shard
        dev = clusters_full_or_shard.W_perm.device
        self.rec = 2 + 2 * k_t
        self.records = torch.empty((B, self.rec), dtype=torch.float32, device=dev)
        self.gathered = torch.empty((world, B, self.rec), dtype=torch.float32, device=dev)
        self.ws = D.Workspace(D.lib().dynaspec_head_forward_ws(self.c.struct(), B, k_t), dev)

    def __call__(self, h_prev, e, h_new, t, k_max, k_min):
        import torch.distributed as dist
        D = self.D
        k = D.budget(t, k_max, k_min)
        scores = D.meta_score(self.router, h_prev, e)
        sel, cnt, off = D.select(scores, self.c, k, shared=self.shared)
        rs, rc, ro = D.restrict_selection(sel, cnt, off, self.c, self.c.m_lo, self.c.m_hi)
        D.head_partial(self.c, h_new, rs, rc, ro, self.k_t, shared=self.shared, ws=self.ws, records=self.records)
        if self.world > 1:
            dist.all_gather_into_tensor(self.gathered, self.records, group=self.group)
        else:
            self.gathered[0].copy_(self.records)
        return D.merge_records(self.gathered, self.k_t)
