"""Test-side builders of the cluster-sharded record protocol in the byte layout include/dynaspec.h
fixes for dynaspec_head_partial / dynaspec_merge_records: per row 2 + 2 k_t float32 words
{max z, sum exp(z - max), (z, id) x k_t by (z desc, id asc), padded with (-inf, INT_MAX)}, ids
bit-cast into the float words.  Records are built from ORACLE logits (never from the CUDA path),
so the gloo world-2 test and the GPU merge test share one reference of the protocol."""
import math

import numpy as np

INT_MAX = np.iinfo(np.int32).max


def oracle_record(z, ids, k):
    """One rank's record for one row from its shortlist logits z over token ids `ids` (fp64 in,
    float32 words out, the layout dynaspec_merge_records reads)."""
    z = np.asarray(z, dtype=np.float64)
    ids = np.asarray(ids, dtype=np.int64)
    vals = np.full(2 + 2 * k, -np.inf, dtype=np.float32)
    idw = np.full(2 + 2 * k, 0, dtype=np.int32)
    idw[3::2] = INT_MAX
    if z.size:
        m = z.max()
        vals[0], vals[1] = np.float32(m), np.float32(np.exp(z - m).sum())
        order = np.lexsort((ids, -z))[:k]
        for q, j in enumerate(order):
            vals[2 + 2 * q] = np.float32(z[j])
            idw[3 + 2 * q] = ids[j]
    else:
        vals[1] = 0.0
    out = vals.copy()
    out[3::2] = idw[3::2].view(np.float32)
    return out


def record_ids(rec, k):
    return np.asarray(rec, dtype=np.float32)[3:3 + 2 * k:2].view(np.int32)


def merge(records, k):
    """Rank-order merge of one row's G records [G][2 + 2k] (the protocol dynaspec_merge_records
    implements): lse = M + log sum_g S_g e^{m_g - M}; top-k of the candidates by (z desc, id asc)."""
    records = np.asarray(records, dtype=np.float32)
    ms = records[:, 0].astype(np.float64)
    fin = np.isfinite(ms)
    M = ms[fin].max()
    S = sum(float(r[1]) * math.exp(float(r[0]) - M) for r in records if np.isfinite(r[0]))
    cand = []
    for r in records:
        ids = record_ids(r, k)
        for q in range(k):
            if np.isfinite(r[2 + 2 * q]):
                cand.append((float(r[2 + 2 * q]), int(ids[q])))
    cand.sort(key=lambda x: (-x[0], x[1]))
    return M + math.log(S), [c[1] for c in cand[:k]], [c[0] for c in cand[:k]]
