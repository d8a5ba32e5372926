"""Summarise a scripts/trace_cta.py dump: per-step phase times (us from the earliest start, median
over reps) and the merger's phases."""
import sys

import numpy as np

z = np.load(sys.argv[1])
ns, cy, k = z["ns"], z["cy"], z["k"]
act = ns[0, 0, :, 0] > 0
ns, cy = ns[:, :, act], cy[:, :, act]
names = {0: "start", 1: "pdl", 2: "L1done", 8: "a1_x", 12: "sc_x", 13: "mask", 4: "stream0", 5: "streamed",
         9: "cta_rec", 14: "recs_seen", 17: "all_seen", 15: "T2", 7: "merged"}
prev_m = None
for t in range(ns.shape[1]):
    t0 = np.where(ns[:, t, :, 0] > 0, ns[:, t, :, 0], np.inf).min(1)  # per rep
    line = []
    for sl, n in names.items():
        x = ns[:, t, :, sl]
        if not (x > 0).any():
            continue
        mx = np.median(np.where(x > 0, x, -np.inf).max(1) - t0) / 1e3
        line.append(f"{n}={mx:.2f}")
    print(f"t={t} k={k[t]} (max over CTAs, us): " + " ".join(line))
    seen = ns[:, t, :, 16]
    if (seen > 0).any():
        print("    record seen (us from t0): median over records %.2f max %.2f; slowest record ids %s" % (
            np.median(np.median(np.where(seen > 0, seen, np.nan) - t0[:, None], 1)) / 1e3,
            np.median(np.nanmax(np.where(seen > 0, seen, np.nan), 1) - t0) / 1e3,
            np.argsort(-np.nanmedian(np.where(seen > 0, seen, np.nan), 0))[:5].tolist()))
    c = cy[:, t, 0]
    print("    merger CTA0 cycles: streamed->rec %d rec->seen %d seen->T2 %d T2->merged %d" % tuple(
        np.median(c[:, b] - c[:, a]) for a, b in [(5, 9), (9, 14), (14, 15), (15, 7)]))
