"""A/B of the lse pass's knobs on the bench's verification workload (Llama-3 vocabulary, 64 chains x
gamma = 8 and one chain, shortlist 7k): DS_VERIFY_POLY (FMA-pipe exp2 share) or, with --pf, DS_VERIFY_PF
(L2 bulk-prefetch distance) or, with --pdl, DS_VERIFY_PDL (the residual pass as a programmatic dependent
launch); alternates settings, median of the per-round medians."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2510_13847_b200 import dynaspec as D  # noqa: E402
from synth import inputs as S  # noqa: E402

dev = torch.device("cuda:0")
C = S.CONFIGS["llama3"]
flush = bench.L2Flush(dev)
res = {}
knob, vals = (("DS_VERIFY_PF", ["0", "1", "2", "3", "5"]) if "--pf" in sys.argv else
              ("DS_VERIFY_PDL", ["0", "1"]) if "--pdl" in sys.argv else ("DS_VERIFY_POLY", ["0", "2", "4", "6", "8"]))
for rnd in range(3):
    for np_ in vals:
        os.environ[knob] = np_
        for B in (64, 1):
            out = bench.verify_run(D, C, dev, flush, 7000, B=B, reps=20)
            res.setdefault(f"B{B}_{knob[10:].lower()}{np_}", []).append(out["us_per_call"])
            res.setdefault(f"B{B}_{knob[10:].lower()}{np_}_acc", []).append(out["mean_accepted"])
summary = {k: (statistics.median(v) if not k.endswith("_acc") else v[0]) for k, v in res.items()}
print(json.dumps(summary, indent=1))
