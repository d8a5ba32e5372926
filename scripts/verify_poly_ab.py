"""A/B of the lse pass's FMA-pipe exp2 share (DS_VERIFY_POLY) on the bench's verification workload
(Llama-3 vocabulary, 64 chains x gamma = 8, shortlist 7k); alternates settings, median of medians."""
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
for rnd in range(3):
    for np_ in ["0", "2", "4", "6", "8"]:
        os.environ["DS_VERIFY_POLY"] = np_
        for B in (64, 1):
            out = bench.verify_run(D, C, dev, flush, 7000, B=B, reps=20)
            res.setdefault(f"B{B}_poly{np_}", []).append(out["us_per_call"])
            res.setdefault(f"B{B}_poly{np_}_acc", []).append(out["mean_accepted"])
summary = {k: (statistics.median(v) if not k.endswith("_acc") else v[0]) for k, v in res.items()}
print(json.dumps(summary, indent=1))
