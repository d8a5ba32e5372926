"""Bisect a grid-step mismatch: the exact-regime case of test_grid_step_exact_bit_exact, with and
without the phase trace, printing the first wrong outputs."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import dynaspec_oracle as O  # noqa: E402
from paper_2510_13847_b200 import dynaspec as D  # noqa: E402
from synth import inputs as S  # noqa: E402
from tests.parity import Rows, f64  # noqa: E402

DEV = "cuda"
import os
V, d, M, h_r, dt, k_t = 7919, 384, 40, int(os.environ.get("HR", 16)), "bf16", int(os.environ.get("KT", 8))
W = S.lm_head(V, d, 0, dt, "exact")
rt = S.router(d, h_r, M, 1, dt, "exact")
tau = S.random_partition(V, M, 2)
perm, off = O.layout(tau, M)
part = {"perm": perm, "offsets": off}
c = D.Clusters.from_tau(W.to(DEV), torch.as_tensor(tau, dtype=torch.int32, device=DEV), M)
r = D.Router(*[x.to(DEV) for x in rt])
Wo, ro = Rows(W), tuple(f64(x) for x in rt)
G = torch.cuda.get_device_properties(0).multi_processor_count
for trace in (False, True):
    st = D.DraftStep(c, r, 1, k_t, z_out=True)
    for t in range(3):
        hp, e, hn = [x.to(DEV) for x in S.step_inputs(1, d, t, dt, "exact", h_r=h_r)]
        buf = torch.zeros(G * 64 + G * 40, dtype=torch.int64, device=DEV)
        if trace:
            D.debug_set_trace(buf)
        st(hp, e, hn, t=t, k_max=16, k_min=4)
        torch.cuda.synchronize()
        D.debug_set_trace(None)
        ref = O.draft_step(part, ro, Wo, f64(hp), f64(e), f64(hn), t, 16, 4, k_t)[0]
        ok_sel = st.sel[0, :st.sel_count[0]].cpu().tolist() == ref["sel"].tolist()
        n = len(ref["V_S"])
        ok_z = np.array_equal(st.z[0, :n].cpu().numpy(), ref["z"].astype(np.float32))
        ids = st.top_ids[0].cpu().numpy()
        print(f"trace={trace} t={t} sel_ok={ok_sel} z_ok={ok_z} ids={ids.tolist()} ref={ref['top_ids'].tolist()} "
              f"lse={st.lse[0].item():.6f} ref_lse={ref['lse']:.6f} err={st.ws.error()}")
        zmap = dict(zip(ref["V_S"].tolist(), ref["z"].tolist()))
        if False:
            rec = buf[G * 64:G * 64 + G * (2 + k_t)].view(G, 2 + k_t).cpu().numpy().astype(np.uint64)
            vs = set(ref["V_S"].tolist())
            allk = {}
            for g in range(G):
                for k in rec[g, 2:2 + int(rec[g, 1]) - 1]:
                    allk.setdefault(int(k), []).append(g)
            dups = {hex(k): v for k, v in allk.items() if len(v) > 1}
            print("   records: total keys", sum(len(v) for v in allk.values()), "cross-record duplicates", list(dups.items())[:5])
            heads = sorted([int(rec[g, 2]) for g in range(G) if rec[g, 1] > 1], reverse=True)
            print("   best heads (hi)", [h >> 32 for h in heads[:10]], "merger ns, T =",
                  buf[G * 64 + G * (2 + k_t)].item(), buf[G * 64 + G * (2 + k_t) + 1].item())
            for g in range(G):
                keys = rec[g, 2:]
                cnt = int(rec[g, 1]) - 1
                ids = [int(~np.uint32(k & np.uint64(0xffffffff)) & 0xffffffff) for k in keys[:cnt]]
                bad = [i for i in ids if i not in vs]
                srt = all(keys[i] > keys[i + 1] for i in range(cnt - 1))
                if bad or not srt:
                    print(f"   CTA {g}: cnt {cnt} keys-not-in-V_S {bad} sorted {srt} ids {ids}")
        print("   gpu logits", st.top_logits[0].cpu().numpy().tolist(), "ref", ref["top_logits"].tolist())
