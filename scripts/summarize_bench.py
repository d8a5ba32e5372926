"""Print a one-line summary of bench JSON lines (files given on the command line)."""
import json
import sys

for p in sys.argv[1:]:
    try:
        j = json.loads(open(p).read().strip().splitlines()[-1])
        c = j["config"]
        rf = j.get("roofline") or {}
        print(f"{p}: value={j['value']:.0f} {j['unit']} us/step={c.get('us_per_draft_step', float('nan')):.1f} "
              f"dense_us={c.get('dense_us_per_draft_step', float('nan')):.1f} speedup={c.get('speedup_vs_dense')} "
              f"frac={rf.get('frac')} rows={c.get('mean_shortlist_rows')} mode={c.get('step_mode')} "
              f"e2e={(j.get('e2e') or {}).get('value')}")
    except Exception as ex:  # noqa: BLE001
        print(p, "unreadable:", ex)
