"""Attribute ncu warp-stall samples (--page source --print-source sass) to CUDA source lines using
the line table of `nvdisasm -gi` (innermost line and the kernel-level call site of inlined code).

Usage: ncu_lines.py REPORT.ncu-rep OBJ.o KERNEL_SUBSTRING [top]"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, obj, kname = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, check=True, capture_output=True)
cubin = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
sass = subprocess.run(["nvdisasm", "-gi", os.path.join(tmp, cubin)], capture_output=True, text=True).stdout
# offset -> (innermost file:line, kernel-level line)
linemap, fn, group = {}, None, []
for ln in sass.splitlines():
    mf = re.match(r"\s*\.text\.(\S+):", ln)
    if mf:
        fn = mf.group(1)
        continue
    if fn is None or kname not in fn:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        group.append(f"{os.path.basename(m.group(1))}:{m.group(2)}")
        continue
    mi = re.search(r"/\*([0-9a-f]{4,})\*/\s+\S", ln)
    if mi:
        off = int(mi.group(1), 16)
        if group:
            linemap[off] = (group[0], group[-1])
            last = linemap[off]
            group = []
        else:
            linemap[off] = last
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hdr_i]
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
samp_i = hdr.index("Warp Stall Sampling (All Samples)")
ex_i = hdr.index("Instructions Executed")
data = [r for r in rows[hdr_i + 1:] if len(r) == len(hdr) and r[0].startswith("0x")]
base = int(data[0][0], 16)
by_inner, by_outer = collections.defaultdict(collections.Counter), collections.defaultdict(collections.Counter)
total = 0
for r in data:
    off = int(r[0], 16) - base
    inner, outer = linemap.get(off, ("?", "?"))
    s = int(r[samp_i] or 0)
    total += s
    for d in (by_inner[inner], by_outer[outer]):
        d["samples"] += s
        d["instr_exec"] += int(r[ex_i] or 0)
        for i in stall_cols:
            v = int(r[i] or 0)
            if v:
                d[hdr[i]] += v
print(f"total samples {total}")
for title, dd in (("kernel-level line", by_outer), ("innermost line", by_inner)):
    print(f"\n== by {title}")
    for k, c in sorted(dd.items(), key=lambda kv: -kv[1]["samples"])[:top]:
        stalls = sorted(((n[6:], v) for n, v in c.items() if n.startswith("stall_")), key=lambda x: -x[1])[:4]
        print(f"{k:16s} samples {c['samples']:6d} ({100 * c['samples'] / max(total, 1):5.1f}%) exec {c['instr_exec']:8d}  "
              + " ".join(f"{n}={v}" for n, v in stalls))
