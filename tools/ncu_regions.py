#!/usr/bin/env python3
"""Per-address-range instruction counts and warp-stall samples of one ncu capture.

usage: ncu_regions.py <report.ncu-rep> name:lo:hi [name:lo:hi ...]
lo/hi are SASS offsets (hex) from the kernel start, e.g. the loops found in
`cuobjdump -sass` of the same build.
"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = []
for r in rows[2:]:
    try:
        data.append((int(r[0], 16), r))
    except (ValueError, IndexError):
        pass
base = data[0][0]
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
regions = [("all", 0, 1 << 40)] + [(a.split(":")[0], int(a.split(":")[1], 16), int(a.split(":")[2], 16))
                                   for a in sys.argv[2:]]
for name, lo, hi in regions:
    sel = [r for a, r in data if lo <= a - base <= hi]
    ie = sum(int(r[ix["Instructions Executed"]] or 0) for r in sel)
    ops = Counter()
    for r in sel:
        op = r[1].split()
        op = [t for t in op if not t.startswith("@")][0].split(".")[0]
        ops[op] += int(r[ix["Instructions Executed"]] or 0)
    samp = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in sel)
    st = {s: sum(int(r[ix[s]] or 0) for r in sel) for s in stalls}
    fp = ops["DFMA"] + ops["DADD"] + ops["DMUL"]
    print(f"{name}: warp-inst {ie:.4g}  fp64 {fp / max(ie, 1):.1%}  samples {samp}")
    print("   stalls:", ", ".join(f"{k[6:]}={v / max(samp, 1):.2f}" for v, k in
                                  sorted(((v, k) for k, v in st.items() if v), reverse=True)[:10]))
    print("   mix:", ", ".join(f"{k}={v / max(ie, 1):.1%}" for k, v in ops.most_common(14)))
