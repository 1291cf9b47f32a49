#!/usr/bin/env python3
"""Attribute ncu per-instruction execution counts to CUDA source lines.

usage: sass_lines.py <report.ncu-rep> <kernel.cubin> <function-substring>
Needs the cubin built with -lineinfo (nvdisasm -g prints the line table).
"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, cubin, fsub = sys.argv[1:4]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ix, isrc = hdr.index("Instructions Executed"), hdr.index("Source")
counts = []
for r in rows[2:]:
    if len(r) > ix:
        counts.append((r[isrc].strip(), int(r[ix] or 0)))
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
# split per function, pick the one matching fsub
funcs = re.split(r"\n\s*\.text\.", dis)
body = None
for f in funcs:
    if fsub in f.split("\n", 1)[0]:
        body = f
        break
if body is None:
    sys.exit("function not found")
line = None
seq = []
for ln in body.split("\n"):
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        line = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
    if m:
        seq.append((line, m.group(2).strip()))
if len(seq) != len(counts):
    print(f"warning: {len(seq)} sass vs {len(counts)} counted instructions", file=sys.stderr)
per = collections.Counter()
kind = collections.defaultdict(collections.Counter)
for (l, ins), (_, n) in zip(seq, counts):
    per[l] += n
    op = ins.split()[0]
    if op.startswith("@"):
        op = ins.split()[1]
    kind[l][op.split(".")[0]] += n
tot = sum(per.values())
src = {}
for l, n in per.most_common(int(sys.argv[4]) if len(sys.argv) > 4 else 40):
    if l is None:
        continue
    fn, no = l
    print(f"{100 * n / tot:5.1f}%  {fn}:{no:<5} " + " ".join(f"{k}:{100 * v / n:.0f}" for k, v in kind[l].most_common(4)))
