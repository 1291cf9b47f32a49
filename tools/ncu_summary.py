#!/usr/bin/env python3
"""Summarise an ncu --set full report: throughputs, stalls, DRAM bytes, instruction mix."""
import collections
import csv
import io
import subprocess
import sys


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        res.append({h: (v, u) for h, u, v in zip(hdr, units, r)})
    return res


def mix(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ix = hdr.index("Instructions Executed")
    isrc = hdr.index("Source")
    ist = hdr.index("Warp Stall Sampling (All Samples)")
    cnt, stall = collections.Counter(), collections.Counter()
    for r in rows[2:]:
        if len(r) <= ix or not r[ix].strip().isdigit():  # multi-kernel reports repeat the header
            continue
        op = r[isrc].strip().split()
        if not op:
            continue
        o = op[1] if op[0].startswith("@") else op[0]
        base = o.split(".")[0]
        cnt[base] += int(r[ix] or 0)
        stall[base] += int(r[ist] or 0)
    return cnt, stall


KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__inst_executed.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
]


def main(rep):
    for k in raw(rep):
        print("kernel:", k.get("Kernel Name", ("?", ""))[0][:90])
        for key in KEYS:
            if key in k:
                print(f"  {key:70s} {k[key][0]} {k[key][1]}")
        st = {h: v for h, v in k.items() if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("per_issue_active.ratio")}
        top = sorted(st.items(), key=lambda kv: -float(kv[1][0] or 0))[:8]
        print("  stalls/issue:", ", ".join(f"{h.split('stalled_')[1].split('_per')[0]}={float(v[0]):.2f}" for h, v in top))
    cnt, stall = mix(rep)
    tot = sum(cnt.values())
    tots = max(1, sum(stall.values()))
    print("  instruction mix (dynamic):")
    for k, v in cnt.most_common(16):
        print(f"    {k:8s} {100 * v / tot:6.2f}%   stall samples {100 * stall[k] / tots:6.2f}%")


if __name__ == "__main__":
    main(sys.argv[1])
