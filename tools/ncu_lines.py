#!/usr/bin/env python
"""Per CUDA source line: warp instructions executed and stall samples of the
FIRST kernel in an ncu report (captured with --import-source on, built with
-lineinfo).  Usage: ncu_lines.py rep.ncu-rep [n_lines] [file_substring]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
want = sys.argv[3] if len(sys.argv) > 3 else ""
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
first_fn = None
cur_file = None
hdr = None
lines = {}  # (file, line) -> [inst, samples, text]
for r in rows:
    if not r:
        continue
    if r[0] == "Function Name":
        if first_fn is None:
            first_fn = r[1]
        elif r[1] != first_fn:
            break  # the next kernel
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0]:  # a CUDA source line with its aggregated metrics
        try:
            inst = int(r[hdr.index("Instructions Executed")] or 0)
            smp = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        except ValueError:
            continue
        if want and want not in (cur_file or ""):
            continue
        lines[(cur_file, int(r[0]))] = [inst, smp, r[1].strip()]
ti = sum(v[0] for v in lines.values()) or 1
ts = sum(v[1] for v in lines.values()) or 1
print(f"warp instructions {ti}, stall samples {ts}")
for (f, ln), (inst, smp, txt) in sorted(lines.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{100*inst/ti:5.1f}% inst {100*smp/ts:5.1f}% smp  {f}:{ln:<5d} {txt[:90]}")
