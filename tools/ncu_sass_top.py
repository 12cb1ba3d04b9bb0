#!/usr/bin/env python
"""Top stalled SASS lines and the opcode mix of one kernel in an ncu report.
Usage: ncu_sass_top.py rep.ncu-rep [n]"""
import collections, csv, io, subprocess, sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
raw = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
i = 0
while rows[i][0] != 'Address':
    i += 1
hdr = rows[i]
data = []
for r in rows[i + 1:]:
    if r and r[0] == 'Address':
        break  # a second kernel's section: only the first is summarised
    if len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
key = 'Warp Stall Sampling (All Samples)'
iv = lambda d, k: int(d.get(k) or 0)
tot = sum(iv(d, key) for d in data) or 1
stalls = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
agg = {h: sum(iv(d, h) for d in data) for h in stalls}
print('samples', tot, 'stalls:', ', '.join(f'{k[6:]} {100*v/tot:.1f}%' for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
op = collections.Counter()
for d in data:
    src = d['Source'].strip()
    if src.startswith('@'):
        src = src.split(None, 1)[1]
    op[src.split()[0] if src else '?'] += iv(d, 'Instructions Executed')
ti = sum(op.values()) or 1
print('warp instructions', ti, 'top opcodes:', ', '.join(f'{o} {100*c/ti:.1f}%' for o, c in op.most_common(14)))
for d in sorted(data, key=lambda d: -iv(d, key))[:n]:
    st = max(stalls, key=lambda h: iv(d, h))
    print(f"{iv(d, key):6d} {100*iv(d, key)/tot:5.1f}% {d['Address'][-5:]} {st[6:]:14s} {d['Source'][:80]}")
