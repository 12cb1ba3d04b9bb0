#!/usr/bin/env python
"""Sum ncu's per-launch metrics of every (workload, op) NVTX range (launches
renamed "ncu|<workload>|<op>" by tools/ncu_ops.py under
--print-nvtx-rename kernel) into profiles/<tag>_ncu_rows.json for bench.py.

Usage: ncu_rows.py ncu_ops.csv out.json [git-head]"""
import csv
import json
import sys
import time
from collections import defaultdict

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "msecond": 1e-3, "ms": 1e-3, "nsecond": 1e-9, "second": 1.0, "s": 1.0}


def main():
    src, dst = sys.argv[1], sys.argv[2]
    lines = [l for l in open(src) if l.startswith('"')]
    rows = list(csv.DictReader(lines))
    per = defaultdict(lambda: defaultdict(dict))  # (workload, op) -> launch id -> metric -> value
    for r in rows:
        name = r["Kernel Name"]
        if not name.startswith("ncu|"):
            continue
        _, wl, rest = name.split("|", 2)
        op, kern = rest.split("/", 1) if "/" in rest else (rest, "")
        try:
            v = float(r["Metric Value"].replace(",", ""))
        except ValueError:
            continue
        unit = r["Metric Unit"]
        v *= SCALE.get(unit, 1.0)
        per[(wl, op)][r["ID"]][r["Metric Name"]] = v
        per[(wl, op)][r["ID"]]["kernel"] = kern
    out = []
    for (wl, op), launches in sorted(per.items()):
        L = [dict(m) for m in launches.values()]
        kern = [m.pop("kernel", "") for m in L]
        dur = sum(m.get("gpu__time_duration.sum", 0.0) for m in L)
        rd = sum(m.get("dram__bytes_read.sum", 0.0) for m in L)
        wr = sum(m.get("dram__bytes_write.sum", 0.0) for m in L)
        lts = sum(m.get("lts__t_bytes.sum", 0.0) for m in L)
        # L2 hit rate weighted by the launch's L2 traffic
        hit = (sum(m.get("lts__t_sector_hit_rate.pct", 0.0) * m.get("lts__t_bytes.sum", 0.0) for m in L) / lts
               if lts else None)
        out.append({"workload": wl, "op": op, "launches": len(L), "duration_s": dur,
                    "dram_bytes": rd + wr, "dram_read_bytes": rd, "dram_write_bytes": wr,
                    "dram_GB/s_under_ncu": (rd + wr) / dur / 1e9 if dur else None,
                    "l2_bytes": lts, "l2_hit_pct": hit,
                    "per_launch": [dict(m, kernel=k) for m, k in zip(L, kern)]})
    json.dump({"tool": "ncu --nvtx --print-nvtx-rename kernel --clock-control none --cache-control all --metrics ...",
               "driver": "tools/ncu_ops.py", "head": sys.argv[3] if len(sys.argv) > 3 else None,
               "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()), "rows": out}, open(dst, "w"), indent=1)
    for r in out:
        print(f"{r['workload']:24s} {r['op']:22s} launches {r['launches']:2d}  {r['duration_s'] * 1e3:8.3f} ms  "
              f"DRAM {r['dram_bytes'] / 1e9:8.3f} GB  L2 hit {r['l2_hit_pct'] or 0:5.1f}%")


if __name__ == "__main__":
    main()
