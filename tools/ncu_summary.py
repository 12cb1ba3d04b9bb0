#!/usr/bin/env python
"""Summarise an ncu --set full report (one kernel) into JSON: the metrics the
bench roofline and DESIGN.md cite.  Usage: ncu_summary.py rep.ncu-rep [workload]"""
import csv, io, json, subprocess, sys

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_sectors.sum',
        'lts__t_sector_hit_rate.pct', 'l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum',
        'l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'l1tex__throughput.avg.pct_of_peak_sustained_elapsed', 'launch__registers_per_thread',
        'smsp__inst_executed.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'launch__grid_size', 'launch__block_size',
        'sm__cycles_elapsed.avg.per_second', 'dram__cycles_elapsed.avg.per_second',
        'launch__shared_mem_per_block_dynamic', 'launch__occupancy_limit_registers',
        'sm__maximum_warps_per_active_cycle_pct']


def main():
    rep = sys.argv[1]
    raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        d = {'kernel': vals[hdr.index('Kernel Name')]}
        for k in KEYS:
            if k in hdr:
                v = vals[hdr.index(k)]
                try:
                    v = float(v.replace(',', ''))
                except ValueError:
                    pass
                d[k] = [v, units[hdr.index(k)]]
        stalls = {}
        for i, h in enumerate(hdr):
            if h.startswith('smsp__average_warps_issue_stalled_') and h.endswith('_per_issue_active.ratio'):
                try:
                    v = float(vals[i])
                except ValueError:
                    continue
                if v > 0.05:
                    stalls[h[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]] = v
        d['stalls_per_issue'] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
        def gb(k):
            v = d.get(k, [0])[0]
            return v * {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}.get(d.get(k, [0, 'byte'])[1], 1)
        d['dram_bytes_per_launch'] = gb('dram__bytes_read.sum') + gb('dram__bytes_write.sum')
        if len(sys.argv) > 2:
            d['workload'] = sys.argv[2]
        out.append(d)
    print(json.dumps(out[0] if len(out) == 1 else out, indent=1))


if __name__ == '__main__':
    main()
