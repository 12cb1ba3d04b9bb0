#!/usr/bin/env python
"""bench.py -- SpMM GE/s and HBM GB/s of the CogDL sparse hot path on B200.

Headline (BASELINE.json metric): C4, a Chung-Lu power-law
graph with Reddit's node / edge counts (232,965 nodes, 11,606,919 undirected
pairs -> nnz(A^) = 23,446,803), 602 fp32 features (ld 608, rows on whole 128-byte lines).  One STEP is
Y = A^ X through gsp_spmm; A^ is built (gsp_coo_to_csr) and normalised
(gsp_sym_normalize) once before timing (reported as rows a1 / a2).

Besides the headline the default run reports one row per (config, op) of
SURVEY §8(d)7 for C1, C2, C2g, C3, C4, C5 (C6 with --with-c6): cold / warm
times, GE/s, algorithmic and ncu-measured DRAM bytes against the HBM peak,
an in-run parity check against the fp64 oracle (full output where the
oracle is fast, sampled rows + hubs otherwise), and the oracle's own
throughput on one core and on all host cores.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C4]
  N > 1 without torchrun: bench.py re-executes itself under torch.distributed.run
  (one process per GPU, NCCL, row partition + chunked all-gather).

Timing: W untimed warm-ups, then K steps each bracketed by CUDA events on the
launching stream with an L2 flush (256 MB memset, untimed) before every step;
barrier + synchronize around the timed loop; max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
TF32_MMA_PEAK = 1035.7  # TFLOP/s, profiles/r2i_mma_peak_probe.txt (tcgen05 kind::tf32, 128x128x8, 148 SMs)
L2_GATHER_PEAK_GBS = 20264.7  # profiles/r1_probes.txt: ldg U=8, x_MB=17 (random 512-B row gathers from L2)
FALLBACK_HBM = 6650.0   # GB/s, B200_PROFILING.md fallback
NOMINAL_HBM = 8000.0    # GB/s, B200 nominal


def hbm_peak():
    try:
        return float(json.load(open(PEAKS_PATH))["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------------------
# byte models
# ---------------------------------------------------------------------------

def spmm_bytes(n, nnz, f):
    """(gather model, compulsory) bytes of one Y = A X: one X row per nonzero
    (gather) or X once (compulsory), + Y write + col / val + row_ptr."""
    csr = 8 * nnz + 8 * (n + 1)
    return 4 * nnz * f + 4 * n * f + csr, 8 * n * f + csr


def gat_bytes(n, nnz, H, D):
    """Fused GAT aggregate: Z gathers + Y + col + row_ptr + gathered er + el."""
    g = 4 * nnz * H * D + 4 * n * H * D + 4 * nnz + 8 * (n + 1) + 4 * nnz * H + 4 * n * H
    m = 8 * n * H * D + 4 * nnz + 8 * (n + 1) + 8 * n * H
    return g, m


def mh_bytes(n, nnz, H, D):
    g = 4 * nnz * H * D + 4 * n * H * D + 4 * nnz + 4 * nnz * H + 8 * (n + 1)
    m = 8 * n * H * D + 4 * nnz + 4 * nnz * H + 8 * (n + 1)
    return g, m


def softmax_bytes(n, nnz, H):
    b = 8 * nnz * H + 8 * (n + 1)
    return b, b


def attn_bytes(n, H, D):
    b = 4 * n * H * D + 8 * n * H
    return b, b


# ---------------------------------------------------------------------------
# measurement helpers
# ---------------------------------------------------------------------------

class Clocks:
    """nvidia-smi sampler for the timed region (B200_PROFILING.md clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.p = None
        self.out = ""

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "50", "-i", str(self.index)], stdout=subprocess.PIPE,
                                      stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        time.sleep(0.15)
        return self

    def __exit__(self, *a):
        if self.p is not None:
            time.sleep(0.1)
            self.p.terminate()
            try:
                self.out, _ = self.p.communicate(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in (self.out or "").strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)), "reasons": sorted(reasons),
                "samples": len(sm)}


class Timer:
    """Cold (L2 flushed before each rep, untimed) and warm (back to back) CUDA
    event timings on the current stream."""

    def __init__(self, dev):
        import torch
        self.torch = torch
        self.flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def cold(self, fn, warmup, reps):
        torch = self.torch
        for _ in range(warmup):
            fn()
        st = torch.cuda.current_stream()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
        torch.cuda.synchronize()
        for a0, a1 in ev:
            self.flush.zero_()
            a0.record(st)
            fn()
            a1.record(st)
        torch.cuda.synchronize()
        return [a0.elapsed_time(a1) for a0, a1 in ev]

    def warm(self, fn, reps):
        torch = self.torch
        st = torch.cuda.current_stream()
        fn()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(st)
        for _ in range(reps):
            fn()
        a1.record(st)
        torch.cuda.synchronize()
        return a0.elapsed_time(a1) / reps


def tstats(ts):
    return {"t_cold_median_ms": float(np.median(ts)), "t_cold_mean_ms": float(np.mean(ts)),
            "t_cold_min_ms": float(np.min(ts)), "t_cold_p90_ms": float(np.percentile(ts, 90))}


def ncu_table():
    """(workload, op) -> ncu summary of that op's launches, from the committed
    profiles/*ncu_rows*.json (tools/ncu_rows.py); the latest file wins."""
    import glob
    out = {}
    for p in sorted(glob.glob(os.path.join(ROOT, "profiles", "*ncu_rows*.json"))):
        try:
            d = json.load(open(p))
        except Exception:
            continue
        for r in d.get("rows", []):
            r = dict(r)
            r["source"] = os.path.relpath(p, ROOT)
            out[(r["workload"], r["op"])] = r
    return out


def sample_rows(row_ptr, k, seed=0):
    deg = np.diff(row_ptr)
    rng = np.random.default_rng(seed)
    rows = set(rng.choice(deg.size, size=min(k, deg.size), replace=False).tolist())
    rows |= set(np.argsort(deg)[-16:].tolist())
    return np.array(sorted(rows), np.int64)


def err_ratio(y, yref, cond, rel=1e-5, abs_=1e-6):
    """max |y - y_ref| / (rel * cond + abs) -- parity passes when <= 1."""
    y = np.asarray(y, np.float64)
    return float(np.max(np.abs(y - yref) / (rel * cond + abs_))) if y.size else 0.0


# ---------------------------------------------------------------------------
# the oracle (cpu_baseline, in-run parity, --impl reference): as it stands
# ---------------------------------------------------------------------------

def oracle_rate(row_ptr, col, a64, x, f, budget_ge, omp=False, start_row=0):
    """GE/s of the fp64 oracle SpMM over a contiguous row sample of about
    budget_ge edge x feature units (single thread, or all host cores)."""
    import oracle as orc
    n = row_ptr.size - 1
    r0 = start_row % n
    r1 = int(np.searchsorted(row_ptr, row_ptr[r0] + max(1, int(budget_ge // max(f, 1))), side="left"))
    r1 = max(r0 + 1, min(r1, n))
    ge = int(row_ptr[r1] - row_ptr[r0]) * f
    t0 = time.perf_counter()
    orc.spmm(row_ptr, col, a64, x, f=f, r0=r0, r1=r1, want_cond=False, omp=omp)
    dt = time.perf_counter() - t0
    return {"GE/s": ge / dt, "s": dt, "rows": [r0, r1], "GE": ge}


def oracle_mh_rate(row_ptr, col, alpha, z, H, D, budget_ge, omp=False):
    import oracle as orc
    n = row_ptr.size - 1
    r1 = int(np.searchsorted(row_ptr, max(1, int(budget_ge // (H * D))), side="left"))
    r1 = max(1, min(r1, n))
    ge = int(row_ptr[r1]) * H * D
    t0 = time.perf_counter()
    orc.multihead_spmm(row_ptr, col, alpha, z, H, D, r0=0, r1=r1, want_cond=False, omp=omp)
    dt = time.perf_counter() - t0
    return {"GE/s": ge / dt, "s": dt, "rows": [0, r1], "GE": ge}


def oracle_legs(fn, budget_1t, budget_nt):
    import oracle as orc
    one = fn(budget_1t, False)
    allc = fn(budget_nt, True)
    cores = orc.usable_cores()
    return {"oracle_1t": one, "oracle_nt": dict(allc, threads=int(os.environ.get("OMP_NUM_THREADS", cores))),
            "cores": cores}


def run_reference(args):
    """--impl reference: there is no reference implementation (the paper ships
    no code); the oracle is timed on the host cores, same metric / config."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle as orc
    from synth import CONFIGS, features, graph_for
    cfg = CONFIGS[args.config]
    s, d = graph_for(cfg, seed=1)
    g = orc.build_csr(cfg.n, s, d, None, True, 1.0)
    _, a64, _ = orc.sym_norm(g)
    x = features(cfg.n, cfg.f, cfg.ld, seed=2)
    orc.lib_omp()
    threads = int(os.environ.get("OMP_NUM_THREADS", orc.usable_cores()))
    times, ges = [], []
    for i in range(args.warmup + args.steps):
        r = oracle_rate(g.row_ptr, g.col, a64, x, cfg.f, args.ref_budget_ge, omp=True, start_row=i * 7919)
        if i >= args.warmup:
            times.append(r["s"])
            ges.append(r["GE"])
    value = float(sum(ges) / sum(times))
    sample = (f"each step: a contiguous row range of {cfg.name} with {np.mean(ges) / 1e9:.2f} G edge x feature "
              f"units (of {cfg.nnz * cfg.f / 1e9:.2f} G per full SpMM), fp64 oracle on {threads} threads "
              f"({orc.cpu_model()})")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GE/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(times)),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg.name, "n": cfg.n, "nnz": cfg.nnz, "f": cfg.f,
                   "graph": "chung-lu gamma=2.5 seed=1", "sample": sample},
        "cpu_baseline": {"value": value, "unit": "GE/s", "cores": threads, "kind": "oracle", "sample": sample,
                         "cpu_model": orc.cpu_model()},
        "e2e": {"value": value, "unit": "GE/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0}), flush=True)
    return 0


# ---------------------------------------------------------------------------
# per-config rows (single GPU)
# ---------------------------------------------------------------------------

PAPER_CONTEXT = {
    "C3": "Table spmm_time GAT Flickr: CogDL 9 ms end-to-end inference on RTX 3090 (P:691)",
    "C4": "Table spmm_time GCN Reddit: CogDL 22 ms end-to-end inference on RTX 3090 (P:679); "
          "GSpMM sum/mean 1.70-4.04x DGL (P:1355)",
    "C5": "Table spmm_time GCN Yelp: CogDL 23 ms end-to-end on RTX 3090 (P:680)",
    "C6": "Yelp x10: no paper number (SURVEY §8(d)2)",
}


class Ctx:
    def __init__(self, args, dev, peak):
        import torch
        self.args, self.dev, self.peak = args, dev, peak
        self.timer = Timer(dev)
        self.ncu = ncu_table()
        self.torch = torch


def build_config(ctx, key, oracle_csr=True):
    """Device CSR (+ the oracle's own host CSR for the parity / oracle legs)."""
    import oracle as orc
    import paper_2103_00959_b200 as G
    from synth import CONFIGS, graph_for
    torch = ctx.torch
    cfg = CONFIGS[key]
    s, d = graph_for(cfg, seed=1)
    st, dt = torch.from_numpy(s).to(ctx.dev), torch.from_numpy(d).to(ctx.dev)
    g = G.gsp_coo_to_csr(cfg.n, st, dt, None, True, 1.0)
    gn = G.gsp_sym_normalize(g)
    host = None
    if oracle_csr:
        go = orc.build_csr(cfg.n, s, d, None, True, 1.0)
        deg, a64, a32 = orc.sym_norm(go)
        exact = bool(gn.nnz == go.nnz and np.array_equal(gn.row_ptr.cpu().numpy(), go.row_ptr)
                     and np.array_equal(gn.col.cpu().numpy(), go.col)
                     and np.array_equal(gn.val.cpu().numpy().view(np.uint32), a32.view(np.uint32))
                     and np.array_equal(gn.deg.cpu().numpy(), deg))
        host = {"go": go, "deg": deg, "a64": a64, "csr_bit_exact": exact}
    return cfg, (st, dt), g, gn, host


def report_row(ctx, cfg, op, P, ts, warm, ge, bytes_, extra=None):
    alg, bmin = bytes_
    t = float(np.median(ts)) * 1e-3
    r = {"config": cfg.name, "op": op, "P": P, "graph_seed": 1, "generator": "chung-lu gamma=2.5",
         "n": cfg.n, "nnz": cfg.nnz, **tstats(ts), "t_warm_ms": warm,
         "GE/s": ge / t if ge else None, "B_alg": alg, "B_min": bmin,
         "B_alg/t GB/s": alg / t / 1e9, "B_alg/t frac_measured_peak": alg / t / 1e9 / ctx.peak,
         "B_alg/t frac_nominal": alg / t / 1e9 / NOMINAL_HBM,
         "B_min/t frac_measured_peak": bmin / t / 1e9 / ctx.peak}
    nc = ctx.ncu.get((cfg.name, op))
    if nc and nc.get("dram_bytes"):
        r["ncu_dram_bytes"] = nc["dram_bytes"]
        r["ncu_dram_GB/s"] = nc["dram_bytes"] / t / 1e9
        r["ncu_dram_frac_measured_peak"] = r["ncu_dram_GB/s"] / ctx.peak
        r["ncu_dram_frac_nominal"] = r["ncu_dram_GB/s"] / NOMINAL_HBM
        r["ncu_l2_hit_pct"] = nc.get("l2_hit_pct")
        r["ncu_source"] = nc.get("source")
    if extra:
        r.update(extra)
    if cfg.name[:2] in PAPER_CONTEXT:
        r["paper_context"] = PAPER_CONTEXT[cfg.name[:2]]
    return r


def gcn_rows(ctx, key, full_parity, budget_1t, budget_nt, with_build=False):
    """a3 SpMM (+ a1 build, a2 normalise) on a GCN config."""
    import oracle as orc
    import paper_2103_00959_b200 as G
    from synth import features
    torch, a = ctx.torch, ctx.args
    cfg, (st, dt), g, gn, host = build_config(ctx, key)
    n, nnz, f = cfg.n, gn.nnz, cfg.f
    rows = []
    if with_build:
        tb = ctx.timer.cold(lambda: G.gsp_coo_to_csr(n, st, dt, None, True, 1.0), 1, 3)
        tn = ctx.timer.cold(lambda: G.gsp_sym_normalize(g), 1, 5)
        m = st.numel()
        rows.append(report_row(ctx, cfg, "a1_build", 1, tb, None, None,
                               (16 * m + 8 * (n + 1) + 8 * nnz, 16 * m + 8 * (n + 1) + 8 * nnz),
                               {"model": "read int64 pairs 16m + write row_ptr, col, val once (sort passes excluded)",
                                "csr_bit_exact": host["csr_bit_exact"]}))
        rows.append(report_row(ctx, cfg, "a2_normalize", 1, tn, None, None,
                               (8 * (n + 1) + 12 * nnz + 8 * n, 8 * (n + 1) + 12 * nnz + 8 * n),
                               {"model": "row_ptr + col, val read + val write + degree write",
                                "csr_bit_exact": host["csr_bit_exact"]}))
    del st, dt
    x_host = features(n, f, cfg.ld, seed=2)
    # the library's feature layout: rows on whole 128-byte L2 lines
    x = G.empty_features(n, f, ctx.dev)
    x.copy_(torch.from_numpy(x_host[:, :f]))
    y = G.empty_features(n, f, ctx.dev)

    def step():
        G.gsp_spmm(gn, x, f=f, y=y)
    ts = ctx.timer.cold(step, a.warmup, max(10, a.steps // 2))
    warm = ctx.timer.warm(step, 10)
    step()
    yh = y.cpu().numpy()
    # column blocks (gsp_spmm_blocked) where G.colblock_bounds chooses more than one
    bounds = G.colblock_bounds(gn, f)
    blocks, yb = None, None
    if len(bounds) > 2:
        tplan = ctx.timer.cold(lambda: G.gsp_csr_colblock(gn, bounds), 1, 3)
        blocks = G.gsp_csr_colblock(gn, bounds)

        def step_b():
            G.gsp_spmm_blocked(blocks, x, f=f, y=y)
        tsb = ctx.timer.cold(step_b, a.warmup, max(10, a.steps // 2))
        warmb = ctx.timer.warm(step_b, 10)
        step_b()
        yb = y.cpu().numpy()
    go, a64 = host["go"], host["a64"]
    outs = {"plain": yh} if yb is None else {"plain": yh, "blocked": yb}
    pars = {}
    if full_parity:
        yref, cond = orc.spmm(go.row_ptr, go.col, a64, x_host, f=f, omp=True)
        for k, yy in outs.items():
            pars[k] = {"max_err_over_bound": err_ratio(yy, yref, cond), "checked": "full output"}
        del yref, cond
    else:
        rs = sample_rows(go.row_ptr, 400, seed=7)
        worst = {k: 0.0 for k in outs}
        for r in rs:
            yr, cr = orc.spmm(go.row_ptr, go.col, a64, x_host, f=f, r0=int(r), r1=int(r) + 1)
            for k, yy in outs.items():
                worst[k] = max(worst[k], err_ratio(yy[r:r + 1], yr, cr))
        for k in outs:
            pars[k] = {"max_err_over_bound": worst[k], "checked": f"{rs.size} sampled rows incl. the 16 heaviest hubs"}
    for par in pars.values():
        par["csr_bit_exact"] = host["csr_bit_exact"]
        par["pass"] = bool(par["max_err_over_bound"] <= 1.0 and par["csr_bit_exact"])
    legs = oracle_legs(lambda b, omp: oracle_rate(go.row_ptr, go.col, a64, x_host, f, b, omp=omp),
                       budget_1t, budget_nt)
    plan = G.gsp_spmm_plan_info(gn, x, f)
    rows.append(report_row(ctx, cfg, "a3_spmm", 1, ts, warm, nnz * f, spmm_bytes(n, nnz, f),
                           {"F": f, "parity": pars["plain"], **legs, "launches": plan[0],
                            "plan": {"slab_cols": plan[1], "tail_slab_cols": plan[2]}}))
    if blocks is not None:
        nl = sum(G.gsp_spmm_plan_info(blocks.block(k), x, f)[0] for k in range(len(blocks)))
        rows.append(report_row(ctx, cfg, "a3_spmm_colblocked", 1, tsb, warmb, nnz * f, spmm_bytes(n, nnz, f),
                               {"F": f, "parity": pars["blocked"], "launches": nl,
                                "plan": {"column_blocks": len(blocks), "col_bounds": bounds,
                                         "block_nnz": blocks.nnz, "plan_ms_one_off": float(np.median(tplan)),
                                         "slab_cols": plan[1], "tail_slab_cols": plan[2]},
                                "note": "Y = A_0 X, Y += A_1 X over column halves (gsp_csr_colblock + "
                                        "gsp_spmm_blocked): each launch gathers from half of X's rows"}))
    return rows, (cfg, g, gn, host, x, x_host, y, blocks)


def gat_rows(ctx, key, H, D, full_parity, budget_1t, budget_nt):
    """a4 attention projection, a5-a7 fused aggregate, a6 edge softmax, a7
    multi-head SpMM on a GAT config."""
    import oracle as orc
    import paper_2103_00959_b200 as G
    from synth import uniform
    import dataclasses
    torch, a = ctx.torch, ctx.args
    cfg, _, g, gn, host = build_config(ctx, key)
    if "-gat" in cfg.name:  # the row names the head shape it ran (C2g runs 8 x 8 and 8 x 64)
        cfg = dataclasses.replace(cfg, name=f"{cfg.name.split('-gat')[0]}-gat{H}x{D}")
    n, nnz = cfg.n, g.nnz
    z_h = uniform((n, H * D), seed=3)
    al_h, ar_h = uniform((H, D), seed=6), uniform((H, D), seed=7)
    z = torch.from_numpy(z_h).to(ctx.dev)
    al = torch.from_numpy(al_h.reshape(-1)).to(ctx.dev)
    ar = torch.from_numpy(ar_h.reshape(-1)).to(ctx.dev)
    el, er = G.gsp_attn_project(z, al, ar, H, D)
    y = G.empty_features(n, H * D, ctx.dev)
    ws = torch.empty(G.gsp_gat_workspace(g, H), dtype=torch.uint8, device=ctx.dev)
    reps = max(10, a.steps // 2)
    t_ap = ctx.timer.cold(lambda: G.gsp_attn_project(z, al, ar, H, D, el=el, er=er), a.warmup, reps)
    w_ap = ctx.timer.warm(lambda: G.gsp_attn_project(z, al, ar, H, D, el=el, er=er), 10)
    fused = lambda: G.gsp_gat_aggregate(g, el, er, z, H, D, 0.2, y=y, ws=ws)
    t_g = ctx.timer.cold(fused, a.warmup, reps)
    w_g = ctx.timer.warm(fused, 10)
    t_g1 = ctx.timer.cold(lambda: G.gsp_gat_aggregate(g, el, er, z, H, D, 0.2, y=y, single_launch=True),
                          a.warmup, reps)
    _, alpha = G.gsp_gat_aggregate(g, el, er, z, H, D, 0.2, y=y, alpha_out=True, ws=ws)
    logits = alpha.clone()
    t_sm = ctx.timer.cold(lambda: G.gsp_edge_softmax(g, logits, H, alpha=alpha), a.warmup, reps)
    w_sm = ctx.timer.warm(lambda: G.gsp_edge_softmax(g, logits, H, alpha=alpha), 10)
    t_mh = ctx.timer.cold(lambda: G.gsp_multihead_spmm(g, alpha, z, H, D, y=y), a.warmup, reps)
    w_mh = ctx.timer.warm(lambda: G.gsp_multihead_spmm(g, alpha, z, H, D, y=y), 10)
    # parity (in-run): el / er on every row; alpha on every entry; Y full or sampled rows
    go = host["go"]
    el_r, er_r, elc, erc = orc.attn_project(z_h, al_h, ar_h, H, D)
    p_ap = max(err_ratio(el.cpu().numpy(), el_r, elc), err_ratio(er.cpu().numpy(), er_r, erc))
    _, alpha = G.gsp_gat_aggregate(g, el, er, z, H, D, 0.2, y=y, alpha_out=alpha, ws=ws)
    yh, ah = y.cpu().numpy(), alpha.cpu().numpy()
    sc = orc.gat_scores(go.row_ptr, go.col, el.cpu().numpy(), er.cpu().numpy(), H, 0.2)
    aref = orc.edge_softmax(go.row_ptr, sc, H)
    p_alpha = float(np.max(np.abs(ah - aref) / (1e-5 * aref + 1e-9)))
    if full_parity:
        yref, cond = orc.multihead_spmm(go.row_ptr, go.col, aref, z_h, H, D, omp=True)
        p_y, how = err_ratio(yh, yref, cond), "full output; alpha on every entry"
        del yref, cond
    else:
        rs = sample_rows(go.row_ptr, 300, seed=8)
        p_y = 0.0
        for r in rs:
            yr, cr = orc.multihead_spmm(go.row_ptr, go.col, aref, z_h, H, D, r0=int(r), r1=int(r) + 1)
            p_y = max(p_y, err_ratio(yh[r:r + 1], yr, cr))
        how = f"{rs.size} sampled rows incl. the 16 heaviest hubs; alpha on every entry"
    par = {"max_err_over_bound": max(p_y, p_alpha), "y": p_y, "alpha": p_alpha, "checked": how,
           "csr_bit_exact": host["csr_bit_exact"]}
    par["pass"] = bool(par["max_err_over_bound"] <= 1.0 and par["csr_bit_exact"])
    # standalone a6 (softmax of the given logits, every entry) and a7 (given alpha)
    lg_h = logits.cpu().numpy()
    G.gsp_edge_softmax(g, logits, H, alpha=alpha)
    a6ref = orc.edge_softmax(go.row_ptr, lg_h.astype(np.float64), H)
    p6 = float(np.max(np.abs(alpha.cpu().numpy() - a6ref) / (1e-5 * a6ref + 1e-9)))
    par6 = {"max_err_over_bound": p6, "checked": "alpha on every entry", "pass": p6 <= 1.0}
    a_h = alpha.cpu().numpy()
    G.gsp_multihead_spmm(g, alpha, z, H, D, y=y)
    y7 = y.cpu().numpy()
    if full_parity:
        y7r, c7 = orc.multihead_spmm(go.row_ptr, go.col, a_h.astype(np.float64), z_h, H, D, omp=True)
        p7, how7 = err_ratio(y7, y7r, c7), "full output"
        del y7r, c7
    else:
        p7 = 0.0
        for r in rs:
            yr, cr = orc.multihead_spmm(go.row_ptr, go.col, a_h.astype(np.float64), z_h, H, D, r0=int(r), r1=int(r) + 1)
            p7 = max(p7, err_ratio(y7[r:r + 1], yr, cr))
        how7 = f"{rs.size} sampled rows"
    par7 = {"max_err_over_bound": p7, "checked": how7, "pass": p7 <= 1.0}
    legs = oracle_legs(lambda b, omp: oracle_mh_rate(go.row_ptr, go.col, aref, z_h, H, D, b, omp=omp),
                       budget_1t, budget_nt)
    ge = nnz * H * D
    common = {"H": H, "D": D}
    rows = [
        report_row(ctx, cfg, "a4_attn_project", 1, t_ap, w_ap, None, attn_bytes(n, H, D),
                   {**common, "parity": {"max_err_over_bound": p_ap, "checked": "el, er on every row",
                                         "pass": p_ap <= 1.0}, "launches": 1}),
        report_row(ctx, cfg, "a5-a7_gat_fused", 1, t_g, w_g, ge, gat_bytes(n, nnz, H, D),
                   {**common, "parity": par, **legs, "launches": 2,
                    "single_launch_schedule": tstats(t_g1),
                    "kernels": "row_stats_warp (softmax statistics, all heads) + engine_kernel<WeightGatT<1>>"}),
        report_row(ctx, cfg, "a6_edge_softmax", 1, t_sm, w_sm, None, softmax_bytes(n, nnz, H),
                   {**common, "edge-heads/s": nnz * H / (float(np.median(t_sm)) * 1e-3), "launches": 1,
                    "parity": par6}),
        report_row(ctx, cfg, "a7_multihead_spmm", 1, t_mh, w_mh, ge, mh_bytes(n, nnz, H, D),
                   {**common, "launches": 1, "parity": par7}),
    ]
    return rows, (cfg, g, el, er, z, y, ws, alpha, logits)


# ---------------------------------------------------------------------------
# secondaries (NEXT rows of §8(f)); reported, not the headline
# ---------------------------------------------------------------------------

def secondaries(ctx, c4, c3):
    import paper_2103_00959_b200 as G
    from synth import CONFIGS, features, graph_for
    torch, a = ctx.torch, ctx.args
    out = {}
    cfg, g, gn, host, x, x_host, y, _ = c4
    n, nnz, f = cfg.n, gn.nnz, cfg.f
    red = {}
    for r_ in ("mean", "max", "min"):
        ts = ctx.timer.cold(lambda: G.gsp_gspmm(gn, x, r_, f=f, y=y), a.warmup, 10)
        red[r_] = {"ms": float(np.median(ts)), "GE/s": nnz * f / (np.median(ts) * 1e-3)}
    out["NEXT2_C4_gspmm_reduce"] = red
    ld16 = (f + 3) // 4 * 4
    x16 = torch.zeros((n, ld16), dtype=torch.float16, device=ctx.dev)
    x16[:, :f] = x[:, :f].half()
    t16 = ctx.timer.cold(lambda: G.gsp_spmm_f16(gn, x16, f=f, y=y), a.warmup, 10)
    b16 = 2 * nnz * f + 4 * n * f + 8 * nnz + 8 * (n + 1)
    out["NEXT4_C4_spmm_f16_storage"] = {
        "ms": float(np.median(t16)), "GE/s": nnz * f / (np.median(t16) * 1e-3),
        "alg_GB/s": b16 / (np.median(t16) * 1e-3) / 1e9,
        "note": "x stored in fp16, converted exactly, fp32 products and sums (gsp_spmm_f16); not the headline"}
    del x16
    fk, K = 41, 10
    xk = G.empty_features(n, fk, ctx.dev)
    xk.copy_(torch.from_numpy(features(n, fk, fk, seed=9)))
    yk = G.empty_features(n, fk, ctx.dev)
    th = [0.1 * 0.9 ** k for k in range(K + 1)]
    tk = ctx.timer.cold(lambda: G.gsp_propagate(gn, xk, th, f=fk, y=yk), a.warmup, 5)
    out["NEXT4_C4_appnp_K10_f41"] = {"ms": float(np.median(tk)), "GE/s": K * nnz * fk / (np.median(tk) * 1e-3),
                                     "launches": K}
    del xk, yk
    c3cfg, g3, el, er, z, y3, ws, alpha3, logits3 = c3
    H, D = c3cfg.heads, c3cfg.d
    at3, perm3 = G.gsp_csr_transpose(g3)
    t_tr = ctx.timer.cold(lambda: G.gsp_csr_transpose(g3), 1, 3)
    t_sd = ctx.timer.cold(lambda: G.gsp_sddmm(g3, y3, z, heads=H, out=logits3), a.warmup, 10)
    t_sb = ctx.timer.cold(lambda: G.gsp_edge_softmax_backward(g3, alpha3, logits3, H, ds=logits3), a.warmup, 10)
    t_gb = ctx.timer.cold(lambda: G.gsp_gat_aggregate_backward(g3, at3, perm3, el, er, z, y3, H, D), a.warmup, 5)
    out["NEXT3_C3_gat_backward"] = {"csr_transpose_ms": float(np.median(t_tr)), "sddmm_ms": float(np.median(t_sd)),
                                    "softmax_backward_ms": float(np.median(t_sb)),
                                    "aggregate_backward_ms": float(np.median(t_gb))}
    del at3, perm3
    # NEXT-1 dense step alone: C4 layer 1 (232,965 x 602 -> 128) on the tcgen05
    # 3xTF32 GEMM, against the measured TF32 MMA rate (tools/mma_peak_probe.cu)
    # and the HBM copy peak; the x_lo * w_hi, x_hi * w_lo, x_hi * w_hi products
    # are the work the tensor pipe does
    fin, fout = f, 128
    xl = x[:, :fin]
    wl = torch.from_numpy(features(fin, fout, fout, seed=3)).to(ctx.dev)
    yl = G.empty_features(n, fout, ctx.dev)
    import ctypes
    nbl = ctypes.c_size_t(0)
    G.lib().gsp_linear_workspace(fin, fout, ctypes.byref(nbl))
    wsl = torch.empty(max(nbl.value, 16), dtype=torch.uint8, device=ctx.dev)
    tl_ = ctx.timer.cold(lambda: G.gsp_linear(xl, wl, y=yl, ws=wsl), a.warmup, 20)
    ml = float(np.median(tl_))
    tf = 3 * 2.0 * n * fin * fout / (ml * 1e-3) / 1e12
    bl = 4.0 * (n * fin + n * fout + 2 * fin * fout)
    out["NEXT1_C4_layer1_dense_step"] = {
        "ms": ml, "shape": [n, fin, fout], "TFLOPs_tf32_products": tf,
        "tf32_peak_TFLOPs": TF32_MMA_PEAK, "tf32_frac": tf / TF32_MMA_PEAK,
        "tf32_peak_kind": "measured tcgen05.mma kind::tf32 M=128 N=128 issue rate (profiles/r2i_mma_peak_probe.txt)",
        "hbm_GB/s": bl / (ml * 1e-3) / 1e9, "hbm_frac": bl / (ml * 1e-3) / 1e9 / ctx.peak,
        "kernel": "linear_tc_kernel<true, 2> (3xTF32, CTA pairs sharing W)"}
    del xl, wl, yl, wsl
    # NEXT-1: the paper's Table spmm_time workload (2-layer GCN / GAT inference,
    # hidden 128, GAT 4 heads; both readings of A20: 4 x 32 and 4 x 128 per head)
    from paper_2103_00959_b200.inference import GATParams, GCNParams, gat_inference, gcn_inference
    paper = {"C3": ("Flickr", 500, 7, 0.002, 0.009), "C4": ("Reddit", 602, 41, 0.022, 0.080),
             "C5": ("Yelp", 300, 100, 0.023, 0.081)}  # (name, feats, classes, GCN s, GAT s) P:24-26
    table = {}
    for key, (dname, fin, ncls, t_gcn, t_gat) in paper.items():
        cfg_k = CONFIGS[key]
        if key == "C4":
            gk = gn
        else:
            sk, dk = graph_for(cfg_k, seed=1)
            gk = G.gsp_sym_normalize(G.gsp_coo_to_csr(cfg_k.n, torch.from_numpy(sk).to(ctx.dev),
                                                      torch.from_numpy(dk).to(ctx.dev), None, True, 1.0))
        xk = G.empty_features(cfg_k.n, fin, ctx.dev)
        xk.copy_(torch.from_numpy(features(cfg_k.n, fin, fin, seed=2)))
        pg = GCNParams.init(fin, 128, ncls, ctx.dev, seed=1)
        pa = GATParams.init(fin, 128, 4, ncls, ctx.dev, seed=1)
        pa4 = GATParams.init(fin, 512, 4, ncls, ctx.dev, seed=1)
        res = {}
        for mname, fn_ in (("gcn", lambda: gcn_inference(gk, xk, pg)), ("gat_4x32", lambda: gat_inference(gk, xk, pa)),
                           ("gat_4x128", lambda: gat_inference(gk, xk, pa4))):
            res[mname + "_ms"] = float(np.median(ctx.timer.cold(fn_, a.warmup, 10)))
        res["paper_3090_gcn_ms"] = 1e3 * t_gcn
        res["paper_3090_gat_ms"] = 1e3 * t_gat
        table[f"{key}-{dname}"] = res
        del xk
    out["NEXT1_table_spmm_time"] = {
        "workload": "2-layer GCN (hidden 128, ReLU) and GAT (4 heads x 32 and 4 heads x 128 per head, ELU; 1 output "
                    "head) inference, random weights, synthetic graphs with the paper's node/edge/feature/class counts",
        "note": "paper times are CogDL on an RTX 3090 (P:678-693), fp32, context only (other hardware)",
        "results": table}
    return out


def e2e_single(ctx, c4):
    import paper_2103_00959_b200 as G
    from paper_2103_00959_b200.host import HostSpMM
    torch, a = ctx.torch, ctx.args
    cfg, g, gn, host, x, x_host, y, blocks = c4
    n, f = cfg.n, cfg.f
    xh = torch.from_numpy(x_host).pin_memory()
    yh = torch.empty((n, cfg.ld), dtype=torch.float32).pin_memory()
    hs = HostSpMM(gn, f, G.feature_ld(f), device=ctx.dev, blocks=blocks)
    st = torch.cuda.current_stream()
    ts = []
    for i in range(a.warmup + max(3, a.steps // 3)):
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(st)
        hs(xh, yh)
        a1.record(st)
        torch.cuda.synchronize()
        if i >= a.warmup:
            ts.append(a0.elapsed_time(a1))
    te = float(np.mean(ts))
    y_chk = G.gsp_spmm_blocked(blocks, x, f=f) if blocks is not None else G.gsp_spmm(gn, x, f=f)
    return {"value": gn.nnz * f / (te * 1e-3), "unit": "GE/s", "ms_per_step": te,
            "h2d_bytes_per_step": int(n * f * 4), "d2h_bytes_per_step": int(n * f * 4),
            "bitwise_equal_to_device_path": bool(torch.equal(yh[:, :f], y_chk.cpu())),
            "launches_per_step": hs.launches(),
            "api": "paper_2103_00959_b200.host.HostSpMM: per-128-column slab H2D (2-D DMA) || " +
                   ("gsp_spmm_blocked" if blocks is not None else "gsp_spmm") + " || D2H"}


def main_single(args):
    import torch
    import oracle as orc
    import paper_2103_00959_b200 as G
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    G.lib()  # fail loudly if the extension is missing
    peak, peak_kind = hbm_peak()
    ctx = Ctx(args, dev, peak)
    # --- headline config: a1 + a2 + a3 rows; the timed loop below is the headline
    rows, c4 = gcn_rows(ctx, args.config, full_parity=not args.sampled_parity, budget_1t=args.cpu_budget_ge,
                        budget_nt=args.cpu_budget_ge * 8, with_build=True)
    cfg, g, gn, host, x, x_host, y, blocks = c4
    n, nnz, f = cfg.n, gn.nnz, cfg.f
    launches, plan_slab, plan_tail = G.gsp_spmm_plan_info(gn, x, f)
    # the step: the column-blocked SpMM when G.colblock_bounds chose blocks for
    # this graph (A split once, before timing, like the CSR build), else gsp_spmm
    head_op = "a3_spmm_colblocked" if blocks is not None else "a3_spmm"
    if blocks is not None:
        launches = sum(G.gsp_spmm_plan_info(blocks.block(k), x, f)[0] for k in range(len(blocks)))

    def step():
        if blocks is not None:
            G.gsp_spmm_blocked(blocks, x, f=f, y=y)
        else:
            G.gsp_spmm(gn, x, f=f, y=y)
    for _ in range(args.warmup):
        step()
    flush = ctx.timer.flush
    st = torch.cuda.current_stream()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with Clocks(0) as clk:
        torch.cuda.synchronize()
        for i in range(args.steps):
            flush.zero_()  # L2 flush (untimed: outside the events)
            starts[i].record(st)
            step()
            ends[i].record(st)
        torch.cuda.synchronize()
    times = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    t_ms = float(np.mean(times))
    warm = ctx.timer.warm(step, args.steps)
    ge = nnz * f
    alg, bmin = spmm_bytes(n, nnz, f)
    a3 = [r for r in rows if r["op"] == "a3_spmm"][0]
    a3h = [r for r in rows if r["op"] == head_op][0]
    nc = ctx.ncu.get((cfg.name, head_op))
    dram = nc.get("dram_bytes") if nc else None
    # The SpMM is a gather through L2 (57 GB of row-slab gathers per step
    # against 1.3 GB of compulsory traffic, 86% L2 hits): its roofline is the
    # measured service rate of random 512-byte row gathers from an L2-resident
    # X (8 LDG.128 in flight per lane, 32 warps/SM; profiles/r1_probes.txt,
    # profiles/r2c_gather_ceiling_probe.txt: more parallelism does not raise
    # it).  achieved = the algorithmic (gather-model) bytes / the step time.
    # The HBM view (ncu DRAM bytes / time against the copy peak) is kept in
    # roofline["hbm"]; it FALLS as the L2 hit rate rises.
    roof = {"bound": "l2", "achieved": alg / (t_ms * 1e-3) / 1e9, "peak": L2_GATHER_PEAK_GBS, "unit": "GB/s",
            "frac": alg / (t_ms * 1e-3) / 1e9 / L2_GATHER_PEAK_GBS, "traffic": dram,
            "achieved_kind": "algorithmic bytes (gather model 4*nnz*F + 4*n*F + 8*nnz + 8*(n+1): one X row-slab "
                             "per nonzero, Y, CSR) / mean step time",
            "peak_kind": "measured random 512-byte row-gather rate from an L2-resident X (profiles/r1_probes.txt)",
            "traffic_kind": "ncu dram__bytes_read.sum + dram__bytes_write.sum of the step's launches",
            "traffic_source": nc.get("source") if nc else None,
            "kernel": "engine_kernel<4,32,WeightVal,RedSum,XF32<4>> (" +
                      ("gsp_spmm_blocked: one launch per column block" if blocks is not None else "gsp_spmm") + ")",
            "alg_bytes_gather_model": alg, "alg_bytes_compulsory": bmin,
            "compulsory_GB/s": bmin / (t_ms * 1e-3) / 1e9}
    l2b = nc.get("l2_bytes") if nc else None
    if l2b:
        roof["l2_traffic_GB/s"] = l2b / (t_ms * 1e-3) / 1e9
        roof["l2_traffic_kind"] = "ncu lts__t_bytes.sum of the step's launches / mean step time"
    roof["hbm"] = {"peak": peak, "unit": "GB/s", "peak_kind": peak_kind,
                   "achieved": dram / (t_ms * 1e-3) / 1e9 if dram else None,
                   "frac": dram / (t_ms * 1e-3) / 1e9 / peak if dram else None,
                   "achieved_kind": "ncu DRAM bytes of the step's launches / mean step time",
                   "compulsory_frac": bmin / (t_ms * 1e-3) / 1e9 / peak}
    out = {
        "metric": METRIC, "value": ge / (t_ms * 1e-3), "unit": "GE/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_ms, "ms_per_step_median": float(np.median(times)),
        "ms_per_step_min": float(np.min(times)), "ms_per_step_p90": float(np.percentile(times, 90)),
        "ms_per_step_warm_no_flush": warm, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": cfg.name, "n": n, "nnz": nnz, "f": f, "ldx": x.stride(0), "ldy": y.stride(0),
                   "layout": "row-major fp32, rows padded to whole 128-byte lines (G.feature_ld)",
                   "graph": f"chung-lu gamma=2.5 seed=1 ({cfg.note}; node/pair counts P:18-26)",
                   "l2": "flushed before every step (256 MB memset, untimed); X (562 MB) > L2 as well",
                   "parallelism": "single GPU",
                   "plan": {"launches": launches, "slab_cols": plan_slab, "tail_slab_cols": plan_tail,
                            **({"column_blocks": len(blocks), "col_bounds": blocks.bounds,
                                "plan_ms_one_off": a3h["plan"]["plan_ms_one_off"]} if blocks is not None else {})}},
        "roofline": roof,
        "clocks": clk.summary(),
        "gpu_launches": launches * args.steps,
        "parity": a3h["parity"],
        "ms_per_step_gsp_spmm_unblocked": a3["t_cold_median_ms"],
    }
    report = list(rows)
    if not args.no_e2e:
        out["e2e"] = e2e_single(ctx, c4)
    # --- cpu_baseline: the oracle (as it stands) on all host cores, plus one core
    out["cpu_baseline"] = {
        "value": a3["oracle_nt"]["GE/s"], "unit": "GE/s", "cores": a3["oracle_nt"]["threads"], "kind": "oracle",
        "sample": f"rows {a3['oracle_nt']['rows']} of {cfg.name} ({a3['oracle_nt']['GE'] / 1e9:.2f} G GE, "
                  f"{a3['oracle_nt']['s']:.1f} s), fp64 oracle (liboracle_omp.so, OpenMP row loop)",
        "cpu_model": orc.cpu_model(), "usable_cores": orc.usable_cores(),
        "compiler": "gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math [-fopenmp]",
        "single_thread": {"value": a3["oracle_1t"]["GE/s"], "cores": 1,
                          "sample": f"rows {a3['oracle_1t']['rows']} ({a3['oracle_1t']['GE'] / 1e9:.2f} G GE, "
                                    f"{a3['oracle_1t']['s']:.1f} s)"}}
    # --- the other configs' rows
    c3 = None
    if not args.no_rows:
        for key in ("C1", "C2", "C5") + (("C6",) if args.with_c6 else ()):
            if key == args.config:
                continue
            r_, ctx_k = gcn_rows(ctx, key, full_parity=key != "C6" and not args.sampled_parity,
                                 budget_1t=min(args.cpu_budget_ge, 0.5e9), budget_nt=min(args.cpu_budget_ge, 2e9))
            report += r_
            del ctx_k
            torch.cuda.empty_cache()
        for key, H, D in (("C2g", 8, 8), ("C2g", 8, 64), ("C3", 8, 64)):
            r_, ctx_k = gat_rows(ctx, key, H, D, full_parity=True, budget_1t=0.3e9, budget_nt=1e9)
            report += r_
            if key == "C3":
                c3 = ctx_k
    if not args.no_secondary and c3 is not None:
        out["secondary"] = secondaries(ctx, c4, c3)
    out["parity_all_pass"] = bool(all(r["parity"]["pass"] for r in report if "parity" in r))
    out["report"] = report
    if args.report:
        with open(args.report, "w") as fh:
            for r in report:
                fh.write(json.dumps(r) + "\n")
    print(json.dumps(out), flush=True)
    return 0


# ---------------------------------------------------------------------------
# multi-GPU: one process per GPU (NCCL), row partition + chunked all-gather
# ---------------------------------------------------------------------------

def main_dist(args):
    import torch
    import torch.distributed as dist
    import paper_2103_00959_b200 as G
    from paper_2103_00959_b200.dist import RowPartitionedGAT, RowPartitionedSpMM
    from synth import CONFIGS, features, graph_for, uniform
    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    gloo = args.dist_backend == "gloo"
    if gloo:  # functional check of this path on a one-GPU box: ranks share the GPUs, host-staged all-gathers
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if gloo:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=dev)
    G.lib()

    def staged_gather(out, inp):
        parts = [torch.empty_like(inp, device="cpu") for _ in range(world)]
        dist.all_gather(parts, inp.cpu())
        out.copy_(torch.cat(parts, 0))
    ag = staged_gather if gloo else None
    peak, peak_kind = hbm_peak()
    cfg = CONFIGS[args.config]
    s, d = graph_for(cfg, seed=1)
    g = G.gsp_coo_to_csr(cfg.n, torch.from_numpy(s).to(dev), torch.from_numpy(d).to(dev), None, True, 1.0)
    gn = G.gsp_sym_normalize(g)
    del s, d
    n, nnz, f = cfg.n, gn.nnz, cfg.f
    # each rank generates the full X deterministically and keeps its own rows
    x_host = features(n, f, cfg.ld, seed=2)
    cb = G.colblock_bounds(gn, f)  # the single-GPU headline's column blocks (global bounds)
    op = RowPartitionedSpMM(gn, rank, world, f, chunks=args.chunks, device=dev, all_gather=ag,
                            col_blocks=cb if len(cb) > 2 else None)
    xs = torch.from_numpy(np.ascontiguousarray(x_host[op.r0:op.r1, :f])).to(dev)
    op.load_shard(xs)
    y = G.empty_features(op.rows, f, dev)
    timer = Timer(dev)

    def step():
        op(y)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    st = torch.cuda.current_stream()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with Clocks(local) as clk:
        torch.cuda.synchronize()
        for i in range(args.steps):
            timer.flush.zero_()
            dist.barrier()
            starts[i].record(st)
            step()
            ends[i].record(st)
        torch.cuda.synchronize()
    dist.barrier()
    t_ms = float(np.mean([a.elapsed_time(b) for a, b in zip(starts, ends)]))

    def allmax(v):
        t = torch.tensor([v], device="cpu" if gloo else dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())
    t_max = allmax(t_ms)
    # components: the all-gather alone and the local SpMM alone (same chunks)
    nch = len(op.cols) - 1
    t_comm = allmax(float(np.median(timer.cold(lambda: [op.exchange(k) for k in range(nch)], 2, 5))))
    t_comp = allmax(float(np.median(timer.cold(lambda: [op._local(k, y) for k in range(nch)], 2, 5))))
    # bitwise check of this rank's rows against the single-GPU gsp_spmm
    xfull = G.empty_features(n, f, dev)
    xfull.copy_(torch.from_numpy(x_host[:, :f]))
    step()
    torch.cuda.synchronize()
    y1 = G.gsp_spmm_blocked(G.gsp_csr_colblock(gn, cb), xfull, f=f) if len(cb) > 2 else G.gsp_spmm(gn, xfull, f=f)
    bitwise = allmax(0.0 if torch.equal(y, y1[op.r0:op.r1]) else 1.0) == 0.0
    del xfull, y1
    torch.cuda.empty_cache()
    alg, bmin = spmm_bytes(n, nnz, f)
    ge = nnz * f
    recv = 4 * n * f * (world - 1) / world
    # e2e: pinned host X shard -> device, all-gather + local SpMM, Y shard -> host
    xh = torch.from_numpy(np.ascontiguousarray(x_host[op.r0:op.r1, :f])).pin_memory()
    yh = torch.empty((op.rows, f), dtype=torch.float32).pin_memory()
    te_l = []
    for i in range(args.warmup + max(3, args.steps // 3)):
        dist.barrier()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(st)
        xs.copy_(xh, non_blocking=True)
        op.load_shard(xs)
        op(y)
        yh.copy_(y, non_blocking=True)
        a1.record(st)
        torch.cuda.synchronize()
        if i >= args.warmup:
            te_l.append(a0.elapsed_time(a1))
    te = allmax(float(np.mean(te_l)))
    # GAT (C3, 8 x 64): RowPartitionedGAT, all-gather Z and er, el local
    gat = None
    if not args.no_rows:
        c3 = CONFIGS["C3"]
        H, D = c3.heads, c3.d
        s3, d3 = graph_for(c3, seed=1)
        g3 = G.gsp_coo_to_csr(c3.n, torch.from_numpy(s3).to(dev), torch.from_numpy(d3).to(dev), None, True, 1.0)
        z = torch.from_numpy(uniform((c3.n, H * D), seed=3)).to(dev)
        al = torch.from_numpy(uniform((H, D), seed=6).reshape(-1)).to(dev)
        ar = torch.from_numpy(uniform((H, D), seed=7).reshape(-1)).to(dev)
        gt = RowPartitionedGAT(g3, rank, world, H, D, head_groups=1, device=dev, all_gather=ag)
        gt.load_shard(z[gt.r0:gt.r1])
        y3 = torch.empty((gt.rows, H * D), dtype=torch.float32, device=dev)
        ts3 = timer.cold(lambda: gt(al, ar, y3), args.warmup, 10)
        el, er = G.gsp_attn_project(z, al, ar, H, D)
        y3ref = G.gsp_gat_aggregate(g3, el, er, z, H, D, 0.2)
        gt(al, ar, y3)
        torch.cuda.synchronize()
        ok3 = allmax(0.0 if torch.equal(y3, y3ref[gt.r0:gt.r1]) else 1.0) == 0.0
        t3 = allmax(float(np.median(ts3)))
        gat = {"workload": c3.name, "ms": t3, "GE/s": g3.nnz * H * D / (t3 * 1e-3),
               "bitwise_equal_to_1gpu": ok3, "exchange": "all-gather Z (n x 512) and er (n x 8); el local"}
    out = {
        "metric": METRIC, "value": ge / (t_max * 1e-3), "unit": "GE/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_max, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": cfg.name, "n": n, "nnz": nnz, "f": f, "ldy": y.stride(0),
                   "layout": "row-major fp32, rows padded to whole 128-byte lines (G.feature_ld); shards chunk-packed",
                   "graph": f"chung-lu gamma=2.5 seed=1 ({cfg.note})",
                   "l2": "flushed before every step (256 MB memset, untimed)",
                   "parallelism": f"row partition x{world} (nnz-balanced) + NCCL all-gather of X, "
                                  f"{nch} column chunks overlapped with the local SpMM"},
        "roofline": {"bound": "hbm", "achieved": None, "peak": peak, "unit": "GB/s", "frac": None, "traffic": None,
                     "effective_GB/s_per_gpu": alg / world / (t_max * 1e-3) / 1e9,
                     "note": "per-rank DRAM traffic is not captured under multi-rank runs (ncu is single-GPU)"},
        "components": {"allgather_ms": t_comm, "local_spmm_ms": t_comp, "overlapped_step_ms": t_max,
                       "allgather_recv_bytes_per_rank": recv,
                       "allgather_GB/s_per_rank": recv / (t_comm * 1e-3) / 1e9 if world > 1 else None,
                       "rows_per_rank_max": op.npad, "bounds": op.bounds},
        "bitwise_equal_to_1gpu": bitwise,
        "dist_backend": args.dist_backend,
        "e2e": {"value": ge / (te * 1e-3), "unit": "GE/s", "ms_per_step": te,
                "h2d_bytes_per_step": int(n * f * 4), "d2h_bytes_per_step": int(n * f * 4),
                "api": "RowPartitionedSpMM (gsp_csr_slice + NCCL all-gather + gsp_spmm), pinned host shards"},
        "clocks": clk.summary(),
        "gpu_launches": sum(G.gsp_spmm_plan_info(op.local, gg, c1 - c0)[0]
                            for gg, c0, c1 in zip(op.gathered, op.cols[:-1], op.cols[1:])) * args.steps,
        "gat_row_partitioned": gat,
    }
    if rank == 0:
        print(json.dumps(out), flush=True)
    dist.destroy_process_group()
    return 0


def _json_stdout():
    """Keep stdout for the one JSON line: libraries that print banners to fd 1
    (NCCL prints its version at communicator creation) are moved to stderr;
    the JSON line goes to the saved original stdout."""
    sys.stdout.flush()
    saved = os.dup(1)
    os.dup2(2, 1)
    global print
    out = os.fdopen(saved, "w", buffering=1)
    _builtin_print = print

    def _print(*a, **k):
        if "file" not in k:
            k["file"] = out
        _builtin_print(*a, **k)
    print = _print


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--chunks", type=int, default=5, help="feature chunks (128-col aligned) for comm/compute overlap")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: run the N-rank path on fewer GPUs (functional check, host-staged all-gathers)")
    ap.add_argument("--no-rows", action="store_true", help="headline only (skip the other configs' rows)")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--with-c6", action="store_true", help="add the C6 (Yelp x10, 147M nnz) row")
    ap.add_argument("--sampled-parity", action="store_true", help="sampled rows instead of the full output")
    ap.add_argument("--cpu-budget-ge", type=float, default=1.0e9)
    ap.add_argument("--ref-budget-ge", type=float, default=4e9)
    ap.add_argument("--report", default="", help="also write the §8(d)7 rows as JSONL to this path")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    return args


if __name__ == "__main__":
    args = parse()
    if args.impl == "ours" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-execute under torch.distributed.run (before stdout is redirected)
        import socket
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
        sk.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    _json_stdout()
    if args.impl == "reference":
        sys.exit(run_reference(args))
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        sys.exit(main_dist(args))
    sys.exit(main_single(args))
