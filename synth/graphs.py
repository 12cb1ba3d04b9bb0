"""Seeded synthetic inputs shaped like the paper's datasets.

This module is shared by the oracle tests and the CUDA path.  It holds NONE of
the method's arithmetic (no CSR build, no normalisation, no aggregation): it
only draws random graphs (as undirected COO pair lists) and random feature
matrices, following the recipe in DESIGN.md §"Input recipe".

Shapes (node / pair counts) come from the paper's Table node_dataset,
PAPER.md:11-38 (Cora, Pubmed, Flickr, Reddit, Yelp rows P:18-26); see DESIGN.md
reading A18 for the directed/undirected edge-count reading.
"""
from __future__ import annotations

import dataclasses
import os
from typing import Optional

import numpy as np

# --------------------------------------------------------------------------
# Workload table (BASELINE.json configs)
# --------------------------------------------------------------------------


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    n: int            # nodes
    m: int            # undirected pairs (each listed once)
    f: int            # feature width (GCN) or H*D (GAT)
    heads: int = 1    # GAT heads (1 = GCN SpMM)
    d: int = 0        # GAT per-head width
    note: str = ""

    @property
    def ld(self) -> int:
        return (self.f + 3) // 4 * 4

    @property
    def nnz(self) -> int:
        """nnz of Â for a simple undirected graph with self-loops."""
        return 2 * self.m + self.n


CONFIGS = {
    # P:18 Cora 2,708 nodes; BASELINE "~10.6K directed edges" -> 5,278 pairs (A18)
    "C1": Config("C1-cora-gcn", 2708, 5278, 1433, note="Cora-shaped, GCN SpMM"),
    # P:20 Pubmed 19,717 nodes, 44,338 pairs
    "C2": Config("C2-pubmed-gcn", 19717, 44338, 500, note="Pubmed-shaped, GCN SpMM"),
    "C2g": Config("C2g-pubmed-gat8x8", 19717, 44338, 64, heads=8, d=8, note="Pubmed-shaped, GAT 8x8"),
    # P:24 Flickr 89,350 nodes, 899,756 edges
    "C3": Config("C3-flickr-gat8x64", 89350, 899756, 512, heads=8, d=64, note="Flickr-shaped, GAT 8x64"),
    # P:25 Reddit 232,965 nodes, 11,606,919 edges, 602 features
    "C4": Config("C4-reddit-gcn", 232965, 11606919, 602, note="Reddit-shaped, GCN SpMM"),
    # P:26 Yelp 716,847 nodes, 6,977,410 edges, 300 features
    "C5": Config("C5-yelp-gcn", 716847, 6977410, 300, note="Yelp-shaped, GCN SpMM"),
    "C6": Config("C6-yelp10x-gcn", 7168470, 69774100, 300, note="Yelp x10 power-law"),
    # calibration probes (not paper shapes): uniform random graphs whose X is
    # L2-resident (P1: 60K x 128 fp32 = 31 MB) or far larger than L2 (P2: 2M x 128 = 1 GB)
    "P1": Config("P1-probe-l2resident", 60000, 11600000, 128, note="L2-resident gather probe (ER)"),
    "P2": Config("P2-probe-dram", 2000000, 11600000, 128, note="DRAM gather probe (ER)"),
}

GENERATOR = {"P1": "er", "P2": "er"}  # default generator per config (else chung_lu)


# --------------------------------------------------------------------------
# Graph generators (undirected simple pair lists, ids randomly permuted)
# --------------------------------------------------------------------------


def _collect_unique_pairs(draw, n: int, m: int, rng: np.random.Generator):
    """Draw batches of endpoint pairs via draw(k) until m distinct unordered
    non-loop pairs exist; keep first occurrences in generation order."""
    keys_all = np.empty(0, dtype=np.int64)
    first = True
    uniq = 0
    while True:
        k = (int(1.25 * m) + 1024) if first else (int(1.5 * (m - uniq)) + 1024)
        first = False
        a, b = draw(k)
        keep = a != b
        a, b = a[keep], b[keep]
        lo = np.minimum(a, b)
        hi = np.maximum(a, b)
        keys_all = np.concatenate([keys_all, lo * np.int64(n) + hi])
        # distinct keys in order of first occurrence (hash-based; the same
        # sequence as np.unique(return_index) sorted by first index)
        uk = _unique_first(keys_all)
        uniq = uk.size
        if uniq >= m:
            keys = uk[:m]
            return keys // n, keys % n


def _unique_first(keys: np.ndarray) -> np.ndarray:
    try:
        import pandas as pd
        return pd.unique(keys)
    except ImportError:  # pragma: no cover
        _, idx = np.unique(keys, return_index=True)
        idx.sort()
        return keys[idx]


def _searchsorted_right(cdf: np.ndarray, u: np.ndarray) -> np.ndarray:
    """np.searchsorted(cdf, u, side="right") for u in [0, 1), cdf ascending:
    a guide table over 2^22 equal buckets of [0, 1) gives each u its first
    candidate, then a few vectorised steps advance while cdf[idx] <= u
    (exact: the count of cdf entries <= u)."""
    B = 1 << 22
    edges = np.arange(B + 1, dtype=np.float64) / B
    start = np.searchsorted(cdf, edges, side="right")
    j = np.minimum((u * B).astype(np.int64), B - 1)
    idx = start[j]
    n = cdf.size
    act = np.flatnonzero(idx < n)
    while act.size:
        adv = cdf[idx[act]] <= u[act]
        act = act[adv]
        idx[act] += 1
        act = act[idx[act] < n]
    return idx


def chung_lu(n: int, m: int, seed: int = 1, gamma: float = 2.5):
    """Chung-Lu power-law graph (primary generator).

    w_i = (i + i0 + 1)^(-1/(gamma-1)); i0 chosen by 60-step bisection so the
    expected max degree 2m*w_0/sum(w) equals min(n/4, 4*sqrt(2m)).
    Returns int64 arrays (src, dst) of m undirected pairs, ids permuted.
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    ex = -1.0 / (gamma - 1.0)
    i = np.arange(n, dtype=np.float64)
    target = min(n / 4.0, 4.0 * np.sqrt(2.0 * m))

    def max_deg(i0):
        w = (i + i0 + 1.0) ** ex
        return 2.0 * m * w[0] / w.sum()

    lo, hi = 0.0, float(n)
    if max_deg(0.0) <= target:
        i0 = 0.0
    else:
        for _ in range(60):
            mid = 0.5 * (lo + hi)
            if max_deg(mid) > target:
                lo = mid
            else:
                hi = mid
        i0 = 0.5 * (lo + hi)
    w = (i + i0 + 1.0) ** ex
    cdf = np.cumsum(w / w.sum())

    def draw(k):
        u = rng.random(2 * k)
        ab = np.minimum(_searchsorted_right(cdf, u), n - 1).astype(np.int64)
        return ab[:k], ab[k:]

    a, b = _collect_unique_pairs(draw, n, m, rng)
    perm = rng.permutation(n).astype(np.int64)
    return perm[a], perm[b]


def rmat(n: int, m: int, seed: int = 1, probs=(0.57, 0.19, 0.19, 0.05)):
    """R-MAT stress generator: scale ceil(log2 n), reject ids >= n."""
    rng = np.random.Generator(np.random.PCG64(seed))
    scale = max(1, int(np.ceil(np.log2(max(n, 2)))))
    p = np.asarray(probs, dtype=np.float64)
    cp = np.cumsum(p / p.sum())

    def draw(k):
        a = np.zeros(k, dtype=np.int64)
        b = np.zeros(k, dtype=np.int64)
        for _ in range(scale):
            q = np.searchsorted(cp, rng.random(k), side="right")
            a = (a << 1) | (q >> 1)
            b = (b << 1) | (q & 1)
        ok = (a < n) & (b < n)
        return a[ok], b[ok]

    a, b = _collect_unique_pairs(draw, n, m, rng)
    perm = rng.permutation(n).astype(np.int64)
    return perm[a], perm[b]


def erdos_renyi(n: int, m: int, seed: int = 1):
    """Uniform random simple graph (small parity cases)."""
    rng = np.random.Generator(np.random.PCG64(seed))

    def draw(k):
        return rng.integers(0, n, k, dtype=np.int64), rng.integers(0, n, k, dtype=np.int64)

    return _collect_unique_pairs(draw, n, m, rng)


_CACHE_DIR = os.environ.get("GSP_DATA_DIR", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "data"))


def graph_for(cfg: Config, seed: int = 1, gen: str = "chung_lu", cache: bool = True):
    """(src, dst) int64 undirected pairs for a config; cached as .npz under data/."""
    path = os.path.join(_CACHE_DIR, f"{gen}_{cfg.n}_{cfg.m}_s{seed}.npz")
    if cache and os.path.exists(path):
        z = np.load(path)
        return z["src"], z["dst"]
    fn = {"chung_lu": chung_lu, "rmat": rmat, "er": erdos_renyi}[gen]
    src, dst = fn(cfg.n, cfg.m, seed)
    if cache:
        try:
            os.makedirs(_CACHE_DIR, exist_ok=True)
            tmp = path + f".tmp{os.getpid()}.npz"
            np.savez(tmp, src=src, dst=dst)
            os.replace(tmp, path)
        except OSError:
            pass
    return src, dst


# --------------------------------------------------------------------------
# Dense inputs
# --------------------------------------------------------------------------


def features(n: int, f: int, ld: Optional[int] = None, seed: int = 2, low=-1.0, high=1.0) -> np.ndarray:
    """X ~ U[low, high) fp32, shape [n, ld], padding columns zero."""
    ld = f if ld is None else ld
    rng = np.random.Generator(np.random.PCG64(seed))
    x = np.zeros((n, ld), dtype=np.float32)
    # filled in row chunks (the same stream as one rng.random((n, f)) call) so
    # the 8.6 GB C6 matrix needs no full-size temporaries
    step = max(1, (1 << 24) // max(f, 1))
    for r0 in range(0, n, step):
        r1 = min(n, r0 + step)
        x[r0:r1, :f] = low + (high - low) * rng.random((r1 - r0, f), dtype=np.float32)
    return x


def uniform(shape, seed: int, low=-1.0, high=1.0) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed))
    return (low + (high - low) * rng.random(shape, dtype=np.float64)).astype(np.float32)


def weights(m: int, seed: int = 5) -> np.ndarray:
    """Positive edge weights U(0, 2] fp32 (weighted-path parity variant)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return (2.0 - 2.0 * rng.random(m)).astype(np.float32)


def bag_of_words(n: int, f: int, density: float = 0.02, seed: int = 2) -> np.ndarray:
    """Binary bag-of-words features (P:233 'sparse bag-of-words feature vectors')."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return (rng.random((n, f)) < density).astype(np.float32)
