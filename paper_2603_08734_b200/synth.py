"""Seeded synthetic inputs: the five BASELINE.json workloads (bench and parity-test inputs).

Recipes follow SURVEY.md Appendix B exactly (same numpy Generator call sequence), so the
counts quoted there reproduce: config 2 -> nnz 16,086,387, 546,921 touched columns, etc.
``rmat_sNN`` names the weak-scaling R-MAT graphs (scale NN, edge factor 16, seed 0) of the
multi-GPU run.  The reference's power-law test corpus lives in oracle/corpus.py (test
infrastructure).
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

from .core import CsrMatrix


def _csr_from_keys(n_rows: int, n_cols: int, keys: np.ndarray, values: np.ndarray) -> CsrMatrix:
    """keys = row * n_cols + col, sorted and unique."""
    rows = keys // n_cols
    cols = (keys - rows * n_cols).astype(np.int32)
    rp = np.zeros(n_rows + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n_rows), out=rp[1:])
    return CsrMatrix(n_rows, n_cols, rp, cols, values)


def sorted_unique(x: np.ndarray) -> np.ndarray:
    """np.unique for a 1-D integer array (sort + adjacent-difference mask: numpy 2.3's
    np.unique is ~50x slower on 10^7 int64 keys)."""
    x = np.sort(x)
    if x.size < 2:
        return x
    keep = np.empty(x.size, dtype=bool)
    keep[0] = True
    np.not_equal(x[1:], x[:-1], out=keep[1:])
    return x[keep]


def _threads() -> int:
    return max(1, min(16, len(os.sched_getaffinity(0))))


def rmat_keys(scale: int, edge_factor: int, seed: int, a=0.57, b=0.19, c=0.19) -> tuple[np.ndarray, np.random.Generator]:
    """R-MAT edge keys (row * n + col), deduplicated and sorted, and the generator positioned
    after the draws.  The recipe draws ``u = rng.random(m)`` once per
    bit from ``default_rng(seed)`` and sets row bit (u >= a+b), column bit ((a <= u < a+b) or
    u >= a+b+c).  The same stream is produced here in parallel: PCG64 advances in O(log n), so
    each thread draws its slice [lo, hi) of every bit's m doubles from a copy advanced to
    bit * m + lo (Generator.random consumes one 64-bit output per double)."""
    n = 1 << scale
    m = edge_factor * n
    r = np.zeros(m, dtype=np.int64)
    q = np.zeros(m, dtype=np.int64)
    nt = _threads()
    cuts = [m * i // nt for i in range(nt + 1)]
    ta, tab, tabc = a, a + b, a + b + c

    def work(i):
        lo, hi = cuts[i], cuts[i + 1]
        if hi <= lo:
            return
        rs, qs = r[lo:hi], q[lo:hi]
        for bit in range(scale):
            g = np.random.Generator(np.random.PCG64(seed).advance(bit * m + lo))
            u = g.random(hi - lo)
            # category (u >= a) + (u >= a+b) + (u >= a+b+c): row bit = cat >= 2, column bit = cat odd
            cat = (u >= ta).view(np.uint8)
            cat += (u >= tab).view(np.uint8)
            cat += (u >= tabc).view(np.uint8)
            del u
            rs |= (cat >> 1).astype(np.int64) << bit
            qs |= (cat & 1).astype(np.int64) << bit

    with ThreadPoolExecutor(nt) as ex:
        list(ex.map(work, range(nt)))
    keys = r
    keys *= n
    keys += q
    del q
    rng = np.random.Generator(np.random.PCG64(seed).advance(scale * m))
    return sorted_unique(keys), rng


def rmat(scale: int, edge_factor: int, seed: int) -> CsrMatrix:
    keys, rng = rmat_keys(scale, edge_factor, seed)
    n = 1 << scale
    vals = rng.uniform(-1.0, 1.0, keys.size).astype(np.float32)
    return _csr_from_keys(n, n, keys, vals)


def uniform_4096() -> CsrMatrix:
    rng = np.random.default_rng(0)
    n = 4096
    flat = np.sort(rng.choice(n * n, 167_772, replace=False))
    vals = rng.uniform(-1.0, 1.0, flat.size).astype(np.float32)
    return _csr_from_keys(n, n, flat.astype(np.int64), vals)


def stencil27(nx: int = 128) -> CsrMatrix:
    n = nx ** 3
    idx = np.arange(n, dtype=np.int64)
    x, y, z = idx % nx, (idx // nx) % nx, idx // (nx * nx)
    rows_l, cols_l = [], []
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                ok = ((x + dx >= 0) & (x + dx < nx) & (y + dy >= 0) & (y + dy < nx)
                      & (z + dz >= 0) & (z + dz < nx))
                rows_l.append(idx[ok])
                cols_l.append(idx[ok] + dx + dy * nx + dz * nx * nx)
    keys = np.concatenate(rows_l) * n + np.concatenate(cols_l)
    keys.sort()
    vals = np.random.default_rng(0).uniform(-1.0, 1.0, keys.size).astype(np.float32)
    return _csr_from_keys(n, n, keys, vals)


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round float32 -> bfloat16 (round to nearest even), returned as float32."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def heavy_tail_4m() -> CsrMatrix:
    scale = 22
    n = 1 << scale
    keys, _ = rmat_keys(scale, 16, 0)
    rng1 = np.random.default_rng(1)
    dense = np.sort(rng1.choice(n, 8, replace=False))
    extra = np.concatenate([r * n + rng1.choice(n, n // 4, replace=False) for r in dense])
    keys = sorted_unique(np.concatenate([keys, extra]))  # np.union1d
    vals = bf16_round(np.random.default_rng(2).uniform(-1.0, 1.0, keys.size).astype(np.float32))
    return _csr_from_keys(n, n, keys, vals)


@dataclass(frozen=True)
class Workload:
    name: str
    description: str
    n_features: int
    dtype: str  # "f32" (TF32/FP32 math) or "bf16"
    b_seed: int


WORKLOADS = {
    "uniform4k": Workload("uniform4k", "uniform 4096x4096, 1% density, N=32, fp32", 32, "f32", 1),
    "rmat1m": Workload("rmat1m", "R-MAT scale 20 ef16, N=128, fp32", 128, "f32", 1),
    "stencil2m": Workload("stencil2m", "27-point stencil 128^3, N=64, fp32", 64, "f32", 1),
    "heavytail4m": Workload("heavytail4m", "R-MAT scale 22 + 8 rows@25%, N=256, bf16", 256, "bf16", 3),
    "rmat16m": Workload("rmat16m", "R-MAT scale 24 ef16, N=128, fp32", 128, "f32", 1),
}


def workload_spec(name: str) -> Workload:
    """WORKLOADS[name], plus ``rmat_sNN`` (R-MAT scale NN, ef16, N=128, fp32)."""
    if name in WORKLOADS:
        return WORKLOADS[name]
    if name.startswith("rmat_s") and name[6:].isdigit():
        s = int(name[6:])
        return Workload(name, f"R-MAT scale {s} ef16, N=128, fp32", 128, "f32", 1)
    raise KeyError(name)


def workload_matrix(name: str) -> CsrMatrix:
    if name.startswith("rmat_s") and name[6:].isdigit():
        return rmat(int(name[6:]), 16, 0)
    if name == "uniform4k":
        return uniform_4096()
    if name == "rmat1m":
        return rmat(20, 16, 0)
    if name == "stencil2m":
        return stencil27(128)
    if name == "heavytail4m":
        return heavy_tail_4m()
    if name == "rmat16m":
        return rmat(24, 16, 0)
    raise KeyError(name)


def workload_b(name: str, n_rows: int, rows=None) -> np.ndarray:
    """B = uniform(-1, 1, (n, N)) from default_rng(b_seed); bf16 workloads are rounded to bf16.
    ``rows`` restricts generation to a prefix (the full draw is made, as the recipe does)."""
    w = workload_spec(name)
    b = np.random.default_rng(w.b_seed).uniform(-1.0, 1.0, (n_rows, w.n_features)).astype(np.float32)
    if w.dtype == "bf16":
        b = bf16_round(b)
    return b
