"""Seeded synthetic inputs: the five BASELINE.json workloads and the reference's power-law corpus.

Recipes follow SURVEY.md Appendix B exactly (same numpy Generator call sequence), so the
counts quoted there reproduce: config 2 -> nnz 16,086,387, 546,921 touched columns, etc.
``generate_power_law`` reproduces the reference generator (core.py:300-373) draw for draw so
the reference test corpora (conftest.py:22-45, test_acceptance.py:62-89) can be rebuilt on a
machine without the reference installed.
"""

from __future__ import annotations

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


def rmat_keys(scale: int, edge_factor: int, rng: np.random.Generator, a=0.57, b=0.19, c=0.19) -> np.ndarray:
    """R-MAT edge keys (row * n + col), deduplicated and sorted."""
    n = 1 << scale
    m = edge_factor * n
    r = np.zeros(m, dtype=np.int64)
    q = np.zeros(m, dtype=np.int64)
    for bit in range(scale):
        u = rng.random(m)
        down = u >= a + b
        right = ((u >= a) & (u < a + b)) | (u >= a + b + c)
        r |= down.astype(np.int64) << bit
        q |= right.astype(np.int64) << bit
        del u, down, right
    return np.unique(r * n + q)


def rmat(scale: int, edge_factor: int, seed: int) -> CsrMatrix:
    rng = np.random.default_rng(seed)
    keys = rmat_keys(scale, edge_factor, rng)
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
    keys = rmat_keys(scale, 16, np.random.default_rng(0))
    rng1 = np.random.default_rng(1)
    dense = np.sort(rng1.choice(n, 8, replace=False))
    extra = np.concatenate([r * n + rng1.choice(n, n // 4, replace=False) for r in dense])
    keys = np.union1d(keys, extra)
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


def workload_matrix(name: str) -> CsrMatrix:
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
    w = WORKLOADS[name]
    b = np.random.default_rng(w.b_seed).uniform(-1.0, 1.0, (n_rows, w.n_features)).astype(np.float32)
    if w.dtype == "bf16":
        b = bf16_round(b)
    return b


# ---------------------------------------------------------------------------------------------
# the reference's power-law generator (core.py:300-373), reproduced draw for draw
# ---------------------------------------------------------------------------------------------

_SCATTER_NNZ = 1      # rows with <= this many nonzeros scatter over all columns
_ROWS_PER_COMMUNITY = 8
_POOL_SCALE = 1.5


def _scaled_counts(raw: np.ndarray, target: int, cap: int) -> np.ndarray:
    """Smallest scale (by 80-step bisection after doubling) whose clipped rounded counts reach
    the target; returns those counts."""
    if target == 0:
        return np.zeros(raw.size, dtype=np.int64)

    def at(scale):
        return np.minimum(np.rint(raw * scale), cap)

    hi = 1.0
    while at(hi).sum() < target and hi < 1e18:
        hi *= 2.0
    lo = 0.0
    for _ in range(80):
        mid = (lo + hi) / 2
        if at(mid).sum() >= target:
            hi = mid
        else:
            lo = mid
    return at(hi).astype(np.int64)


def _interleave_gaps(counts: np.ndarray) -> np.ndarray:
    """Runs of 8 long rows (draw order) alternating with evenly cut bursts of short rows."""
    long_rows = counts[counts > _SCATTER_NNZ]
    short_rows = counts[counts <= _SCATTER_NNZ]
    if long_rows.size == 0 or short_rows.size == 0:
        return counts
    groups = -(-long_rows.size // _ROWS_PER_COMMUNITY)
    edges = np.round(np.linspace(0, short_rows.size, groups + 1)).astype(np.int64)
    parts = []
    for g in range(groups):
        parts.append(long_rows[g * _ROWS_PER_COMMUNITY:(g + 1) * _ROWS_PER_COMMUNITY])
        parts.append(short_rows[edges[g]:edges[g + 1]])
    return np.concatenate(parts)


def generate_power_law(n_rows: int, n_cols: int, target_nnz: int, skew: float, seed: int) -> CsrMatrix:
    if skew <= 0:
        raise ValueError("skew must be positive")
    if target_nnz < 0 or target_nnz > n_rows * n_cols:
        raise ValueError("target_nnz infeasible for the given dimensions")
    rng = np.random.default_rng(seed)
    if 0 in (n_rows, n_cols, target_nnz):
        return CsrMatrix(n_rows, n_cols, np.zeros(n_rows + 1, np.int64), np.empty(0), np.empty(0))
    counts = _interleave_gaps(_scaled_counts(rng.pareto(skew, n_rows) + 1.0, target_nnz, n_cols))
    is_long = counts > _SCATTER_NNZ
    n_long = int(is_long.sum())
    if n_long:
        comm = np.zeros(n_rows, dtype=np.int64)
        comm[is_long] = np.arange(n_long) // _ROWS_PER_COMMUNITY
        n_comm = int(comm[is_long].max()) + 1
        pool = int(min(n_cols, max(16, round(_POOL_SCALE * _ROWS_PER_COMMUNITY * float(counts[is_long].mean())))))
        spread = n_cols - pool
        if n_comm > 1:
            origin = np.round(np.arange(n_comm) * spread / max(1, n_comm - 1)).astype(np.int64)
        else:
            origin = np.zeros(1, dtype=np.int64)
    everything = np.arange(n_cols)
    per_row = []
    for r in range(n_rows):
        k = int(counts[r])
        if k == 0:
            per_row.append(np.empty(0, dtype=np.int64))
        elif k <= _SCATTER_NNZ:
            per_row.append(np.sort(rng.choice(n_cols, size=k, replace=False)))
        else:
            o = int(origin[comm[r]])
            window = np.arange(o, o + pool)
            if k <= pool:
                picked = rng.choice(window, size=k, replace=False)
            else:
                outside = np.concatenate([everything[:o], everything[o + pool:]])
                picked = np.concatenate([window, rng.choice(outside, size=k - pool, replace=False)])
            per_row.append(np.sort(picked))
    cols = np.concatenate(per_row)
    rp = np.zeros(n_rows + 1, dtype=np.int64)
    np.cumsum(counts, out=rp[1:])
    vals = rng.uniform(-1.0, 1.0, size=cols.size).astype(np.float32)
    return CsrMatrix(n_rows, n_cols, rp, cols, vals)


def small_corpus() -> list[CsrMatrix]:
    """The reference's 24-matrix fixture (conftest.py:22-45)."""
    out, i = [], 0
    for n in (32, 48, 64, 96, 128, 192):
        for delta in (0, 1):
            n_cols = n if delta == 0 else max(16, n // 2)
            dens = (0.01, 0.03, 0.08)[(i + delta) % 3]
            out.append(generate_power_law(n, n_cols, max(1, int(round(dens * n * n_cols))),
                                          (1.2, 1.5, 2.0)[i % 3], seed=100 + i))
            i += 1
        for delta in (2, 3):
            n_cols = min(256, 2 * n) if delta == 2 else n
            dens = (0.01, 0.03, 0.08)[i % 3]
            out.append(generate_power_law(n, n_cols, max(1, int(round(dens * n * n_cols))),
                                          (1.2, 1.5, 2.0)[(i + 1) % 3], seed=200 + i))
            i += 1
    return out


def acceptance_cases() -> list[tuple]:
    """(n_rows, n_cols, nnz, skew, seed, d) of the reference acceptance corpus
    (test_acceptance.py:62-89)."""
    rng = np.random.default_rng(990099)
    sizes = [64, 96, 128, 192, 256, 384, 512]
    rows = [sizes[i % 7] for i in range(150)] + [768 if i % 2 else 1024 for i in range(40)]
    rows += [2048] * 8 + [4096] * 2
    cases = []
    for i, nr in enumerate(rows):
        nc = 3 * nr // 4 if i % 4 == 1 else (2 * nr if i % 7 == 3 else nr)
        dens = 10 ** rng.uniform(-3.0, -1.0)
        nnz = max(16, min(int(round(dens * nr * nc)), 150_000, int(0.4 * nr * nc)))
        cases.append((nr, nc, nnz, (1.2, 1.5, 2.0)[i % 3], i, (16, 64, 128)[i % 3]))
    return cases
