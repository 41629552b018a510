"""The reference's power-law generator and test corpora -- TEST INFRASTRUCTURE ONLY.

``generate_power_law`` restates rstile core.py:240-373 (``_fit_counts``, ``_rearrange_counts``,
``generate_power_law``) draw for draw: the golden digests under tests/golden/ are keyed on the
matrices it produces, so the draw order must be the reference's.  ``small_corpus`` is the
reference's 24-matrix fixture (tests/conftest.py:22-45) and ``acceptance_cases`` its acceptance
corpus parameters (tests/test_acceptance.py:62-89).  Only tests/, smoke() and the golden
generators import this module; the product package does not.
"""

from __future__ import annotations

import numpy as np

from paper_2603_08734_b200.core import CsrMatrix

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
