"""CPU oracle for the RSH-SpMM hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / ``--impl
reference`` leg may import this package, and only as the checker (or the timed CPU baseline),
never as the thing measured for the GPU arm.  The product package ``paper_2603_08734_b200``
never imports it.

It restates the reference package ``rstile`` 0.1.0 (``/root/reference/pkg/src/rstile``):

* integer/byte work (partition scan, column increment, block counts, bitmap build, f64 SpMM)
  in plain C, ``oracle/rsh_oracle.c`` (built by ``oracle/build_oracle.sh``);
* the scalar glue (thresholds, split map, entry arrays, residual gather, validation, decode)
  in numpy below, each function citing the reference file:line it follows;
* ``port_hybrid_spmm`` -- a numpy restatement of the reference executor (per-window
  bitmap expansion, B-row gather, one dense GEMM per window; execute.py:155-226), which is
  what ``bench.py --impl reference`` times as the reference CPU path.

Parity pinned: ``tests/golden/`` holds fixtures produced by importing the reference itself
(``tests/golden/make_golden.py``); ``tests/test_oracle_golden.py`` checks this restatement
against every one of them (known-answer vectors from the reference's own tests plus digests
of the reference's outputs over seeded corpora).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "librsh_oracle.so")
_lib = None

_i64p = ctypes.POINTER(ctypes.c_int64)


def compile_lib() -> str:
    """Compile the C restatement (gcc, no GPU needed)."""
    subprocess.run(["bash", os.path.join(_HERE, "build_oracle.sh")], check=True)
    return _SO


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            compile_lib()
        L = ctypes.CDLL(_SO)
        vp = ctypes.c_void_p
        L.orc_column_increment.restype = ctypes.c_int64
        L.orc_column_increment.argtypes = [vp, vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64]
        L.orc_partition.restype = ctypes.c_int64
        L.orc_partition.argtypes = [vp, vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                    ctypes.c_int64, vp, vp, vp, vp]
        L.orc_window_nblocks.restype = None
        L.orc_window_nblocks.argtypes = [vp, vp, ctypes.c_int64, vp, vp, vp, vp]
        L.orc_build_windows.restype = None
        L.orc_build_windows.argtypes = [vp, vp, vp, ctypes.c_int64, vp, vp, vp, vp, vp, vp, vp]
        L.orc_spmm_f64.restype = None
        L.orc_spmm_f64.argtypes = [vp, vp, vp, ctypes.c_int64, ctypes.c_int64, vp,
                                   ctypes.c_int64, vp, vp]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


@dataclass
class Csr:
    """Plain CSR triple with the reference dtypes (core.py:26-47)."""

    n_rows: int
    n_cols: int
    row_ptr: np.ndarray  # int64
    col_idx: np.ndarray  # int32
    values: np.ndarray   # float32

    def __post_init__(self):
        self.row_ptr = np.ascontiguousarray(self.row_ptr, dtype=np.int64)
        self.col_idx = np.ascontiguousarray(self.col_idx, dtype=np.int32)
        self.values = np.ascontiguousarray(self.values, dtype=np.float32)

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    @classmethod
    def of(cls, a) -> "Csr":
        """Accept any object with the CsrMatrix attribute names (reference or product)."""
        return cls(int(a.n_rows), int(a.n_cols), np.asarray(a.row_ptr), np.asarray(a.col_idx),
                   np.asarray(a.values))


# ---------------------------------------------------------------------------------------------
# partition.py
# ---------------------------------------------------------------------------------------------

def thresholds(n_rows: int, nnz: int, tau_nnz=None, tau_inc=None) -> tuple[int, int]:
    """partition.py:44-49 + 91-98: tau_nnz = clamp(round(nnz/n/2), 2, 6) with Python's
    half-to-even round on the double quotient; tau_inc defaults to 2; explicit values win."""
    if tau_nnz is not None and tau_inc is not None:
        return int(tau_nnz), int(tau_inc)
    n = max(n_rows, 1)
    est = min(6, max(2, round(nnz / n / 2)))
    return (est if tau_nnz is None else int(tau_nnz)), (2 if tau_inc is None else int(tau_inc))


def column_increment(a: Csr, r: int, w: int) -> int:
    """partition.py:101-116 (C restatement)."""
    return int(lib().orc_column_increment(_p(a.row_ptr), _p(a.col_idx), a.n_rows, r, w))


def partition(a: Csr, window_size=8, tau_nnz=None, tau_inc=None):
    """partition.py:119-141 -> (windows tuple of (start, count), residual int64 array)."""
    if a.n_rows == 0:
        return (), np.empty(0, np.int64)
    tn, ti = thresholds(a.n_rows, a.nnz, tau_nnz, tau_inc)
    ws = np.empty(a.n_rows, np.int64)
    wc = np.empty(a.n_rows, np.int64)
    rs = np.empty(a.n_rows, np.int64)
    nr = np.zeros(1, np.int64)
    nw = lib().orc_partition(_p(a.row_ptr), _p(a.col_idx), a.n_rows, window_size, tn, ti,
                             _p(ws), _p(wc), _p(rs), _p(nr))
    windows = tuple(zip(ws[:nw].tolist(), wc[:nw].tolist()))
    return windows, rs[: int(nr[0])].copy()


def window_blocks(a: Csr, windows) -> tuple[np.ndarray, np.ndarray]:
    """ceil(|window_columns|/8) per window (partition.py:144-146,167) and the longest row."""
    n = len(windows)
    ws = np.array([s for s, _ in windows], np.int64)
    wc = np.array([c for _, c in windows], np.int64)
    nb = np.zeros(n, np.int64)
    lg = np.zeros(n, np.int64)
    if n:
        lib().orc_window_nblocks(_p(a.row_ptr), _p(a.col_idx), n, _p(ws), _p(wc), _p(nb), _p(lg))
    return nb, lg


def split_map(a: Csr, windows, max_blocks_per_item=64, split_on_row_nnz=False,
              split_factor=4.0) -> dict:
    """partition.py:149-180: windows over the block bound get (b, min(b+bound, nblocks))
    segments; with split_on_row_nnz a long-row window gets ceil(nblocks/ceil(longest/cap))."""
    bound = max_blocks_per_item
    if bound is None and not split_on_row_nnz:
        return {}
    nb, lg = window_blocks(a, windows)
    mean = a.nnz / a.n_rows if a.n_rows else 0.0
    out = {}
    for i in range(len(windows)):
        nblocks = int(nb[i])
        chunk = 0
        if bound is not None and nblocks > bound:
            chunk = bound
        elif split_on_row_nnz and nblocks > 1 and mean > 0.0:
            longest = int(lg[i])
            cap = split_factor * mean
            if longest > cap:
                chunk = max(1, -(-nblocks // math.ceil(longest / cap)))
        if chunk and chunk < nblocks:
            out[i] = tuple((b, min(b + chunk, nblocks)) for b in range(0, nblocks, chunk))
    return out


# ---------------------------------------------------------------------------------------------
# tile.py
# ---------------------------------------------------------------------------------------------

@dataclass
class Tile:
    """The RS-Tile arrays with the reference dtypes (tile.py:43-91)."""

    n_rows: int
    n_cols: int
    row_window_id: np.ndarray      # int32
    row_window_offset: np.ndarray  # int64
    bitmaps: np.ndarray            # uint64
    col_id: np.ndarray             # int32
    values: np.ndarray             # float32
    res_row_id: np.ndarray         # int32
    res_offset: np.ndarray         # int64
    res_col_id: np.ndarray         # int32
    res_values: np.ndarray         # float32
    window_size: int

    ARRAYS = ("row_window_id", "row_window_offset", "bitmaps", "col_id", "values",
              "res_row_id", "res_offset", "res_col_id", "res_values")

    @classmethod
    def of(cls, m) -> "Tile":
        """From an RsTileMatrix-shaped object (reference or product host format)."""
        return cls(int(m.n_rows), int(m.n_cols),
                   np.asarray(m.tc.row_window_id), np.asarray(m.tc.row_window_offset),
                   np.asarray(m.tc.bitmaps), np.asarray(m.tc.col_id), np.asarray(m.tc.values),
                   np.asarray(m.residual.row_id), np.asarray(m.residual.row_nnz_offset),
                   np.asarray(m.residual.col_id), np.asarray(m.residual.values),
                   int(m.window_size))

    def arrays(self) -> dict:
        return {k: getattr(self, k) for k in self.ARRAYS}


def build(a: Csr, windows, residual, smap: dict) -> Tile:
    """tile.py:102-173 restated: per-window bitmap blocks (C), one entry per segment sharing
    the window's start row, offsets = [0]+cumsum(entry blocks), residual rows copied in plan
    order, window_size = max window row count or 8."""
    n = len(windows)
    ws = np.array([s for s, _ in windows], np.int64)
    wc = np.array([c for _, c in windows], np.int64)
    nb, _ = window_blocks(a, windows)
    block_base = np.zeros(n + 1, np.int64)
    np.cumsum(nb, out=block_base[1:])
    wnnz = a.row_ptr[ws + wc] - a.row_ptr[ws] if n else np.zeros(0, np.int64)
    value_base = np.zeros(n + 1, np.int64)
    np.cumsum(wnnz, out=value_base[1:])
    total_blocks = int(block_base[-1])
    bitmaps = np.zeros(total_blocks, np.uint64)
    col_id = np.zeros(8 * total_blocks, np.int32)
    values = np.zeros(int(value_base[-1]), np.float32)
    if n:
        lib().orc_build_windows(_p(a.row_ptr), _p(a.col_idx), _p(a.values), n, _p(ws), _p(wc),
                                _p(block_base), _p(value_base), _p(bitmaps), _p(col_id),
                                _p(values))
    rwid, eblocks = [], []
    for i in range(n):
        for bs, be in smap.get(i, ((0, int(nb[i])),)):
            rwid.append(int(ws[i]))
            eblocks.append(be - bs)
    offsets = np.zeros(len(rwid) + 1, np.int64)
    np.cumsum(np.array(eblocks, np.int64), out=offsets[1:])

    res = np.asarray(residual, np.int64)
    counts = a.row_ptr[res + 1] - a.row_ptr[res]
    r_off = np.zeros(res.size + 1, np.int64)
    np.cumsum(counts, out=r_off[1:])
    if res.size:
        starts = np.repeat(a.row_ptr[res] - r_off[:-1], counts)
        gather = starts + np.arange(int(r_off[-1]), dtype=np.int64)
        r_cols, r_vals = a.col_idx[gather], a.values[gather]
    else:
        r_cols, r_vals = np.empty(0, np.int32), np.empty(0, np.float32)
    wsize = int(wc.max()) if n else 0
    return Tile(a.n_rows, a.n_cols, np.array(rwid, np.int32), offsets, bitmaps, col_id, values,
                res.astype(np.int32), r_off, r_cols.astype(np.int32), r_vals.astype(np.float32),
                wsize if wsize else 8)


def build_format(a: Csr, window_size=8, tau_nnz=None, tau_inc=None, max_blocks_per_item=64,
                 split_on_row_nnz=False, split_factor=4.0) -> Tile:
    """partition -> split -> build, the reference conftest.py:11-19 pipeline."""
    windows, residual = partition(a, window_size, tau_nnz, tau_inc)
    smap = split_map(a, windows, max_blocks_per_item, split_on_row_nnz, split_factor)
    return build(a, windows, residual, smap)


def popcounts(bitmaps: np.ndarray) -> np.ndarray:
    """tile.py:94-99: set-bit count per 64-bit mask."""
    b = np.ascontiguousarray(bitmaps, dtype="<u8").view(np.uint8)
    return np.unpackbits(b).reshape(-1, 64).sum(axis=1).astype(np.int64) if b.size else \
        np.zeros(0, np.int64)


def decode(t: Tile) -> Csr:
    """tile.py:270-307: expand bitmaps (bit b -> row b>>3, col slot b&7; values in ascending
    (block, bit) order), append residual runs, sort by (row, col)."""
    if t.bitmaps.size:
        eob = np.repeat(np.arange(t.row_window_id.size), np.diff(t.row_window_offset))
        base = t.row_window_id[eob].astype(np.int64)
        bits = np.unpackbits(np.ascontiguousarray(t.bitmaps, "<u8").view(np.uint8),
                             bitorder="little").reshape(-1, 64)
        blk, bit = np.nonzero(bits)
        rows = base[blk] + (bit >> 3)
        cols = t.col_id[blk * 8 + (bit & 7)].astype(np.int64)
        vals = t.values
    else:
        rows = cols = np.empty(0, np.int64)
        vals = np.empty(0, np.float32)
    rr = np.repeat(t.res_row_id.astype(np.int64), np.diff(t.res_offset))
    rows = np.concatenate([rows, rr])
    cols = np.concatenate([cols, t.res_col_id.astype(np.int64)])
    vals = np.concatenate([vals, t.res_values])
    order = np.lexsort((cols, rows))
    rp = np.zeros(t.n_rows + 1, np.int64)
    np.cumsum(np.bincount(rows, minlength=t.n_rows), out=rp[1:])
    return Csr(t.n_rows, t.n_cols, rp, cols[order], vals[order])


def tiles_equal(x: Tile, y: Tile) -> list[str]:
    """Names of the fields that differ (bit-exact array comparison)."""
    bad = []
    for k in ("n_rows", "n_cols", "window_size"):
        if getattr(x, k) != getattr(y, k):
            bad.append(k)
    for k in Tile.ARRAYS:
        a, b = getattr(x, k), getattr(y, k)
        if a.dtype != b.dtype or a.shape != b.shape or not np.array_equal(a, b):
            bad.append(k)
    return bad


# ---------------------------------------------------------------------------------------------
# core.py
# ---------------------------------------------------------------------------------------------

def spmm_f64(a: Csr, b: np.ndarray, row_lo=0, row_hi=None, want64=True):
    """core.py:380-395: per-row f64 accumulation, f32 store.  Returns (c32, c64 or None)."""
    row_hi = a.n_rows if row_hi is None else row_hi
    b = np.ascontiguousarray(b, np.float32)
    d = b.shape[1]
    c32 = np.empty((row_hi - row_lo, d), np.float32)
    c64 = np.empty((row_hi - row_lo, d), np.float64) if want64 else None
    lib().orc_spmm_f64(_p(a.row_ptr), _p(a.col_idx), _p(a.values), row_lo, row_hi, _p(b), d,
                       _p(c32), _p(c64) if want64 else None)
    return c32, c64


def max_relative_error(c, ref) -> float:
    """core.py:398-408: max |c-ref| / max(|ref|, 1)."""
    c = np.asarray(c, np.float64)
    ref = np.asarray(ref, np.float64)
    if c.size == 0:
        return 0.0
    return float((np.abs(c - ref) / np.maximum(np.abs(ref), 1.0)).max())


def rel_frobenius(c, ref64) -> float:
    """||c - ref||_F / ||ref||_F in f64 (the north-star FP gate)."""
    c = np.asarray(c, np.float64)
    ref64 = np.asarray(ref64, np.float64)
    den = float(np.linalg.norm(ref64))
    num = float(np.linalg.norm(c - ref64))
    return num / den if den > 0 else num


# ---------------------------------------------------------------------------------------------
# execute.py -- the reference CPU executor, restated (the reference arm / cpu_baseline)
# ---------------------------------------------------------------------------------------------

def port_hybrid_spmm(t: Tile, b: np.ndarray, num_workers: int = 1, entry_range=None,
                     residual_range=None) -> np.ndarray:
    """execute.py:155-226 restated in numpy: consecutive entries sharing a row_window_id are one
    logical window (execute.py:136-152); each window expands its bitmap blocks to dense 8x8
    fragments (execute.py:65-77), gathers its 8*k B rows (execute.py:92-95) and runs one
    (8 x 8k) @ (8k x d) f32 GEMM whose first min(window_size, n-rid) rows are assigned to C
    (execute.py:171-182); residual rows are values @ B[cols] (execute.py:184-193).  Worker
    threads split the work the same way the reference's ThreadPoolExecutor does.

    ``entry_range``/``residual_range`` restrict the work to a bounded sample (bench.py).
    """
    b = np.ascontiguousarray(b, np.float32)
    d = b.shape[1]
    c = np.zeros((t.n_rows, d), np.float32)
    rwid = t.row_window_id
    off = t.row_window_offset
    e_lo, e_hi = (0, rwid.size) if entry_range is None else entry_range
    groups = []
    e = e_lo
    while e < e_hi:
        f = e + 1
        while f < e_hi and rwid[f] == rwid[e]:
            f += 1
        groups.append((int(rwid[e]), int(off[e]), int(off[f])))
        e = f
    vstart = np.zeros(t.bitmaps.size + 1, np.int64)
    np.cumsum(popcounts(t.bitmaps), out=vstart[1:])

    def window(g):
        rid, bs, be = g
        if bs == be:
            return
        nb = be - bs
        bits = np.unpackbits(np.ascontiguousarray(t.bitmaps[bs:be], "<u8").view(np.uint8),
                             bitorder="little").reshape(nb, 64)
        frag = np.zeros((nb, 64), np.float32)
        kb, kbit = np.nonzero(bits)
        frag[kb, kbit] = t.values[vstart[bs]:vstart[be]]
        a_rows = frag.reshape(nb, 8, 8).transpose(1, 0, 2).reshape(8, 8 * nb)
        prod = a_rows @ b[t.col_id[8 * bs:8 * be]]
        avail = min(t.window_size, t.n_rows - rid)
        c[rid:rid + avail] = prod[:avail]

    r_lo, r_hi = (0, t.res_row_id.size) if residual_range is None else residual_range

    def residual(lo, hi):
        for i in range(lo, hi):
            s, e2 = int(t.res_offset[i]), int(t.res_offset[i + 1])
            if s < e2:
                c[int(t.res_row_id[i])] = t.res_values[s:e2] @ b[t.res_col_id[s:e2]]

    if num_workers <= 1:
        for g in groups:
            window(g)
        residual(r_lo, r_hi)
    else:
        cuts = np.linspace(r_lo, r_hi, num_workers + 1).astype(int)
        with ThreadPoolExecutor(max_workers=num_workers) as pool:
            futs = [pool.submit(window, g) for g in groups]
            futs += [pool.submit(residual, int(x), int(y)) for x, y in zip(cuts[:-1], cuts[1:])
                     if x < y]
            for f in futs:
                f.result()
    return c
