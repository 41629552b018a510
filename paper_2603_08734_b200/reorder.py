"""Locality-aware row reordering (rstile reorder.py, PAPER Alg. 3) on device.

The reference pipeline -- column weights d^-alpha, candidate rows through an inverted index,
top-k weighted-Jaccard kNN graph, Kruskal forest linearised depth-first, windowed 2-opt -- runs
as sm_100a kernels (csrc/reorder.cu) with the two sequential steps (forest + DFS, the
objective's left-to-right sum) as host C++ in the same library:

    column_weights     reorder.py:33-42     rsh_column_weights
    build_knn          reorder.py:158-230   rsh_knn (A^T from rsh_transpose_csr)
    mst_order          reorder.py:268-321   rsh_mst_order (host C++, exact restatement)
    isolation_adjust   reorder.py:386-446   rsh_isolation_adjust (host C++, exact restatement)
    refine_2opt        reorder.py:328-380   rsh_two_opt_sweep (disjoint windows in parallel)
    permutation_objective  reorder.py:96-101  rsh_pair_dis + rsh_sum_sequential
    permute_rows       reorder.py:138-151   rsh_permute_rows

Differences from the reference, all on the side of the search, none on the objective: the
2-opt sweeps process disjoint windows in parallel (each window keeps the reference's
sequential first-improvement scan), so the refined order differs but never has a larger
objective than its input; candidate walks skip columns above ``hub_cap`` rows (default: none)
and keep at most 1024 distinct candidates per row (overflow is counted).  The isolation pass
(reorder.py:386-446) is an exact host C++ restatement (rsh_isolation_adjust), kept only when it
does not worsen the objective, as in the reference.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import CsrMatrix


@dataclass(frozen=True)
class ColumnWeights:
    """reorder.py:26-30: float64 per column, 0.0 for unused columns."""

    weights: np.ndarray
    alpha: float


@dataclass(frozen=True)
class KnnGraph:
    """reorder.py:196-216: neighbors[r] = at most k (row, similarity) pairs, similarity > 0,
    sorted by descending similarity then ascending row."""

    n_rows: int
    neighbors: list
    k: int

    def undirected_edges(self) -> list:
        edges = {}
        for r, lst in enumerate(self.neighbors):
            for u, sim in lst:
                edges[(r, u) if r < u else (u, r)] = sim
        return [(u, v, edges[(u, v)]) for u, v in sorted(edges)]


@dataclass(frozen=True)
class ReorderParams:
    """reorder.py:454-461 plus ``hub_cap`` (candidate walks skip columns with more rows; None =
    walk every column, as the reference)."""

    alpha: float = 0.5
    k: int = 8
    max_candidates: int = 256
    two_opt_window: int = 64
    two_opt_passes: int = 3
    iso_threshold: float = 0.05
    hub_cap: int | None = None


@dataclass(frozen=True)
class Permutation:
    """reorder.py:95-107: a bijective row order; order[i] is the source row at position i."""

    order: np.ndarray
    objective: float

    def __post_init__(self) -> None:
        order = np.ascontiguousarray(self.order, dtype=np.int64)
        if not np.array_equal(np.sort(order), np.arange(order.size)):
            raise ValueError("order is not a permutation of 0..n-1")
        order.flags.writeable = False
        object.__setattr__(self, "order", order)

    def __len__(self) -> int:
        return int(self.order.size)


def permute_rows_device(a, order):
    """reorder.py:138-151 on device: DeviceCsr with row i taken from source row order[i]."""
    import torch
    from ._lib import call, lib
    from .device import DeviceCsr, _ptr, _stream, _ws
    dev = a.device
    o = order if isinstance(order, torch.Tensor) else torch.from_numpy(np.array(order, dtype=np.int64))
    o = o.to(device=dev, dtype=torch.int64)
    if o.numel() != a.n_rows:
        raise ValueError("order length must equal n_rows")
    rp = torch.empty(a.n_rows + 1, dtype=torch.int64, device=dev)
    ci = torch.empty(max(a.nnz, 1), dtype=torch.int32, device=dev)
    va = torch.empty(max(a.nnz, 1), dtype=torch.float32, device=dev)
    nbytes = lib().rsh_permute_workspace(a.n_rows)
    ws = _ws(nbytes, dev)
    call("rsh_permute_rows", _ptr(a.row_ptr), _ptr(a.col_idx), _ptr(a.values), a.n_rows, _ptr(o), _ptr(rp),
         _ptr(ci), _ptr(va), _ptr(ws), nbytes, _stream())
    return DeviceCsr(a.n_rows, a.n_cols, rp, ci[:a.nnz], va[:a.nnz])


def permute_rows(a: CsrMatrix, order) -> CsrMatrix:
    """reorder.py:138-151: CSR with row i taken from source row order[i] (computed on device)."""
    from .partition import _dev
    if isinstance(order, Permutation):
        order = order.order
    order = np.ascontiguousarray(order, dtype=np.int64)
    if order.size != a.n_rows:
        raise ValueError("order length must equal n_rows")
    d = permute_rows_device(_dev(a), order)
    return CsrMatrix(a.n_rows, a.n_cols, d.row_ptr.cpu().numpy(), d.col_idx.cpu().numpy(), d.values.cpu().numpy())


# ---------------------------------------------------------------------------------------------
# device pipeline
# ---------------------------------------------------------------------------------------------

class _Ctx:
    """Device-resident state shared by the reorder steps of one matrix: the CSR, its weights and
    row weight sums."""

    def __init__(self, a, alpha: float):
        import torch
        from ._lib import call, lib
        from .device import DeviceCsr, _ptr, _stream, _ws
        from .partition import _dev
        if not (alpha > 0):
            raise ValueError("alpha must be positive")
        self.d = a if isinstance(a, DeviceCsr) else _dev(a)
        d = self.d
        self.w = torch.empty(max(d.n_cols, 1), dtype=torch.float64, device=d.device)
        self.wsum = torch.empty(max(d.n_rows, 1), dtype=torch.float64, device=d.device)
        nbytes = lib().rsh_reorder_workspace(d.n_rows, d.n_cols)
        ws = _ws(nbytes, d.device)
        call("rsh_column_weights", _ptr(d.row_ptr), _ptr(d.col_idx), d.n_rows, d.n_cols, d.nnz, float(alpha),
             _ptr(self.w), _ptr(self.wsum), _ptr(ws), nbytes, _stream())
        self.alpha = alpha

    def objective(self, order_dev) -> float:
        import torch
        from ._lib import call, lib
        from .device import _ptr, _stream
        m = int(order_dev.numel())
        if m < 2:
            return 0.0
        dis = torch.empty(m - 1, dtype=torch.float64, device=order_dev.device)
        call("rsh_pair_dis", _ptr(self.d.row_ptr), _ptr(self.d.col_idx), _ptr(self.w), _ptr(self.wsum),
             _ptr(order_dev), m, _ptr(dis), _stream())
        h = dis.cpu().numpy()
        return float(lib().rsh_sum_sequential(h.ctypes.data, h.size))


def column_weights(a: CsrMatrix, alpha: float = 0.5) -> ColumnWeights:
    """reorder.py:33-42 on device: d_j**(-alpha), 0 for unused columns."""
    c = _Ctx(a, alpha)
    return ColumnWeights(c.w[:a.n_cols].cpu().numpy(), alpha)


def knn_device(ctx: "_Ctx", k: int = 8, max_candidates: int = 256, hub_cap: int | None = None):
    """rsh_knn: device (nbr int32[n,k], sim float64[n,k], count int32[n], overflowed rows)."""
    import torch
    from ._lib import call
    from .device import _ptr, _stream
    from .gnn import transpose_device
    if k < 1:
        raise ValueError("k must be at least 1")
    if max_candidates < 1:
        raise ValueError("max_candidates must be at least 1")
    d = ctx.d
    at = transpose_device(d)
    dev = d.device
    n = d.n_rows
    nbr = torch.zeros((max(n, 1), k), dtype=torch.int32, device=dev)
    sim = torch.zeros((max(n, 1), k), dtype=torch.float64, device=dev)
    cnt = torch.zeros(max(n, 1), dtype=torch.int32, device=dev)
    stats = torch.zeros(1, dtype=torch.int64, device=dev)
    call("rsh_knn", _ptr(d.row_ptr), _ptr(d.col_idx), n, _ptr(at.row_ptr), _ptr(at.col_idx), _ptr(ctx.w),
         _ptr(ctx.wsum), k, max_candidates, (1 << 62) if hub_cap is None else int(hub_cap), _ptr(nbr), _ptr(sim),
         _ptr(cnt), _ptr(stats), _stream())
    return nbr[:n], sim[:n], cnt[:n], int(stats.item())


def build_candidates(a: CsrMatrix, max_candidates: int = 256, hub_cap: int | None = None) -> list:
    """reorder.py:168-194 on device (rsh_candidates): for every row, the rows sharing at least one
    column with it (never itself), the max_candidates with the largest shared-column count when
    there are more (ties to the lower row index), ascending, as int64 arrays.  Raises ValueError
    when a row's candidate set overflows the device's per-row table (pass ``hub_cap`` to skip
    columns of higher degree, as build_knn does)."""
    import torch
    from ._lib import call
    from .device import _ptr, _stream
    from .gnn import transpose_device
    if max_candidates < 1:
        raise ValueError("max_candidates must be at least 1")
    ctx = _Ctx(a, 0.5)
    d = ctx.d
    n = d.n_rows
    if n == 0:
        return []
    at = transpose_device(d)
    cand = torch.zeros((n, max_candidates), dtype=torch.int32, device=d.device)
    cnt = torch.zeros(n, dtype=torch.int32, device=d.device)
    stats = torch.zeros(1, dtype=torch.int64, device=d.device)
    call("rsh_candidates", _ptr(d.row_ptr), _ptr(d.col_idx), n, _ptr(at.row_ptr), _ptr(at.col_idx), max_candidates,
         (1 << 62) if hub_cap is None else int(hub_cap), _ptr(cand), _ptr(cnt), _ptr(stats), _stream())
    if int(stats.item()):
        raise ValueError(f"{int(stats.item())} rows have more distinct candidate rows than the device table holds; "
                         "pass hub_cap to bound the columns walked")
    cn, cd = cnt.cpu().numpy(), cand.cpu().numpy()
    return [cd[r, :cn[r]].astype(np.int64) for r in range(n)]


def build_knn(a: CsrMatrix, w: ColumnWeights | None = None, candidates=None, k: int = 8,
              max_candidates: int = 256, hub_cap: int | None = None) -> KnnGraph:
    """reorder.py:158-230 (build_candidates + build_knn) on device.  ``candidates`` is accepted
    for signature compatibility and ignored: candidates are generated on device."""
    ctx = _Ctx(a, 0.5 if w is None else w.alpha)
    nbr, sim, cnt, _ = knn_device(ctx, k, max_candidates, hub_cap)
    nb, sm, ct = nbr.cpu().numpy(), sim.cpu().numpy(), cnt.cpu().numpy()
    return KnnGraph(a.n_rows, [[(int(nb[r, t]), float(sm[r, t])) for t in range(ct[r])] for r in range(a.n_rows)], k)


def _mst_host(n: int, k: int, nbr: np.ndarray, sim: np.ndarray, cnt: np.ndarray) -> np.ndarray:
    from ._lib import call
    order = np.empty(n, np.int64)
    nbr = np.ascontiguousarray(nbr, np.int32)
    sim = np.ascontiguousarray(sim, np.float64)
    cnt = np.ascontiguousarray(cnt, np.int32)
    call("rsh_mst_order", n, k, nbr.ctypes.data, sim.ctypes.data, cnt.ctypes.data, order.ctypes.data)
    return order


def mst_order(g: KnnGraph, a: CsrMatrix | None = None, w: ColumnWeights | None = None) -> Permutation:
    """reorder.py:268-321: Kruskal forest + depth-first linearisation (host C++ in librsh.so).
    With the matrix the objective is recomputed on device; otherwise absent pairs count 0."""
    n, k = g.n_rows, max(1, g.k)
    nbr = np.zeros((max(n, 1), k), np.int32)
    sim = np.zeros((max(n, 1), k), np.float64)
    cnt = np.zeros(max(n, 1), np.int32)
    for r, lst in enumerate(g.neighbors):
        cnt[r] = len(lst)
        for t, (u, s_) in enumerate(lst):
            nbr[r, t], sim[r, t] = u, s_
    order = _mst_host(n, k, nbr, sim, cnt)
    if a is not None and w is not None:
        return Permutation(order, permutation_objective(a, w, order))
    simmap = {(u, v): s_ for u, v, s_ in g.undirected_edges()}
    obj = 0.0
    for x, y in zip(order[:-1], order[1:]):
        obj += 1.0 - simmap.get((x, y) if x < y else (y, x), 0.0)
    return Permutation(order, obj)


def permutation_objective(a: CsrMatrix, w: ColumnWeights, order) -> float:
    """reorder.py:96-101: sum of (1 - similarity) over adjacent pairs (terms on device, summed
    left to right)."""
    import torch
    ctx = _Ctx(a, w.alpha)
    o = torch.from_numpy(np.array(order, dtype=np.int64)).to(ctx.d.device)
    return ctx.objective(o)


def two_opt_device(ctx: "_Ctx", order_dev, window: int = 64, max_passes: int = 3) -> int:
    """In-place windowed 2-opt on a device order; returns the number of sweeps that improved."""
    import torch
    from ._lib import call
    from .device import _ptr, _stream
    if window < 2:
        raise ValueError("window must be at least 2")
    if max_passes < 0:
        raise ValueError("max_passes must be non-negative")
    m = int(order_dev.numel())
    flag = torch.zeros(1, dtype=torch.int64, device=order_dev.device)
    improving = 0
    for _ in range(max_passes):
        flag.zero_()
        for off in (0, max(1, window // 2)):
            call("rsh_two_opt_sweep", _ptr(ctx.d.row_ptr), _ptr(ctx.d.col_idx), _ptr(ctx.w), _ptr(ctx.wsum),
                 _ptr(order_dev), m, window, off, _ptr(flag), _stream())
        if int(flag.item()) == 0:
            break
        improving += 1
    return improving


def refine_2opt(a: CsrMatrix, w: ColumnWeights, p: Permutation, window: int = 64, max_passes: int = 3) -> Permutation:
    """reorder.py:328-380 on device (disjoint windows in parallel; strict improvements only, so
    the objective never increases).  max_passes = 0 returns the input verbatim."""
    import torch
    if window < 2:
        raise ValueError("window must be at least 2")
    if max_passes < 0:
        raise ValueError("max_passes must be non-negative")
    if max_passes == 0:
        return p
    ctx = _Ctx(a, w.alpha)
    o = torch.from_numpy(np.array(p.order, np.int64)).to(ctx.d.device)
    two_opt_device(ctx, o, window, max_passes)
    return Permutation(o.cpu().numpy(), ctx.objective(o))


def w_jaccard(a: CsrMatrix, w: ColumnWeights, r: int, u: int) -> float:
    """reorder.py:45-57: weighted Jaccard of rows r and u (the device pair kernel)."""
    if r == u:
        return 1.0
    return 1.0 - permutation_objective(a, w, [r, u])


def save_permutation(path, p: Permutation) -> None:
    """reorder.py:110-114 (same text format)."""
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(f"# objective={p.objective!r}\n")
        for r in p.order:
            fh.write(f"{int(r)}\n")


def load_permutation(path) -> Permutation:
    """reorder.py:117-132."""
    objective = 0.0
    order = []
    with open(path, "r", encoding="utf-8") as fh:
        for line in fh:
            t = line.strip()
            if not t:
                continue
            if t.startswith("#"):
                if "objective=" in t:
                    objective = float(t.split("objective=", 1)[1])
                continue
            order.append(int(t))
    return Permutation(np.array(order, dtype=np.int64), objective)


def _isolation_host(ctx: "_Ctx", order: np.ndarray, iso_threshold: float, hub_cap: int | None):
    from ._lib import call
    d = ctx.d
    rp, ci = d.row_ptr.cpu().numpy(), d.col_idx.cpu().numpy()
    w, ws = ctx.w.cpu().numpy(), ctx.wsum.cpu().numpy()
    src = np.ascontiguousarray(order, np.int64)
    out = np.empty_like(src)
    n_iso = np.zeros(1, np.int64)
    call("rsh_isolation_adjust", d.n_rows, d.n_cols, rp.ctypes.data, ci.ctypes.data, w.ctypes.data, ws.ctypes.data,
         src.ctypes.data, float(iso_threshold), -1 if hub_cap is None else int(hub_cap), out.ctypes.data,
         n_iso.ctypes.data)
    return out, int(n_iso[0])


def isolation_adjust(a: CsrMatrix, w: ColumnWeights, p: Permutation, iso_threshold: float = 0.05,
                     hub_cap: int | None = None) -> Permutation:
    """reorder.py:386-446: rows dissimilar to both sequence neighbours are reinserted after their
    most similar non-isolated row (host C++ restatement, rsh_isolation_adjust; weights on
    device).  iso_threshold = 0 returns the input verbatim."""
    import torch
    if not (0.0 <= iso_threshold <= 1.0):
        raise ValueError("iso_threshold must lie in [0, 1]")
    if len(p) <= 1 or iso_threshold == 0.0:
        return p
    ctx = _Ctx(a, w.alpha)
    out, n_iso = _isolation_host(ctx, p.order, iso_threshold, hub_cap)
    if n_iso == 0:
        return p
    return Permutation(out, ctx.objective(torch.from_numpy(out).to(ctx.d.device)))


def reorder_device(a, params: ReorderParams = ReorderParams()):
    """The pipeline on device: returns (order int64 device tensor, {"mst": objective,
    "refined": objective, "overflow_rows": n, "ms": {...}})."""
    import time
    import torch
    t0 = time.perf_counter()
    ctx = _Ctx(a, params.alpha)
    d = ctx.d
    nbr, sim, cnt, overflow = knn_device(ctx, params.k, params.max_candidates, params.hub_cap)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    order = _mst_host(d.n_rows, params.k, nbr.cpu().numpy(), sim.cpu().numpy(), cnt.cpu().numpy()) \
        if d.n_rows else np.empty(0, np.int64)
    t2 = time.perf_counter()
    o = torch.from_numpy(order).to(d.device)
    mst_obj = ctx.objective(o)
    two_opt_device(ctx, o, params.two_opt_window, params.two_opt_passes)
    refined = ctx.objective(o)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    # isolation pass (reorder.py:386-446), kept only when it does not worsen the objective
    final, n_iso = refined, 0
    if d.n_rows > 1 and params.iso_threshold > 0.0:
        adj, n_iso = _isolation_host(ctx, o.cpu().numpy(), params.iso_threshold, params.hub_cap)
        if n_iso:
            oa = torch.from_numpy(adj).to(d.device)
            obj = ctx.objective(oa)
            if obj <= refined:
                o, final = oa, obj
    t4 = time.perf_counter()
    return o, {"mst": mst_obj, "refined": refined, "final": final, "isolated_rows": n_iso, "overflow_rows": overflow,
               "ms": {"knn": 1e3 * (t1 - t0), "mst_host": 1e3 * (t2 - t1), "two_opt": 1e3 * (t3 - t2),
                      "isolation_host": 1e3 * (t4 - t3)}}


def reorder_pipeline(a: CsrMatrix, params: ReorderParams = ReorderParams()):
    """reorder.py:464-481: (Permutation, permuted matrix); the objective never exceeds the MST
    stage's."""
    o, info = reorder_device(a, params)
    best = Permutation(o.cpu().numpy(), info["final"])
    return best, permute_rows(a, best.order)


__all__ = ["ColumnWeights", "KnnGraph", "Permutation", "ReorderParams", "build_knn", "column_weights",
           "isolation_adjust", "knn_device", "load_permutation", "mst_order", "permutation_objective", "permute_rows",
           "permute_rows_device", "refine_2opt", "reorder_device", "reorder_pipeline", "save_permutation",
           "two_opt_device", "w_jaccard"]
