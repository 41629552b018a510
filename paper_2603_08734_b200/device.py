"""Device-resident RSH-SpMM pipeline: CSR -> partition -> split -> RS-Tile -> schedule -> SpMM.

Every step runs as sm_100a kernels from librsh.so (C ABI, include/rsh.h) on the current torch
CUDA stream; torch only allocates device memory (caller-owned buffers and workspaces, as the
ABI requires) and provides the stream.  The host reads back a handful of sizes between the
build phases (window / block / entry / residual counts) -- nothing else leaves the device.
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import call, lib

_U64 = np.uint64


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _stream(stream=None) -> int:
    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream


def _ws(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device)


def _upload(arr, dtype, dev) -> torch.Tensor:
    x = np.ascontiguousarray(arr, dtype=dtype)
    if not x.flags.writeable:  # reference containers are read-only; torch wants writable memory
        x = x.copy()
    return torch.from_numpy(x).to(dev)


def require_cuda(device=None) -> torch.device:
    """The product has no CPU path: fail loudly without a CUDA device or the library."""
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2603_08734_b200 needs a CUDA device (sm_100a); none is available")
    lib()
    return torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())


# ---------------------------------------------------------------------------------------------
# containers
# ---------------------------------------------------------------------------------------------

@dataclass
class DeviceCsr:
    """CSR resident in HBM with the reference dtypes (int64 row_ptr, int32 col_idx, f32 values)."""

    n_rows: int
    n_cols: int
    row_ptr: torch.Tensor
    col_idx: torch.Tensor
    values: torch.Tensor

    @property
    def nnz(self) -> int:
        return int(self.col_idx.numel())

    @property
    def device(self) -> torch.device:
        return self.row_ptr.device

    @classmethod
    def from_host(cls, a, device=None) -> "DeviceCsr":
        dev = require_cuda(device)
        return cls(int(a.n_rows), int(a.n_cols), _upload(a.row_ptr, np.int64, dev),
                   _upload(a.col_idx, np.int32, dev), _upload(a.values, np.float32, dev))


TILE_FIELDS = ("row_window_id", "row_window_offset", "bitmaps", "col_id", "values",
               "res_row_id", "res_offset", "res_col_id", "res_values")


@dataclass
class DeviceTile:
    """An RS-Tile matrix (tile.py:43-91) resident in HBM.  ``bitmaps`` is stored as int64 bits
    (torch's uint64 support is partial); ``to_host`` reinterprets them as uint64."""

    n_rows: int
    n_cols: int
    window_size: int
    row_window_id: torch.Tensor      # int32 [E]
    row_window_offset: torch.Tensor  # int64 [E+1]
    bitmaps: torch.Tensor            # int64 (u64 bits) [nb]
    col_id: torch.Tensor             # int32 [8 nb]
    values: torch.Tensor             # float32 [tc nnz]
    res_row_id: torch.Tensor         # int32 [R]
    res_offset: torch.Tensor         # int64 [R+1]
    res_col_id: torch.Tensor         # int32 [res nnz]
    res_values: torch.Tensor         # float32 [res nnz]
    _plan: "dict | SpmmPlan | None" = field(default=None, repr=False)

    @property
    def n_entries(self) -> int:
        return int(self.row_window_id.numel())

    @property
    def n_blocks(self) -> int:
        return int(self.bitmaps.numel())

    @property
    def n_res(self) -> int:
        return int(self.res_row_id.numel())

    @property
    def device(self) -> torch.device:
        return self.row_window_offset.device

    def nbytes(self) -> int:
        return sum(getattr(self, f).numel() * getattr(self, f).element_size() for f in TILE_FIELDS)

    def host_arrays(self) -> dict:
        out = {f: getattr(self, f).cpu().numpy() for f in TILE_FIELDS}
        out["bitmaps"] = out["bitmaps"].view(_U64)
        return out

    @classmethod
    def from_arrays(cls, n_rows, n_cols, window_size, arrays: dict, device=None) -> "DeviceTile":
        dev = require_cuda(device)
        dt = {"row_window_id": np.int32, "row_window_offset": np.int64, "bitmaps": np.uint64,
              "col_id": np.int32, "values": np.float32, "res_row_id": np.int32,
              "res_offset": np.int64, "res_col_id": np.int32, "res_values": np.float32}
        ts = {}
        for f in TILE_FIELDS:
            a = np.ascontiguousarray(arrays[f], dtype=dt[f])
            if f == "bitmaps":
                a = a.view(np.int64)
            ts[f] = _upload(a, a.dtype, dev)
        return cls(int(n_rows), int(n_cols), int(window_size), **ts)


# ---------------------------------------------------------------------------------------------
# build pipeline
# ---------------------------------------------------------------------------------------------

def partition_device(a: DeviceCsr, window_size: int, tau_nnz: int, tau_inc: int, stream=None):
    """partition.py:119-141 on device -> (win_start int32, resid_rows int32)."""
    dev = a.device
    n = a.n_rows
    win = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    res = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    counts = torch.zeros(2, dtype=torch.int64, device=dev)
    nbytes = lib().rsh_partition_workspace(n)
    ws = _ws(nbytes, dev)
    call("rsh_partition", _ptr(a.row_ptr), _ptr(a.col_idx), n, window_size, tau_nnz, tau_inc,
         _ptr(win), _ptr(res), _ptr(counts), _ptr(ws), nbytes, _stream(stream))
    nw, nr = (int(x) for x in counts.cpu())
    return win[:nw], res[:nr]


@dataclass
class WindowPlan:
    """Per-window planning state shared by split_long_work and the build (partition.py:144-180)."""

    win_start: torch.Tensor   # int32 [nw]
    win_count: torch.Tensor | None  # int32 [nw] explicit row counts, None = min(W, n - start)
    row_win: torch.Tensor     # int32 [n_rows]
    prefix: torch.Tensor      # int32 [nnz+1] exclusive scan of first-occurrence flags
    nblocks: torch.Tensor     # int64 [nw]
    longest: torch.Tensor     # int64 [nw]
    chunk: torch.Tensor       # int64 [nw], 0 = unsplit
    entry_base: torch.Tensor  # int64 [nw+1]
    block_base: torch.Tensor  # int64 [nw+1]
    n_entries: int
    n_blocks: int


def plan_windows(a: DeviceCsr, win_start: torch.Tensor, window_size: int, max_blocks_per_item,
                 split_on_row_nnz: bool = False, split_factor: float = 4.0, stream=None,
                 win_count: torch.Tensor | None = None) -> WindowPlan:
    dev = a.device
    nw = int(win_start.numel())
    bound = 0 if max_blocks_per_item is None else int(max_blocks_per_item)
    t64 = lambda k: torch.empty(max(k, 1), dtype=torch.int64, device=dev)  # noqa: E731
    row_win = torch.empty(max(a.n_rows, 1), dtype=torch.int32, device=dev)
    prefix = torch.empty(a.nnz + 1, dtype=torch.int32, device=dev)
    nblocks, longest, chunk = t64(nw), t64(nw), t64(nw)
    entry_base, block_base = t64(nw + 1), t64(nw + 1)
    nbytes = lib().rsh_plan_workspace(a.n_rows, a.nnz, nw)
    ws = _ws(nbytes, dev)
    call("rsh_plan_windows", _ptr(a.row_ptr), _ptr(a.col_idx), a.n_rows, a.nnz, window_size,
         _ptr(win_start), _ptr(win_count), nw, bound, int(bool(split_on_row_nnz)), float(split_factor),
         _ptr(row_win), _ptr(prefix), _ptr(nblocks), _ptr(longest), _ptr(chunk), _ptr(entry_base),
         _ptr(block_base), _ptr(ws), nbytes, _stream(stream))
    tot = torch.stack([entry_base[nw], block_base[nw]]).cpu()
    return WindowPlan(win_start, win_count, row_win, prefix, nblocks[:nw], longest[:nw], chunk[:nw],
                      entry_base[:nw + 1], block_base[:nw + 1], int(tot[0]), int(tot[1]))


def fill_tile(a: DeviceCsr, plan: WindowPlan, resid: torch.Tensor, window_size: int,
              entries: tuple[np.ndarray, np.ndarray] | None = None, stream=None) -> DeviceTile:
    """tile.py:102-173 on device.  ``entries`` = explicit (row_window_id, row_window_offset)
    host arrays for a caller-supplied split map; None = derive them from plan.chunk."""
    dev = a.device
    st = _stream(stream)
    nw = int(plan.win_start.numel())
    nb = plan.n_blocks
    if entries is None:
        ne = plan.n_entries
        rwid = torch.empty(max(ne, 1), dtype=torch.int32, device=dev)
        rwoff = torch.empty(ne + 1, dtype=torch.int64, device=dev)
    else:
        rwid = torch.from_numpy(np.ascontiguousarray(entries[0], np.int32)).to(dev)
        rwoff = torch.from_numpy(np.ascontiguousarray(entries[1], np.int64)).to(dev)
        ne = int(rwid.numel())
    bitmaps = torch.empty(max(nb, 1), dtype=torch.int64, device=dev)
    col_id = torch.empty(max(8 * nb, 1), dtype=torch.int32, device=dev)
    wn = torch.zeros(1, dtype=torch.int64, device=dev)
    call("rsh_window_nnz", _ptr(a.row_ptr), a.n_rows, _ptr(plan.win_start), _ptr(plan.win_count), nw, window_size,
         _ptr(wn), st)
    tc_nnz = int(wn.item())
    values = torch.empty(max(tc_nnz, 1), dtype=torch.float32, device=dev)
    nbytes = lib().rsh_fill_workspace(a.nnz, nb)
    ws = _ws(nbytes, dev)
    call("rsh_build_fill", _ptr(a.row_ptr), _ptr(a.col_idx), _ptr(a.values), a.n_rows, a.nnz,
         window_size, _ptr(plan.win_start), _ptr(plan.win_count), nw, _ptr(plan.row_win), _ptr(plan.prefix),
         _ptr(plan.block_base), nb, None if entries is not None else _ptr(plan.chunk),
         _ptr(plan.entry_base), _ptr(rwid), _ptr(rwoff), _ptr(bitmaps), _ptr(col_id), _ptr(values),
         _ptr(ws), nbytes, st)
    # residual part
    nr = int(resid.numel())
    r_off = torch.empty(nr + 1, dtype=torch.int64, device=dev)
    nbytes = lib().rsh_residual_workspace(nr)
    ws2 = _ws(nbytes, dev)
    call("rsh_residual_offsets", _ptr(a.row_ptr), _ptr(resid), nr, _ptr(r_off), _ptr(ws2), nbytes, st)
    r_nnz = int(r_off[nr].item())
    r_col = torch.empty(max(r_nnz, 1), dtype=torch.int32, device=dev)
    r_val = torch.empty(max(r_nnz, 1), dtype=torch.float32, device=dev)
    call("rsh_residual_gather", _ptr(a.row_ptr), _ptr(a.col_idx), _ptr(a.values), _ptr(resid), nr,
         _ptr(r_off), _ptr(r_col), _ptr(r_val), st)
    # window_size = max window row count, 8 when there are no windows (tile.py:169-173); only
    # the last window can be clamped by the matrix edge
    if nw == 0:
        wsize = 8
    elif plan.win_count is not None:
        wsize = int(plan.win_count.max().item())
    elif nw >= 2:
        wsize = window_size
    else:
        wsize = min(window_size, a.n_rows - int(plan.win_start[0].item()))
    return DeviceTile(a.n_rows, a.n_cols, wsize, rwid[:ne], rwoff, bitmaps[:nb], col_id[:8 * nb],
                      values[:tc_nnz], resid.clone(), r_off, r_col[:r_nnz], r_val[:r_nnz])


def build_device(a: DeviceCsr, window_size=8, tau_nnz=None, tau_inc=None, max_blocks_per_item=64,
                 split_on_row_nnz=False, split_factor=4.0, stream=None) -> DeviceTile:
    """partition_rows -> split_long_work -> build_rstile, entirely on device."""
    from .partition import estimate_thresholds
    if a.n_rows == 0:
        tn, ti = 0, 0
    else:
        est = estimate_thresholds(a.n_rows, a.nnz)
        tn = est[0] if tau_nnz is None else int(tau_nnz)
        ti = est[1] if tau_inc is None else int(tau_inc)
    win, res = partition_device(a, window_size, tn, ti, stream)
    plan = plan_windows(a, win, window_size, max_blocks_per_item, split_on_row_nnz, split_factor, stream)
    return fill_tile(a, plan, res, window_size, None, stream)


# ---------------------------------------------------------------------------------------------
# SpMM
# ---------------------------------------------------------------------------------------------

_BDT = {torch.float32: 0, torch.bfloat16: 1, torch.float16: 2}


CHUNK_CC = 32    # blocks per work unit for the CUDA-core kernel walking bitmaps (csrc/sched.cuh kChunkCC)
# ... for the streaming kernel reading the pre-decoded row-major list (RSH_CC_LIST_CHUNK overrides)
CHUNK_CC_LIST = int(os.environ.get("RSH_CC_LIST_CHUNK", "128"))
CHUNK_TC = 256   # ... and for the tensor-core kernel (kChunkTC)


def _tile_stamp(t: DeviceTile) -> tuple:
    """Identity of a tile's arrays (address + torch version counter): a cached schedule and its
    row-major list snapshot col_id / values, so they are rebuilt when an array is replaced or
    modified in place."""
    return tuple((getattr(t, f).data_ptr(), getattr(t, f)._version, getattr(t, f).numel()) for f in TILE_FIELDS)


class SpmmPlan:
    """Persistent-kernel work schedule of one DeviceTile for one unit size (built once, reused).

    The schedule is read-only during SpMM launches; each launch's mutable state (work counter,
    window tickets, chunk partials) lives in a workspace from ``workspace()``, one per (N,
    accumulation, stream), so launches on different streams never share one."""

    def __init__(self, t: DeviceTile, chunk: int = CHUNK_CC, stream=None):
        from .tile import FormatError, structural_issues
        issues = structural_issues(t)
        if issues:  # the kernels index with these arrays: refuse a malformed format up front
            raise FormatError("; ".join(issues))
        dev = t.device
        self.chunk = chunk
        self.stamp = _tile_stamp(t)
        self.n_entries = t.n_entries
        self.nbytes = lib().rsh_schedule_bytes(t.n_rows, t.n_entries, t.n_blocks, t.n_res)
        self.buf = _ws(self.nbytes, dev)
        hdr = torch.zeros(8, dtype=torch.int64, device=dev)
        call("rsh_schedule", t.n_rows, t.window_size, _ptr(t.row_window_id), _ptr(t.row_window_offset),
             t.n_entries, _ptr(t.bitmaps), t.n_blocks, _ptr(t.res_row_id), t.n_res, chunk, _ptr(self.buf),
             self.nbytes, _ptr(hdr), _stream(stream))
        h = hdr.cpu().tolist()
        self.groups, self.window_units, self.units, self.partial_slots, self.uncovered = h[:5]
        self.fixup_windows = h[6]
        self._ws = {}
        self._frags = {}
        self.ulist = None
        if chunk == CHUNK_CC_LIST:
            # the streaming kernel's pre-decoded window list (8 bytes per tc nonzero)
            tc_nnz = int(t.values.numel())
            lb = lib().rsh_rowmajor_bytes(t.n_rows, t.n_entries, t.n_blocks, t.n_res, tc_nnz)
            self.ulist = torch.empty((lb + 7) // 8, dtype=torch.int64, device=dev)
            call("rsh_schedule_rowmajor", t.n_rows, t.n_entries, _ptr(t.bitmaps), _ptr(t.col_id), _ptr(t.values),
                 t.n_blocks, tc_nnz, t.n_res, _ptr(self.buf), self.nbytes, _ptr(self.ulist), 8 * self.ulist.numel(),
                 _stream(stream))

    def fragments(self, t: DeviceTile, b_dtype: int, stream=None) -> torch.Tensor:
        """The tensor-core kernel's schedule-time fragments for one operand type (rsh_tc_fragments),
        built on first use."""
        if b_dtype not in self._frags:
            nbytes = lib().rsh_tc_fragment_bytes(t.n_blocks, b_dtype)
            fr = torch.empty((nbytes + 15) // 16 * 16, dtype=torch.uint8, device=t.device)
            call("rsh_tc_fragments", t.n_rows, t.n_entries, _ptr(t.bitmaps), _ptr(t.values), t.n_blocks, t.n_res,
                 b_dtype, _ptr(self.buf), self.nbytes, _ptr(fr), fr.numel(), _stream(stream))
            self._frags[b_dtype] = fr
        return self._frags[b_dtype]

    def workspace(self, N: int, accum: int, dev, stream=None) -> torch.Tensor:
        """Zero-filled SpMM workspace (control block + chunk partials) for one stream."""
        sid = _stream(stream)
        key = (N, accum, sid)
        if key not in self._ws:
            nbytes = lib().rsh_partials_bytes(self.n_entries, self.partial_slots, N, accum)
            self._ws[key] = torch.zeros(max(int(nbytes), 16), dtype=torch.uint8, device=dev)
        return self._ws[key]

    partials = workspace  # round-1 name


# the streaming kernel reads a pre-decoded row-major window list (rsh_schedule_rowmajor)
ROWMAJOR_LIST = os.environ.get("RSH_ROWMAJOR_LIST", "1") != "0"
# rsh_spmm_cc tuning knobs (accum bits 1..): development override through RSH_CC_VARIANT
CC_VARIANT = int(os.environ.get("RSH_CC_VARIANT", "0"))
NO_FIXUP = 8192  # cc variant bit: the schedule has no window the fix-up kernels must reduce
# rsh_spmm_tc perf-probe knobs (bits 0-2 skip gathers / decode / MMA: results invalid); development only
TC_FLAGS = int(os.environ.get("RSH_TC_FLAGS", "0"))


def spmm_plan(t: DeviceTile, chunk: int = CHUNK_CC) -> SpmmPlan:
    """The cached schedule of ``t`` for units of ``chunk`` blocks (rebuilt when the tile's arrays
    were replaced or modified in place since it was built)."""
    if t._plan is None:
        t._plan = {}
    elif isinstance(t._plan, SpmmPlan):  # a single prebuilt schedule handed over by a caller
        t._plan = {t._plan.chunk: t._plan}
    pl = t._plan.get(chunk)
    if pl is None or pl.stamp != _tile_stamp(t):
        pl = t._plan[chunk] = SpmmPlan(t, chunk)
    return pl


TC_N = {torch.float32: (32, 64, 128, 256), torch.bfloat16: (64, 128, 256), torch.float16: (64, 128, 256)}


def tc_eligible(t: DeviceTile, b: torch.Tensor, accumulate: str = "f32") -> bool:
    """The tensor-core kernel handles N in {32, 64, 128, 256} (fp32 B; {64, 128, 256} for half B)
    with f32 accumulation and 16-B aligned rows (csrc/spmm_tc.cu)."""
    n = int(b.shape[1])
    eb = b.element_size()
    return (accumulate == "f32" and n in TC_N.get(b.dtype, ()) and b.data_ptr() % 16 == 0
            and (b.stride(0) * eb) % 16 == 0)


def resolve_math(math: str, b: torch.Tensor, t: DeviceTile, accumulate: str) -> str:
    """"tc" (tcgen05 window path) or "cc" (CUDA-core streaming kernel).  "auto" runs the CUDA
    cores for every dtype: the window path's cost is the B-row gather, and the streaming kernel
    gathers faster than the tensor-core pipeline can stage (measured on every BASELINE config,
    DESIGN.md section 3.3).  "tf32" / "tc" ask for the tensor cores (TF32 for fp32 B, BF16/FP16
    MMA for half B); "fp32" is the exact-FP32 CUDA-core path."""
    if math not in ("auto", "fp32", "tf32", "tc"):
        raise ValueError(f"unknown math mode {math!r}")
    if math in ("auto", "fp32") or accumulate != "f32":
        return "cc"
    if not tc_eligible(t, b, accumulate):
        raise ValueError(f"math={math!r} needs N in {TC_N.get(b.dtype, ())} for {b.dtype}, f32 accumulation and "
                         "16-byte aligned B rows")
    return "tc"


def spmm_device(t: DeviceTile, b: torch.Tensor, out: torch.Tensor | None = None, accumulate: str = "f32",
                stream=None, math: str = "auto", cc_variant: int | None = None) -> torch.Tensor:
    """C = A @ B with A an RS-Tile on device; B [n_cols, N] f32/bf16/f16 row-major on device.
    Returns (or fills) C [n_rows, N] float32.  accumulate: "f32" | "f64" (execute.py:33-49);
    math: "auto" / "fp32" (CUDA-core FMA) | "tf32" / "tc" (tensor cores, see resolve_math)."""
    if b.dim() != 2 or b.shape[0] != t.n_cols:
        raise ValueError(f"dimension mismatch: matrix has {t.n_cols} columns, B has {tuple(b.shape)}")
    if b.dtype not in _BDT:
        raise ValueError(f"unsupported B dtype {b.dtype}")
    if not b.is_cuda:
        raise ValueError("B must be a CUDA tensor (use hybrid_spmm for host operands)")
    if b.stride(1) != 1:
        b = b.contiguous()
    N = int(b.shape[1])
    if out is None:
        out = torch.empty((t.n_rows, N), dtype=torch.float32, device=b.device)
    elif out.shape != (t.n_rows, N) or out.dtype != torch.float32 or out.stride(1) != 1:
        raise ValueError("out must be a float32 [n_rows, N] tensor with unit column stride")
    if t.n_rows == 0 or N == 0:
        return out
    acc = {"f32": 0, "f64": 1}[accumulate]
    if cc_variant is None:
        cc_variant = CC_VARIANT
    path = resolve_math(math, b, t, accumulate)
    if path == "tc":
        chunk = CHUNK_TC
    elif acc == 0 and ROWMAJOR_LIST and not (cc_variant & (64 | 4096)):
        # long units + the row-major list; cc_variant bits 64 / 4096 select 32-block units without
        # the list (the bitmap-decoding stream; tests/test_gpu_parity.py compares the variants)
        chunk = CHUNK_CC_LIST
    else:
        chunk = CHUNK_CC
    plan = spmm_plan(t, chunk)
    part = plan.workspace(N, acc, b.device, stream)
    res = (_ptr(t.res_row_id), _ptr(t.res_offset), _ptr(t.res_col_id), _ptr(t.res_values), t.n_res)
    if path == "tc":
        flags = (NO_FIXUP if plan.fixup_windows == 0 else 0) | TC_FLAGS
        fr = plan.fragments(t, _BDT[b.dtype], stream)
        call("rsh_spmm_tc", t.n_rows, t.window_size, t.n_entries, _ptr(t.bitmaps), _ptr(t.col_id), _ptr(fr),
             fr.numel(), t.n_blocks, *res, _ptr(b), int(b.shape[0]), b.stride(0), _BDT[b.dtype], N, _ptr(out),
             out.stride(0), flags, _ptr(plan.buf), plan.nbytes, _ptr(part), part.numel(), _stream(stream))
    else:
        fmt = (t.n_rows, t.window_size, t.n_entries, _ptr(t.bitmaps), _ptr(t.col_id), _ptr(t.values), t.n_blocks,
               *res)
        flags = acc | (cc_variant << 1)
        if plan.fixup_windows == 0:
            flags |= NO_FIXUP << 1
        call("rsh_spmm_cc", *fmt, _ptr(b), b.stride(0), _BDT[b.dtype], N, _ptr(out), out.stride(0),
             flags, _ptr(plan.buf), plan.nbytes, _ptr(part), part.numel(), _stream(stream))
    return out


def max_relative_error_device(c: torch.Tensor, ref: torch.Tensor, stream=None) -> float:
    out = torch.zeros(1, dtype=torch.float64, device=c.device)
    call("rsh_max_relative_error", _ptr(c), _ptr(ref), c.shape[0], c.shape[1], c.stride(0), _ptr(out),
         _stream(stream))
    return float(out.item())


# ---------------------------------------------------------------------------------------------
# host-resident operands, streamed
# ---------------------------------------------------------------------------------------------

TILE_HOST_FIELDS = ("row_window_id", "row_window_offset", "bitmaps", "col_id", "values", "res_row_id", "res_offset",
                    "res_col_id", "res_values")


class HostStream:
    """SpMMs whose format, B and C live in (pinned) host memory: every step copies the format and
    B in, runs ``spmm_device`` (schedule rebuilt: the arrays are new data) and copies C out.
    Steps are pipelined over three CUDA streams with two device buffer sets: step i+1's inputs
    are enqueued before step i's SpMM (whose schedule build waits on the host for step i's
    inputs), so the host-to-device engine never idles, and step i's C copy overlaps step i+1's
    input copies (PCIe is full duplex).

    ``host``: dict of pinned host tensors keyed by TILE_HOST_FIELDS; ``b_host`` pinned B;
    ``n_rows`` / ``n_cols`` / ``window_size`` describe the format; results land in the two pinned
    ``c_host`` buffers alternately (``result(i)`` after ``run``)."""

    def __init__(self, host: dict, b_host: torch.Tensor, n_rows: int, n_cols: int, window_size: int,
                 device=None, math: str = "auto"):
        dev = require_cuda(device)
        self.host, self.b_host, self.math = host, b_host, math
        self.c_host = [torch.empty((n_rows, int(b_host.shape[1])), dtype=torch.float32).pin_memory() for _ in range(2)]
        self.sets = []
        for _ in range(2):
            bufs = {k: torch.empty_like(v, device=dev) for k, v in host.items()}
            self.sets.append((DeviceTile(n_rows, n_cols, window_size, **bufs), bufs,
                              torch.empty_like(b_host, device=dev),
                              torch.empty((n_rows, int(b_host.shape[1])), dtype=torch.float32, device=dev)))
        self.s_in, self.s_comp, self.s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    @property
    def h2d_bytes(self) -> int:
        return sum(v.numel() * v.element_size() for v in self.host.values()) + \
            self.b_host.numel() * self.b_host.element_size()

    @property
    def d2h_bytes(self) -> int:
        return self.c_host[0].numel() * 4

    def result(self, i: int) -> torch.Tensor:
        """Host C of step i of the last ``run`` (the last two steps' results are kept)."""
        return self.c_host[i % 2]

    def run(self, n_steps: int, pipelined: bool = True) -> float:
        """n_steps steps; returns milliseconds per step (device events from the first input copy
        to the last C copy).  pipelined=False runs one step at a time (one buffer set)."""
        torch.cuda.synchronize()
        ev = lambda: torch.cuda.Event(enable_timing=False)  # noqa: E731
        comp_done, out_done, in_done = [None, None], [None, None], [None, None]
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(self.s_in)

        def stage_inputs(i: int) -> None:
            k = i % 2 if pipelined else 0
            _, bufs, b_dev, _ = self.sets[k]
            if comp_done[k] is not None:
                self.s_in.wait_event(comp_done[k])      # set k's inputs are free again
            with torch.cuda.stream(self.s_in):
                for f, v in self.host.items():
                    bufs[f].copy_(v, non_blocking=True)
                b_dev.copy_(self.b_host, non_blocking=True)
                in_done[k] = ev()
                in_done[k].record(self.s_in)

        stage_inputs(0)
        for i in range(n_steps):
            k = i % 2 if pipelined else 0
            t, _, b_dev, c_dev = self.sets[k]
            if pipelined and i + 1 < n_steps:
                stage_inputs(i + 1)                     # before this step's host-blocking schedule
            self.s_comp.wait_event(in_done[k])
            if out_done[k] is not None:
                self.s_comp.wait_event(out_done[k])     # set k's C has reached the host
            with torch.cuda.stream(self.s_comp):
                spmm_device(t, b_dev, out=c_dev, math=self.math, stream=self.s_comp)
                comp_done[k] = ev()
                comp_done[k].record(self.s_comp)
            self.s_out.wait_event(comp_done[k])
            with torch.cuda.stream(self.s_out):
                self.c_host[i % 2].copy_(c_dev, non_blocking=True)
                out_done[k] = ev()
                out_done[k].record(self.s_out)
            if not pipelined:
                torch.cuda.synchronize()
                if i + 1 < n_steps:
                    stage_inputs(i + 1)
        for e in out_done:
            if e is not None:
                self.s_out.wait_event(e)
        t1.record(self.s_out)
        torch.cuda.synchronize()
        return t0.elapsed_time(t1) / n_steps
