"""Hybrid SpMM executor (rstile execute.py) -- same entry point, one persistent GPU launch.

``hybrid_spmm(m, b, cfg)`` keeps execute.py:155-226's contract: dimension check (ValueError),
a fresh float32 C, every row written once (window rows assigned, residual rows assigned, all
other rows zero), optional verification against an f64 reference (VerificationError above
ORACLE_TOLERANCE max-relative error).  The work runs on the GPU:

* host operands (RsTileMatrix + DenseMatrix) are uploaded, the product runs, C comes back as a
  DenseMatrix -- a drop-in for the reference call;
* device operands (DeviceTile + a CUDA tensor) stay on the device and a CUDA tensor is
  returned (``out=`` reuses a caller buffer).

``ExecConfig.num_workers`` is accepted for API compatibility (the reference's thread count);
the GPU path is a single persistent launch whose result is independent of any worker count.
``check_against_oracle`` recomputes C on device with f64 accumulation over the same format
(the reference decodes and runs oracle_spmm on the CPU, execute.py:219-225) and compares with
the device max-relative-error kernel.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import DenseMatrix

ORACLE_TOLERANCE = 1e-5  # execute.py:26


class VerificationError(ArithmeticError):
    """The executor's result diverged from the reference beyond tolerance (execute.py:29-30)."""


@dataclass(frozen=True)
class ExecConfig:
    """execute.py:33-49 plus the GPU arithmetic mode.

    math: "fp32"  CUDA-core FP32 FMA (exact f32 products; the reference's f32 semantics)
          "tf32"  tensor-core window path, TF32 operands, f32 accumulation (north-star (2));
                  "tc" is the same request for any B dtype (BF16/FP16 MMA for half B)
          "auto"  the CUDA-core streaming kernel for every dtype (the faster path, measured)
    """

    num_workers: int = 1
    check_against_oracle: bool = False
    accumulate_precision: str = "f32"
    math: str = "auto"

    def __post_init__(self) -> None:
        if self.num_workers < 1:
            raise ValueError(f"num_workers must be >= 1, got {self.num_workers}")
        if self.accumulate_precision not in ("f32", "f64"):
            raise ValueError(
                f"accumulate_precision must be f32 or f64, got {self.accumulate_precision!r}")
        if self.math not in ("auto", "fp32", "tf32", "tc"):
            raise ValueError(f"math must be auto, fp32, tf32 or tc, got {self.math!r}")

    @property
    def dtype(self) -> np.dtype:
        return np.dtype(np.float64 if self.accumulate_precision == "f64" else np.float32)


def _device_spmm(t, b, cfg: ExecConfig, out=None):
    from .device import spmm_device
    math = "fp32" if cfg.math == "fp32" else cfg.math
    return spmm_device(t, b, out=out, accumulate=cfg.accumulate_precision, math=math)


def _verify(t, b, c) -> None:
    from .device import max_relative_error_device, spmm_device
    ref = spmm_device(t, b, accumulate="f64")
    err = max_relative_error_device(c, ref)
    if err > ORACLE_TOLERANCE:
        raise VerificationError(f"max relative error {err:.3e} exceeds {ORACLE_TOLERANCE:.0e}")


def hybrid_spmm(m, b, cfg: ExecConfig | None = None, out=None):
    """C = A @ B over the RS-Tile format (execute.py:155-226)."""
    import torch
    from .device import DeviceTile
    from .tile import FormatError, RsTileMatrix, tile_to_device
    cfg = cfg or ExecConfig()
    if isinstance(m, DeviceTile):
        t = m
        if not isinstance(b, torch.Tensor):
            raise ValueError("a DeviceTile multiplies a CUDA tensor B")
        if b.dim() != 2 or b.shape[0] != t.n_cols:
            raise ValueError(f"dimension mismatch: matrix has {t.n_cols} columns, B has {tuple(b.shape)}")
        c = _device_spmm(t, b, cfg, out)
        if cfg.check_against_oracle:
            _verify(t, b, c)
        return c
    if not isinstance(m, RsTileMatrix):
        raise TypeError("hybrid_spmm expects an RsTileMatrix or a DeviceTile")
    bd = b.data if isinstance(b, DenseMatrix) else np.asarray(b, dtype=np.float32)
    if bd.ndim != 2 or bd.shape[0] != m.n_cols:
        raise ValueError(
            f"dimension mismatch: matrix has {m.n_cols} columns, B has {bd.shape[0] if bd.ndim else 0} rows")
    # execute.py:93-95, 196-200: column ids must address rows of B
    for ids in (m.tc.col_id, m.residual.col_id):
        if ids.size and (int(ids.min()) < 0 or int(ids.max()) >= bd.shape[0]):
            raise FormatError("col_id references a column outside B's row range")
    t = tile_to_device(m)
    bt = torch.from_numpy(np.array(bd, np.float32, order="C", copy=True)).to(t.device)
    c = _device_spmm(t, bt, cfg)
    if cfg.check_against_oracle:
        _verify(t, bt, c)
    return DenseMatrix.from_array(c.cpu().numpy())


__all__ = ["ExecConfig", "VerificationError", "hybrid_spmm", "ORACLE_TOLERANCE"]


# ---------------------------------------------------------------------------------------------
# per-block / per-entry executor pieces (execute.py:52-133) -- each runs the device SpMM on a
# one-window or residual-only sub-format, so the arithmetic is the product kernel's
# ---------------------------------------------------------------------------------------------

def oracle_spmm(a, b) -> DenseMatrix:
    """core.py:380-395 on device: C = A @ B with every row accumulated in f64 in CSR order (A's
    values and B widened exactly), stored as f32; empty rows are zero.  ``a`` is a CsrMatrix (or
    a DeviceCsr), ``b`` a DenseMatrix (or a CUDA tensor; a CUDA tensor is returned)."""
    import torch

    from ._lib import call
    from .device import DeviceCsr, _ptr, _stream, require_cuda
    host = not isinstance(a, DeviceCsr)
    n_b = b.n_rows if isinstance(b, DenseMatrix) else int(b.shape[0])
    if a.n_cols != n_b:
        raise ValueError(f"dimension mismatch: A is {a.n_rows}x{a.n_cols}, B has {n_b} rows")
    dev = require_cuda()
    d = DeviceCsr.from_host(a, dev) if host else a
    if isinstance(b, DenseMatrix):
        bt = torch.from_numpy(np.array(b.data, np.float32, order="C", copy=True)).to(d.device)
    else:
        bt = b.float().contiguous()
    n_feat = int(bt.shape[1])
    c = torch.empty((d.n_rows, n_feat), dtype=torch.float32, device=d.device)
    call("rsh_csr_spmm_f64", _ptr(d.row_ptr), _ptr(d.col_idx), _ptr(d.values), d.n_rows, _ptr(bt), bt.stride(0),
         n_feat, _ptr(c), c.stride(0), _stream())
    if not isinstance(b, DenseMatrix):
        return c
    return DenseMatrix(d.n_rows, n_feat, c.cpu().numpy())


@dataclass(frozen=True)
class Fragment8x8:
    """execute.py:52-62: dense row-major 8x8 expansion of one bitmap block."""

    data: np.ndarray

    def __post_init__(self) -> None:
        arr = np.ascontiguousarray(self.data, dtype=np.float32)
        if arr.shape != (8, 8):
            raise ValueError(f"fragment must be 8x8, got {arr.shape}")
        arr.flags.writeable = False
        object.__setattr__(self, "data", arr)


def _window_tile(bitmaps, col_id, values, n_cols: int):
    """A one-window RS-Tile (rows 0..7) holding the given blocks."""
    from .tile import ResidualPart, RsTileMatrix, TcPart
    nb = int(np.asarray(bitmaps).size)
    z32, z64 = np.zeros(0, np.int32), np.zeros(1, np.int64)
    return RsTileMatrix(8, n_cols, TcPart(np.zeros(1 if nb else 0, np.int32), np.array([0, nb] if nb else [0], np.int64),
                                          bitmaps, col_id, values),
                        ResidualPart(z32, z64, z32, np.zeros(0, np.float32)), 8)


def decode_tile(bitmap: int, values) -> Fragment8x8:
    """execute.py:80-89: expand one bitmap block (bit b -> row b >> 3, column b & 7); on device,
    as the block times the 8x8 identity."""
    from .tile import TcPart  # noqa: F401
    bm = np.array([bitmap], dtype=np.uint64)
    vals = np.asarray(values, dtype=np.float32).ravel()
    expected = bin(int(bitmap) & (2 ** 64 - 1)).count("1")
    if vals.size != expected:
        raise ValueError(f"bitmap has {expected} set bits but {vals.size} values were given")
    m = _window_tile(bm, np.arange(8, dtype=np.int32), vals, 8)
    eye = DenseMatrix.from_array(np.eye(8, dtype=np.float32))
    return Fragment8x8(hybrid_spmm(m, eye, ExecConfig(math="fp32")).data)


def exec_tc_window(m, entry: int, b: DenseMatrix, c_out: np.ndarray) -> None:
    """execute.py:98-114: accumulate one window entry's block products into a local 8 x d
    array (f32 or f64 by c_out's dtype)."""
    from ._lib import FormatError
    if not 0 <= entry < m.tc.n_entries:
        raise IndexError(f"entry {entry} out of range")
    bs, be = int(m.tc.row_window_offset[entry]), int(m.tc.row_window_offset[entry + 1])
    if bs == be:
        return
    cols = np.asarray(m.tc.col_id[bs * 8:be * 8])
    if cols.size and (int(cols.min()) < 0 or int(cols.max()) >= b.n_rows):
        raise FormatError("col_id references a column outside B's row range")
    pc = np.unpackbits(np.ascontiguousarray(m.tc.bitmaps, "<u8").view(np.uint8)).reshape(-1, 64).sum(1)
    vs = int(pc[:bs].sum())
    sub = _window_tile(m.tc.bitmaps[bs:be], cols, m.tc.values[vs:vs + int(pc[bs:be].sum())], b.n_rows)
    prec = "f64" if c_out.dtype == np.float64 else "f32"
    r = hybrid_spmm(sub, b, ExecConfig(math="fp32", accumulate_precision=prec)).data
    c_out += r.astype(c_out.dtype)


def exec_residual(m, b: DenseMatrix, c: np.ndarray) -> None:
    """execute.py:117-133: c[r] += v . B[cols] for every residual row (on device)."""
    from ._lib import FormatError
    from .tile import RsTileMatrix, TcPart
    res = m.residual
    if res.col_id.size and (int(res.col_id.min()) < 0 or int(res.col_id.max()) >= b.n_rows):
        raise FormatError("residual col_id references a column outside B")
    if res.n_rows == 0:
        return
    sub = RsTileMatrix(m.n_rows, m.n_cols, TcPart(np.zeros(0, np.int32), np.zeros(1, np.int64),
                                                  np.zeros(0, np.uint64), np.zeros(0, np.int32),
                                                  np.zeros(0, np.float32)), res, 8)
    prec = "f64" if c.dtype == np.float64 else "f32"
    r = hybrid_spmm(sub, b, ExecConfig(math="fp32", accumulate_precision=prec)).data
    rows = np.asarray(res.row_id, np.int64)
    c[rows] += r[rows].astype(c.dtype)
