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
    bt = torch.from_numpy(np.ascontiguousarray(bd, np.float32)).to(t.device)
    c = _device_spmm(t, bt, cfg)
    if cfg.check_against_oracle:
        _verify(t, bt, c)
    return DenseMatrix.from_array(c.cpu().numpy())


__all__ = ["ExecConfig", "VerificationError", "hybrid_spmm", "ORACLE_TOLERANCE"]
