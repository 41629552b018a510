"""Host-side matrix containers with the reference's contracts (rstile core.py).

These are the drop-in boundary types: the same class names, fields, dtypes, immutability and
ValueError checks as the reference (core.py:26-100 CsrMatrix, core.py:190-213 DenseMatrix),
so code written against ``rstile`` can pass its matrices straight in.  They hold numpy arrays;
the compute entry points move them to the GPU (see device.py) -- nothing here computes a
product.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

INDEX_LIMIT = 2 ** 31  # core.py:18


def _frozen(arr: np.ndarray) -> np.ndarray:
    arr.flags.writeable = False
    return arr


@dataclass(frozen=True)
class CsrMatrix:
    """Canonical CSR: int64 row_ptr[n_rows+1], int32 col_idx, float32 values, columns strictly
    increasing inside every row, all arrays read-only (core.py:26-71)."""

    n_rows: int
    n_cols: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray

    def __post_init__(self) -> None:
        if self.n_rows < 0 or self.n_cols < 0:
            raise ValueError("matrix dimensions must be non-negative")
        rp = np.ascontiguousarray(self.row_ptr, dtype=np.int64)
        ci = np.ascontiguousarray(self.col_idx, dtype=np.int32)
        va = np.ascontiguousarray(self.values, dtype=np.float32)
        nnz = va.size
        if max(self.n_rows, self.n_cols, nnz) >= INDEX_LIMIT:
            raise ValueError("dimensions or nnz exceed the 32-bit index limit")
        if rp.shape != (self.n_rows + 1,):
            raise ValueError("row_ptr must have length n_rows + 1")
        if ci.shape != va.shape:
            raise ValueError("col_idx and values must have equal length")
        if rp[0] != 0 or rp[-1] != nnz:
            raise ValueError("row_ptr must start at 0 and end at nnz")
        if nnz:
            if (rp[1:] < rp[:-1]).any():
                raise ValueError("row_ptr must be monotone")
            if int(ci.min()) < 0 or int(ci.max()) >= self.n_cols:
                raise ValueError("column index out of range")
            # strictly increasing within a row: every step that does not start a new row
            step_ok = ci[1:] > ci[:-1]
            row_start = np.zeros(nnz, dtype=bool)
            starts = rp[1:-1]
            row_start[starts[starts < nnz]] = True
            if not (step_ok | row_start[1:]).all():
                raise ValueError("column indices must increase strictly within a row")
        object.__setattr__(self, "row_ptr", _frozen(rp))
        object.__setattr__(self, "col_idx", _frozen(ci))
        object.__setattr__(self, "values", _frozen(va))

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def row_nnz(self) -> np.ndarray:
        return self.row_ptr[1:] - self.row_ptr[:-1]

    def row_cols(self, r: int) -> np.ndarray:
        return self.col_idx[self.row_ptr[r]:self.row_ptr[r + 1]]

    def row_values(self, r: int) -> np.ndarray:
        return self.values[self.row_ptr[r]:self.row_ptr[r + 1]]

    @classmethod
    def from_dense(cls, dense) -> "CsrMatrix":
        arr = np.asarray(dense, dtype=np.float32)
        if arr.ndim != 2:
            raise ValueError("expected a 2-d array")
        mask = arr != 0
        rp = np.zeros(arr.shape[0] + 1, dtype=np.int64)
        rp[1:] = np.cumsum(mask.sum(axis=1))
        rows, cols = np.nonzero(mask)
        return cls(arr.shape[0], arr.shape[1], rp, cols, arr[rows, cols])

    def to_dense(self) -> np.ndarray:
        out = np.zeros((self.n_rows, self.n_cols), dtype=np.float32)
        rows = np.repeat(np.arange(self.n_rows), self.row_nnz())
        out[rows, self.col_idx] = self.values
        return out


def csr_equal(a: CsrMatrix, b: CsrMatrix) -> bool:
    """Exact equality of shape, structure and values (core.py:103-111)."""
    return (a.n_rows, a.n_cols) == (b.n_rows, b.n_cols) and all(
        np.array_equal(x, y) for x, y in ((a.row_ptr, b.row_ptr), (a.col_idx, b.col_idx),
                                          (a.values, b.values)))


@dataclass(frozen=True)
class DenseMatrix:
    """Row-major float32 matrix whose entries must all be finite (core.py:190-213)."""

    n_rows: int
    n_cols: int
    data: np.ndarray

    def __post_init__(self) -> None:
        d = np.ascontiguousarray(self.data, dtype=np.float32)
        if d.shape != (self.n_rows, self.n_cols):
            raise ValueError("data shape does not match dimensions")
        if not np.isfinite(d).all():
            raise ValueError("dense matrix entries must be finite")
        object.__setattr__(self, "data", _frozen(d))

    @classmethod
    def from_array(cls, arr) -> "DenseMatrix":
        a = np.asarray(arr, dtype=np.float32)
        return cls(a.shape[0], a.shape[1], a)

    @classmethod
    def zeros(cls, n_rows: int, n_cols: int) -> "DenseMatrix":
        return cls(n_rows, n_cols, np.zeros((n_rows, n_cols), dtype=np.float32))


def max_relative_error(c, ref) -> float:
    """max |c - ref| / max(|ref|, 1) over all entries (core.py:398-408)."""
    x = c.data if isinstance(c, DenseMatrix) else np.asarray(c)
    y = ref.data if isinstance(ref, DenseMatrix) else np.asarray(ref)
    if x.shape != y.shape:
        raise ValueError(f"shape mismatch: {x.shape} vs {y.shape}")
    if x.size == 0:
        return 0.0
    x = x.astype(np.float64)
    y = y.astype(np.float64)
    return float((np.abs(x - y) / np.maximum(np.abs(y), 1.0)).max())
