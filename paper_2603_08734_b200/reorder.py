"""Row permutation (rstile reorder.py:95-151) -- the part of the reorder subsystem the hot path
needs: formats are built "for the same permutation", so a permutation produced anywhere (the
reference's reorder_pipeline, a file, a graph library) is applied on device before partitioning.

The locality-aware search itself (reorder.py:168-481) is SURVEY §8(f) "next" and not part of
this package yet.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import CsrMatrix


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
    o = order if isinstance(order, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(order, np.int64))
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


__all__ = ["Permutation", "permute_rows", "permute_rows_device"]
