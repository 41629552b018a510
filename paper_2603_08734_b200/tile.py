"""RS-Tile format (rstile tile.py) -- same host dataclasses, built on device.

``build_rstile(a, plan)`` mirrors tile.py:102-166: it checks the plan (ValueError on a
mismatch), then the bitmap blocks, padded col_id, bit-ordered values, entry arrays and the
residual part are produced by the sm_100a builder (csrc/builder.cu) and copied back into the
reference's TcPart / ResidualPart / RsTileMatrix types, bit-exact with the reference.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from ._lib import FormatError
from .core import CsrMatrix
from .partition import PartitionPlan, _dev, _max_rows, _win_tensors, validate_plan


def _ro(a, dt) -> np.ndarray:
    x = np.ascontiguousarray(a, dtype=dt)
    x.flags.writeable = False
    return x


@dataclass(frozen=True)
class TcPart:
    """tile.py:43-62: int32 row_window_id[E], int64 row_window_offset[E+1], uint64 bitmaps[nb],
    int32 col_id[8 nb], float32 values (bit order)."""

    row_window_id: np.ndarray
    row_window_offset: np.ndarray
    bitmaps: np.ndarray
    col_id: np.ndarray
    values: np.ndarray

    def __post_init__(self) -> None:
        for name, dt in (("row_window_id", np.int32), ("row_window_offset", np.int64),
                         ("bitmaps", np.uint64), ("col_id", np.int32), ("values", np.float32)):
            object.__setattr__(self, name, _ro(getattr(self, name), dt))

    @property
    def n_entries(self) -> int:
        return int(self.row_window_id.size)

    @property
    def n_blocks(self) -> int:
        return int(self.bitmaps.size)


@dataclass(frozen=True)
class ResidualPart:
    """tile.py:65-82: int32 row_id, int64 row_nnz_offset[R+1], int32 col_id, float32 values."""

    row_id: np.ndarray
    row_nnz_offset: np.ndarray
    col_id: np.ndarray
    values: np.ndarray

    def __post_init__(self) -> None:
        for name, dt in (("row_id", np.int32), ("row_nnz_offset", np.int64), ("col_id", np.int32),
                         ("values", np.float32)):
            object.__setattr__(self, name, _ro(getattr(self, name), dt))

    @property
    def n_rows(self) -> int:
        return int(self.row_id.size)


@dataclass(frozen=True)
class RsTileMatrix:
    """tile.py:85-91."""

    n_rows: int
    n_cols: int
    tc: TcPart
    residual: ResidualPart
    window_size: int


def tile_from_device(t) -> RsTileMatrix:
    """Copy a DeviceTile back into the reference host types."""
    h = t.host_arrays()
    return RsTileMatrix(t.n_rows, t.n_cols,
                        TcPart(h["row_window_id"], h["row_window_offset"], h["bitmaps"], h["col_id"],
                               h["values"]),
                        ResidualPart(h["res_row_id"], h["res_offset"], h["res_col_id"], h["res_values"]),
                        t.window_size)


def tile_to_device(m: RsTileMatrix, device=None):
    """Upload a host RsTileMatrix (cached on the instance; the instance is immutable)."""
    from .device import DeviceTile
    d = m.__dict__.get("_device_tile")
    if d is None:
        d = DeviceTile.from_arrays(m.n_rows, m.n_cols, m.window_size, {
            "row_window_id": m.tc.row_window_id, "row_window_offset": m.tc.row_window_offset,
            "bitmaps": m.tc.bitmaps, "col_id": m.tc.col_id, "values": m.tc.values,
            "res_row_id": m.residual.row_id, "res_offset": m.residual.row_nnz_offset,
            "res_col_id": m.residual.col_id, "res_values": m.residual.values}, device)
        object.__setattr__(m, "_device_tile", d)
    return d


def build_rstile_device(a: CsrMatrix, plan: PartitionPlan):
    """tile.py:102-166 on device, returning the DeviceTile (no copy back)."""
    import torch
    from .device import fill_tile, plan_windows
    issues = validate_plan(a, plan)
    if issues:
        raise ValueError(f"plan does not match matrix: {issues[0]}")
    dev = _dev(a)
    res = torch.from_numpy(np.ascontiguousarray(plan.residual_rows, np.int32)).to(dev.device)
    if not plan.windows:
        starts = torch.zeros(0, dtype=torch.int32, device=dev.device)
        counts = starts
    else:
        starts, counts = _win_tensors(a, plan)
    wp = plan_windows(dev, starts, min(8, _max_rows(plan)), None, win_count=counts)
    # one entry per segment, all sharing the window's start row (tile.py:135-144)
    nblocks = wp.nblocks.cpu().numpy()
    rwid, eblocks = [], []
    for i, (s, _c) in enumerate(plan.windows):
        segs = plan.split_map.get(i)
        if segs is None:
            rwid.append(s)
            eblocks.append(int(nblocks[i]))
        else:
            for bs, be in segs:
                rwid.append(s)
                eblocks.append(be - bs)
    offsets = np.zeros(len(rwid) + 1, np.int64)
    np.cumsum(np.asarray(eblocks, np.int64), out=offsets[1:])
    return fill_tile(dev, wp, res, min(8, _max_rows(plan)),
                     entries=(np.asarray(rwid, np.int32), offsets))


def build_rstile(a: CsrMatrix, plan: PartitionPlan) -> RsTileMatrix:
    """tile.py:102-166: materialise the format for a matrix under a partition plan."""
    return tile_from_device(build_rstile_device(a, plan))


__all__ = ["FormatError", "TcPart", "ResidualPart", "RsTileMatrix", "build_rstile",
           "build_rstile_device", "tile_from_device", "tile_to_device"]
