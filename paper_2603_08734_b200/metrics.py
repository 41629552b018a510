"""Structure metrics of the RS-Tile format (rstile metrics.py:28-88) computed on device.

``tile_density`` counts real nonzeros only (padding slots never contribute), treats a window
split into segments as one window, and takes row fractions relative to rows holding at least one
nonzero (metrics.py:28-63).  ``threshold_sweep`` rebuilds the format on device once per
row-nnz threshold (metrics.py:66-78).  Window and occupied-row counts come from
``rsh_tile_density`` (csrc/tile_ops.cu); the rest are array sizes.
"""

from __future__ import annotations

from dataclasses import dataclass, replace

from .core import CsrMatrix
from .partition import PartitionParams

SWEEP_CSV_HEADER = "tau,mean_nnz_per_block,mean_nnz_per_window,residual_nnz_fraction"


@dataclass(frozen=True)
class TileDensityReport:
    """metrics.py:18-25."""

    mean_nnz_per_block: float
    mean_nnz_per_window: float
    block_count: int
    window_count: int
    residual_nnz_fraction: float
    residual_row_fraction: float


def tile_density_device(t) -> TileDensityReport:
    """tile_density of a DeviceTile (device.py)."""
    import torch

    from ._lib import call
    from .device import _ptr, _stream
    out = torch.zeros(2, dtype=torch.int64, device=t.device)
    call("rsh_tile_density", _ptr(t.row_window_id), _ptr(t.row_window_offset), t.n_entries, _ptr(t.bitmaps),
         _ptr(out), _stream())
    window_count, occupied_rows = (int(x) for x in out.cpu().tolist())
    tc_nnz = int(t.values.numel())
    res_nnz = int(t.res_values.numel())
    total = tc_nnz + res_nnz
    nonzero_rows = occupied_rows + t.n_res
    n_blocks = t.n_blocks
    return TileDensityReport(
        mean_nnz_per_block=tc_nnz / n_blocks if n_blocks else 0.0,
        mean_nnz_per_window=tc_nnz / window_count if window_count else 0.0,
        block_count=n_blocks,
        window_count=window_count,
        residual_nnz_fraction=res_nnz / total if total else 0.0,
        residual_row_fraction=t.n_res / nonzero_rows if nonzero_rows else 0.0,
    )


def tile_density(m) -> TileDensityReport:
    """metrics.py:28-63: density of an RsTileMatrix (uploaded) or a DeviceTile."""
    from .device import DeviceTile
    if isinstance(m, DeviceTile):
        return tile_density_device(m)
    from .tile import tile_to_device
    return tile_density_device(tile_to_device(m))


def threshold_sweep(a: CsrMatrix, tau_values: list[int], p: PartitionParams | None = None) -> list:
    """metrics.py:66-78: the format rebuilt (on device) once per row-nnz threshold tau, with its
    density report: [(tau, TileDensityReport), ...]."""
    if not tau_values:
        raise ValueError("tau_values must be non-empty")
    from .device import DeviceCsr, build_device
    from .partition import resolve_thresholds
    p = p or PartitionParams()
    d = DeviceCsr.from_host(a)
    out = []
    for tau in tau_values:
        params = replace(p, tau_nnz=int(tau))
        tn, ti = resolve_thresholds(a, params)
        t = build_device(d, window_size=params.window_size, tau_nnz=tn, tau_inc=ti,
                         max_blocks_per_item=params.max_blocks_per_item, split_on_row_nnz=params.split_on_row_nnz,
                         split_factor=params.split_factor)
        out.append((int(tau), tile_density_device(t)))
    return out


def sweep_csv(rows: list) -> str:
    """metrics.py:81-88."""
    lines = [SWEEP_CSV_HEADER]
    for tau, rep in rows:
        lines.append(f"{tau},{rep.mean_nnz_per_block!r},{rep.mean_nnz_per_window!r},{rep.residual_nnz_fraction!r}")
    return "\n".join(lines) + "\n"
