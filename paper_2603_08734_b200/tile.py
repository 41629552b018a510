"""RS-Tile format (rstile tile.py) -- same host dataclasses, built on device.

``build_rstile(a, plan)`` mirrors tile.py:102-166: it checks the plan (ValueError on a
mismatch), then the bitmap blocks, padded col_id, bit-ordered values, entry arrays and the
residual part are produced by the sm_100a builder (csrc/builder.cu) and copied back into the
reference's TcPart / ResidualPart / RsTileMatrix types, bit-exact with the reference.
"""

from __future__ import annotations

import struct
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


# ---------------------------------------------------------------------------------------------
# validation and decoding (tile.py:176-307).  The structural facts are computed on device by
# rsh_validate (csrc/tile_ops.cu); this host side only turns them into the reference's messages,
# in the reference's order, including its two early returns and its two "only when clean" checks.
# ---------------------------------------------------------------------------------------------

# report slots, csrc/tile_ops.cu enum Rep
(_OFF0, _OFF_LAST, _OFF_NONMONO, _COL_MIN, _COL_MAX, _RWID_MIN, _RWID_MAX, _POP_SUM, _POP_OVER,
 _BIT_BEYOND, _ROFF0, _ROFF_LAST, _ROFF_NONMONO, _RROW_NONINC, _RROW_MIN, _RROW_MAX, _RCOL_MIN,
 _RCOL_MAX, _RES_IN_WINDOW, _DUP_HEAD, _N_SLOTS) = range(21)
_NONE = np.iinfo(np.int64).max


def _report(t, res_ok: bool, check_bits: bool, check_cover: bool) -> np.ndarray:
    import torch
    from ._lib import call, lib
    from .device import _ptr, _stream, _ws
    dev = t.device
    if lib().rsh_report_slots() != _N_SLOTS:
        raise RuntimeError("librsh.so report layout does not match this package")
    rep = torch.empty(_N_SLOTS, dtype=torch.int64, device=dev)
    if res_ok:
        rr, ro, rc, n_res, n_rc = t.res_row_id, t.res_offset, t.res_col_id, t.n_res, t.res_col_id.numel()
    else:  # the reference stops before the residual checks; give the kernel an empty residual part
        ro = torch.zeros(1, dtype=torch.int64, device=dev)
        rr, rc, n_res, n_rc = None, None, 0, 0
    nbytes = lib().rsh_validate_workspace(t.n_rows, t.n_entries, t.n_blocks)
    ws = _ws(nbytes, dev)
    call("rsh_validate", t.n_rows, t.n_cols, t.window_size, _ptr(t.row_window_id), _ptr(t.row_window_offset),
         t.n_entries, _ptr(t.bitmaps), _ptr(t.col_id), t.col_id.numel(), t.n_blocks, t.values.numel(),
         _ptr(rr), _ptr(ro), n_res, _ptr(rc), n_rc, int(check_bits), int(check_cover), _ptr(rep), _ptr(ws),
         nbytes, _stream())
    return rep.cpu().numpy()


def structural_issues(t) -> list[str]:
    """The subset of validate_rstile's checks the SpMM kernels rely on for memory safety (array
    lengths, offsets monotone and in bounds, row / column ids in range, popcount sum = value
    count).  One device pass; the schedule build refuses a format that fails any of them (the
    reference executor would raise IndexError / FormatError or read garbage from numpy arrays
    on such input, never write out of bounds)."""
    E, nb, R = t.n_entries, t.n_blocks, t.n_res
    if not (1 <= t.window_size <= 8):
        return [f"window_size {t.window_size} outside 1..8"]
    if t.row_window_offset.numel() != E + 1:
        return ["row_window_offset length must be entries + 1"]
    if t.res_offset.numel() != R + 1:
        return ["residual offset length must be rows + 1"]
    if t.col_id.numel() != nb * 8:
        return ["col_id length must be 8 per block"]
    r = _report(t, True, False, False)
    out: list[str] = []
    if r[_OFF0] != 0 or r[_OFF_NONMONO] != _NONE or r[_OFF_LAST] != nb:
        out.append("row_window_offset must run monotonically from 0 to the block count")
    if t.col_id.numel() and (r[_COL_MIN] < 0 or r[_COL_MAX] >= t.n_cols):
        out.append("col_id entry out of range")
    if E and (r[_RWID_MIN] < 0 or r[_RWID_MAX] >= t.n_rows):
        out.append("row_window_id out of range")
    if r[_POP_SUM] != t.values.numel():
        out.append(f"bitmap popcount sum {int(r[_POP_SUM])} does not match value count {t.values.numel()}")
    if r[_ROFF0] != 0 or r[_ROFF_NONMONO] != _NONE or r[_ROFF_LAST] != t.res_values.numel() \
            or t.res_col_id.numel() != t.res_values.numel():
        out.append("residual offsets must run monotonically from 0 to the residual entry count")
    if R and (r[_RROW_MIN] < 0 or r[_RROW_MAX] >= t.n_rows):
        out.append("residual row_id out of range")
    if t.res_col_id.numel() and (r[_RCOL_MIN] < 0 or r[_RCOL_MAX] >= t.n_cols):
        out.append("residual col_id out of range")
    if t.values.numel() >= 2 ** 31 or t.res_values.numel() >= 2 ** 31:
        out.append("more than 2^31 - 1 nonzeros in one part (int32 value offsets)")
    return out


def validate_rstile_device(t) -> list[str]:
    """tile.py:176-267 for a DeviceTile: every structural invariant, checked on device; an empty
    list means valid.  Messages and their order are the reference's."""
    issues: list[str] = []
    E, nb, R = t.n_entries, t.n_blocks, t.n_res
    n_values, n_rc = t.values.numel(), t.res_col_id.numel()
    if not (1 <= t.window_size <= 8):
        issues.append(f"window_size {t.window_size} outside 1..8")
    if t.row_window_offset.numel() != E + 1:
        issues.append("row_window_offset length must be entries + 1")
        return issues
    res_ok = t.res_offset.numel() == R + 1
    r = _report(t, res_ok, False, False)

    def tc_checks(r) -> list[str]:
        out: list[str] = []
        if r[_OFF0] != 0:
            out.append("row_window_offset must start at 0")
        if r[_OFF_NONMONO] != _NONE:
            out.append("row_window_offset not monotone")
        if r[_OFF_LAST] != nb:
            out.append("row_window_offset end does not equal block count")
        if t.col_id.numel() != nb * 8:
            out.append("col_id length must be 8 per block")
        if t.col_id.numel() and (r[_COL_MIN] < 0 or r[_COL_MAX] >= t.n_cols):
            out.append("col_id entry out of range")
        if E:
            if r[_RWID_MIN] < 0 or r[_RWID_MAX] >= t.n_rows:
                out.append("row_window_id out of range")
            if r[_DUP_HEAD] != _NONE:
                rid = int(t.row_window_id[int(r[_DUP_HEAD])].item())
                out.append(f"entries sharing row window {rid} are not consecutive segments")
        if r[_POP_SUM] != n_values:
            where = int(r[_POP_OVER]) if r[_POP_OVER] != _NONE else nb - 1
            out.append(f"bitmap popcount sum {int(r[_POP_SUM])} does not match value count "
                       f"{n_values} (first divergence at block {where})")
        return out

    def res_checks(r) -> list[str]:
        out: list[str] = []
        if r[_ROFF0] != 0:
            out.append("residual offsets must start at 0")
        if r[_ROFF_NONMONO] != _NONE:
            out.append("residual offsets not monotone")
        if r[_ROFF_LAST] != t.res_values.numel() or n_rc != t.res_values.numel():
            out.append("residual offsets do not match entry count")
        if R:
            if r[_RROW_NONINC] != _NONE:
                out.append("residual row_id not strictly increasing")
            if r[_RROW_MIN] < 0 or r[_RROW_MAX] >= t.n_rows:
                out.append("residual row_id out of range")
        if n_rc and (r[_RCOL_MIN] < 0 or r[_RCOL_MAX] >= t.n_cols):
            out.append("residual col_id out of range")
        return out

    issues += tc_checks(r)
    rest = res_checks(r) if res_ok else []
    check_bits = bool(nb) and not issues
    check_cover = res_ok and bool(R) and bool(E) and not issues and not rest
    if check_bits or check_cover:  # second pass: the checks that need a clean format
        r = _report(t, res_ok, check_bits, check_cover)
    if check_bits and r[_BIT_BEYOND] != _NONE:
        issues.append(f"block {int(r[_BIT_BEYOND])} has a bit beyond its window's last row")
    if not res_ok:
        issues.append("residual offset length must be rows + 1")
        return issues
    issues += rest
    if check_cover and not issues and r[_RES_IN_WINDOW] != _NONE:
        row = int(t.res_row_id[int(r[_RES_IN_WINDOW])].item())
        issues.append(f"residual row {row} lies inside a window's row range")
    return issues


def validate_rstile(m: RsTileMatrix) -> list[str]:
    """tile.py:176-267: check every structural invariant; an empty list means valid."""
    return validate_rstile_device(tile_to_device(m))


def decode_rstile_device(t):
    """tile.py:270-307 for a DeviceTile -> (DeviceCsr, first duplicate position or -1).  The
    format must be valid (validate_rstile_device); padding contributes nothing."""
    import torch
    from ._lib import call, lib
    from .device import DeviceCsr, _ptr, _stream, _ws
    dev = t.device
    tc_nnz, res_nnz = t.values.numel(), t.res_values.numel()
    nnz = tc_nnz + res_nnz
    rp = torch.empty(t.n_rows + 1, dtype=torch.int64, device=dev)
    ci = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
    va = torch.empty(max(nnz, 1), dtype=torch.float32, device=dev)
    dup = torch.empty(1, dtype=torch.int64, device=dev)
    nbytes = lib().rsh_decode_workspace(t.n_rows, nnz, t.n_blocks)
    ws = _ws(nbytes, dev)
    call("rsh_decode", t.n_rows, t.n_cols, _ptr(t.row_window_id), _ptr(t.row_window_offset), t.n_entries,
         _ptr(t.bitmaps), _ptr(t.col_id), _ptr(t.values), t.n_blocks, tc_nnz, _ptr(t.res_row_id),
         _ptr(t.res_offset), t.n_res, _ptr(t.res_col_id), _ptr(t.res_values), res_nnz, _ptr(rp), _ptr(ci),
         _ptr(va), _ptr(dup), _ptr(ws), nbytes, _stream())
    return DeviceCsr(t.n_rows, t.n_cols, rp, ci[:nnz], va[:nnz]), int(dup.item())


def decode_rstile(m: RsTileMatrix) -> CsrMatrix:
    """tile.py:270-307: reconstruct the original CSR exactly (decoded on device)."""
    issues = validate_rstile(m)
    if issues:
        raise FormatError(issues[0])
    d, _dup = decode_rstile_device(tile_to_device(m))
    try:  # the reference's canonical-CSR check and its message
        return CsrMatrix(m.n_rows, m.n_cols, d.row_ptr.cpu().numpy(), d.col_idx.cpu().numpy(),
                         d.values.cpu().numpy())
    except ValueError as exc:
        raise FormatError(f"decoded arrays are not canonical: {exc}") from exc


# ---------------------------------------------------------------------------------------------
# serialization (tile.py:314-388) and storage accounting (tile.py:394-440)
# ---------------------------------------------------------------------------------------------

RSTILE_MAGIC = b"RSTL"
RSTILE_VERSION = 1
# magic, version, window_size, n_rows, n_cols, entries, blocks, tc nnz, residual rows, residual nnz
_HEADER = struct.Struct("<4sHHIIIQQIQ")
HEADER_BYTES = _HEADER.size
# on-disk dtypes of the nine arrays, in file order (offsets are stored as u32)
_FILE_LAYOUT = (("tc", "row_window_id", "<u4"), ("tc", "row_window_offset", "<u4"), ("tc", "bitmaps", "<u8"),
                ("tc", "col_id", "<u4"), ("tc", "values", "<f4"), ("residual", "row_id", "<u4"),
                ("residual", "row_nnz_offset", "<u4"), ("residual", "col_id", "<u4"),
                ("residual", "values", "<f4"))


def rstile_bytes(m: RsTileMatrix) -> bytes:
    """The .rst byte image of a format (no validation): the reference's header then the nine
    arrays little-endian, offsets narrowed to u32 exactly as tile.py:318-341 writes them."""
    tc, res = m.tc, m.residual
    head = _HEADER.pack(RSTILE_MAGIC, RSTILE_VERSION, m.window_size, m.n_rows, m.n_cols, tc.n_entries,
                        tc.n_blocks, tc.values.size, res.n_rows, res.values.size)
    return head + b"".join(getattr(getattr(m, part), name).astype(dt).tobytes() for part, name, dt in _FILE_LAYOUT)


def save_rstile(path, m: RsTileMatrix) -> None:
    """tile.py:314-341: validate (on device), then write the .rst file."""
    issues = validate_rstile(m)
    if issues:
        raise FormatError(issues[0])
    with open(path, "wb") as fh:
        fh.write(rstile_bytes(m))


def save_rstile_device(path, t) -> None:
    """Serialize a DeviceTile: validated in HBM, then copied out once and written."""
    issues = validate_rstile_device(t)
    if issues:
        raise FormatError(issues[0])
    with open(path, "wb") as fh:
        fh.write(rstile_bytes(tile_from_device(t)))


def parse_rstile(blob: bytes, name: str = "<bytes>") -> RsTileMatrix:
    """The structural half of load_rstile (tile.py:344-382): header, sizes, truncation and
    trailing-byte checks, with the reference's messages.  No semantic validation."""
    if len(blob) < _HEADER.size:
        raise FormatError(f"{name}: truncated header")
    magic, version, wsize, n_rows, n_cols, entries, blocks, tc_nnz, r_rows, r_nnz = _HEADER.unpack_from(blob)
    if magic != RSTILE_MAGIC:
        raise FormatError(f"{name}: bad magic {magic!r}")
    if version != RSTILE_VERSION:
        raise FormatError(f"{name}: unsupported version {version}")
    pos = _HEADER.size
    fields = []
    for count, dt in ((entries, "<u4"), (entries + 1, "<u4"), (blocks, "<u8"), (blocks * 8, "<u4"),
                      (tc_nnz, "<f4"), (r_rows, "<u4"), (r_rows + 1, "<u4"), (r_nnz, "<u4"), (r_nnz, "<f4")):
        width = int(count) * np.dtype(dt).itemsize
        if pos + width > len(blob):
            raise FormatError(f"{name}: truncated at byte {pos}")
        fields.append(np.frombuffer(blob, dtype=dt, count=int(count), offset=pos))
        pos += width
    if pos != len(blob):
        raise FormatError(f"{name}: {len(blob) - pos} trailing bytes")
    return RsTileMatrix(n_rows, n_cols, TcPart(*fields[:5]), ResidualPart(*fields[5:]), wsize)


def load_rstile(path) -> RsTileMatrix:
    """tile.py:344-388: parse, then validate on device (FormatError with the first issue)."""
    with open(path, "rb") as fh:
        blob = fh.read()
    m = parse_rstile(blob, str(path))
    issues = validate_rstile(m)
    if issues:
        raise FormatError(f"{path}: {issues[0]}")
    return m


@dataclass(frozen=True)
class StorageReport:
    """tile.py:398-407."""

    coo_bytes: int
    csr_bytes: int
    rstile_bytes: int
    tc_bytes: int
    residual_bytes: int
    bitmap_bytes: int
    colid_bytes: int
    offset_bytes: int


def storage_report(a: CsrMatrix, m: RsTileMatrix) -> StorageReport:
    """tile.py:410-440: byte counts under 32-bit indices, 32-bit values, 64-bit bitmaps; the
    .rst file is exactly HEADER_BYTES + rstile_bytes."""
    entries, blocks = m.tc.n_entries, m.tc.n_blocks
    r_rows, r_nnz = m.residual.n_rows, int(m.residual.values.size)
    bitmap_bytes, colid_bytes, offset_bytes = blocks * 8, blocks * 32, (entries + 1) * 4
    tc_bytes = entries * 4 + offset_bytes + bitmap_bytes + colid_bytes + int(m.tc.values.size) * 4
    residual_bytes = r_rows * 4 + r_nnz * 8 + (r_rows + 1) * 4
    return StorageReport(coo_bytes=a.nnz * 12, csr_bytes=a.nnz * 8 + (a.n_rows + 1) * 4,
                         rstile_bytes=tc_bytes + residual_bytes, tc_bytes=tc_bytes, residual_bytes=residual_bytes,
                         bitmap_bytes=bitmap_bytes, colid_bytes=colid_bytes, offset_bytes=offset_bytes)


__all__ = ["FormatError", "HEADER_BYTES", "RSTILE_MAGIC", "RSTILE_VERSION", "ResidualPart", "RsTileMatrix",
           "StorageReport", "TcPart", "build_rstile", "build_rstile_device", "decode_rstile", "decode_rstile_device",
           "load_rstile", "parse_rstile", "rstile_bytes", "save_rstile", "save_rstile_device", "storage_report",
           "tile_from_device", "tile_to_device", "validate_rstile", "validate_rstile_device"]
