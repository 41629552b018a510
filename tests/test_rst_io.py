""".rst serialization (reference tile.py:314-388) and storage accounting (tile.py:410-440).

tests/golden/rst_cases.json holds the SHA-256 of the files the REFERENCE's save_rstile wrote
for seeded formats (make_rst_golden.py).  CPU: the byte image of the oracle-built format (the
oracle is pinned bit-exact to the reference's builder) matches those digests, and parsing
round-trips.  GPU: the product path (device build -> device validate -> save) writes the same
bytes and load_rstile reads them back; the reference's structural errors keep their messages.
"""

from __future__ import annotations

import dataclasses
import hashlib
import json
import os

import numpy as np
import pytest

from rsh_testlib import GOLDEN, corpus_matrix


def _cases():
    with open(os.path.join(GOLDEN, "rst_cases.json")) as fh:
        return json.load(fh)


def _oracle_matrix(rec):
    import oracle as O
    from paper_2603_08734_b200.tile import ResidualPart, RsTileMatrix, TcPart
    a = corpus_matrix(rec["recipe"])
    t = O.build_format(O.Csr.of(a), **rec["params"])
    m = RsTileMatrix(t.n_rows, t.n_cols, TcPart(t.row_window_id, t.row_window_offset, t.bitmaps, t.col_id, t.values),
                     ResidualPart(t.res_row_id, t.res_offset, t.res_col_id, t.res_values), t.window_size)
    return a, m


def test_header_size():
    from paper_2603_08734_b200 import HEADER_BYTES
    assert HEADER_BYTES == _cases()["header_bytes"] == 48


@pytest.mark.parametrize("rec", _cases()["cases"], ids=lambda r: r["case"])
def test_byte_image_matches_reference(rec):
    from paper_2603_08734_b200 import storage_report
    from paper_2603_08734_b200.tile import HEADER_BYTES, parse_rstile, rstile_bytes
    a, m = _oracle_matrix(rec)
    blob = rstile_bytes(m)
    assert hashlib.sha256(blob).hexdigest() == rec["sha256"]
    rep = storage_report(a, m)
    assert dataclasses.asdict(rep) == rec["storage"]
    assert len(blob) == HEADER_BYTES + rep.rstile_bytes  # test_acceptance.py:281
    back = parse_rstile(blob)
    assert rstile_bytes(back) == blob


def test_structural_errors_keep_reference_messages():
    from paper_2603_08734_b200 import FormatError
    from paper_2603_08734_b200.tile import parse_rstile, rstile_bytes
    _, m = _oracle_matrix(_cases()["cases"][5])
    blob = rstile_bytes(m)
    with pytest.raises(FormatError, match="truncated header"):
        parse_rstile(blob[:20], "f")
    with pytest.raises(FormatError, match="bad magic"):
        parse_rstile(b"XXXX" + blob[4:], "f")
    with pytest.raises(FormatError, match="unsupported version 2"):
        parse_rstile(blob[:4] + (2).to_bytes(2, "little") + blob[6:], "f")
    with pytest.raises(FormatError, match="truncated at byte"):
        parse_rstile(blob[:-3], "f")
    with pytest.raises(FormatError, match="3 trailing bytes"):
        parse_rstile(blob + b"abc", "f")


@pytest.mark.gpu
@pytest.mark.parametrize("rec", _cases()["cases"], ids=lambda r: r["case"])
def test_save_load_on_device(rec, tmp_path):
    from paper_2603_08734_b200 import (PartitionParams, build_rstile, load_rstile, partition_rows, save_rstile,
                                       split_long_work)
    from paper_2603_08734_b200.device import DeviceCsr, build_device
    from paper_2603_08734_b200.tile import rstile_bytes, save_rstile_device
    a = corpus_matrix(rec["recipe"])
    p = PartitionParams(**rec["params"])
    m = build_rstile(a, split_long_work(a, partition_rows(a, p), p))
    path = tmp_path / "m.rst"
    save_rstile(path, m)
    assert hashlib.sha256(path.read_bytes()).hexdigest() == rec["sha256"]
    back = load_rstile(path)
    assert rstile_bytes(back) == path.read_bytes()
    # straight from HBM: device build -> device validate -> one copy out
    kw = {k: v for k, v in rec["params"].items()}
    t = build_device(DeviceCsr.from_host(a), **kw)
    save_rstile_device(tmp_path / "d.rst", t)
    assert (tmp_path / "d.rst").read_bytes() == path.read_bytes()


@pytest.mark.gpu
def test_load_rejects_invalid_format(tmp_path):
    from paper_2603_08734_b200 import FormatError, load_rstile
    from paper_2603_08734_b200.tile import RsTileMatrix, TcPart, rstile_bytes
    _, m = _oracle_matrix(_cases()["cases"][6])
    bad = np.array(m.tc.col_id)
    bad[0] = m.n_cols + 5  # out-of-range column (tile.py:229-231)
    mm = RsTileMatrix(m.n_rows, m.n_cols, TcPart(m.tc.row_window_id, m.tc.row_window_offset, m.tc.bitmaps, bad,
                                                 m.tc.values), m.residual, m.window_size)
    path = tmp_path / "bad.rst"
    path.write_bytes(rstile_bytes(mm))
    with pytest.raises(FormatError, match=str(path)):
        load_rstile(path)
