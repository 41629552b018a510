"""validate_rstile / decode_rstile on device (csrc/tile_ops.cu) against the reference.

The golden cases (tests/golden/make_validate_golden.py) hold reference-built formats with one
tampering each and the REFERENCE's full issue list and decode outcome (tile.py:176-307); the
device path must reproduce both exactly.  At full size the round trip decode(build(A)) == A is
the size-independent property (reference test_tile.py:118-153).
"""

from __future__ import annotations

import dataclasses
import json
import os

import numpy as np
import pytest

from rsh_testlib import GOLDEN, digest

pytestmark = pytest.mark.gpu


def _cases():
    with open(os.path.join(GOLDEN, "validate_cases.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="module")
def arrays():
    return np.load(os.path.join(GOLDEN, "validate_cases.npz"))


def _matrix(rec, arrays):
    from paper_2603_08734_b200.tile import ResidualPart, RsTileMatrix, TcPart
    k = rec["case"]
    tc = TcPart(*(arrays[f"{k}/tc.{f}"] for f in ("row_window_id", "row_window_offset", "bitmaps", "col_id",
                                                  "values")))
    res = ResidualPart(*(arrays[f"{k}/residual.{f}"] for f in ("row_id", "row_nnz_offset", "col_id", "values")))
    return RsTileMatrix(rec["n_rows"], rec["n_cols"], tc, res, rec["window_size"])


@pytest.mark.parametrize("rec", _cases(), ids=lambda r: r["case"])
def test_validate_and_decode_match_reference(rec, arrays):
    from paper_2603_08734_b200 import FormatError, decode_rstile, validate_rstile
    m = _matrix(rec, arrays)
    assert validate_rstile(m) == rec["issues"]
    if "error" in rec["decode"]:
        with pytest.raises(FormatError) as ei:
            decode_rstile(m)
        assert str(ei.value) == rec["decode"]["error"]
    else:
        d = decode_rstile(m)
        got = digest(np.array([d.n_rows, d.n_cols]), d.row_ptr, d.col_idx, d.values)
        assert got == rec["decode"]["csr"]


def test_reference_tamper_tests():
    """test_tile.py:165-214 restated on the product types."""
    from paper_2603_08734_b200 import (CsrMatrix, PartitionParams, build_rstile, partition_rows,
                                       split_long_work, validate_rstile)

    def build(a, p=None):
        p = p or PartitionParams()
        return build_rstile(a, split_long_work(a, partition_rows(a, p), p))

    def tamper(m, part, mutate):
        arrs = {f.name: np.array(getattr(getattr(m, part), f.name)) for f in dataclasses.fields(getattr(m, part))}
        mutate(arrs)
        return dataclasses.replace(m, **{part: type(getattr(m, part))(**arrs)})

    force_tc = PartitionParams(tau_nnz=0)
    m = build(CsrMatrix.from_dense(np.ones((8, 8), np.float32)), force_tc)
    issues = validate_rstile(tamper(m, "tc", lambda a: a["bitmaps"].__setitem__(0, a["bitmaps"][0] & np.uint64(
        0xFFFFFFFFFFFFFFFE))))
    assert any("block 0" in s for s in issues)
    m = build(CsrMatrix.from_dense(np.eye(16, dtype=np.float32)))

    def swap(a):
        a["row_nnz_offset"][1], a["row_nnz_offset"][2] = 2, 1
    assert any("monotone" in s or "offset" in s for s in validate_rstile(tamper(m, "residual", swap)))

    def scramble(a):
        a["row_id"][0], a["row_id"][1] = a["row_id"][1], a["row_id"][0]
    assert validate_rstile(tamper(m, "residual", scramble)) != []
    m = build(CsrMatrix.from_dense(np.asarray([[1.0, 2.0]], np.float32)), force_tc)
    assert validate_rstile(tamper(m, "tc", lambda a: a["col_id"].__setitem__(0, 99))) != []


@pytest.mark.parametrize("kw", [{}, {"max_blocks_per_item": 2}, {"window_size": 5}, {"tau_nnz": 0}])
def test_round_trip_small_corpus(kw):
    from paper_2603_08734_b200 import (PartitionParams, build_rstile, csr_equal, decode_rstile,
                                       partition_rows, split_long_work, validate_rstile)
    from paper_2603_08734_b200 import synth
    from oracle import corpus  # noqa: E402
    p = PartitionParams(**kw)
    for a in corpus.small_corpus():
        m = build_rstile(a, split_long_work(a, partition_rows(a, p), p))
        assert validate_rstile(m) == []
        assert csr_equal(decode_rstile(m), a)


@pytest.mark.parametrize("name", ["uniform4k", "rmat1m", "stencil2m"])
def test_round_trip_full_size_on_device(name):
    """decode(build(A)) == A bit-exactly at the benchmark sizes, device resident throughout."""
    import torch
    from paper_2603_08734_b200 import synth
    from oracle import corpus  # noqa: E402
    from paper_2603_08734_b200.device import DeviceCsr, build_device
    from paper_2603_08734_b200.tile import decode_rstile_device, validate_rstile_device
    a = synth.workload_matrix(name)
    d = DeviceCsr.from_host(a)
    t = build_device(d)
    assert validate_rstile_device(t) == []
    out, dup = decode_rstile_device(t)
    assert dup == -1
    assert torch.equal(out.row_ptr, d.row_ptr)
    assert torch.equal(out.col_idx, d.col_idx)
    assert torch.equal(out.values.view(torch.int32), d.values.view(torch.int32))
