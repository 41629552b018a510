"""CPU: pin the oracle (oracle/, test infrastructure) to the reference's own outputs.

Every digest in tests/golden/formats.json and every known answer in known_answers.json was
produced by running the reference rstile 0.1.0 (tests/golden/make_golden.py).  The oracle must
reproduce all of them bit-exactly before it is trusted as the GPU checker.
"""

from __future__ import annotations

import json
import os

import numpy as np
import pytest

import oracle as O
from rsh_testlib import GOLDEN, digest


def test_generated_inputs_match_reference_inputs(golden_corpus):
    for name, (a, entry) in golden_corpus.items():
        got = digest(np.array([a.n_rows, a.n_cols]), a.row_ptr, a.col_idx, a.values)
        assert got == entry["input"], name


def _record(t: O.Tile, windows, residual, smap) -> dict:
    wins = np.array(windows, dtype=np.int64).reshape(-1, 2)
    import hashlib
    sm = sorted((int(k), [list(s) for s in v]) for k, v in smap.items())
    return {
        "windows": digest(wins), "residual": digest(np.asarray(residual, np.int64)),
        "split_map": hashlib.sha256(json.dumps(sm).encode()).hexdigest(),
        "n_windows": len(windows), "n_residual": int(len(residual)),
        "n_entries": int(t.row_window_id.size), "n_blocks": int(t.bitmaps.size),
        "window_size": t.window_size,
        "arrays": {k: digest(getattr(t, k)) for k in O.Tile.ARRAYS},
    }


def test_oracle_formats_match_reference_digests(golden_corpus, golden_formats):
    checked = 0
    for name, (a, entry) in golden_corpus.items():
        c = O.Csr.of(a)
        for pname, want in entry["formats"].items():
            p = golden_formats["param_sets"][pname]
            windows, residual = O.partition(c, p.get("window_size", 8), p.get("tau_nnz"), p.get("tau_inc"))
            smap = O.split_map(c, windows, p.get("max_blocks_per_item", 64), p.get("split_on_row_nnz", False))
            t = O.build(c, windows, residual, smap)
            got = _record(t, windows, residual, smap)
            assert got == want, (name, pname, [k for k in want if got.get(k) != want[k]])
            checked += 1
    assert checked > 300


def test_oracle_known_answers(known_answers):
    from paper_2603_08734_b200.core import CsrMatrix
    for name, case in known_answers.items():
        if "tc" not in case:
            continue
        a = O.Csr.of(CsrMatrix.from_dense(np.asarray(case["dense"], np.float32)))
        p = case["params"]
        t = O.build_format(a, p.get("window_size", 8), p.get("tau_nnz"), p.get("tau_inc"),
                           p.get("max_blocks_per_item", 64))
        assert t.row_window_id.tolist() == case["tc"]["row_window_id"], name
        assert t.row_window_offset.tolist() == case["tc"]["row_window_offset"], name
        assert [str(int(x)) for x in t.bitmaps] == case["tc"]["bitmaps"], name
        assert t.col_id.tolist() == case["tc"]["col_id"], name
        assert t.values.tolist() == case["tc"]["values"], name
        assert t.res_row_id.tolist() == case["residual_rows"], name
        if "c_f64" in case:
            c32, _ = O.spmm_f64(a, np.asarray(case["b"], np.float32))
            assert O.max_relative_error(c32, case["c_f64"]) == 0.0, name


def test_oracle_thresholds_and_increments(known_answers):
    from paper_2603_08734_b200.core import CsrMatrix
    for n, z, want in known_answers["thresholds"]["cases"]:
        assert list(O.thresholds(n, z)) == want
    for c in known_answers["column_increment"]["cases"]:
        a = O.Csr.of(CsrMatrix.from_dense(np.asarray(c["dense"], np.float32)))
        assert O.column_increment(a, c["r"], c["w"]) == c["delta"]


def test_oracle_spmm_matches_reference_oracle(small_corpus):
    ref = np.load(os.path.join(GOLDEN, "small_spmm.npz"))
    for i, a in enumerate(small_corpus):
        b = np.random.default_rng(a.nnz).uniform(-1, 1, (a.n_cols, 16)).astype(np.float32)
        c32, c64 = O.spmm_f64(O.Csr.of(a), b)
        assert O.max_relative_error(c32, ref[f"c{i:02d}"]) <= 1e-7
        assert O.rel_frobenius(ref[f"c{i:02d}"], c64) <= 1e-7


def test_oracle_round_trip(small_corpus):
    for a in small_corpus:
        for kw in ({}, {"max_blocks_per_item": 2}, {"tau_nnz": 0}):
            c = O.Csr.of(a)
            back = O.decode(O.build_format(c, **kw))
            assert np.array_equal(back.row_ptr, c.row_ptr)
            assert np.array_equal(back.col_idx, c.col_idx)
            assert np.array_equal(back.values, c.values)


def test_port_executor_matches_oracle(small_corpus):
    """The numpy restatement of the reference executor (the reference arm in bench.py) agrees
    with the f64 oracle at the reference's own 1e-5 gate on the small corpus."""
    for a in small_corpus:
        c = O.Csr.of(a)
        t = O.build_format(c)
        b = np.random.default_rng(7).uniform(-1, 1, (a.n_cols, 8)).astype(np.float32)
        got = O.port_hybrid_spmm(t, b)
        got4 = O.port_hybrid_spmm(t, b, num_workers=4)
        ref, _ = O.spmm_f64(c, b)
        assert O.max_relative_error(got, ref) <= 1e-5
        assert got.tobytes() == got4.tobytes()


@pytest.mark.parametrize("name,expect", [("uniform4k", (512, 0, 20451)), ])
def test_config1_routing_matches_survey(name, expect):
    """config 1 -> 512 windows, 0 residual, 20,451 blocks (reference output)."""
    from paper_2603_08734_b200 import synth
    a = O.Csr.of(synth.workload_matrix(name))
    t = O.build_format(a)
    assert (t.row_window_id.size, t.res_row_id.size, t.bitmaps.size) == expect


def test_oracle_decode_matches_reference_validate_cases():
    """The oracle decode reproduces the reference's decode of every valid golden format
    (tests/golden/validate_cases.*, made by running the reference)."""
    with open(os.path.join(GOLDEN, "validate_cases.json")) as fh:
        cases = json.load(fh)
    arrs = np.load(os.path.join(GOLDEN, "validate_cases.npz"))
    n_ok = 0
    for rec in cases:
        if "csr" not in rec["decode"]:
            continue
        k = rec["case"]
        t = O.Tile(rec["n_rows"], rec["n_cols"],
                   *(arrs[f"{k}/tc.{f}"] for f in ("row_window_id", "row_window_offset", "bitmaps", "col_id",
                                                    "values")),
                   *(arrs[f"{k}/residual.{f}"] for f in ("row_id", "row_nnz_offset", "col_id", "values")),
                   rec["window_size"])
        d = O.decode(t)
        assert digest(np.array([d.n_rows, d.n_cols]), d.row_ptr, d.col_idx.astype(np.int32),
                      d.values) == rec["decode"]["csr"], k
        n_ok += 1
    assert n_ok >= 7
