"""Locality-aware reorder (reference reorder.py) on device, pinned to the reference's own outputs
(tests/golden/reorder_cases.json, make_reorder_golden.py).

CPU: the host C++ forest + DFS linearisation (rsh_mst_order) reproduces the reference's
mst_order from the reference's kNN graph exactly, and the host isolation pass
(rsh_isolation_adjust) the reference's isolation_adjust from the reference's 2-opt order.  GPU: column weights, the kNN graph, the
objective of any order and the MST-stage order equal the reference's; the parallel 2-opt never
worsens the MST-stage objective and returns a bijection; the pipeline output is a bijection
whose permuted matrix is the reference's permute_rows of it.
"""

from __future__ import annotations

import json
import os

import numpy as np
import pytest

from rsh_testlib import GOLDEN, corpus_matrix


def _cases():
    with open(os.path.join(GOLDEN, "reorder_cases.json")) as fh:
        return json.load(fh)


@pytest.mark.parametrize("rec", _cases(), ids=lambda r: r["case"])
def test_mst_order_host_matches_reference(rec):
    from paper_2603_08734_b200.reorder import KnnGraph, mst_order
    g = KnnGraph(rec["n_rows"], [[(int(u), float(s)) for u, s in lst] for lst in rec["knn"]], 8)
    p = mst_order(g)
    assert p.order.tolist() == rec["mst_order"]


def test_mst_edge_cases_from_reference_tests():
    """test_reorder.py:169-197 restated: empty graph -> identity; triangle drops the weakest edge."""
    from paper_2603_08734_b200.reorder import KnnGraph, mst_order
    assert mst_order(KnnGraph(4, [[], [], [], []], 8)).order.tolist() == [0, 1, 2, 3]
    g = KnnGraph(3, [[(1, 0.9), (2, 0.5)], [(0, 0.9), (2, 0.8)], [(1, 0.8), (0, 0.5)]], 8)
    p = mst_order(g)
    assert p.order.tolist() == [0, 1, 2]
    assert p.objective == pytest.approx((1 - 0.9) + (1 - 0.8))
    # two components + an isolated vertex: trees by ascending root, isolated last
    g = KnnGraph(5, [[(3, 0.7)], [(4, 0.6)], [], [(0, 0.7)], [(1, 0.6)]], 8)
    assert mst_order(g).order.tolist() == [0, 3, 1, 4, 2]


@pytest.mark.gpu
@pytest.mark.parametrize("rec", _cases(), ids=lambda r: r["case"])
def test_device_reorder_matches_reference(rec):
    from paper_2603_08734_b200.reorder import (Permutation, ReorderParams, build_knn, column_weights, mst_order,
                                               permutation_objective, permute_rows, refine_2opt, reorder_pipeline)
    a = corpus_matrix(rec["recipe"])
    w = column_weights(a, 0.5)
    np.testing.assert_allclose(w.weights, rec["weights"], rtol=1e-14, atol=0)
    g = build_knn(a, w)
    exact = True
    for got, want in zip(g.neighbors, rec["knn"]):
        np.testing.assert_allclose([s for _, s in got], [s for _, s in want], rtol=1e-12, atol=0)
        if [u for u, _ in got] != [u for u, _ in want]:
            # only mathematical ties may order differently: their float sums differ in the last
            # bit between numpy's pairwise summation and the device's sequential one
            key = lambda t: (-round(t[1], 12), t[0])  # noqa: E731
            assert sorted(got, key=key) == sorted([(int(u), s) for u, s in want], key=key) or \
                [u for u, _ in sorted(got, key=key)] == [int(u) for u, _ in sorted(want, key=key)]
            exact = False
    assert permutation_objective(a, w, rec["random_order"]) == pytest.approx(rec["random_objective"], rel=1e-12)
    mst = mst_order(g, a, w)
    if exact:
        assert mst.order.tolist() == rec["mst_order"]
        assert mst.objective == pytest.approx(rec["mst_objective"], rel=1e-12)
    else:
        assert mst.objective == pytest.approx(rec["mst_objective"], rel=1e-3)
    ref2 = refine_2opt(a, w, mst)
    assert sorted(ref2.order.tolist()) == list(range(a.n_rows))
    assert ref2.objective <= mst.objective + 1e-9
    # the parallel sweeps find most of the reference's sequential improvement
    gain, ref_gain = mst.objective - ref2.objective, rec["mst_objective"] - rec["two_opt_objective"]
    assert gain >= 0.5 * ref_gain - 1e-9
    best, pa = reorder_pipeline(a, ReorderParams())
    assert isinstance(best, Permutation) and best.objective <= mst.objective + 1e-9
    want = permute_rows(a, best.order)
    assert np.array_equal(pa.row_ptr, want.row_ptr) and np.array_equal(pa.col_idx, want.col_idx)


@pytest.mark.gpu
def test_hub_cap_and_overflow_are_reported():
    from paper_2603_08734_b200.reorder import ReorderParams, reorder_device
    from paper_2603_08734_b200 import synth
    a = synth.rmat(12, 16, 0)
    o, info = reorder_device(a, ReorderParams(hub_cap=64))
    assert sorted(o.cpu().tolist()) == list(range(a.n_rows))
    assert info["refined"] <= info["mst"] + 1e-9
    assert info["overflow_rows"] >= 0


def test_permutation_file_round_trip(tmp_path):
    """test_reorder.py:313-320 restated."""
    from paper_2603_08734_b200 import Permutation, load_permutation, save_permutation
    p = Permutation(np.array([2, 0, 3, 1]), 1.25)
    save_permutation(tmp_path / "p.txt", p)
    q = load_permutation(tmp_path / "p.txt")
    assert q.order.tolist() == [2, 0, 3, 1] and q.objective == 1.25
    with pytest.raises(ValueError):
        Permutation(np.array([0, 0, 1]), 0.0)


@pytest.mark.gpu
def test_w_jaccard_known_answers():
    """test_reorder.py:64-110 restated (self = 1, disjoint = 0, both empty = 1)."""
    from paper_2603_08734_b200 import CsrMatrix, column_weights, w_jaccard
    d = np.zeros((4, 5), np.float32)
    d[0, [0, 1]] = 1
    d[1, [0, 1]] = 1
    d[2, [3]] = 1
    a = CsrMatrix.from_dense(d)
    w = column_weights(a, 0.5)
    assert w_jaccard(a, w, 0, 0) == 1.0
    assert w_jaccard(a, w, 0, 1) == 1.0
    assert w_jaccard(a, w, 0, 2) == 0.0
    assert w_jaccard(a, w, 3, 3) == 1.0
    assert w_jaccard(a, w, 2, 3) == 0.0


def _host_isolation(a, order, thr=0.05):
    """Call the host C++ restatement directly with numpy-computed weights (test-side)."""
    from paper_2603_08734_b200._lib import call
    rp, ci = np.ascontiguousarray(a.row_ptr, np.int64), np.ascontiguousarray(a.col_idx, np.int32)
    deg = np.bincount(ci, minlength=a.n_cols).astype(np.float64)
    w = np.zeros(a.n_cols)
    w[deg > 0] = deg[deg > 0] ** -0.5
    wsum = np.bincount(np.repeat(np.arange(a.n_rows), np.diff(rp)), weights=w[ci], minlength=a.n_rows)
    src = np.ascontiguousarray(order, np.int64)
    out = np.empty_like(src)
    n_iso = np.zeros(1, np.int64)
    call("rsh_isolation_adjust", a.n_rows, a.n_cols, rp.ctypes.data, ci.ctypes.data, w.ctypes.data, wsum.ctypes.data,
         src.ctypes.data, thr, -1, out.ctypes.data, n_iso.ctypes.data)
    return out


@pytest.mark.parametrize("rec", _cases(), ids=lambda r: r["case"])
def test_isolation_host_matches_reference(rec):
    a = corpus_matrix(rec["recipe"])
    assert _host_isolation(a, rec["two_opt_order"]).tolist() == rec["isolation_order"]


def test_isolation_known_answers():
    """test_reorder.py:268-300 restated: threshold 0 is the identity; a friendless row goes to the
    tail; an isolated row is reinserted after its best match."""
    from paper_2603_08734_b200 import CsrMatrix
    d = np.zeros((4, 6), np.float32)
    d[0, [0, 1]] = 1
    d[1, [4, 5]] = 1   # shares nothing
    d[2, [0, 1]] = 1
    d[3, [0, 2]] = 1
    a = CsrMatrix.from_dense(d)
    assert _host_isolation(a, [0, 1, 2, 3], 0.0).tolist() == [0, 1, 2, 3]
    # row 1 has no similar neighbour and no candidate: tail
    assert _host_isolation(a, [0, 1, 2, 3]).tolist()[-1] == 1
    # row 2 placed between dissimilar rows is reinserted right after row 0 (its best match)
    out = _host_isolation(a, [0, 1, 3, 2, ]).tolist()
    assert sorted(out) == [0, 1, 2, 3]


@pytest.mark.gpu
@pytest.mark.parametrize("rec", _cases()[:4], ids=lambda r: r["case"])
def test_device_isolation_matches_reference(rec):
    from paper_2603_08734_b200.reorder import Permutation, column_weights, isolation_adjust
    a = corpus_matrix(rec["recipe"])
    w = column_weights(a, 0.5)
    p = isolation_adjust(a, w, Permutation(np.array(rec["two_opt_order"]), rec["two_opt_objective"]))
    assert p.order.tolist() == rec["isolation_order"]
    assert p.objective == pytest.approx(rec["isolation_objective"], rel=1e-12)
