"""GPU: drop-in API functions beyond the SpMM path -- oracle_spmm (core.py:380-395),
build_candidates (reorder.py:168-194), tile_density / threshold_sweep / sweep_csv
(metrics.py:28-88) -- against fixtures the reference itself produced
(tests/golden/make_api_golden.py) and the reference tests' known answers."""

from __future__ import annotations

import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2603_08734_b200")
torch = pytest.importorskip("torch")

from rsh_testlib import corpus_matrix  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def api_cases(small_corpus):
    with open(os.path.join(HERE, "golden", "api_cases.json")) as fh:
        cases = json.load(fh)
    arrays = np.load(os.path.join(HERE, "golden", "api_oracle.npz"))
    return [(c, corpus_matrix(c["recipe"], small_corpus), arrays[c["name"] + "_b"], arrays[c["name"] + "_c"])
            for c in cases]


def test_oracle_spmm_matches_reference_outputs(api_cases):
    for case, a, b, ref in api_cases:
        c = P.oracle_spmm(a, P.DenseMatrix.from_array(b)).data
        # f64 accumulation in CSR order vs the reference's BLAS dot: at most one f32 ulp apart
        assert np.all(np.abs(c - ref) <= np.spacing(np.abs(ref))), case["name"]


def test_oracle_spmm_known_answers():
    # test_core.py:191-233
    eye = P.CsrMatrix.from_dense(np.eye(4, dtype=np.float32))
    b = P.DenseMatrix.from_array(np.arange(8, dtype=np.float32).reshape(4, 2))
    assert np.array_equal(P.oracle_spmm(eye, b).data, b.data)
    z = P.CsrMatrix.from_dense(np.zeros((3, 4), np.float32))
    assert np.array_equal(P.oracle_spmm(z, b).data, np.zeros((3, 2), np.float32))
    a = P.CsrMatrix.from_dense(np.array([[1, 1], [0, 3]], np.float32))
    assert P.oracle_spmm(a, P.DenseMatrix.from_array(np.ones((2, 2), np.float32))).data.tolist() == [[2.0, 2.0],
                                                                                                   [3.0, 3.0]]
    d = np.random.default_rng(0).uniform(-1, 1, (5, 5)).astype(np.float32)
    d[d < 0] = 0
    assert np.array_equal(P.oracle_spmm(P.CsrMatrix.from_dense(d), P.DenseMatrix.from_array(np.eye(5, dtype=np.float32))).data, d)
    with pytest.raises(ValueError):
        P.oracle_spmm(eye, P.DenseMatrix.from_array(np.ones((3, 2), np.float32)))


def test_build_candidates_matches_reference(api_cases):
    for case, a, _, _ in api_cases:
        for mc, want in case["candidates"].items():
            got = P.build_candidates(a, int(mc))
            assert len(got) == len(want), case["name"]
            for r, (g, w) in enumerate(zip(got, want)):
                assert g.tolist() == w, (case["name"], mc, r)
    with pytest.raises(ValueError):
        P.build_candidates(api_cases[0][1], 0)


def test_tile_density_and_sweep_match_reference(api_cases):
    for case, a, _, _ in api_cases:
        m = P.build_rstile(a, P.split_long_work(a, P.partition_rows(a)))
        assert P.tile_density(m).__dict__ == case["tile_density"], case["name"]
        sweep = P.threshold_sweep(a, [0, 2, 4, 6])
        assert [[t, r.__dict__] for t, r in sweep] == case["threshold_sweep"], case["name"]
        assert P.sweep_csv(P.threshold_sweep(a, [0, 4])) == case["sweep_csv"], case["name"]


def test_tile_density_known_answers():
    # test_metrics.py: full block, residual-only matrix, planted two-block window
    force_tc = P.PartitionParams(tau_nnz=0)

    def build(a, p=P.PartitionParams()):
        return P.build_rstile(a, P.split_long_work(a, P.partition_rows(a, p), p))

    rep = P.tile_density(build(P.CsrMatrix.from_dense(np.ones((8, 8), np.float32)), force_tc))
    assert (rep.block_count, rep.window_count, rep.mean_nnz_per_block, rep.mean_nnz_per_window,
            rep.residual_nnz_fraction) == (1, 1, 64.0, 64.0, 0.0)
    rep = P.tile_density(build(P.CsrMatrix.from_dense(np.eye(16, dtype=np.float32))))
    assert (rep.block_count, rep.window_count, rep.residual_nnz_fraction, rep.residual_row_fraction) == (0, 0, 1.0, 1.0)
    dense = np.zeros((2, 16), np.float32)
    dense[0, :10] = 1.0
    dense[1, 6:16] = 1.0
    rep = P.tile_density(build(P.CsrMatrix.from_dense(dense), force_tc))
    assert (rep.window_count, rep.block_count, rep.mean_nnz_per_window, rep.mean_nnz_per_block) == (1, 2, 20.0, 10.0)
    with pytest.raises(ValueError):
        P.threshold_sweep(P.CsrMatrix.from_dense(dense), [])
