"""GPU parity: the sm_100a path against the reference's golden outputs and the CPU oracle.

Metadata (partition windows, residual rows, split map, all nine RS-Tile arrays, window_size)
must be BIT-EXACT with the reference (digests from tests/golden/make_golden.py).  SpMM results
are compared with the f64 oracle: the exact-FP32 CUDA-core path is held to the reference's own
max-relative-error gate of 1e-5 (execute.py:26); f64 accumulation to 1e-7.
"""

from __future__ import annotations

import hashlib
import json

import numpy as np
import pytest

import oracle as O
from rsh_testlib import digest

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2603_08734_b200")


def _params(golden_formats, pname):
    return P.PartitionParams(**golden_formats["param_sets"][pname])


def _record(plan, split, m) -> dict:
    wins = np.array(plan.windows, dtype=np.int64).reshape(-1, 2)
    sm = sorted((int(k), [list(s) for s in v]) for k, v in split.split_map.items())
    return {
        "windows": digest(wins), "residual": digest(plan.residual_rows),
        "split_map": hashlib.sha256(json.dumps(sm).encode()).hexdigest(),
        "n_windows": len(plan.windows), "n_residual": int(plan.residual_rows.size),
        "n_entries": m.tc.n_entries, "n_blocks": m.tc.n_blocks, "window_size": m.window_size,
        "arrays": {
            "row_window_id": digest(m.tc.row_window_id), "row_window_offset": digest(m.tc.row_window_offset),
            "bitmaps": digest(m.tc.bitmaps), "col_id": digest(m.tc.col_id), "values": digest(m.tc.values),
            "res_row_id": digest(m.residual.row_id), "res_offset": digest(m.residual.row_nnz_offset),
            "res_col_id": digest(m.residual.col_id), "res_values": digest(m.residual.values)},
    }


def build(a, p=None):
    p = p or P.PartitionParams()
    return P.build_rstile(a, P.split_long_work(a, P.partition_rows(a, p), p))


def rand_b(n, d, seed):
    return np.random.default_rng(seed).uniform(-1, 1, (n, d)).astype(np.float32)


# ---------------------------------------------------------------------------------------------
# metadata: bit-exact with the reference
# ---------------------------------------------------------------------------------------------

def test_formats_bit_exact_with_reference(golden_corpus, golden_formats):
    checked = 0
    for name, (a, entry) in golden_corpus.items():
        for pname, want in entry["formats"].items():
            p = _params(golden_formats, pname)
            plan = P.partition_rows(a, p)
            split = P.split_long_work(a, plan, p)
            m = P.build_rstile(a, split)
            got = _record(plan, split, m)
            assert got == want, (name, pname, [k for k in want if got.get(k) != want[k]])
            checked += 1
    assert checked > 300


def test_device_pipeline_matches_oracle(golden_corpus):
    """build_device (no host round trip of the plan) == oracle arrays, default and split params."""
    from paper_2603_08734_b200.device import DeviceCsr, build_device
    for name, (a, _entry) in golden_corpus.items():
        for kw in ({}, {"max_blocks_per_item": 2}, {"tau_nnz": 0, "window_size": 3}):
            t = build_device(DeviceCsr.from_host(a), **kw)
            want = O.build_format(O.Csr.of(a), **kw)
            h = t.host_arrays()
            got = O.Tile(t.n_rows, t.n_cols, *(h[k] for k in O.Tile.ARRAYS), t.window_size)
            assert O.tiles_equal(got, want) == [], (name, kw)


def test_known_answer_formats(known_answers):
    for name, case in known_answers.items():
        if "tc" not in case:
            continue
        a = P.CsrMatrix.from_dense(np.asarray(case["dense"], np.float32))
        p = P.PartitionParams(**case["params"])
        plan = P.split_long_work(a, P.partition_rows(a, p), p)
        assert [list(w) for w in plan.windows] == case["plan_windows"], name
        assert plan.residual_rows.tolist() == case["plan_residual"], name
        assert {str(k): [list(s) for s in v] for k, v in plan.split_map.items()} == case["plan_split_map"], name
        m = P.build_rstile(a, plan)
        assert m.tc.row_window_id.tolist() == case["tc"]["row_window_id"], name
        assert m.tc.row_window_offset.tolist() == case["tc"]["row_window_offset"], name
        assert [str(int(x)) for x in m.tc.bitmaps] == case["tc"]["bitmaps"], name
        assert m.tc.col_id.tolist() == case["tc"]["col_id"], name
        assert m.tc.values.tolist() == case["tc"]["values"], name


def test_empty_and_degenerate_matrices():
    for dense in (np.zeros((10, 10)), np.zeros((1, 1)), np.eye(1), np.ones((1, 1))):
        a = P.CsrMatrix.from_dense(np.asarray(dense, np.float32))
        want = O.build_format(O.Csr.of(a))
        m = build(a)
        got = O.Tile.of(m)
        assert O.tiles_equal(got, want) == []
        b = rand_b(a.n_cols, 3, 0)
        c = P.hybrid_spmm(m, P.DenseMatrix.from_array(b)).data
        assert np.array_equal(c, O.spmm_f64(O.Csr.of(a), b)[0])
    a = P.CsrMatrix(0, 5, np.zeros(1, np.int64), np.empty(0), np.empty(0))
    assert P.partition_rows(a).windows == ()


def test_arbitrary_valid_plan_builds_like_reference():
    """A hand-made plan with uneven window sizes (validate_plan accepts it) builds bit-exactly."""
    a = P.CsrMatrix.from_dense(np.ones((12, 20), np.float32))
    plan = P.PartitionPlan(((0, 3), (3, 5), (8, 4)), np.empty(0, np.int64), {1: ((0, 1), (1, 3))})
    m = P.build_rstile(a, plan)
    assert m.window_size == 5
    assert m.tc.row_window_id.tolist() == [0, 3, 3, 8]
    assert m.tc.row_window_offset.tolist() == [0, 3, 4, 6, 9]
    with pytest.raises(ValueError):
        P.build_rstile(a, P.PartitionPlan(((0, 8), (4, 8)), np.empty(0, np.int64)))


def test_validate_plan_flags_broken_segments():
    a = P.CsrMatrix.from_dense(np.ones((1, 1037), np.float32))
    p = P.PartitionParams(tau_nnz=0)
    plan = P.partition_rows(a, p)
    bad = P.PartitionPlan(plan.windows, plan.residual_rows, {0: ((0, 64), (64, 100))})
    assert any("segments" in m for m in P.validate_plan(a, bad))
    good = P.split_long_work(a, plan, P.PartitionParams(tau_nnz=0, max_blocks_per_item=64))
    assert good.split_map == {0: ((0, 64), (64, 128), (128, 130))}
    assert P.validate_plan(a, good) == []


# ---------------------------------------------------------------------------------------------
# SpMM: against the f64 oracle
# ---------------------------------------------------------------------------------------------

@pytest.mark.parametrize("d", [16, 64])
def test_spmm_small_corpus_vs_oracle(small_corpus, d):
    for a in small_corpus:
        m = build(a)
        b = rand_b(a.n_cols, d, a.nnz)
        got = P.hybrid_spmm(m, P.DenseMatrix.from_array(b))
        ref, _ = O.spmm_f64(O.Csr.of(a), b)
        assert P.max_relative_error(got, ref) <= 1e-5
        got64 = P.hybrid_spmm(m, P.DenseMatrix.from_array(b), P.ExecConfig(accumulate_precision="f64"))
        assert P.max_relative_error(got64, ref) <= 1e-7


def test_spmm_matches_reference_oracle_outputs(small_corpus):
    import os
    from rsh_testlib import GOLDEN
    ref = np.load(os.path.join(GOLDEN, "small_spmm.npz"))
    for i, a in enumerate(small_corpus):
        b = np.random.default_rng(a.nnz).uniform(-1, 1, (a.n_cols, 16)).astype(np.float32)
        got = P.hybrid_spmm(build(a), P.DenseMatrix.from_array(b))
        assert P.max_relative_error(got, ref[f"c{i:02d}"]) <= 1e-5


def test_known_answer_products(known_answers):
    for name, case in known_answers.items():
        if "b" not in case:
            continue
        a = P.CsrMatrix.from_dense(np.asarray(case["dense"], np.float32))
        m = build(a, P.PartitionParams(**case["params"]))
        b = P.DenseMatrix.from_array(np.asarray(case["b"], np.float32))
        c64 = P.hybrid_spmm(m, b, P.ExecConfig(accumulate_precision="f64")).data
        assert np.array_equal(c64, np.asarray(case["c_f64"], np.float32)), name
        c32 = P.hybrid_spmm(m, b).data
        assert P.max_relative_error(c32, np.asarray(case["c_f32"], np.float32)) <= 1e-5, name


@pytest.mark.parametrize("force_tc", [False, True])
def test_identity_returns_b_exactly(force_tc):
    p = P.PartitionParams(tau_nnz=0) if force_tc else P.PartitionParams()
    m = build(P.CsrMatrix.from_dense(np.eye(16, dtype=np.float32)), p)
    assert (m.residual.n_rows == 0) if force_tc else (m.tc.n_blocks == 0)
    b = rand_b(16, 4, 7)
    assert np.array_equal(P.hybrid_spmm(m, P.DenseMatrix.from_array(b)).data, b)


def test_uncovered_rows_are_zero():
    dense = np.zeros((20, 16), np.float32)
    dense[:8] = 1.0
    dense[19, 0] = 5.0
    m = build(P.CsrMatrix.from_dense(dense))
    c = P.hybrid_spmm(m, P.DenseMatrix.from_array(rand_b(16, 3, 9))).data
    assert not c[8:19].any() and c[19].any()


def test_cancellation_f32_fails_check_f64_exact():
    dense = np.zeros((1, 4), np.float32)
    dense[0] = [2.0 ** 24, 1.0, 1.0, -(2.0 ** 24)]
    m = build(P.CsrMatrix.from_dense(dense), P.PartitionParams(tau_nnz=0))
    ones = P.DenseMatrix.from_array(np.ones((4, 1), np.float32))
    with pytest.raises(P.VerificationError):
        P.hybrid_spmm(m, ones, P.ExecConfig(check_against_oracle=True))
    out = P.hybrid_spmm(m, ones, P.ExecConfig(accumulate_precision="f64", check_against_oracle=True))
    assert out.data.ravel().tolist() == [2.0]


@pytest.mark.parametrize("precision", ["f32", "f64"])
def test_split_granularity_is_bitwise_invisible(precision):
    a = P.CsrMatrix(*(lambda x: (x.n_rows, x.n_cols, x.row_ptr, x.col_idx, x.values))(
        __import__("oracle.corpus", fromlist=["x"]).generate_power_law(128, 512, 4000, 2.0, seed=11)))
    b = P.DenseMatrix.from_array(rand_b(512, 16, 11))
    cfg = P.ExecConfig(accumulate_precision=precision)
    blobs = {P.hybrid_spmm(build(a, P.PartitionParams(max_blocks_per_item=k)), b, cfg).data.tobytes()
             for k in (1, 4, 64, None)}
    assert len(blobs) == 1


def test_long_window_multi_chunk_reduction():
    """A 1 x 20000 dense row: 2500 blocks -> 79 fixed chunks reduced in order; repeated launches
    reuse the tickets and give identical bits."""
    a = P.CsrMatrix.from_dense(np.random.default_rng(3).uniform(-1, 1, (2, 20000)).astype(np.float32))
    m = build(a, P.PartitionParams(tau_nnz=0))
    b = rand_b(20000, 32, 4)
    ref, _ = O.spmm_f64(O.Csr.of(a), b)
    outs = [P.hybrid_spmm(m, P.DenseMatrix.from_array(b)).data for _ in range(3)]
    assert all(o.tobytes() == outs[0].tobytes() for o in outs)
    # 20000-term f32 sums: the reference's own f32 path also exceeds 1e-5 max-rel on long rows
    # (SURVEY.md §8(c)); the f64 path is held to the oracle exactly
    assert O.max_relative_error(outs[0], ref) <= 1e-4
    c64 = P.hybrid_spmm(m, P.DenseMatrix.from_array(b), P.ExecConfig(accumulate_precision="f64")).data
    assert O.max_relative_error(c64, ref) <= 1e-7


@pytest.mark.parametrize("d", [1, 3, 5, 7, 32, 33, 96, 128, 256, 384])
def test_feature_widths(d):
    from paper_2603_08734_b200 import synth
    from oracle import corpus  # noqa: E402
    a = corpus.generate_power_law(300, 200, 3000, 1.5, seed=d)
    m = build(a)
    b = rand_b(200, d, d)
    ref, _ = O.spmm_f64(O.Csr.of(a), b)
    assert P.max_relative_error(P.hybrid_spmm(m, P.DenseMatrix.from_array(b)), ref) <= 1e-5


@pytest.mark.parametrize("dt", ["bfloat16", "float16"])
def test_half_precision_b(dt):
    import torch
    from paper_2603_08734_b200 import synth
    from oracle import corpus  # noqa: E402
    from paper_2603_08734_b200.device import DeviceCsr, build_device, spmm_device
    a = corpus.generate_power_law(512, 400, 8000, 1.5, seed=5)
    t = build_device(DeviceCsr.from_host(a))
    b = torch.from_numpy(rand_b(400, 256, 1)).cuda().to(getattr(torch, dt))
    c = spmm_device(t, b, math="fp32")  # CUDA-core path: half B, fp32 A values, exact products
    ref, ref64 = O.spmm_f64(O.Csr.of(a), b.float().cpu().numpy())
    assert O.rel_frobenius(c.cpu().numpy(), ref64) <= 1e-6


def test_device_api_out_buffer_and_errors():
    import torch
    from paper_2603_08734_b200 import synth
    from oracle import corpus  # noqa: E402
    from paper_2603_08734_b200.device import DeviceCsr, build_device
    a = corpus.generate_power_law(256, 128, 2000, 1.5, seed=2)
    t = build_device(DeviceCsr.from_host(a))
    b = torch.from_numpy(rand_b(128, 64, 2)).cuda()
    out = torch.full((256, 64), float("nan"), device="cuda")
    c = P.hybrid_spmm(t, b, out=out)
    assert c.data_ptr() == out.data_ptr()
    ref, _ = O.spmm_f64(O.Csr.of(a), b.cpu().numpy())
    assert O.max_relative_error(out.cpu().numpy(), ref) <= 1e-5
    with pytest.raises(ValueError):
        P.hybrid_spmm(t, torch.zeros(127, 64, device="cuda"))
    m = build(a)
    with pytest.raises(ValueError):
        P.hybrid_spmm(m, P.DenseMatrix.from_array(rand_b(129, 4, 0)))


def test_permute_rows_matches_reference_semantics(small_corpus):
    """reorder.py:138-151: row i <- source row order[i]; formats built for the same permutation
    are bit-exact with the oracle's build of the permuted matrix."""
    for i, a in enumerate(small_corpus[:8]):
        order = np.random.default_rng(i).permutation(a.n_rows)
        got = P.permute_rows(a, P.Permutation(order, 0.0))
        dense = a.to_dense()[order]
        assert P.csr_equal(got, P.CsrMatrix.from_dense(dense))
        m = build(got)
        want = O.build_format(O.Csr.of(got))
        assert O.tiles_equal(O.Tile.of(m), want) == []
    with pytest.raises(ValueError):
        P.Permutation(np.array([0, 0, 1]), 0.0)


@pytest.mark.parametrize("dtype", ["float32", "bfloat16"])
def test_stream_kernel_bit_identical_across_variants(dtype):
    """The streaming kernel's list pieces (kCap 256 / 320 / 448), pipeline depths, unit setup (header
    read or the chained lookups, flag 128) and the row-walk
    kernel accumulate every row in the same order: C must be bitwise equal across them for one
    schedule (and across lane-group splits of narrow rows, flag 2048),
    including multi-chunk windows (partials + ticket / fix-up reduction) and a near-dense row."""
    import torch
    from paper_2603_08734_b200 import synth
    from oracle import corpus  # noqa: E402
    from paper_2603_08734_b200.device import DeviceCsr, build_device, spmm_device
    a = corpus.generate_power_law(3000, 2500, 60000, 1.3, seed=21)
    dense = np.zeros((a.n_rows, a.n_cols), np.float32)
    rows = np.repeat(np.arange(a.n_rows), np.diff(np.asarray(a.row_ptr)))
    dense[rows, np.asarray(a.col_idx)] = np.asarray(a.values)
    rng = np.random.default_rng(4)
    dense[17, rng.choice(a.n_cols, 2000, replace=False)] = rng.uniform(-1, 1, 2000).astype(np.float32)
    a = P.CsrMatrix.from_dense(dense)
    t = build_device(DeviceCsr.from_host(a))
    for n in (64, 128, 256):
        b = torch.from_numpy(rand_b(a.n_cols, n, n)).cuda().to(getattr(torch, dtype))
        if dtype == "bfloat16" and n == 64:
            continue
        # 256-block units + row-major list (the default schedule): every stream variant agrees
        base = spmm_device(t, b, math="fp32", cc_variant=0)
        for v in (8, 16, 24, 32, 40, 48, 128, 1024, 2048):
            got = spmm_device(t, b, math="fp32", cc_variant=v)
            assert torch.equal(got.view(torch.int32), base.view(torch.int32)), (n, v)
        # 32-block units (bitmap decode, flag 4096): the stream and the row walk agree -- the row
        # walk sums in the same order except its narrow-row (N <= 64 fp32) lane-group mode
        base32 = spmm_device(t, b, math="fp32", cc_variant=4096)
        for v in (4096 | 8, 4096 | 2048) + ((64,) if n >= 128 or dtype != "float32" else ()):
            got = spmm_device(t, b, math="fp32", cc_variant=v)
            assert torch.equal(got.view(torch.int32), base32.view(torch.int32)), (n, v)
        # both schedules against the fp64 oracle (chunk partials change the rounding, not the sum)
        ref = O.spmm_f64(O.Csr.of(a), b.float().cpu().numpy())[1]
        for c in (base, base32):
            assert O.rel_frobenius(c.cpu().numpy(), ref) <= 1e-6
