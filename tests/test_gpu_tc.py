"""GPU: the tensor-core (tcgen05) window path.

North-star tolerances (BASELINE.json): relative Frobenius error <= 1e-3 for TF32 operands and
<= 1e-2 for BF16/FP16 operands against the reference's fp64 result.  Both tensor-core kinds
also keep the structural contracts: every row written once, zero rows exact, split-granularity
invariance and run-to-run determinism.
"""

from __future__ import annotations

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2603_08734_b200")
torch = pytest.importorskip("torch")

TF32_TOL = 1e-3  # BASELINE.json north_star: TF32 rel-Frobenius vs fp64
HALF_TOL = 1e-2  # BF16 / FP16


def _tile(a, **kw):
    from paper_2603_08734_b200.device import DeviceCsr, build_device
    return build_device(DeviceCsr.from_host(a), **kw)


def _b(n, d, seed, dtype=torch.float32):
    x = np.random.default_rng(seed).uniform(-1, 1, (n, d)).astype(np.float32)
    return torch.from_numpy(x).cuda().to(dtype)


@pytest.mark.parametrize("d", [32, 64, 128, 256])
def test_tf32_matches_fp64_oracle(small_corpus, d):
    from paper_2603_08734_b200.device import spmm_device
    for a in small_corpus:
        t = _tile(a)
        b = _b(a.n_cols, d, a.nnz)
        c = spmm_device(t, b, math="tf32").cpu().numpy()
        _, ref64 = O.spmm_f64(O.Csr.of(a), b.cpu().numpy())
        assert O.rel_frobenius(c, ref64) <= TF32_TOL
        # rows outside windows and residual rows are written exactly like the CUDA-core path
        cc = spmm_device(t, b, math="fp32").cpu().numpy()
        zero = ~np.abs(ref64).any(axis=1)
        assert not c[zero].any()
        assert np.abs(c - cc).max() <= 1e-2 * max(1.0, np.abs(cc).max())


@pytest.mark.parametrize("dt", ["bfloat16", "float16"])
@pytest.mark.parametrize("d", [64, 128, 256])
def test_half_operands_on_tensor_cores(dt, d):
    from paper_2603_08734_b200 import synth
    from oracle import corpus  # noqa: E402
    from paper_2603_08734_b200.device import resolve_math, spmm_device
    a = corpus.generate_power_law(700, 500, 9000, 1.5, seed=3)
    t = _tile(a)
    b = _b(500, d, 5, getattr(torch, dt))
    assert resolve_math("auto", b, t, "f32") == "cc"  # the streaming CUDA-core kernel is faster
    assert resolve_math("tc", b, t, "f32") == "tc"
    c = spmm_device(t, b, math="tc").cpu().numpy()
    _, ref64 = O.spmm_f64(O.Csr.of(a), b.float().cpu().numpy())
    err = O.rel_frobenius(c, ref64)
    assert err <= HALF_TOL
    # A values of this corpus are not bf16-exact, so the tensor cores see them rounded; the
    # CUDA-core path keeps them in fp32
    assert err <= 5e-3


def test_tf32_rounding_is_not_truncation():
    """A values are rounded to tf32 with cvt.rna before the MMA; with a bf16-exact A and B the
    TF32 product is exact."""
    from paper_2603_08734_b200 import synth
    from oracle import corpus  # noqa: E402
    from paper_2603_08734_b200.device import spmm_device
    a = corpus.generate_power_law(256, 256, 4000, 1.5, seed=9)
    vals = synth.bf16_round(np.asarray(a.values))
    a = P.CsrMatrix(a.n_rows, a.n_cols, a.row_ptr, a.col_idx, vals)
    t = _tile(a)
    b = _b(256, 128, 1, torch.bfloat16).float()
    c = spmm_device(t, b, math="tf32").cpu().numpy()
    _, ref64 = O.spmm_f64(O.Csr.of(a), b.cpu().numpy())
    assert O.rel_frobenius(c, ref64) <= 1e-6


@pytest.mark.parametrize("d", [64, 128])
def test_tc_split_invariance_and_determinism(d):
    from paper_2603_08734_b200 import synth
    from oracle import corpus  # noqa: E402
    from paper_2603_08734_b200.device import spmm_device
    a = corpus.generate_power_law(128, 4096, 40000, 2.0, seed=11)
    b = _b(4096, d, 11)
    outs = set()
    for k in (1, 4, 64, None):
        t = _tile(a, max_blocks_per_item=k)
        for _ in range(2):
            outs.add(spmm_device(t, b, math="tf32").cpu().numpy().tobytes())
    assert len(outs) == 1


def test_tc_long_windows_and_residual_mix():
    """Multi-chunk windows (partials + ordered ticket reduction), residual rows and uncovered
    rows in one launch."""
    from paper_2603_08734_b200.device import spmm_device
    rng = np.random.default_rng(2)
    dense = np.zeros((300, 6000), np.float32)
    dense[0, :] = rng.uniform(-1, 1, 6000)           # 750 blocks -> 24 chunks
    dense[17, rng.choice(6000, 3000, replace=False)] = 1.0
    for r in range(40, 300, 7):  # single-nonzero rows: delta <= 1 < tau_inc -> residual
        dense[r, rng.integers(6000)] = rng.uniform(-1, 1)
    a = P.CsrMatrix.from_dense(dense)
    t = _tile(a)
    assert t.n_res > 0
    b = _b(6000, 256, 3)
    _, ref64 = O.spmm_f64(O.Csr.of(a), b.cpu().numpy())
    for _ in range(3):
        c = spmm_device(t, b, math="tf32").cpu().numpy()
        assert O.rel_frobenius(c, ref64) <= TF32_TOL
        zero = ~dense.any(axis=1)
        assert not c[zero].any()


def test_exec_config_tf32_through_host_api(small_corpus):
    a = small_corpus[5]
    m = P.build_rstile(a, P.split_long_work(a, P.partition_rows(a)))
    b = np.random.default_rng(0).uniform(-1, 1, (a.n_cols, 128)).astype(np.float32)
    c = P.hybrid_spmm(m, P.DenseMatrix.from_array(b), P.ExecConfig(math="tf32")).data
    _, ref64 = O.spmm_f64(O.Csr.of(a), b)
    assert O.rel_frobenius(c, ref64) <= TF32_TOL
    with pytest.raises(ValueError):
        P.hybrid_spmm(m, P.DenseMatrix.from_array(b[:, :100]), P.ExecConfig(math="tf32"))


@pytest.mark.parametrize("math", ["fp32", "tf32"])
def test_spmm_device_is_cuda_graph_capturable(small_corpus, math):
    """bench.py times CUDA-graph replays of spmm_device: a captured step equals a direct call
    bitwise (no host synchronisation or allocation inside a warmed-up call)."""
    from paper_2603_08734_b200.device import spmm_device
    a = small_corpus[3]
    t = _tile(a)
    b = _b(a.n_cols, 128, 4)
    ref = spmm_device(t, b, math=math)
    out = torch.empty_like(ref)
    spmm_device(t, b, out=out, math=math)  # warm-up: schedule, fragments, workspace
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        spmm_device(t, b, out=out, math=math)
    out.zero_()
    g.replay()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, ref)


@pytest.mark.parametrize("d", [32, 64, 128, 256])
def test_tc_edge_cases(d):
    """Degenerate formats on the tensor-core path: identity through windows (B tf32-exact, so C
    is B exactly), identity through residual rows only (no blocks at all), an all-zero matrix,
    a single element, and padding slots next to a B row of large values (zero-filled by the
    TMA's out-of-bounds rows, never multiplied in)."""
    from paper_2603_08734_b200.device import spmm_device
    rng = np.random.default_rng(d)
    bq = (rng.integers(-64, 64, (16, d)) / 8.0).astype(np.float32)  # exact in tf32
    b = torch.from_numpy(bq).cuda()
    eye = P.CsrMatrix.from_dense(np.eye(16, dtype=np.float32))
    t_win = _tile(eye, tau_nnz=0)
    assert t_win.n_blocks > 0 and t_win.n_res == 0
    assert torch.equal(spmm_device(t_win, b, math="tf32"), b)
    t_res = _tile(eye)
    assert t_res.n_blocks == 0 and t_res.n_res == 16
    assert torch.equal(spmm_device(t_res, b, math="tf32"), b)
    zero = P.CsrMatrix.from_dense(np.zeros((16, 16), np.float32))
    assert not spmm_device(_tile(zero), b, math="tf32").any()
    one = P.CsrMatrix.from_dense(np.full((1, 1), 2.0, np.float32))
    assert torch.equal(spmm_device(_tile(one, tau_nnz=0), b[:1], math="tf32"), 2.0 * b[:1])
    # one row using columns 1 and 9 (one block, 6 padding slots whose col_id is 0): B row 0 is NaN,
    # but padding rows arrive as zeros from the TMA's out-of-bounds fill and never reach the MMA
    dense = np.zeros((8, 16), np.float32)
    dense[0, 1] = dense[0, 9] = 1.0
    big = b.clone()
    big[0] = float("nan")
    c = spmm_device(_tile(P.CsrMatrix.from_dense(dense), tau_nnz=0), big, math="tf32")
    assert torch.equal(c[0], big[1] + big[9]) and not c[1:].any()
