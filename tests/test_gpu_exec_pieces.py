"""decode_tile / Fragment8x8 / exec_tc_window / exec_residual (reference execute.py:52-133),
restating the reference's own tests (test_execute.py:48-180) on the product, which runs them as
device SpMMs over one-window / residual-only sub-formats."""

from __future__ import annotations

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2603_08734_b200")


def _b(n, d, seed):
    return P.DenseMatrix.from_array(np.random.default_rng(seed).uniform(-1, 1, (n, d)).astype(np.float32))


def _build(a, p=None):
    p = p or P.PartitionParams()
    return P.build_rstile(a, P.split_long_work(a, P.partition_rows(a, p), p))


def test_decode_known_answers():
    assert not P.decode_tile(0, np.zeros(0, np.float32)).data.any()
    vals = np.arange(1, 65, dtype=np.float32)
    assert np.array_equal(P.decode_tile(0xFFFFFFFFFFFFFFFF, vals).data, vals.reshape(8, 8))
    f = P.decode_tile(0x201, np.array([3.0, 4.0], np.float32))
    assert f.data[0, 0] == 3.0 and f.data[1, 1] == 4.0 and np.count_nonzero(f.data) == 2
    with pytest.raises(ValueError):
        P.decode_tile(0x201, np.array([1.0], np.float32))
    with pytest.raises(ValueError):
        P.Fragment8x8(np.zeros((4, 4), np.float32))


@pytest.mark.parametrize("seed", range(5))
def test_decode_positions_follow_set_bits(seed):
    rng = np.random.default_rng(seed)
    bitmap = int(rng.integers(1, 2 ** 64, dtype=np.uint64))
    vals = rng.uniform(1, 2, bin(bitmap).count("1")).astype(np.float32)
    f = P.decode_tile(bitmap, vals)
    for bit in range(64):
        assert bool(f.data[bit // 8, bit % 8]) == bool(bitmap >> bit & 1)
    assert np.array_equal(f.data[f.data != 0], vals)  # values in bit order


def test_exec_tc_window_identity_and_dense():
    force_tc = P.PartitionParams(tau_nnz=0)
    m = _build(P.CsrMatrix.from_dense(np.eye(8, dtype=np.float32)), force_tc)
    b = _b(8, 5, 0)
    c = np.zeros((8, 5), np.float32)
    P.exec_tc_window(m, 0, b, c)
    assert np.array_equal(c, b.data)
    with pytest.raises(IndexError):
        P.exec_tc_window(m, 1, b, c)
    from paper_2603_08734_b200 import synth
    from oracle import corpus  # noqa: E402
    a = corpus.generate_power_law(8, 16, 50, 1.5, seed=3)
    m = _build(a, force_tc)
    assert m.tc.n_entries == 1 and m.residual.n_rows == 0
    b = _b(16, 7, 3)
    c = np.zeros((8, 7), np.float32)
    P.exec_tc_window(m, 0, b, c)
    ref, _ = O.spmm_f64(O.Csr.of(a), b.data)
    assert O.max_relative_error(c, ref) <= 1e-5
    c64 = np.zeros((8, 7), np.float64)
    P.exec_tc_window(m, 0, b, c64)
    assert O.max_relative_error(c64.astype(np.float32), ref) <= 1e-7


def test_exec_residual_identity():
    m = _build(P.CsrMatrix.from_dense(np.eye(16, dtype=np.float32)))
    assert m.tc.n_entries == 0 and m.residual.n_rows == 16
    b = _b(16, 4, 2)
    c = np.zeros((16, 4), np.float32)
    P.exec_residual(m, b, c)
    assert np.array_equal(c, b.data)
    P.exec_residual(m, b, c)  # accumulates
    assert np.array_equal(c, 2 * b.data)


def test_host_stream_pipelined_steps_match_device_result(small_corpus):
    """device.HostStream (host-resident format + B, pipelined copies): every step's host C equals
    the device-resident product bitwise."""
    import torch
    from paper_2603_08734_b200.device import TILE_HOST_FIELDS, DeviceCsr, HostStream, build_device, spmm_device
    a = small_corpus[7]
    t = build_device(DeviceCsr.from_host(a))
    b = torch.from_numpy(np.random.default_rng(5).uniform(-1, 1, (a.n_cols, 64)).astype(np.float32)).cuda()
    ref = spmm_device(t, b).cpu()
    hs = HostStream({k: getattr(t, k).cpu().pin_memory() for k in TILE_HOST_FIELDS}, b.cpu().pin_memory(),
                    t.n_rows, t.n_cols, t.window_size)
    assert hs.run(5) > 0
    assert torch.equal(hs.result(3), ref) and torch.equal(hs.result(4), ref)
    assert hs.run(2, pipelined=False) > 0
    assert torch.equal(hs.result(0), ref) and torch.equal(hs.result(1), ref)
