"""GNN aggregation with autograd: A·H forward and Aᵀ·dY backward through the
RS-Tile SpMM, against a dense fp64 torch reference of the same op."""

from __future__ import annotations

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _dense(a) -> np.ndarray:
    d = np.zeros((a.n_rows, a.n_cols), np.float64)
    rows = np.repeat(np.arange(a.n_rows), np.diff(np.asarray(a.row_ptr)))
    d[rows, np.asarray(a.col_idx)] = np.asarray(a.values, np.float64)
    return d


@pytest.mark.parametrize("shape", [(700, 500, 9000), (1500, 1500, 30000), (64, 3000, 4000)])
def test_transpose_is_canonical_and_exact(shape):
    from paper_2603_08734_b200 import synth
    from oracle import corpus  # noqa: E402
    from paper_2603_08734_b200.device import DeviceCsr
    from paper_2603_08734_b200.gnn import transpose_device
    a = corpus.generate_power_law(*shape, 1.5, seed=11)
    t = transpose_device(DeviceCsr.from_host(a))
    rp, ci, va = t.row_ptr.cpu().numpy(), t.col_idx.cpu().numpy(), t.values.cpu().numpy()
    assert t.n_rows == a.n_cols and t.n_cols == a.n_rows
    for r in range(t.n_rows):  # strictly increasing columns in every row
        seg = ci[rp[r]:rp[r + 1]]
        assert np.all(np.diff(seg) > 0)
    dt = np.zeros((t.n_rows, t.n_cols))
    rows = np.repeat(np.arange(t.n_rows), np.diff(rp))
    dt[rows, ci] = va
    assert np.array_equal(dt, _dense(a).T)


@pytest.mark.parametrize("n_feat", [32, 64, 128])
def test_forward_backward_against_dense(n_feat):
    from paper_2603_08734_b200 import synth
    from oracle import corpus  # noqa: E402
    from paper_2603_08734_b200.gnn import SparseOperator
    a = corpus.generate_power_law(1200, 900, 20000, 1.5, seed=5)
    op = SparseOperator.from_csr(a)
    g = torch.Generator().manual_seed(0)
    h = torch.rand((a.n_cols, n_feat), generator=g).mul_(2).sub_(1).cuda().requires_grad_(True)
    dy = torch.rand((a.n_rows, n_feat), generator=g).mul_(2).sub_(1).cuda()
    y = op(h)
    y.backward(dy)
    A = torch.from_numpy(_dense(a))
    y_ref = A @ h.detach().cpu().double()
    dh_ref = A.T @ dy.cpu().double()
    rel = lambda x, r: float((x.cpu().double() - r).norm() / r.norm())  # noqa: E731
    assert rel(y.detach(), y_ref) <= 1e-6
    assert rel(h.grad, dh_ref) <= 1e-6


def test_gcn_layer_trains():
    from paper_2603_08734_b200 import synth
    from oracle import corpus  # noqa: E402
    from paper_2603_08734_b200.gnn import GCNLayer, SparseOperator
    a = corpus.generate_power_law(800, 800, 12000, 1.4, seed=2)
    op = SparseOperator.from_csr(a)
    torch.manual_seed(0)
    layer = GCNLayer(op, 16, 8).cuda()
    x = torch.randn(800, 16, device="cuda")
    target = torch.randn(800, 8, device="cuda")
    opt = torch.optim.SGD(layer.parameters(), lr=0.01)
    losses = []
    for _ in range(20):
        opt.zero_grad()
        loss = ((layer(x) - target) ** 2).mean()
        loss.backward()
        opt.step()
        losses.append(float(loss.detach()))
    assert losses[-1] < losses[0]
    # the weight gradient equals the dense computation's
    A = torch.from_numpy(_dense(a)).float().cuda()
    w = layer.weight.detach().clone().requires_grad_(True)
    ref = ((A @ (x @ w) + layer.bias.detach() - target) ** 2).mean()
    ref.backward()
    layer.zero_grad()
    ((layer(x) - target) ** 2).mean().backward()
    assert torch.allclose(layer.weight.grad, w.grad, rtol=1e-4, atol=1e-6)


def test_shape_errors():
    from paper_2603_08734_b200 import synth
    from oracle import corpus  # noqa: E402
    from paper_2603_08734_b200.gnn import SparseOperator
    a = corpus.generate_power_law(100, 80, 600, 1.5, seed=1)
    op = SparseOperator.from_csr(a)
    with pytest.raises(ValueError):
        op(torch.zeros((81, 4), device="cuda"))
    with pytest.raises(ValueError):
        op(torch.zeros((80, 4), device="cuda", dtype=torch.float64))
