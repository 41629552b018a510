"""GNN aggregation with autograd (the paper's GCN case study).

``SparseOperator`` holds A and Aᵀ as device RS-Tiles (Aᵀ built by ``rsh_transpose_csr`` and the
same on-device builder) so that ``op(H)`` = A·H runs the hybrid SpMM forward and Aᵀ·dY backward,
both through librsh.so.  The gradient flows to H only: the adjacency is data, as in the GCN
case study; its values carry no gradient.

    op = SparseOperator.from_csr(a)            # a: CsrMatrix (host) or DeviceCsr
    y = op(h)                                  # h: [n_cols, N] CUDA tensor, requires_grad ok
    y.sum().backward()                         # h.grad = Aᵀ · 1
"""

from __future__ import annotations

import torch

from ._lib import call, lib
from .device import DeviceCsr, DeviceTile, _ptr, _stream, _ws, build_device, spmm_device


def transpose_device(a: DeviceCsr, stream=None) -> DeviceCsr:
    """Aᵀ as a canonical CSR on device (rsh_transpose_csr)."""
    dev = a.device
    nnz = a.nnz
    rp = torch.empty(a.n_cols + 1, dtype=torch.int64, device=dev)
    ci = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
    va = torch.empty(max(nnz, 1), dtype=torch.float32, device=dev)
    nbytes = lib().rsh_transpose_workspace(a.n_rows, a.n_cols, nnz)
    ws = _ws(nbytes, dev)
    call("rsh_transpose_csr", _ptr(a.row_ptr), _ptr(a.col_idx), _ptr(a.values), a.n_rows, a.n_cols, nnz, _ptr(rp),
         _ptr(ci), _ptr(va), _ptr(ws), nbytes, _stream(stream))
    return DeviceCsr(a.n_cols, a.n_rows, rp, ci[:nnz], va[:nnz])


class _RsTileMatmul(torch.autograd.Function):
    @staticmethod
    def forward(ctx, op: "SparseOperator", h: torch.Tensor) -> torch.Tensor:
        ctx.op = op
        return spmm_device(op.tile, h.detach(), math=op.math)

    @staticmethod
    def backward(ctx, dy: torch.Tensor):
        op = ctx.op
        dh = spmm_device(op.tile_t, dy.contiguous(), math=op.math) if ctx.needs_input_grad[1] else None
        return None, dh


class SparseOperator:
    """A fixed sparse matrix as a differentiable linear map H -> A·H (fp32 accumulation;
    ``math`` as in spmm_device: "auto" = exact-FP32 CUDA-core path)."""

    def __init__(self, tile: DeviceTile, tile_t: DeviceTile, math: str = "auto"):
        self.tile, self.tile_t, self.math = tile, tile_t, math

    @classmethod
    def from_csr(cls, a, math: str = "auto", device=None, **build_kw) -> "SparseOperator":
        d = a if isinstance(a, DeviceCsr) else DeviceCsr.from_host(a, device)
        return cls(build_device(d, **build_kw), build_device(transpose_device(d), **build_kw), math)

    @property
    def shape(self) -> tuple[int, int]:
        return (self.tile.n_rows, self.tile.n_cols)

    def __call__(self, h: torch.Tensor) -> torch.Tensor:
        if h.dim() != 2 or h.shape[0] != self.tile.n_cols:
            raise ValueError(f"dimension mismatch: operator is {self.shape}, H is {tuple(h.shape)}")
        if h.dtype != torch.float32:
            raise ValueError("SparseOperator computes in fp32; pass a float32 H")
        return _RsTileMatmul.apply(self, h.contiguous())


class GCNLayer(torch.nn.Module):
    """One graph-convolution layer Y = Â · (X W) (+ bias) with Â a SparseOperator (the
    normalised adjacency); the dense X W is a library GEMM, the aggregation is the RS-Tile SpMM."""

    def __init__(self, op: SparseOperator, in_features: int, out_features: int, bias: bool = True):
        super().__init__()
        self.op = op
        self.weight = torch.nn.Parameter(torch.empty(in_features, out_features))
        self.bias = torch.nn.Parameter(torch.zeros(out_features)) if bias else None
        torch.nn.init.xavier_uniform_(self.weight)

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        y = self.op(x @ self.weight)
        return y + self.bias if self.bias is not None else y


__all__ = ["GCNLayer", "SparseOperator", "transpose_device"]
