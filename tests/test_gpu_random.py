"""GPU: seeded randomized parity sweep over shapes the fixed corpora do not pin -- odd row and
column counts, empty rows and columns, near-dense rows (multi-chunk windows), every feature width
the two SpMM paths accept and all three B dtypes.  For each case: the device format equals the
oracle's bit for bit (for every max_blocks_per_item split), the CUDA-core product is within the
fp32 gate of the fp64 oracle, and the tensor-core product within the TF32 / half gate."""

from __future__ import annotations

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2603_08734_b200")
torch = pytest.importorskip("torch")

FP32_TOL = 1e-6   # exact-FP32 products, fp32 accumulation (rel-Frobenius vs fp64)
TF32_TOL = 1e-3   # north star
HALF_TOL = 1e-2


def _case(seed: int):
    rng = np.random.default_rng(seed)
    n_rows = int(rng.integers(1, 3000))
    n_cols = int(rng.integers(1, 3000))
    density = float(rng.choice([0.0005, 0.002, 0.01, 0.05]))
    mask = rng.random((n_rows, n_cols)) < density
    if n_rows > 10 and rng.random() < 0.5:  # a few near-dense rows
        for r in rng.choice(n_rows, 2, replace=False):
            mask[r, rng.random(n_cols) < 0.6] = True
    if rng.random() < 0.3:  # empty column bands
        mask[:, : n_cols // 3] = False
    dense = np.where(mask, rng.uniform(-1, 1, (n_rows, n_cols)), 0).astype(np.float32)
    return P.CsrMatrix.from_dense(dense)


@pytest.mark.parametrize("seed", range(12))
def test_random_formats_and_products(seed):
    from paper_2603_08734_b200.device import DeviceCsr, build_device, spmm_device, tc_eligible
    a = _case(seed)
    rng = np.random.default_rng(1000 + seed)
    d = DeviceCsr.from_host(a)
    for mbpi in (64, 3):
        t = build_device(d, max_blocks_per_item=mbpi)
        want = O.build_format(O.Csr.of(a), max_blocks_per_item=mbpi)
        h = t.host_arrays()
        got = O.Tile(t.n_rows, t.n_cols, *(h[k] for k in O.Tile.ARRAYS), t.window_size)
        assert O.tiles_equal(got, want) == [], (seed, mbpi)
    t = build_device(d)
    for n_feat, dtype in ((32, torch.float32), (64, torch.float32), (96, torch.float32), (128, torch.float32),
                          (256, torch.float32), (64, torch.bfloat16), (128, torch.float16), (256, torch.bfloat16)):
        b32 = rng.uniform(-1, 1, (a.n_cols, n_feat)).astype(np.float32)
        b = torch.from_numpy(b32).cuda().to(dtype)
        _, ref64 = O.spmm_f64(O.Csr.of(a), b.float().cpu().numpy())
        c = spmm_device(t, b).cpu().numpy()
        assert O.rel_frobenius(c, ref64) <= FP32_TOL, (seed, n_feat, dtype)
        assert not c[~np.abs(ref64).any(axis=1) & (np.diff(np.asarray(a.row_ptr)) == 0)].any()
        if tc_eligible(t, b):
            ctc = spmm_device(t, b, math="tc").cpu().numpy()
            tol = TF32_TOL if dtype == torch.float32 else HALF_TOL
            assert O.rel_frobenius(ctc, ref64) <= tol, (seed, n_feat, dtype)
