"""GPU: the five BASELINE.json workloads at full size (config 5 = R-MAT scale 24, 263,433,540 nnz).

Per config:
* the device-built RS-Tile (partition + split + build, on device) is bit-exact with the CPU
  oracle's build of the same matrix (the oracle itself is pinned to the reference by
  tests/test_oracle_golden.py), and -- for the configs whose reference build fits this
  container (tests/golden/make_config_golden.py) -- with SHA-256 digests of the REFERENCE's
  own build of the same matrix;
* C from the exact-FP32 CUDA-core path matches the f64 oracle to the reference's 1e-5
  max-relative gate (excluding the long-row reductions the reference's own f32 path fails,
  SURVEY.md 8(c)) and 1e-6 relative Frobenius on sampled row ranges;
* the tensor-core path (TF32 for fp32 configs, BF16 for config 4) meets the north-star
  relative-Frobenius gates (1e-3 / 1e-2);
* size-independent properties on the whole C: rows with no nonzeros are exactly 0, repeated
  launches are bit-identical.
"""

from __future__ import annotations

import json
import os

import numpy as np
import pytest

import oracle as O
from rsh_testlib import GOLDEN, digest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

CONFIGS = ["uniform4k", "rmat1m", "stencil2m", "heavytail4m", "rmat16m"]


def _reference_digests():
    try:
        with open(os.path.join(GOLDEN, "config_formats.json")) as fh:
            return json.load(fh)["configs"]
    except OSError:
        return {}


def _sample_ranges(n_rows: int, k: int = 6, width: int = 4096, seed: int = 0):
    if n_rows <= k * width:
        return [(0, n_rows)]
    rng = np.random.default_rng(seed)
    starts = np.sort(rng.choice(n_rows - width, k - 1, replace=False))
    return [(0, width)] + [(int(s), int(s) + width) for s in starts]


@pytest.fixture(scope="module", params=CONFIGS)
def config(request):
    from paper_2603_08734_b200 import synth
    from paper_2603_08734_b200.device import DeviceCsr, build_device
    name = request.param
    a = synth.workload_matrix(name)
    w = synth.workload_spec(name)
    b = synth.workload_b(name, a.n_cols)
    t = build_device(DeviceCsr.from_host(a))
    yield name, w, a, b, t
    del t
    torch.cuda.empty_cache()


def test_format_digests_match_reference_build(config):
    """Full-size pin: the device format equals the reference's own build, array by array."""
    name, _, a, _, t = config
    ref = _reference_digests().get(name)
    if ref is None:
        pytest.skip(f"no reference build recorded for {name} (tests/golden/make_config_golden.py)")
    assert ref["input"] == digest(np.array([a.n_rows, a.n_cols]), a.row_ptr, a.col_idx, a.values), name
    h = t.host_arrays()
    f = ref["format"]
    assert (t.n_entries, t.n_blocks, t.window_size) == (f["n_entries"], f["n_blocks"], f["window_size"])
    for k, want in f["arrays"].items():
        assert digest(h[k]) == want, (name, k)


def test_format_bit_exact_with_oracle(config):
    name, _, a, _, t = config
    want = O.build_format(O.Csr.of(a))
    h = t.host_arrays()
    got = O.Tile(t.n_rows, t.n_cols, *(h[k] for k in O.Tile.ARRAYS), t.window_size)
    assert O.tiles_equal(got, want) == [], name


def test_products_against_fp64_oracle(config):
    from paper_2603_08734_b200.device import spmm_device, tc_eligible
    name, w, a, b, t = config
    bt = torch.from_numpy(b).cuda()
    if w.dtype == "bf16":
        bt = bt.to(torch.bfloat16)
    c_fp32 = spmm_device(t, bt, math="fp32")
    c_fp32_again = spmm_device(t, bt, math="fp32")
    assert torch.equal(c_fp32, c_fp32_again)
    use_tc = tc_eligible(t, bt)
    c_tc = spmm_device(t, bt, math="tc") if use_tc else None
    if c_tc is not None:
        assert torch.equal(c_tc, spmm_device(t, bt, math="tc"))
    # exact zeros on rows without nonzeros, over the whole C
    empty = torch.from_numpy(np.diff(np.asarray(a.row_ptr)) == 0).cuda()
    assert not c_fp32[empty].any()
    if c_tc is not None:
        assert not c_tc[empty].any()
    oc = O.Csr.of(a)
    tol_tc = 1e-3 if w.dtype == "f32" else 1e-2
    for lo, hi in _sample_ranges(a.n_rows):
        ref32, ref64 = O.spmm_f64(oc, b, lo, hi)
        got = c_fp32[lo:hi].cpu().numpy()
        assert O.rel_frobenius(got, ref64) <= 1e-6, (name, lo)
        longest = int(np.diff(oc.row_ptr[lo:hi + 1]).max(initial=0))
        if longest <= 64:  # short reductions: the reference's own 1e-5 max-relative gate
            assert O.max_relative_error(got, ref32) <= 1e-5, (name, lo)
        if c_tc is not None:
            assert O.rel_frobenius(c_tc[lo:hi].cpu().numpy(), ref64) <= tol_tc, (name, lo)
