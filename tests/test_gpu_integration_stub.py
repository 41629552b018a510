"""GPU: the reference-side ctypes binding INTEGRATION.md shows a maintainer (rstile/_gpu.py) is
executed as written against librsh.so: its hybrid_spmm_gpu reproduces the oracle on seeded
matrices.  Keeps the documented boundary honest."""

from __future__ import annotations

import os
import re

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2603_08734_b200")
torch = pytest.importorskip("torch")

import oracle as O  # noqa: E402
from rsh_testlib import ROOT  # noqa: E402


def _stub_namespace():
    from paper_2603_08734_b200 import _lib
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    block = re.search(r"```python\n(# rstile/_gpu\.py.*?)```", text, re.S).group(1)
    block = block.replace("from .tile import FormatError", "from paper_2603_08734_b200 import FormatError")
    block = block.replace('ctypes.CDLL("librsh.so")', f'ctypes.CDLL({_lib.LIB_PATH!r})')
    ns: dict = {}
    exec(compile(block, "INTEGRATION.md:rstile/_gpu.py", "exec"), ns)
    return ns


def test_integration_stub_runs_against_the_library(small_corpus):
    ns = _stub_namespace()
    for a in small_corpus[:8] + [small_corpus[-1]]:
        m = P.build_rstile(a, P.split_long_work(a, P.partition_rows(a)))
        b = P.DenseMatrix.from_array(np.random.default_rng(a.nnz).uniform(-1, 1, (a.n_cols, 64)).astype(np.float32))
        c = ns["hybrid_spmm_gpu"](m, b)
        _, ref64 = O.spmm_f64(O.Csr.of(a), b.data)
        assert c.shape == (a.n_rows, 64)
        assert O.rel_frobenius(c, ref64) <= 1e-6
