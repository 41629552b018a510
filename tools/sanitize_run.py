"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck / synccheck): the device
builder, the CUDA-core streaming kernel (fp32, bf16, f64 accumulation), the tensor-core window
kernel (TF32 at N = 32/64/128/256, BF16 at N = 64/128), multi-chunk windows with the ticket
reduction and the fix-up kernels, on config 1 (uniform 4096^2) and small seeded corpora.

    compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_08734_b200 as P  # noqa: E402
from oracle import corpus  # noqa: E402
from paper_2603_08734_b200 import synth  # noqa: E402
from paper_2603_08734_b200.device import DeviceCsr, build_device, spmm_device  # noqa: E402


def run(a, name):
    t = build_device(DeviceCsr.from_host(a))
    rng = np.random.default_rng(a.nnz)
    for n in (32, 64, 128, 256):
        b = torch.from_numpy(rng.uniform(-1, 1, (a.n_cols, n)).astype(np.float32)).cuda()
        c0 = spmm_device(t, b, math="fp32")
        c1 = spmm_device(t, b, math="tf32")
        c2 = spmm_device(t, b, accumulate="f64")
        rel = float((c1 - c0).norm() / max(float(c0.norm()), 1e-30))
        assert rel < 1e-3 and torch.allclose(c0, c2, atol=1e-4), (name, n, rel)
        if n >= 64:
            bh = b.to(torch.bfloat16)
            c3 = spmm_device(t, bh, math="tc")
            c4 = spmm_device(t, bh)
            assert float((c3 - c4).norm() / max(float(c4.norm()), 1e-30)) < 1e-2
    torch.cuda.synchronize()
    print(f"{name}: n={a.n_rows} nnz={a.nnz} blocks={t.n_blocks} residual={t.n_res} ok", flush=True)


def main():
    run(synth.uniform_4096(), "config1-uniform4096")
    run(corpus.generate_power_law(2048, 1536, 30000, 1.5, seed=1), "power-law")
    # one near-dense row: a window of 700+ blocks (multi-chunk: partials + tickets), residual rows
    rng = np.random.default_rng(2)
    dense = np.zeros((300, 6000), np.float32)
    dense[0, :] = rng.uniform(-1, 1, 6000)
    dense[17, rng.choice(6000, 3000, replace=False)] = 1.0
    for r in range(40, 300, 7):
        dense[r, rng.integers(6000)] = rng.uniform(-1, 1)
    run(P.CsrMatrix.from_dense(dense), "long-windows")
    print("sanitize workload done")


if __name__ == "__main__":
    main()
