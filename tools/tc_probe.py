"""Tensor-core vs CUDA-core window path on the BASELINE workloads: kernel time (CUDA events,
median of 20 after warm-up) and the TC result's rel-Frobenius distance from the exact-FP32 path.

    python tools/tc_probe.py stencil2m rmat1m
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_08734_b200 import synth  # noqa: E402
from paper_2603_08734_b200.device import DeviceCsr, build_device, spmm_device  # noqa: E402


def timeit(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def main():
    names = sys.argv[1:] or ["stencil2m"]
    dev = torch.device("cuda", 0)
    for name in names:
        w = synth.WORKLOADS[name]
        t0 = time.time()
        a = synth.workload_matrix(name)
        b = synth.workload_b(name, a.n_cols)
        tile = build_device(DeviceCsr.from_host(a, dev))
        bt = torch.from_numpy(b).to(dev)
        if w.dtype == "bf16" or os.environ.get("TC_BF16"):
            bt = bt.to(torch.bfloat16)
        print(f"{name}: nnz {a.nnz} blocks {tile.n_blocks} N {w.n_features} ({time.time() - t0:.1f} s)", flush=True)
        out_cc = torch.empty((a.n_rows, w.n_features), dtype=torch.float32, device=dev)
        out_tc = torch.empty_like(out_cc)
        ms_cc = timeit(lambda: spmm_device(tile, bt, out=out_cc, math="fp32" if bt.dtype == torch.float32 else "auto"))
        ms_tc = timeit(lambda: spmm_device(tile, bt, out=out_tc, math="tc"))
        d = (out_tc - out_cc).double()
        rel = float(d.norm() / out_cc.double().norm())
        flops = 2.0 * a.nnz * w.n_features
        from paper_2603_08734_b200 import device as D
        knobs = [(int(k), k) for k in os.environ.get("TC_KNOBS", "").split(",") if k.strip()]
        for knob, what in knobs:
            if os.environ.get("TC_KNOBS"):
                D.TC_FLAGS = knob
                ms = timeit(lambda: spmm_device(tile, bt, out=out_tc, math="tc"))
                print(f"  tensor-core with {what}: {ms:.3f} ms", flush=True)
        D.TC_FLAGS = 0
        print(f"  cuda-core {ms_cc:.3f} ms ({flops / ms_cc / 1e6:.0f} GFLOP/s)   tensor-core {ms_tc:.3f} ms "
              f"({flops / ms_tc / 1e6:.0f} GFLOP/s)   rel-Frobenius(tc vs fp32) {rel:.2e}", flush=True)


if __name__ == "__main__":
    main()
