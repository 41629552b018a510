"""CUDA-core streaming-kernel variants (rsh_spmm_cc development knobs passed as cc_variant, see
csrc/spmm_cc.cu) on the BASELINE workloads: CUDA-event median of 20 launches + bitwise check
against variant 0.

    python tools/cc_probe.py rmat1m heavytail4m 0 16384 32768 49152
"""
import os
import sys

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
    names = [x for x in sys.argv[1:] if not x.isdigit()] or ["rmat1m"]
    variants = [int(x) for x in sys.argv[1:] if x.isdigit()] or [0]
    dev = torch.device("cuda", 0)
    for name in names:
        w = synth.WORKLOADS[name]
        a = synth.workload_matrix(name)
        b = synth.workload_b(name, a.n_cols)
        tile = build_device(DeviceCsr.from_host(a, dev))
        bt = torch.from_numpy(b).to(dev)
        if w.dtype == "bf16":
            bt = bt.to(torch.bfloat16)
        ref = spmm_device(tile, bt)
        print(f"{name}: nnz {a.nnz} N {w.n_features}", flush=True)
        for v in variants:
            out = torch.empty_like(ref)
            ms = timeit(lambda: spmm_device(tile, bt, out=out, cc_variant=v))
            print(f"  variant {v:6d}: {ms:.3f} ms  bitwise-equal {bool(torch.equal(out, ref))}", flush=True)


if __name__ == "__main__":
    main()
