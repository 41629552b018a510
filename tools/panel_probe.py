"""Feature-panel probe: run the streaming SpMM over B in column panels (each panel's hot B rows
fit the 126 MB L2 better) and compare time and bitwise results against the one-pass kernel.

    python tools/panel_probe.py rmat1m heavytail4m
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_08734_b200 import synth  # noqa: E402
from paper_2603_08734_b200.device import DeviceCsr, build_device, spmm_device  # noqa: E402


def run(tile, bt, out, panels, variant, iters=20):
    N = bt.shape[1]
    w = N // panels

    def step():
        for p in range(panels):
            spmm_device(tile, bt[:, p * w:(p + 1) * w], out=out[:, p * w:(p + 1) * w], cc_variant=variant)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        step()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def main():
    names = sys.argv[1:] or ["rmat1m", "heavytail4m"]
    dev = torch.device("cuda", 0)
    for name in names:
        w = synth.WORKLOADS[name]
        t0 = time.time()
        a = synth.workload_matrix(name)
        b = synth.workload_b(name, a.n_cols)
        tile = build_device(DeviceCsr.from_host(a, dev))
        bt = torch.from_numpy(b).to(dev)
        if w.dtype == "bf16":
            bt = bt.to(torch.bfloat16)
        print(f"{name}: nnz {a.nnz} N {w.n_features} ({time.time() - t0:.1f} s to build)", flush=True)
        ref = torch.empty((a.n_rows, w.n_features), dtype=torch.float32, device=dev)
        spmm_device(tile, bt, out=ref)
        torch.cuda.synchronize()
        for variant in (0, 4):
            for panels in (1, 2, 4, 8):
                if w.n_features // panels < (32 if w.dtype == "f32" else 64):
                    continue
                out = torch.empty_like(ref)
                ms = run(tile, bt, out, panels, variant)
                same = bool(torch.equal(out, ref))
                print(f"  panels {panels} variant {variant}: {ms:.3f} ms  bitwise-equal {same}", flush=True)


if __name__ == "__main__":
    main()
