"""Reorder a BASELINE workload on device and time the SpMM before/after (development tool)."""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2603_08734_b200 import synth  # noqa: E402
from paper_2603_08734_b200.device import DeviceCsr, build_device, spmm_device  # noqa: E402
from paper_2603_08734_b200.reorder import ReorderParams, permute_rows_device, reorder_device  # noqa: E402


def spmm_ms(t, b, iters=20, math="auto"):
    out = torch.empty((t.n_rows, b.shape[1]), dtype=torch.float32, device=b.device)
    for _ in range(3):
        spmm_device(t, b, out=out, math=math)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        spmm_device(t, b, out=out, math=math)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def stats(t):
    nnz_tc = t.values.numel()
    return {"windows": t.n_entries, "blocks": t.n_blocks, "nnz_per_block": nnz_tc / max(t.n_blocks, 1),
            "residual_nnz_share": t.res_values.numel() / max(nnz_tc + t.res_values.numel(), 1)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="rmat1m")
    ap.add_argument("--hub-cap", type=int, default=256)
    ap.add_argument("--passes", type=int, default=3)
    args = ap.parse_args()
    a = synth.workload_matrix(args.workload)
    w = synth.WORKLOADS[args.workload]
    d = DeviceCsr.from_host(a)
    b = torch.from_numpy(synth.workload_b(args.workload, a.n_cols)).cuda()
    if w.dtype == "bf16":
        b = b.to(torch.bfloat16)
    t0 = build_device(d)
    base = spmm_ms(t0, b)
    torch.cuda.synchronize()
    s = time.perf_counter()
    o, info = reorder_device(d, ReorderParams(hub_cap=args.hub_cap, two_opt_passes=args.passes))
    torch.cuda.synchronize()
    rt = time.perf_counter() - s
    dp = permute_rows_device(d, o)
    t1 = build_device(dp)
    after = spmm_ms(t1, b)
    print(f"{args.workload}: reorder {rt:.2f} s {info}")
    print(f"  before: {base:.3f} ms (tensor cores {spmm_ms(t0, b, math='tc'):.3f} ms) {stats(t0)}")
    print(f"  after : {after:.3f} ms (tensor cores {spmm_ms(t1, b, math='tc'):.3f} ms) {stats(t1)}")


if __name__ == "__main__":
    main()
