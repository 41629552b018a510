"""Quick GPU probe: build one BASELINE workload on device, time build phases and the SpMM, and
check a row sample against the f64 oracle.  Development tool (bench.py is the contract)."""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2603_08734_b200 import synth  # noqa: E402
from paper_2603_08734_b200.device import DeviceCsr, build_device, spmm_device, spmm_plan  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="rmat1m")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--check", action="store_true")
    ap.add_argument("--math", default="auto")
    ap.add_argument("--l1", type=int, default=1)
    ap.add_argument("--ccv", type=int, default=0)
    ap.add_argument("--ccflags", type=int, default=0)
    args = ap.parse_args()
    t0 = time.time()
    a = synth.workload_matrix(args.workload)
    w = synth.WORKLOADS[args.workload]
    print(f"{args.workload}: n={a.n_rows} nnz={a.nnz} gen {time.time() - t0:.1f}s", flush=True)
    b = synth.workload_b(args.workload, a.n_cols)
    dev = torch.device("cuda")
    d = DeviceCsr.from_host(a, dev)
    bt = torch.from_numpy(b).to(dev)
    if w.dtype == "bf16":
        bt = bt.to(torch.bfloat16)
    torch.cuda.synchronize()
    for rep in range(2):
        t1 = time.time()
        t = build_device(d)
        torch.cuda.synchronize()
        tb = time.time() - t1
    print(f"build_device {tb * 1e3:.1f} ms: entries={t.n_entries} blocks={t.n_blocks} res={t.n_res} "
          f"ws={t.window_size} tile bytes={t.nbytes() / 1e6:.1f} MB", flush=True)
    t1 = time.time()
    plan = spmm_plan(t)
    from paper_2603_08734_b200.device import CHUNK_TC
    spmm_plan(t, CHUNK_TC)
    torch.cuda.synchronize()
    print(f"schedule {1e3 * (time.time() - t1):.1f} ms: groups={plan.groups} units={plan.units} "
          f"slots={plan.partial_slots} uncovered={plan.uncovered}", flush=True)
    out = torch.empty((a.n_rows, b.shape[1]), dtype=torch.float32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for _ in range(3):
        spmm_device(t, bt, out=out, math=args.math, cc_variant=args.ccv)
    torch.cuda.synchronize()
    times = []
    for _ in range(args.iters):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        spmm_device(t, bt, out=out, math=args.math, cc_variant=args.ccv)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    ms = float(np.median(times))
    flops = 2.0 * a.nnz * b.shape[1]
    print(f"spmm[{args.math}] median {ms:.3f} ms  min {min(times):.3f}  -> {flops / ms / 1e6:.1f} GFLOP/s", flush=True)
    if args.check:
        import oracle as O
        c = out.cpu().numpy()
        rng = np.random.default_rng(0)
        rows = np.sort(rng.choice(a.n_rows, min(a.n_rows, 20000), replace=False))
        oc = O.Csr.of(a)
        errs = []
        for lo in range(0, len(rows), 1):
            pass
        ref32, ref64 = O.spmm_f64(oc, bt.float().cpu().numpy())
        print("max_rel", O.max_relative_error(c, ref32), "relF", O.rel_frobenius(c, ref64), flush=True)


if __name__ == "__main__":
    main()
