"""Role timing of the tensor-core kernel (rsh_spmm_tc with flags bit 4): where each warp role of
each CTA spends its cycles.  Development tool."""

from __future__ import annotations

import argparse
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2603_08734_b200 import synth  # noqa: E402
from paper_2603_08734_b200._lib import lib  # noqa: E402
from paper_2603_08734_b200.device import DeviceCsr, build_device, spmm_device  # noqa: E402

NAMES = ["prod: empty wait", "prod: window loop", "prod: tail units", "mma: full wait", "mma: tempty wait",
         "mma: loop", "epi: tfull wait", "epi: loop", "epi: partials", "kernel (thread 0)"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="rmat1m")
    ap.add_argument("--flags", type=int, default=1)
    args = ap.parse_args()
    a = synth.workload_matrix(args.workload)
    b = torch.from_numpy(synth.workload_b(args.workload, a.n_cols)).cuda()
    t = build_device(DeviceCsr.from_host(a))
    out = torch.empty((a.n_rows, b.shape[1]), device="cuda")
    for _ in range(2):
        spmm_device(t, b, out=out, math="tf32", l1=args.flags)
    torch.cuda.synchronize()
    buf = np.zeros((1024, 16), np.uint64)
    lib().rsh_tc_profile(buf.ctypes.data_as(ctypes.c_void_p))
    spmm_device(t, b, out=out, math="tf32", l1=args.flags | 16)
    torch.cuda.synchronize()
    lib().rsh_tc_profile(buf.ctypes.data_as(ctypes.c_void_p))
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    p = buf[:sms].astype(np.float64)
    per = {"prod": 12, "mma": 4, "epi": 1}
    for i, n in enumerate(NAMES):
        div = per.get(n.split(":")[0], 1)
        col = p[:, i] / div
        print(f"{n:22s} mean {col.mean() / 1e3:9.1f} kcyc  max {col.max() / 1e3:9.1f} kcyc")


if __name__ == "__main__":
    main()
