"""Per-role cycle accounting of the tensor-core kernel (development build: spmm_tc.cu compiled
with -DRSH_TC_PROFILE, see tools/build_tc_profile.sh).  Prints, per warp role, the mean total
cycles and the share spent waiting on each barrier.

    bash tools/build_tc_profile.sh && python tools/tc_role_profile.py stencil2m [flags]
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_08734_b200 import _lib, synth  # noqa: E402
from paper_2603_08734_b200 import device as D  # noqa: E402
from paper_2603_08734_b200.device import DeviceCsr, build_device, spmm_device  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "stencil2m"
    flags = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    w = synth.WORKLOADS[name]
    a = synth.workload_matrix(name)
    b = synth.workload_b(name, a.n_cols)
    tile = build_device(DeviceCsr.from_host(a))
    bt = torch.from_numpy(b).cuda()
    if w.dtype == "bf16":
        bt = bt.to(torch.bfloat16)
    D.TC_FLAGS = flags
    out = spmm_device(tile, bt, math="tc")
    torch.cuda.synchronize()
    L = _lib.lib()
    buf = np.zeros((148 * 40, 8), np.uint64)
    L.rsh_tc_profile_read(buf.ctypes.data_as(ctypes.c_void_p))  # clear
    for _ in range(5):
        spmm_device(tile, bt, out=out, math="tc")
    torch.cuda.synchronize()
    L.rsh_tc_profile_read(buf.ctypes.data_as(ctypes.c_void_p))
    n_feat = w.n_features
    P = 10 if n_feat <= 64 else (8 if n_feat == 128 else 6)
    roles = {"epilogue": range(0, 8), "mma": range(8, 8 + P), "producer": range(8 + P, 8 + 2 * P)}
    per = buf.reshape(148, 40, 8).astype(np.float64) / 5
    for role, ws in roles.items():
        x = per[:, list(ws), :]
        tot = x[..., 0].mean()
        print(f"{role:9s} total {tot / 1.965e3:8.1f} us   wait empty {x[..., 1].mean() / tot:5.1%}  full "
              f"{x[..., 2].mean() / tot:5.1%}  tempty {x[..., 3].mean() / tot:5.1%}  tfull {x[..., 4].mean() / tot:5.1%}")


if __name__ == "__main__":
    main()
