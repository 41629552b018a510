"""Library baseline beside the product kernels: torch.sparse.mm on a CSR tensor (cuSPARSE SpMM)
vs spmm_device on the same matrix and B, CUDA-event median of 20 (results compared).

    python tools/cusparse_probe.py rmat1m stencil2m heavytail4m uniform4k
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
    dev = torch.device("cuda", 0)
    for name in sys.argv[1:] or ["rmat1m"]:
        w = synth.WORKLOADS[name]
        a = synth.workload_matrix(name)
        b = synth.workload_b(name, a.n_cols)
        d = DeviceCsr.from_host(a, dev)
        tile = build_device(d)
        bt = torch.from_numpy(b).to(dev)
        if w.dtype == "bf16":
            bt = bt.to(torch.bfloat16)
        flops = 2.0 * a.nnz * w.n_features
        ours = spmm_device(tile, bt)
        ms_ours = timeit(lambda: spmm_device(tile, bt, out=ours))
        line = f"{name}: ours {ms_ours:.3f} ms ({flops / ms_ours / 1e6:.0f} GFLOP/s)"
        try:
            vals = d.values if w.dtype == "f32" else d.values.to(torch.bfloat16)
            csr = torch.sparse_csr_tensor(d.row_ptr.to(torch.int32), d.col_idx, vals, (a.n_rows, a.n_cols))
            ref = torch.sparse.mm(csr, bt)
            ms_lib = timeit(lambda: torch.sparse.mm(csr, bt))
            rel = float((ref.float() - ours).norm() / max(float(ours.norm()), 1e-30))
            line += f"   torch.sparse.mm (cuSPARSE) {ms_lib:.3f} ms ({flops / ms_lib / 1e6:.0f} GFLOP/s)  " \
                    f"speed-up {ms_lib / ms_ours:.2f}x  rel diff {rel:.1e}"
        except Exception as exc:  # noqa: BLE001
            line += f"   torch.sparse.mm unavailable: {type(exc).__name__}: {str(exc)[:80]}"
        print(line, flush=True)


if __name__ == "__main__":
    main()
