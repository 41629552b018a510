"""L2 residency probe: does reserving L2 for persisting (evict_last) lines change the streaming
SpMM?  The kernel marks every B-row gather L2::evict_last and the format / C streams
evict_first; without a persisting set-aside (cudaLimitPersistingL2CacheSize, default 0) the
hint may have no effect.

    python tools/l2_probe.py rmat1m heavytail4m
"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_08734_b200 import synth  # noqa: E402
from paper_2603_08734_b200.device import DeviceCsr, build_device, spmm_device  # noqa: E402

cudart = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None


def set_persist(nbytes):
    torch.cuda.synchronize()
    rt = cudart or ctypes.CDLL("libcudart.so")
    lim = ctypes.c_size_t(0)
    r = rt.cudaDeviceSetLimit(ctypes.c_int(0x06), ctypes.c_size_t(nbytes))  # cudaLimitPersistingL2CacheSize
    rt.cudaDeviceGetLimit(ctypes.byref(lim), ctypes.c_int(0x06))
    return r, lim.value


def timeit(tile, bt, out, variant, iters=20):
    for _ in range(3):
        spmm_device(tile, bt, out=out, cc_variant=variant)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        spmm_device(tile, bt, out=out, cc_variant=variant)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def main():
    dev = torch.device("cuda", 0)
    props = torch.cuda.get_device_properties(0)
    print("L2 bytes", props.L2_cache_size, "persisting max", getattr(props, "persisting_l2_cache_max_size", None))
    for name in sys.argv[1:] or ["rmat1m", "heavytail4m"]:
        w = synth.WORKLOADS[name]
        a = synth.workload_matrix(name)
        b = synth.workload_b(name, a.n_cols)
        tile = build_device(DeviceCsr.from_host(a, dev))
        bt = torch.from_numpy(b).to(dev)
        if w.dtype == "bf16":
            bt = bt.to(torch.bfloat16)
        out = torch.empty((a.n_rows, w.n_features), dtype=torch.float32, device=dev)
        print(name, flush=True)
        for persist in (0, 32 << 20, 64 << 20, 96 << 20, 1 << 30):
            r, got = set_persist(persist)
            for variant in (0, 4):
                ms = timeit(tile, bt, out, variant)
                print(f"  persist {persist >> 20:5d} MB (rc {r}, limit {got >> 20} MB) variant {variant}: {ms:.3f} ms",
                      flush=True)
        set_persist(0)


if __name__ == "__main__":
    main()
