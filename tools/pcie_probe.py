"""PCIe copy rates on the GPU box: pinned H2D alone, D2H alone, both at once (separate streams),
and the config-2 HostStream breakdown (inputs only / SpMM with schedule rebuild only / all)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def rate(fn, nbytes, iters=5):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(iters):
        fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / iters
    return dt * 1e3, nbytes / dt / 1e9


def main():
    dev = torch.device("cuda", 0)
    n = 512 << 20
    h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
    d_in = torch.empty(n, dtype=torch.uint8, device=dev)
    d_out = torch.empty(n, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def h2d():
        with torch.cuda.stream(s1):
            d_in.copy_(h_in, non_blocking=True)

    def d2h():
        with torch.cuda.stream(s2):
            h_out.copy_(d_out, non_blocking=True)

    def both():
        h2d()
        d2h()
    print("H2D 512 MiB: %.2f ms %.1f GB/s" % rate(h2d, n))
    print("D2H 512 MiB: %.2f ms %.1f GB/s" % rate(d2h, n))
    ms, gbs = rate(both, 2 * n)
    print("both at once: %.2f ms, %.1f GB/s total" % (ms, gbs))
    # chunked copies (8 x 64 MiB) alternating directions
    from paper_2603_08734_b200 import synth
    from paper_2603_08734_b200.device import DeviceCsr, build_device, spmm_device, TILE_HOST_FIELDS, HostStream
    a = synth.workload_matrix("rmat1m")
    b = torch.from_numpy(synth.workload_b("rmat1m", a.n_cols))
    tile = build_device(DeviceCsr.from_host(a, dev))
    host = {k: getattr(tile, k).cpu().pin_memory() for k in TILE_HOST_FIELDS}
    for k, v in host.items():
        print(f"  field {k}: {v.numel() * v.element_size() / 1e6:.1f} MB")
    hs = HostStream(host, b.pin_memory(), tile.n_rows, tile.n_cols, tile.window_size, dev)
    hs.run(2)
    print("HostStream pipelined %.2f ms/step, sequential %.2f" % (hs.run(6), hs.run(4, pipelined=False)))
    t, bufs, b_dev, c_dev = hs.sets[0]
    # SpMM with schedule rebuild each time: fresh tile object over the same buffers
    from paper_2603_08734_b200.device import DeviceTile
    def spmm_fresh():
        tt = DeviceTile(tile.n_rows, tile.n_cols, tile.window_size, **bufs)
        spmm_device(tt, b_dev, out=c_dev)
    for _ in range(2):
        spmm_fresh()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        spmm_fresh()
    torch.cuda.synchronize()
    print("schedule rebuild + SpMM: %.2f ms" % ((time.perf_counter() - t0) / 5 * 1e3))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        spmm_device(tile, b_dev, out=c_dev)
    torch.cuda.synchronize()
    print("SpMM with cached schedule: %.2f ms" % ((time.perf_counter() - t0) / 5 * 1e3))


if __name__ == "__main__":
    main()
