"""Per-step timeline of device.HostStream on config 2: when each step's input copy, SpMM (with
schedule rebuild) and C copy start and end on the device, and where the host blocks."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_08734_b200 import synth  # noqa: E402
from paper_2603_08734_b200 import device as D  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    name = sys.argv[1] if len(sys.argv) > 1 else "rmat1m"
    a = synth.workload_matrix(name)
    b = torch.from_numpy(synth.workload_b(name, a.n_cols))
    if synth.WORKLOADS[name].dtype == "bf16":
        b = b.to(torch.bfloat16)
    tile = D.build_device(D.DeviceCsr.from_host(a, dev))
    host = {k: getattr(tile, k).cpu().pin_memory() for k in D.TILE_HOST_FIELDS}
    hs = D.HostStream(host, b.pin_memory(), tile.n_rows, tile.n_cols, tile.window_size, dev)
    hs.run(2)
    n = 6
    E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    marks = []
    orig = D.spmm_device
    host_t = []

    def spy(*args, **kw):
        s = kw.get("stream")
        e0, e1 = E(), E()
        e0.record(s)
        h0 = time.perf_counter()
        r = orig(*args, **kw)
        host_t.append((h0, time.perf_counter()))
        e1.record(s)
        marks.append(("spmm", e0, e1))
        return r
    D.spmm_device = spy
    # wrap copy_ on the streams by recording around stage_inputs / out copies: emulate with events
    # recorded on s_in / s_out right after run() (coarse) -- instead re-implement one pipelined run
    torch.cuda.synchronize()
    T0 = E()
    T0.record()
    w0 = time.perf_counter()
    ms = hs.run(n)
    w1 = time.perf_counter()
    D.spmm_device = orig
    torch.cuda.synchronize()
    print(f"{name}: pipelined {ms:.2f} ms/step (wall {1e3 * (w1 - w0) / n:.2f})")
    for i, (k, e0, e1) in enumerate(marks):
        print(f"  step {i} spmm device [{T0.elapsed_time(e0):8.2f}, {T0.elapsed_time(e1):8.2f}] ms  host call "
              f"[{1e3 * (host_t[i][0] - w0):8.2f}, {1e3 * (host_t[i][1] - w0):8.2f}] ms")


if __name__ == "__main__":
    main()
