"""Config-2 SpMM timed three ways on one box: 5 back-to-back launches (bench's path probe), 200
launches with per-step events (bench's timed loop), and the same 200 with `nvidia-smi -lms 50`
polling beside them (bench's clock sampler).  Median of 3 repeats each.

    python tools/timing_probe.py [workload]
"""
import os
import subprocess
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_08734_b200 import synth  # noqa: E402
from paper_2603_08734_b200.device import DeviceCsr, build_device, spmm_device  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "rmat1m"
    a = synth.workload_matrix(name)
    b = torch.from_numpy(synth.workload_b(name, a.n_cols)).cuda()
    t = build_device(DeviceCsr.from_host(a))
    out = spmm_device(t, b, math="fp32")
    st = torch.cuda.current_stream()

    def burst(n, per_step_events):
        for _ in range(3):
            spmm_device(t, b, out=out, math="fp32")
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(st)
        for e0, e1 in ev:
            if per_step_events:
                e0.record(st)
            spmm_device(t, b, out=out, math="fp32")
            if per_step_events:
                e1.record(st)
        g1.record(st)
        torch.cuda.synchronize()
        return g0.elapsed_time(g1) / n

    for label, n, evs, smi in [("5 back-to-back", 5, False, False), ("200 + events", 200, True, False),
                               ("200 no events", 200, False, False), ("200 + events + nvidia-smi", 200, True, True),
                               ("5 back-to-back", 5, False, False)]:
        res = []
        for _ in range(3):
            p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader", "-lms", "50"],
                                 stdout=subprocess.DEVNULL) if smi else None
            time.sleep(0.3 if smi else 0)
            res.append(burst(n, evs))
            if p:
                p.terminate()
                p.wait()
        print(f"{name} {label:28s}: {np.median(res):.4f} ms/launch  {['%.4f' % r for r in res]}", flush=True)


if __name__ == "__main__":
    main()
