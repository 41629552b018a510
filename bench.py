"""RSH-SpMM benchmark -- the driver contract (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload rmat1m] [--impl ours|reference]

A step is one hybrid SpMM C = A @ B over the whole workload (BASELINE.json configs[1] by
default: R-MAT scale 20, avg degree 16, N = 128, fp32), inputs resident in HBM.  ``value`` is
SpMM GFLOP/s = 2 nnz N / t over all ranks (max-over-ranks device time).  With N > 1 ranks
(torchrun) the rows of A are sharded by cost across GPUs (dist.py): B is broadcast and C
gathered over NCCL, both timed separately from the kernel and reported beside it.

Extra keys: ``e2e`` (the same metric through the C ABI with host buffers, H2D of the format
and B plus D2H of C inside every step), ``roofline`` (dominant kernel's algorithmic bytes over
its event-timed duration against MEASURED_PEAKS.json HBM bandwidth), ``gather`` (the measured
L2->SM row-gather roof), ``cpu_baseline`` (the reference executor, restated in numpy under
oracle/, timed on this host), ``clocks`` (nvidia-smi during the timed region).

``--impl reference`` times the reference CPU executor (oracle.port_hybrid_spmm, a numpy
restatement of rstile execute.py:155-226) on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SpMM GFLOP/s (2*nnz*N/t)"
# profiles/r01_gather_bw2_microbench.txt: random 512-B B rows gathered with LDG.128 by 148 SMs
GATHER_ROOF_L2_GBS = 18454.0   # 64 MB footprint (L2-resident)
GATHER_ROOF_HBM_GBS = 7291.0   # 2 GB footprint (from HBM)


def _peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except OSError:
        return {"hbm_gbs": 6650.0, "_fallback": True}


def _traffic(workload: str):
    """dram read+write bytes per launch of the SpMM kernel from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            rec = json.load(fh).get(workload)
        return None if rec is None else rec["dram_bytes_per_launch"]
    except (OSError, KeyError, TypeError):
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons, sampled while the timed region runs."""

    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None
        self.window = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={','.join(self.FIELDS)}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append((time.time(), line.strip()))

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        lo, hi = self.window if self.window else (0, 1e30)
        inside = [s for t, s in self.samples if lo <= t <= hi] or [s for _, s in self.samples[-5:]]
        sm, mx, reasons = [], [], set()
        for s in inside:
            parts = [p.strip() for p in s.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, flag in zip(self.NAMES, parts[2:6]):
                if flag.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(inside)}


def algorithmic_bytes(a, n_feat: int, b_elem: int, val_bytes: int = 4) -> tuple[int, int]:
    """nnz*(val+4) + touched_cols*N*E_B + n_rows*N*4 (C f32), and touched cols."""
    touched = int(np.unique(a.col_idx).size) if a.nnz else 0
    return a.nnz * (val_bytes + 4) + touched * n_feat * b_elem + a.n_rows * n_feat * 4, touched


def cpu_reference_sample(a, b, workload: str, target_s: float = 10.0, num_workers: int = 1):
    """Time the reference executor restatement (oracle.port_hybrid_spmm) on a bounded sample:
    a prefix of the format's entries and residual rows holding ~frac of the nnz."""
    import oracle as O
    c = O.Csr.of(a)
    t = O.build_format(c)
    n_ent, n_res = t.row_window_id.size, t.res_row_id.size
    frac = 1.0
    # probe 1% to size the sample
    e_hi = max(1, int(n_ent * 0.01)) if n_ent else 0
    t0 = time.perf_counter()
    O.port_hybrid_spmm(t, b, num_workers, entry_range=(0, e_hi), residual_range=(0, int(n_res * 0.01)))
    dt = time.perf_counter() - t0
    if dt > 0:
        frac = min(1.0, max(0.01, 0.01 * target_s / dt))
    e_hi = int(n_ent * frac)
    # do not cut a split window in two
    while 0 < e_hi < n_ent and t.row_window_id[e_hi] == t.row_window_id[e_hi - 1]:
        e_hi += 1
    r_hi = int(n_res * frac)
    blocks = int(t.row_window_offset[e_hi]) if n_ent else 0
    nnz_s = int(O.popcounts(t.bitmaps[:blocks]).sum()) + int(t.res_offset[r_hi])
    t0 = time.perf_counter()
    O.port_hybrid_spmm(t, b, num_workers, entry_range=(0, e_hi), residual_range=(0, r_hi))
    dt = time.perf_counter() - t0
    gflops = 2.0 * nnz_s * b.shape[1] / dt / 1e9
    sample = (f"{workload}: first {e_hi}/{n_ent} window entries + {r_hi}/{n_res} residual rows "
              f"({nnz_s} of {a.nnz} nnz, {100.0 * nnz_s / max(a.nnz, 1):.1f}%), one pass {dt:.2f} s")
    return gflops, dt, sample, nnz_s


def run_reference(args):
    """--impl reference: the reference CPU executor on this host (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2603_08734_b200 import synth
    import oracle as O
    a = synth.workload_matrix(args.workload)
    w = synth.WORKLOADS[args.workload]
    b = synth.workload_b(args.workload, a.n_cols)
    cores = len(os.sched_getaffinity(0))
    c = O.Csr.of(a)
    t = O.build_format(c)
    n_ent, n_res = t.row_window_id.size, t.res_row_id.size
    # each step: a bounded slice of the work (~2 s), stepping through the matrix
    probe_e = max(1, n_ent // 100)
    t0 = time.perf_counter()
    O.port_hybrid_spmm(t, b, cores, entry_range=(0, probe_e), residual_range=(0, n_res // 100))
    per = max(time.perf_counter() - t0, 1e-6)
    frac = min(1.0, 0.01 * 2.0 / per)
    slices = max(1, int(round(1.0 / frac)))
    step_ent = -(-n_ent // slices) if n_ent else 0
    step_res = -(-n_res // slices) if n_res else 0
    vstart = np.zeros(t.bitmaps.size + 1, np.int64)
    np.cumsum(O.popcounts(t.bitmaps), out=vstart[1:])
    times, flops = [], []
    for it in range(args.warmup + args.steps):
        k = it % slices
        e0, e1 = min(k * step_ent, n_ent), min((k + 1) * step_ent, n_ent)
        while 0 < e0 < n_ent and t.row_window_id[e0] == t.row_window_id[e0 - 1]:
            e0 += 1
        while 0 < e1 < n_ent and t.row_window_id[e1] == t.row_window_id[e1 - 1]:
            e1 += 1
        r0, r1 = min(k * step_res, n_res), min((k + 1) * step_res, n_res)
        nnz_s = int(vstart[t.row_window_offset[e1]] - vstart[t.row_window_offset[e0]]) + \
            int(t.res_offset[r1] - t.res_offset[r0])
        s = time.perf_counter()
        O.port_hybrid_spmm(t, b, cores, entry_range=(e0, e1), residual_range=(r0, r1))
        d = time.perf_counter() - s
        if it >= args.warmup:
            times.append(d)
            flops.append(2.0 * nnz_s * w.n_features)
    value = sum(flops) / sum(times) / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": {"workload": args.workload, "description": w.description,
                                        "n_rows": a.n_rows, "nnz": a.nnz, "n_features": w.n_features},
        "cpu_baseline": {"value": value, "unit": "GFLOP/s", "cores": cores, "kind": "port",
                         "sample": f"each step = 1/{slices} of the {args.workload} window entries and residual "
                                   f"rows (consecutive slices), numpy restatement of rstile hybrid_spmm "
                                   f"(oracle.port_hybrid_spmm), ThreadPoolExecutor({cores}) like the reference"},
        "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="rmat1m")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--math", default="auto", choices=["auto", "fp32", "tf32", "tc"])
    ap.add_argument("--sharded", action="store_true",
                    help="run the row-shard path even on one GPU (config 5 at N=1 under torchrun)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args)
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 or args.gpus > 1 or args.sharded:
        from paper_2603_08734_b200.dist import run_sharded_bench
        run_sharded_bench(args, METRIC, clock_factory=ClockSampler)
        return
    run_single(args)


def run_single(args):
    import torch
    from paper_2603_08734_b200 import synth
    from paper_2603_08734_b200.device import DeviceCsr, build_device, spmm_device, spmm_plan, DeviceTile
    from paper_2603_08734_b200 import _lib

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    w = synth.WORKLOADS[args.workload]
    a = synth.workload_matrix(args.workload)
    b_np = synth.workload_b(args.workload, a.n_cols)
    b_elem = 2 if w.dtype == "bf16" else 4
    alg_bytes, touched = algorithmic_bytes(a, w.n_features, b_elem, 2 if w.dtype == "bf16" else 4)
    flops = 2.0 * a.nnz * w.n_features

    # preprocessing on device (reported separately from the steady-state SpMM); the first build
    # also pays one-time library / allocator initialisation, so the second one is reported
    d = DeviceCsr.from_host(a, dev)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tile = build_device(d)
    torch.cuda.synchronize()
    t_build_first = time.perf_counter() - t0
    del tile
    t0 = time.perf_counter()
    tile = build_device(d)
    torch.cuda.synchronize()
    t_build = time.perf_counter() - t0
    # schedule for the streaming kernel: long units + the pre-decoded row-major window list
    from paper_2603_08734_b200.device import CHUNK_CC_LIST, CHUNK_TC
    t0 = time.perf_counter()
    plan = spmm_plan(tile, CHUNK_CC_LIST)
    torch.cuda.synchronize()
    t_sched = time.perf_counter() - t0
    spmm_plan(tile, CHUNK_TC)  # the tensor-core candidate's schedule
    bt = torch.from_numpy(b_np).to(dev)
    if w.dtype == "bf16":
        bt = bt.to(torch.bfloat16)
    out = torch.empty((a.n_rows, w.n_features), dtype=torch.float32, device=dev)
    st = torch.cuda.current_stream()

    # arithmetic path: fp32 B -> exact FP32 (CUDA cores) or TF32 (tensor cores); bf16 B -> tensor
    # cores when the shape allows.  "auto" times both for a few launches and keeps the faster.
    from paper_2603_08734_b200.device import resolve_math, tc_eligible
    candidates = (["fp32", "tf32"] if w.dtype == "f32" else ["auto", "tc"]) if tc_eligible(tile, bt) else ["auto"]
    if args.math != "auto":
        candidates = [args.math]
    path_ms = {}
    for m in candidates:
        for _ in range(2):
            spmm_device(tile, bt, out=out, math=m)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(5):
            spmm_device(tile, bt, out=out, math=m)
        e1.record(st)
        torch.cuda.synchronize()
        path_ms[m] = e0.elapsed_time(e1) / 5
    math = min(path_ms, key=path_ms.get)
    kernel = "k_spmm_tc" if resolve_math(math, bt, tile, "f32") == "tc" else "k_spmm_cc"

    clocks = ClockSampler(0)
    clocks.start()
    time.sleep(0.3)
    for _ in range(args.warmup):
        spmm_device(tile, bt, out=out, math=math)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    w0 = time.time()
    g0.record(st)
    for e0, e1 in ev:
        e0.record(st)
        spmm_device(tile, bt, out=out, math=math)
        e1.record(st)
    g1.record(st)
    torch.cuda.synchronize()
    w1 = time.time()
    clocks.window = (w0, w1)
    total_ms = g0.elapsed_time(g1)
    kern_ms = [e0.elapsed_time(e1) for e0, e1 in ev]
    clk = clocks.stop()
    ms = total_ms / args.steps
    value = flops / (ms * 1e-3) / 1e9
    kern_avg = float(np.mean(kern_ms))
    achieved = alg_bytes / (kern_avg * 1e-3) / 1e9
    peaks = _peaks()
    peak = float(peaks.get("hbm_gbs", 6650.0))
    gathered = int(plan_gather_bytes(tile, w.n_features, b_elem))

    # end to end through the C ABI with host buffers: H2D(format + B), SpMM, D2H(C) every step
    host = {k: getattr(tile, k).cpu().pin_memory() for k in (
        "row_window_id", "row_window_offset", "bitmaps", "col_id", "values", "res_row_id", "res_offset",
        "res_col_id", "res_values")}
    b_host = bt.cpu().pin_memory()
    c_host = torch.empty((a.n_rows, w.n_features), dtype=torch.float32).pin_memory()
    dev_bufs = {k: torch.empty_like(v, device=dev) for k, v in host.items()}
    b_dev2 = torch.empty_like(b_host, device=dev)
    t2 = DeviceTile(tile.n_rows, tile.n_cols, tile.window_size, **dev_bufs)
    t2._plan = tile._plan  # the schedules are part of the prebuilt operator, like the format itself
    # the schedule's pre-decoded window list is derived from the format: it travels with it
    ulists = [(pl.ulist, pl.ulist.cpu().pin_memory()) for pl in (tile._plan or {}).values()
              if getattr(pl, "ulist", None) is not None]
    h2d = sum(v.numel() * v.element_size() for v in host.values()) + b_host.numel() * b_host.element_size() + \
        sum(h.numel() * h.element_size() for _, h in ulists)
    d2h = c_host.numel() * 4
    e2e_ms = []
    for it in range(args.e2e_steps + 1):
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(st)
        for k, v in host.items():
            dev_bufs[k].copy_(v, non_blocking=True)
        b_dev2.copy_(b_host, non_blocking=True)
        for dst, src in ulists:
            dst.copy_(src, non_blocking=True)
        spmm_device(t2, b_dev2, out=out, math=math)
        c_host.copy_(out, non_blocking=True)
        s1.record(st)
        torch.cuda.synchronize()
        if it:
            e2e_ms.append(s0.elapsed_time(s1))
    e2e_value = flops / (float(np.mean(e2e_ms)) * 1e-3) / 1e9

    cpu = None
    if not args.no_cpu_baseline:
        gf, dt, sample, _ = cpu_reference_sample(a, b_np.astype(np.float32), args.workload)
        cpu = {"value": gf, "unit": "GFLOP/s", "cores": 1, "kind": "port", "sample": sample}

    line = {
        "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16" if w.dtype == "bf16" else ("tf32" if math == "tf32" else "f32"),
        "data": "synthetic",
        "config": {"workload": args.workload, "description": w.description, "n_rows": a.n_rows,
                   "n_cols": a.n_cols, "nnz": a.nnz, "n_features": w.n_features,
                   "parallelism": "single GPU", "math": math, "kernel": kernel,
                   "path_ms": path_ms, "l2": "no flush: per-step inputs (A + B + C = "
                   f"{(alg_bytes + gathered * 0) / 1e9:.2f} GB compulsory) exceed the 126 MB L2",
                   "preprocess_ms": {"build_device": 1e3 * t_build, "build_device_first_call": 1e3 * t_build_first,
                                     "schedule": 1e3 * t_sched},
                   "format": {"entries": tile.n_entries, "blocks": tile.n_blocks, "residual_rows": tile.n_res,
                              "units": plan.units, "uncovered_rows": plan.uncovered}},
        "gpu_launches": 3 * args.steps,  # per step: the SpMM kernel + the two long-window fix-up kernels
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": _traffic(args.workload),
                     "algorithmic_bytes": alg_bytes, "kernel": kernel, "kernel_ms": kern_avg,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "_fallback" not in peaks else "fallback"},
        "gather": {"gathered_bytes": gathered, "achieved_gbs": gathered / (kern_avg * 1e-3) / 1e9,
                   "roof_l2_resident_gbs": GATHER_ROOF_L2_GBS, "roof_hbm_gbs": GATHER_ROOF_HBM_GBS,
                   "frac_of_l2_roof": gathered / (kern_avg * 1e-3) / 1e9 / GATHER_ROOF_L2_GBS,
                   "note": "B rows the window path must move into the SMs (one per occupied col_id slot "
                           "+ one per residual nonzero); roofs measured by tools/microbench/gather_bw2.cu"},
        "e2e": {"value": e2e_value, "unit": "GFLOP/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "ms_per_step": float(np.mean(e2e_ms)),
                "path": f"{kernel} via the C ABI (ctypes), pinned host format + B in, C out"},
        "cpu_baseline": cpu,
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)


def plan_gather_bytes(tile, n_feat: int, b_elem: int) -> int:
    """B bytes the window path must gather: one row per non-padding col_id slot (a slot whose
    bitmap column is empty is skipped), plus one row per residual nonzero."""
    import torch
    bm = tile.bitmaps
    if bm.numel() == 0:
        slots = 0
    else:
        x = bm.clone()
        for sh in (32, 16, 8):
            x = x | (x >> sh) if sh != 32 else x | ((x >> 32) & 0xFFFFFFFF)
        x = x & 0xFF
        slots = int(sum(((x >> j) & 1).sum().item() for j in range(8)))
    return (slots + int(tile.res_col_id.numel())) * n_feat * b_elem


if __name__ == "__main__":
    main()
