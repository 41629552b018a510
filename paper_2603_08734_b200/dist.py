"""Multi-GPU row shard of A (north-star multi-GPU layer), one process per GPU.

The output rows of C are independent, so A is cut into contiguous row ranges, one per rank,
with cut points chosen on a prefix sum of per-row cost (nnz + 1: every nonzero gathers one B
row and every row writes one C row) and snapped to rows the GLOBAL partition scan visits
(window starts and residual rows, partition.py:127-140).  No window straddles a cut, so each
rank's shard format is exactly the global RS-Tile restricted to its rows (row ids rebased), and
every C row is computed by exactly one GPU with the same arithmetic as on one GPU:
C(G GPUs) == C(1 GPU) bit for bit.

Collectives (torch.distributed, NCCL over NVLink/NVSwitch on GPUs, gloo on CPU for tests):
B is broadcast once from rank 0; C shards are gathered to rank 0 with point-to-point sends
(shards are uneven).  Both are timed separately from the SpMM kernel and reported beside it.
"""

from __future__ import annotations

import json
import os
import time

import numpy as np


# ---------------------------------------------------------------------------------------------
# host-side shard planning (pure numpy; shared by the GPU path and the gloo tests)
# ---------------------------------------------------------------------------------------------

def allowed_cuts(win_start: np.ndarray, resid_rows: np.ndarray, n_rows: int) -> np.ndarray:
    """Rows where a shard may begin: rows the global scan visits with an empty window state."""
    return np.unique(np.concatenate([np.asarray(win_start, np.int64), np.asarray(resid_rows, np.int64),
                                     np.array([0, n_rows], np.int64)]))


def shard_cuts(row_nnz: np.ndarray, allowed: np.ndarray, world: int) -> np.ndarray:
    """cuts[0] = 0 < ... < cuts[world] = n_rows (monotone, possibly repeated for tiny inputs)."""
    n = int(row_nnz.size)
    cost = np.zeros(n + 1, np.int64)
    np.cumsum(np.asarray(row_nnz, np.int64) + 1, out=cost[1:])
    total = int(cost[-1])
    cuts = [0]
    acost = cost[allowed]
    for r in range(1, world):
        target = total * r // world
        k = int(np.searchsorted(acost, target, side="left"))
        k = min(k, allowed.size - 1)
        cuts.append(max(cuts[-1], int(allowed[k])))
    cuts.append(n)
    return np.asarray(cuts, np.int64)


def local_plan(win_start: np.ndarray, resid_rows: np.ndarray, r0: int, r1: int):
    """Windows / residual rows of shard [r0, r1), rebased to local row ids."""
    ws = np.asarray(win_start, np.int64)
    rr = np.asarray(resid_rows, np.int64)
    lw = ws[(ws >= r0) & (ws < r1)] - r0
    lr = rr[(rr >= r0) & (rr < r1)] - r0
    return lw, lr


def local_csr(row_ptr: np.ndarray, col_idx: np.ndarray, values: np.ndarray, r0: int, r1: int):
    s, e = int(row_ptr[r0]), int(row_ptr[r1])
    return row_ptr[r0:r1 + 1] - s, col_idx[s:e], values[s:e]


# ---------------------------------------------------------------------------------------------
# collectives
# ---------------------------------------------------------------------------------------------

def gather_rows(c_local, cuts, rank: int, world: int, out=None):
    """Gather row shards of C to rank 0 (uneven sizes -> point-to-point).  Returns the full C on
    rank 0, None elsewhere."""
    import torch
    import torch.distributed as dist
    if rank == 0:
        full = out if out is not None else torch.empty((int(cuts[-1]), c_local.shape[1]), dtype=c_local.dtype,
                                                       device=c_local.device)
        full[int(cuts[0]):int(cuts[1])].copy_(c_local)
        ops = [dist.P2POp(dist.irecv, full[int(cuts[r]):int(cuts[r + 1])], r) for r in range(1, world)
               if cuts[r + 1] > cuts[r]]
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        return full
    if cuts[rank + 1] > cuts[rank]:
        for req in dist.batch_isend_irecv([dist.P2POp(dist.isend, c_local.contiguous(), 0)]):
            req.wait()
    return None


# ---------------------------------------------------------------------------------------------
# device-side synthetic input for the weak-scaling run
# ---------------------------------------------------------------------------------------------

def rmat_device(scale: int, edge_factor: int, seed: int, device, a=0.57, b=0.19, c=0.19):
    """R-MAT (same quadrant probabilities and dedup as synth.rmat) drawn with torch's Philox
    generator on the GPU: the multi-GPU weak-scaling graphs (scale 20 + log2 G) are too large to
    draw with numpy on every rank.  Returns (row_ptr int64, col_idx int32, values f32) on device."""
    import torch
    n = 1 << scale
    m = edge_factor * n
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    r = torch.zeros(m, dtype=torch.int64, device=device)
    q = torch.zeros(m, dtype=torch.int64, device=device)
    for bit in range(scale):
        u = torch.rand(m, generator=g, device=device, dtype=torch.float64)
        r |= (u >= a + b).to(torch.int64) << bit
        q |= (((u >= a) & (u < a + b)) | (u >= a + b + c)).to(torch.int64) << bit
        del u
    keys = torch.unique(r * n + q)
    del r, q
    rows = keys // n
    cols = (keys - rows * n).to(torch.int32)
    counts = torch.bincount(rows, minlength=n)
    row_ptr = torch.zeros(n + 1, dtype=torch.int64, device=device)
    row_ptr[1:] = torch.cumsum(counts, 0)
    vals = (torch.rand(keys.numel(), generator=g, device=device, dtype=torch.float32) * 2.0 - 1.0)
    return n, row_ptr, cols, vals


# ---------------------------------------------------------------------------------------------
# the sharded benchmark (bench.py --gpus N under torchrun)
# ---------------------------------------------------------------------------------------------

def _hbm_peak() -> float:
    """MEASURED_PEAKS.json hbm_gbs (driver-written), else the profiling recipe's fallback."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    try:
        with open(os.path.join(root, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh).get("hbm_gbs", 6650.0))
    except (OSError, ValueError, TypeError):
        return 6650.0


def run_sharded_bench(args, metric: str, clock_factory=None) -> None:
    import torch
    import torch.distributed as dist
    from .device import DeviceCsr, DeviceTile, fill_tile, partition_device, plan_windows, spmm_device, spmm_plan
    from .partition import estimate_thresholds
    from . import synth

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # rank 0's stdout carries only the JSON line: whatever the communicator setup prints (the
    # NCCL version banner) is routed to stderr at the file-descriptor level
    import sys
    sys.stdout.flush()
    saved = os.dup(1)
    os.dup2(2, 1)
    try:
        dist.init_process_group("nccl", device_id=dev)
        dist.barrier()
        torch.cuda.synchronize()
    finally:
        sys.stdout.flush()
        os.dup2(saved, 1)
        os.close(saved)
    w = synth.WORKLOADS[args.workload]
    n_feat = w.n_features
    if args.workload.startswith("rmat"):
        base = 20 if args.workload == "rmat1m" else 24
        scale = base + (world.bit_length() - 1 if args.workload == "rmat1m" else 0)
        n, rp, ci, va = rmat_device(scale, 16, 0, dev)
        desc = f"R-MAT scale {scale} ef16 (device Philox draw), N={n_feat}, fp32, row-sharded over {world} GPUs"
        scaling = "weak" if args.workload == "rmat1m" else "strong"
    else:
        a = synth.workload_matrix(args.workload)
        n = a.n_rows
        rp = torch.from_numpy(np.array(a.row_ptr)).to(dev)
        ci = torch.from_numpy(np.array(a.col_idx)).to(dev)
        va = torch.from_numpy(np.array(a.values)).to(dev)
        desc = w.description + f", row-sharded over {world} GPUs"
        scaling = "strong"
    nnz = int(ci.numel())
    g = DeviceCsr(n, n, rp, ci, va)
    tn, ti = estimate_thresholds(n, nnz)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    win, res = partition_device(g, 8, tn, ti)
    win_h, res_h = win.cpu().numpy(), res.cpu().numpy()
    row_nnz = (rp[1:] - rp[:-1]).cpu().numpy()
    cuts = shard_cuts(row_nnz, allowed_cuts(win_h, res_h, n), world)
    r0, r1 = int(cuts[rank]), int(cuts[rank + 1])
    s, e = int(rp[r0].item()), int(rp[r1].item())
    loc = DeviceCsr(r1 - r0, n, (rp[r0:r1 + 1] - s).contiguous(), ci[s:e].contiguous(), va[s:e].contiguous())
    lw, lr = local_plan(win_h, res_h, r0, r1)
    lw_t = torch.from_numpy(lw.astype(np.int32)).to(dev)
    lr_t = torch.from_numpy(lr.astype(np.int32)).to(dev)
    plan = plan_windows(loc, lw_t, 8, 64)
    tile = fill_tile(loc, plan, lr_t, 8)
    tile.window_size = 8 if len(win_h) != 1 else min(8, n - int(win_h[0]))
    from .device import CHUNK_CC_LIST
    spmm_plan(tile, CHUNK_CC_LIST)  # long units + the row-major window list
    torch.cuda.synchronize()
    t_build = time.perf_counter() - t0
    del g
    # B broadcast from rank 0 (timed separately)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1)
    b = torch.empty((n, n_feat), dtype=torch.float32, device=dev)
    if rank == 0:
        b.uniform_(-1.0, 1.0, generator=gen)
    dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    dist.broadcast(b, 0)
    ev1.record()
    torch.cuda.synchronize()
    bcast_ms = ev0.elapsed_time(ev1)
    out = torch.empty((r1 - r0, n_feat), dtype=torch.float32, device=dev)
    for _ in range(args.warmup):
        spmm_device(tile, b, out=out)
    dist.barrier()
    torch.cuda.synchronize()
    clocks = clock_factory(local) if (clock_factory is not None and rank == 0) else None
    if clocks is not None:
        clocks.start()
        time.sleep(0.3)
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.time()
    g0.record()
    for _ in range(args.steps):
        spmm_device(tile, b, out=out)
    g1.record()
    torch.cuda.synchronize()
    w1 = time.time()
    clk = None
    if clocks is not None:
        clocks.window = (w0, w1)
        clk = clocks.stop()
    dist.barrier()
    local_ms = g0.elapsed_time(g1)
    tmax = torch.tensor([local_ms], dtype=torch.float64, device=dev)
    dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    total_ms = float(tmax.item())
    # C gather (timed separately)
    dist.barrier()
    torch.cuda.synchronize()
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0.record()
    full = gather_rows(out, cuts, rank, world)
    c1.record()
    torch.cuda.synchronize()
    gather_ms = c0.elapsed_time(c1)
    flops = 2.0 * nnz * n_feat
    ms = total_ms / args.steps

    # roofline: SURVEY 8(d) algorithmic bytes of this rank's shard (nnz x (4 + 4) + touched B
    # rows + C rows), summed over ranks, against world x the measured HBM bandwidth
    touched = int(torch.unique(loc.col_idx).numel()) if loc.nnz else 0
    alg = torch.tensor([loc.nnz * 8.0 + touched * n_feat * 4.0 + (r1 - r0) * n_feat * 4.0], dtype=torch.float64,
                       device=dev)
    dist.all_reduce(alg)
    alg_bytes = float(alg.item())
    peak = _hbm_peak() * world

    # end to end through the public device API with host buffers: every step copies this rank's
    # format and B in from pinned host memory and its C rows out (max over ranks)
    host = {k: getattr(tile, k).cpu().pin_memory() for k in (
        "row_window_id", "row_window_offset", "bitmaps", "col_id", "values", "res_row_id", "res_offset",
        "res_col_id", "res_values")}
    b_host = b.cpu().pin_memory()
    c_host = torch.empty(tuple(out.shape), dtype=torch.float32).pin_memory()
    dev_bufs = {k: torch.empty_like(v, device=dev) for k, v in host.items()}
    b_dev2 = torch.empty_like(b_host, device=dev)
    t2 = DeviceTile(tile.n_rows, tile.n_cols, tile.window_size, **dev_bufs)
    t2._plan = tile._plan  # the schedule is part of the prebuilt operator, like the format
    ulists = [(pl.ulist, pl.ulist.cpu().pin_memory()) for pl in (tile._plan or {}).values()
              if getattr(pl, "ulist", None) is not None]
    e2e_steps = max(1, min(args.steps, 5))
    e2e_ms = []
    for it in range(e2e_steps + 1):
        dist.barrier()
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        for k, v in host.items():
            dev_bufs[k].copy_(v, non_blocking=True)
        b_dev2.copy_(b_host, non_blocking=True)
        for dst, src in ulists:
            dst.copy_(src, non_blocking=True)
        spmm_device(t2, b_dev2, out=out)
        c_host.copy_(out, non_blocking=True)
        s1.record()
        torch.cuda.synchronize()
        if it:
            e2e_ms.append(s0.elapsed_time(s1))
    emax = torch.tensor([float(np.mean(e2e_ms))], dtype=torch.float64, device=dev)
    dist.all_reduce(emax, op=dist.ReduceOp.MAX)
    h2d = sum(v.numel() * v.element_size() for v in host.values()) + b_host.numel() * 4 + \
        sum(h.numel() * h.element_size() for _, h in ulists)
    hb = torch.tensor([float(h2d), float(c_host.numel() * 4)], dtype=torch.float64, device=dev)
    dist.all_reduce(hb)
    e2e_ms_max = float(emax.item())
    if rank == 0:
        line = {
            "metric": metric, "value": flops / (ms * 1e-3) / 1e9, "unit": "GFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": args.workload, "description": desc, "n_rows": n, "nnz": nnz,
                       "n_features": n_feat, "parallelism": f"row shard x{world}",
                       "cuts": [int(x) for x in cuts], "preprocess_ms": 1e3 * t_build,
                       "l2": "no flush: inputs exceed the 126 MB L2"},
            "gpu_launches": 3 * args.steps,  # per step: the SpMM kernel + the two long-window fix-up kernels
            "collectives": {"b_broadcast_ms": bcast_ms, "c_gather_ms": gather_ms,
                            "b_bytes": int(b.numel() * 4), "c_bytes": int(n * n_feat * 4)},
            "roofline": {"bound": "hbm", "achieved": alg_bytes / (ms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": alg_bytes / (ms * 1e-3) / 1e9 / peak, "traffic": None,
                         "algorithmic_bytes": alg_bytes, "kernel": "k_spmm_stream",
                         "peak_source": f"MEASURED_PEAKS.json hbm_gbs x {world}"},
            "e2e": {"value": flops / (e2e_ms_max * 1e-3) / 1e9, "unit": "GFLOP/s",
                    "h2d_bytes_per_step": int(hb[0].item()), "d2h_bytes_per_step": int(hb[1].item()),
                    "ms_per_step": e2e_ms_max,
                    "path": "spmm_device per rank, pinned host shard format + B in, C shard out (max over ranks)"},
            "cpu_baseline": None, "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()
