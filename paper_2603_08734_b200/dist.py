"""Multi-GPU row shard of A (north-star multi-GPU layer), one process per GPU.

The output rows of C are independent, so A is cut into contiguous row ranges, one per rank,
with cut points chosen on a prefix sum of per-row cost and snapped to rows the GLOBAL partition
scan visits (window starts and residual rows, partition.py:127-140).  The cost is SURVEY.md
8(e)'s byte model, nnz * (val + 4 + N * E_B * miss) + N * E_C per row: a nonzero streams its
(col, value) pair and gathers a B row that misses L2 with probability ``miss``; every row
writes one C row (R-MAT's low row ids are dense, so nnz-only cuts leave the C writes of the
sparse tail badly imbalanced).  No window straddles a cut, so each
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


def row_cost(row_nnz: np.ndarray, n_feat: int, b_elem: int = 4, c_elem: int = 4, miss: float = 0.35,
             val_bytes: int = 4) -> np.ndarray:
    """bytes per row = nnz * (val + 4 + N * E_B * miss) + N * E_C (float64).
    ``miss`` = fraction of B-row gathers that miss L2 (config 2 measures a 65 % L2 hit rate)."""
    nz = np.asarray(row_nnz, np.float64)
    return nz * (val_bytes + 4 + n_feat * b_elem * miss) + float(n_feat * c_elem)


def shard_cuts(cost: np.ndarray, allowed: np.ndarray, world: int) -> np.ndarray:
    """cuts[0] = 0 < ... < cuts[world] = n_rows (monotone, possibly repeated for tiny inputs):
    shard r ends at the allowed row whose prefix cost is nearest r/world of the total (cost =
    per-row bytes from ``row_cost``; an integer nnz array gives the plain nnz + 1 model)."""
    c = np.asarray(cost)
    n = int(c.size)
    if np.issubdtype(c.dtype, np.integer):
        c = c.astype(np.float64) + 1.0
    pref = np.zeros(n + 1, np.float64)
    np.cumsum(c, out=pref[1:])
    total = float(pref[-1])
    cuts = [0]
    acost = pref[allowed]
    for r in range(1, world):
        target = total * r / world
        k = int(np.searchsorted(acost, target, side="left"))
        k = min(k, allowed.size - 1)
        if k > 0 and abs(acost[k - 1] - target) < abs(acost[k] - target):
            k -= 1  # the nearer of the two allowed rows around the target
        cuts.append(max(cuts[-1], int(allowed[k])))
    cuts.append(n)
    return np.asarray(cuts, np.int64)


def shard_bytes(cost: np.ndarray, cuts: np.ndarray) -> np.ndarray:
    """Predicted bytes of every shard under the cost model."""
    pref = np.zeros(len(cost) + 1, np.float64)
    np.cumsum(np.asarray(cost, np.float64), out=pref[1:])
    return pref[np.asarray(cuts[1:])] - pref[np.asarray(cuts[:-1])]


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


def share_from_rank0(t, rank: int):
    """rank 0's CUDA tensor ``t`` mapped into every rank's address space through CUDA IPC (the
    torch.multiprocessing reduction; peer access over NVLink between GPUs, or the same device
    in another process).  Rank 0 gets ``t`` back; the others get a view of the same memory."""
    import torch.distributed as dist
    from torch.multiprocessing.reductions import reduce_tensor
    obj = [reduce_tensor(t) if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    if rank == 0:
        return t
    fn, args = obj[0]
    return fn(*args)


def spmm_rows_into(tile, b, c_full, r0: int, r1: int, **kw):
    """This rank's shard SpMM with its C rows written straight into ``c_full`` (rank 0's full C,
    possibly a peer-memory view): the epilogue's stores travel over NVLink, so no separate C
    gather follows.  Rows [r0, r1) of c_full receive the shard's rows."""
    from .device import spmm_device
    return spmm_device(tile, b, out=c_full[r0:r1], **kw)


# ---------------------------------------------------------------------------------------------
# device shard build (one rank's part of the global format)
# ---------------------------------------------------------------------------------------------

def global_window_size(win_h: np.ndarray, n_rows: int, window_size: int = 8) -> int:
    """tile.py:169-173 for the GLOBAL plan: every shard format carries the global value."""
    if len(win_h) == 0:
        return 8
    if len(win_h) >= 2:
        return window_size
    return min(window_size, n_rows - int(win_h[0]))


def build_shard(g, win_h: np.ndarray, res_h: np.ndarray, r0: int, r1: int, window_size: int = 8,
                max_blocks_per_item=64):
    """Rows [r0, r1) of the global CSR ``g`` (a DeviceCsr) as a local DeviceCsr and its RS-Tile:
    the global partition's windows / residual rows in the range, rebased, built by the device
    builder with the global parameters.  Column ids stay global (B is replicated)."""
    import torch
    from .device import DeviceCsr, fill_tile, plan_windows
    dev = g.device
    rp = g.row_ptr
    s, e = int(rp[r0].item()), int(rp[r1].item())
    loc = DeviceCsr(r1 - r0, g.n_cols, (rp[r0:r1 + 1] - s).contiguous(), g.col_idx[s:e].contiguous(),
                    g.values[s:e].contiguous())
    lw, lr = local_plan(win_h, res_h, r0, r1)
    lw_t = torch.from_numpy(lw.astype(np.int32)).to(dev)
    lr_t = torch.from_numpy(lr.astype(np.int32)).to(dev)
    plan = plan_windows(loc, lw_t, window_size, max_blocks_per_item)
    tile = fill_tile(loc, plan, lr_t, window_size)
    tile.window_size = global_window_size(win_h, g.n_rows, window_size)
    return loc, tile


def plan_shards(g, world: int, n_feat: int, b_elem: int = 4, miss: float = 0.35, window_size: int = 8):
    """Global partition on device, then cost-model cuts snapped to scan-visited rows.  Returns
    (win_h, res_h, cuts, predicted bytes per shard)."""
    from .device import partition_device
    from .partition import estimate_thresholds
    tn, ti = estimate_thresholds(g.n_rows, g.nnz) if g.n_rows else (0, 0)
    win, res = partition_device(g, window_size, tn, ti)
    win_h, res_h = win.cpu().numpy(), res.cpu().numpy()
    row_nnz = (g.row_ptr[1:] - g.row_ptr[:-1]).cpu().numpy()
    cost = row_cost(row_nnz, n_feat, b_elem, 4, miss)
    cuts = shard_cuts(cost, allowed_cuts(win_h, res_h, g.n_rows), world)
    return win_h, res_h, cuts, shard_bytes(cost, cuts)


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


def sharded_workload(name: str, world: int) -> tuple[str, str]:
    """(matrix name, scaling): rmat1m weak-scales as R-MAT scale 20 + log2(world) (the per-GPU
    share stays config-2-sized); every other workload is a fixed matrix (strong scaling)."""
    if name == "rmat1m" and world > 1:
        return f"rmat_s{20 + (world.bit_length() - 1)}", "weak"
    return name, ("weak" if name == "rmat1m" else "strong")


def _broadcast_csr(rank: int, dev, name: str):
    """Rank 0 draws the workload (synth, the SURVEY Appendix B recipe) and broadcasts the CSR."""
    import torch
    import torch.distributed as dist
    from . import synth
    from .device import DeviceCsr
    if rank == 0:
        a = synth.workload_matrix(name)
        meta = torch.tensor([a.n_rows, a.n_cols, a.nnz], dtype=torch.int64, device=dev)
        rp = torch.from_numpy(np.array(a.row_ptr)).to(dev)
        ci = torch.from_numpy(np.array(a.col_idx)).to(dev)
        va = torch.from_numpy(np.array(a.values)).to(dev)
    else:
        meta = torch.empty(3, dtype=torch.int64, device=dev)
    dist.broadcast(meta, 0)
    n, nc, nnz = (int(x) for x in meta.cpu())
    if rank != 0:
        rp = torch.empty(n + 1, dtype=torch.int64, device=dev)
        ci = torch.empty(nnz, dtype=torch.int32, device=dev)
        va = torch.empty(nnz, dtype=torch.float32, device=dev)
    for t in (rp, ci, va):
        dist.broadcast(t, 0)
    return DeviceCsr(n, nc, rp, ci, va)


def run_sharded_bench(args, metric: str, clock_factory=None, config_factory=None) -> None:
    import torch
    import torch.distributed as dist
    from . import _lib, synth
    from .device import CHUNK_CC_LIST, spmm_device, spmm_plan

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
    name, scaling = sharded_workload(args.workload, world)
    w = synth.workload_spec(name)
    n_feat = w.n_features
    b_elem = 2 if w.dtype == "bf16" else 4
    g = _broadcast_csr(rank, dev, name)
    n, nnz = g.n_rows, g.nnz
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    win_h, res_h, cuts, pred = plan_shards(g, world, n_feat, b_elem)
    r0, r1 = int(cuts[rank]), int(cuts[rank + 1])
    loc, tile = build_shard(g, win_h, res_h, r0, r1)
    plan = spmm_plan(tile, CHUNK_CC_LIST)  # long units + the row-major window list
    torch.cuda.synchronize()
    t_build = time.perf_counter() - t0
    # B broadcast from rank 0 (timed separately); U(-1, 1) drawn on rank 0's device
    gen = torch.Generator(device=dev)
    gen.manual_seed(1)
    b = torch.empty((n, n_feat), dtype=torch.float32, device=dev)
    if rank == 0:
        b.uniform_(-1.0, 1.0, generator=gen)
    if b_elem == 2:
        b = b.to(torch.bfloat16)
    dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    dist.broadcast(b, 0)
    ev1.record()
    torch.cuda.synchronize()
    bcast_ms = ev0.elapsed_time(ev1)
    out = torch.empty((r1 - r0, n_feat), dtype=torch.float32, device=dev)
    # --p2p-gather: every rank's SpMM writes its C rows straight into rank 0's C over peer memory
    # (CUDA IPC), so no gather follows; any failure to map the buffer falls back to NCCL
    c_peer, p2p_note = None, None
    if getattr(args, "p2p_gather", False) and world > 1:
        try:
            c_full = torch.empty((n, n_feat), dtype=torch.float32, device=dev) if rank == 0 else None
            c_peer = share_from_rank0(c_full, rank)
            p2p_note = "C rows stored by each rank's SpMM epilogue into rank 0's buffer over peer memory"
        except Exception as exc:  # noqa: BLE001 -- the NCCL gather below still works
            c_peer, p2p_note = None, f"peer mapping failed ({type(exc).__name__}); NCCL gather"
        ok = torch.tensor([0.0 if c_peer is None else 1.0], device=dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if ok.item() < 1.0:
            c_peer = None
    if c_peer is not None:
        out = c_peer[r0:r1]
    for _ in range(args.warmup):
        spmm_device(tile, b, out=out)
    dist.barrier()
    torch.cuda.synchronize()
    clocks = clock_factory(local) if (clock_factory is not None and rank == 0) else None
    if clocks is not None:
        clocks.start()
        time.sleep(0.3)
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n_launch0 = int(_lib.lib().rsh_launch_count())
    w0 = time.time()
    g0.record()
    for _ in range(args.steps):
        spmm_device(tile, b, out=out)
    g1.record()
    torch.cuda.synchronize()
    w1 = time.time()
    launches = int(_lib.lib().rsh_launch_count()) - n_launch0
    clk = None
    if clocks is not None:
        clocks.window = (w0, w1)
        clk = clocks.stop()
    dist.barrier()
    local_ms = g0.elapsed_time(g1)
    tmax = torch.tensor([local_ms, float(launches)], dtype=torch.float64, device=dev)
    lsum = torch.tensor([float(launches)], dtype=torch.float64, device=dev)
    dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    dist.all_reduce(lsum)
    total_ms = float(tmax[0].item())
    # C gather (timed separately)
    dist.barrier()
    torch.cuda.synchronize()
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0.record()
    if c_peer is None:
        gather_rows(out, cuts, rank, world)
    c1.record()
    torch.cuda.synchronize()
    gather_ms = c0.elapsed_time(c1)
    flops = 2.0 * nnz * n_feat
    ms = total_ms / args.steps

    # roofline: SURVEY 8(d) algorithmic bytes of this rank's shard (nnz x (val + 4) + touched B
    # rows + C rows), summed over ranks, against world x the measured HBM bandwidth
    touched = int(torch.unique(loc.col_idx).numel()) if loc.nnz else 0
    alg = torch.tensor([loc.nnz * (4.0 + b_elem) + touched * n_feat * b_elem + (r1 - r0) * n_feat * 4.0],
                       dtype=torch.float64, device=dev)
    dist.all_reduce(alg)
    alg_bytes = float(alg.item())
    peak = _hbm_peak() * world

    # end to end with host buffers (device.HostStream): every step copies this rank's format and B
    # in from pinned host memory, builds the schedule, runs the SpMM and copies its C rows out,
    # steps pipelined over three streams (max over ranks)
    from .device import TILE_HOST_FIELDS, HostStream
    hs = HostStream({k: getattr(tile, k).cpu().pin_memory() for k in TILE_HOST_FIELDS}, b.cpu().pin_memory(),
                    tile.n_rows, tile.n_cols, tile.window_size, dev)
    e2e_steps = max(2, int(getattr(args, "e2e_steps", 24)))
    hs.run(2)
    dist.barrier()
    e2e_ms = [hs.run(e2e_steps)]
    h2d = hs.h2d_bytes
    emax = torch.tensor([float(np.mean(e2e_ms))], dtype=torch.float64, device=dev)
    dist.all_reduce(emax, op=dist.ReduceOp.MAX)
    hb = torch.tensor([float(h2d), float(hs.d2h_bytes)], dtype=torch.float64, device=dev)
    dist.all_reduce(hb)
    e2e_ms_max = float(emax.item())
    if rank == 0:
        class _A:  # the workload the reference arm prints for the same launch
            workload = name
        if config_factory is not None:
            config = config_factory(_A, g, w)
        else:
            config = {"workload": name, "description": w.description, "n_rows": n, "n_cols": g.n_cols,
                      "nnz": nnz, "n_features": n_feat, "parallelism": f"row shard x{world}"}
        line = {
            "metric": metric, "value": flops / (ms * 1e-3) / 1e9, "unit": "GFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "bf16" if b_elem == 2 else "f32", "data": "synthetic",
            "config": config,
            "details": {"cuts": [int(x) for x in cuts], "preprocess_ms": 1e3 * t_build,
                        "shard_bytes_predicted": [float(x) for x in pred],
                        "shard_bytes_max_over_mean": float(pred.max() / max(pred.mean(), 1.0)),
                        "cost_model": "nnz*(4+4+N*E_B*0.35) + N*E_C per row (SURVEY 8(e))",
                        "b_values": "U(-1,1) drawn on rank 0's device, broadcast"},
            "gpu_launches": int(lsum.item()),
            "collectives": {"b_broadcast_ms": bcast_ms, "c_gather_ms": gather_ms,
                            "c_placement": p2p_note or "NCCL point-to-point gather to rank 0",
                            "b_bytes": int(b.numel() * b.element_size()), "c_bytes": int(n * n_feat * 4)},
            "roofline": {"bound": "hbm", "achieved": alg_bytes / (ms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": alg_bytes / (ms * 1e-3) / 1e9 / peak, "traffic": None,
                         "algorithmic_bytes": alg_bytes, "kernel": "k_spmm_stream",
                         "peak_source": f"MEASURED_PEAKS.json hbm_gbs x {world}"},
            "e2e": {"value": flops / (e2e_ms_max * 1e-3) / 1e9, "unit": "GFLOP/s",
                    "h2d_bytes_per_step": int(hb[0].item()), "d2h_bytes_per_step": int(hb[1].item()),
                    "ms_per_step": e2e_ms_max,
                    "path": "device.HostStream per rank: pinned host shard format + B in, schedule build, "
                            "SpMM, C shard out, steps pipelined on 3 streams (max over ranks)"},
            "cpu_baseline": None, "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    del plan
    dist.barrier()
    dist.destroy_process_group()
