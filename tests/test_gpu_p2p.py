"""GPU, two processes on one device: the B200-first C placement of the row-shard layer.  Each
rank's shard SpMM writes its C rows straight into rank 0's buffer through CUDA IPC (dist.
share_from_rank0 + spmm_rows_into) -- over NVLink between GPUs, the same device here -- and
the assembled C equals the single-process product bit for bit.  The handle exchange runs on
gloo, so the test needs one GPU only."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, world: int, port: int, outdir: str) -> None:
    import torch.distributed as dist

    from paper_2603_08734_b200 import dist as D
    from paper_2603_08734_b200 import synth
    from paper_2603_08734_b200.device import DeviceCsr, build_device, spmm_device
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    a = synth.rmat(14, 16, 0)
    g = DeviceCsr.from_host(a)
    n_feat = 64
    b = torch.from_numpy(np.random.default_rng(3).uniform(-1, 1, (a.n_cols, n_feat)).astype(np.float32)).cuda()
    win_h, res_h, cuts, _ = D.plan_shards(g, world, n_feat)
    r0, r1 = int(cuts[rank]), int(cuts[rank + 1])
    _, tile = D.build_shard(g, win_h, res_h, r0, r1)
    c_full = torch.full((a.n_rows, n_feat), float("nan"), device="cuda") if rank == 0 else None
    c_peer = D.share_from_rank0(c_full, rank)
    D.spmm_rows_into(tile, b, c_peer, r0, r1)
    torch.cuda.synchronize()
    dist.barrier()
    if rank == 0:
        ref = spmm_device(build_device(g), b)
        same = bool(torch.equal(c_full, ref))
        with open(os.path.join(outdir, "result.txt"), "w") as fh:
            fh.write(f"{int(same)} {r0} {r1} {int(cuts[-1])}\n")
    dist.barrier()
    dist.destroy_process_group()


def test_shards_write_c_into_rank0_buffer_over_ipc(tmp_path):
    import torch.multiprocessing as mp
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    same, r0, r1, n = open(tmp_path / "result.txt").read().split()
    assert int(r1) < int(n)  # rank 1 owned rows: its stores crossed processes
    assert same == "1"
