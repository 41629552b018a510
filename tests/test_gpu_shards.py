"""GPU, one process: the multi-GPU row-shard build (dist.py) for world 2 / 4 / 8 on one device.

Exactly the code each rank runs -- global partition on device (partition_device), SURVEY 8(e)
cost-model cuts snapped to scan-visited rows (plan_shards), then the per-rank device build on
the local CSR (build_shard: plan_windows + fill_tile with the global parameters) and the
streaming SpMM -- executed here for every rank in turn.  Checks:

* the shard formats concatenate (row ids / offsets rebased) to the global device format, bit
  for bit (execute.py:163,181-193: every row is owned by exactly one window or residual entry);
* the shard products concatenate to the single-GPU C, bit for bit (the per-row arithmetic
  order does not depend on the shard);
* the cost model keeps the heaviest shard within 5 % of the mean predicted bytes.
"""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

FIELDS = ("row_window_id", "row_window_offset", "bitmaps", "col_id", "values", "res_row_id", "res_offset",
          "res_col_id", "res_values")


def _concat(shards):
    out = {k: [] for k in FIELDS}
    off, roff = [np.zeros(1, np.int64)], [np.zeros(1, np.int64)]
    ob = orr = 0
    for r0, h in shards:
        out["row_window_id"].append(h["row_window_id"] + r0)
        off.append(h["row_window_offset"][1:] + ob)
        ob += int(h["row_window_offset"][-1])
        out["bitmaps"].append(h["bitmaps"])
        out["col_id"].append(h["col_id"])
        out["values"].append(h["values"])
        out["res_row_id"].append(h["res_row_id"] + r0)
        roff.append(h["res_offset"][1:] + orr)
        orr += int(h["res_offset"][-1])
        out["res_col_id"].append(h["res_col_id"])
        out["res_values"].append(h["res_values"])
    res = {k: np.concatenate(v) for k, v in out.items() if v}
    res["row_window_offset"] = np.concatenate(off)
    res["res_offset"] = np.concatenate(roff)
    return res


def _matrices():
    from paper_2603_08734_b200 import synth
    from oracle import corpus
    yield "rmat16", synth.rmat(16, 16, 0), 128
    yield "rmat1m", synth.workload_matrix("rmat1m"), 128
    yield "powerlaw", corpus.generate_power_law(20000, 15000, 400000, 1.4, seed=31), 64


@pytest.mark.parametrize("world", [2, 4, 8])
def test_device_shards_concatenate_to_global(world):
    from paper_2603_08734_b200 import dist as D
    from paper_2603_08734_b200.device import DeviceCsr, build_device, spmm_device
    for name, a, n_feat in _matrices():
        g = DeviceCsr.from_host(a)
        glob = build_device(g)
        b = torch.from_numpy(np.random.default_rng(5).uniform(-1, 1, (a.n_cols, n_feat)).astype(np.float32)).cuda()
        c1 = spmm_device(glob, b)
        win_h, res_h, cuts, pred = D.plan_shards(g, world, n_feat)
        assert cuts[0] == 0 and cuts[-1] == a.n_rows and list(cuts) == sorted(cuts)
        if a.n_rows > 100_000:
            assert pred.max() / pred.mean() <= 1.05, (name, world, pred / pred.mean())
        shards, cparts = [], []
        for rank in range(world):
            r0, r1 = int(cuts[rank]), int(cuts[rank + 1])
            if r1 == r0:
                continue
            loc, tile = D.build_shard(g, win_h, res_h, r0, r1)
            assert tile.window_size == glob.window_size
            shards.append((r0, tile.host_arrays()))
            cparts.append(spmm_device(tile, b))
        cat = _concat(shards)
        want = glob.host_arrays()
        for k in FIELDS:
            assert np.array_equal(cat[k], want[k]), (name, world, k)
        c_sh = torch.cat(cparts, 0)
        assert c_sh.shape == c1.shape
        assert torch.equal(c_sh, c1), (name, world)
        del glob, c1, c_sh, cparts
        torch.cuda.empty_cache()
