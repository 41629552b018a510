"""Generate the golden fixtures by running the REFERENCE package itself (rstile 0.1.0).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Only this script touches /root/reference; its outputs are committed so that the CPU and GPU
test suites (which run where the reference does not exist) are pinned to the reference's own
results:

* known_answers.json  -- the known-answer cases of the reference's tests (test_tile.py,
  test_partition.py, test_execute.py) with the reference's outputs;
* formats.json        -- SHA-256 digests of every array the reference pipeline
  (partition_rows -> split_long_work -> build_rstile) produces over seeded corpora and
  parameter sets, plus digests of the generated inputs themselves;
* small_spmm.npz      -- oracle_spmm outputs of the reference on the 24-matrix small corpus.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import rstile  # noqa: E402  (the reference; PYTHONPATH=/root/reference/pkg/src)
from rstile import core, partition, tile  # noqa: E402

from paper_2603_08734_b200 import synth  # noqa: E402

from oracle import corpus  # noqa: E402

PARAM_SETS = {
    "default": {},
    "tc_only": {"tau_nnz": 0},
    "tau43": {"tau_nnz": 4, "tau_inc": 3},
    "w5": {"window_size": 5},
    "w3_tau0": {"window_size": 3, "tau_nnz": 0},
    "bound2": {"max_blocks_per_item": 2},
    "bound1_tc": {"max_blocks_per_item": 1, "tau_nnz": 0},
    "rownnz": {"split_on_row_nnz": True, "max_blocks_per_item": None},
    "unbounded": {"max_blocks_per_item": None},
    "all_resid": {"tau_nnz": 10 ** 6, "tau_inc": 10 ** 6},
}


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def csr_digest(a) -> str:
    return digest(np.array([a.n_rows, a.n_cols]), a.row_ptr, a.col_idx, a.values)


def format_record(a, params: dict) -> dict:
    p = partition.PartitionParams(**params)
    plan = partition.partition_rows(a, p)
    split = partition.split_long_work(a, plan, p)
    m = tile.build_rstile(a, split)
    wins = np.array(plan.windows, dtype=np.int64).reshape(-1, 2)
    smap = sorted((int(k), [list(s) for s in v]) for k, v in split.split_map.items())
    return {
        "windows": digest(wins),
        "residual": digest(plan.residual_rows),
        "split_map": hashlib.sha256(json.dumps(smap).encode()).hexdigest(),
        "n_windows": len(plan.windows),
        "n_residual": int(plan.residual_rows.size),
        "n_entries": m.tc.n_entries,
        "n_blocks": m.tc.n_blocks,
        "window_size": m.window_size,
        "arrays": {
            "row_window_id": digest(m.tc.row_window_id),
            "row_window_offset": digest(m.tc.row_window_offset),
            "bitmaps": digest(m.tc.bitmaps),
            "col_id": digest(m.tc.col_id),
            "values": digest(m.tc.values),
            "res_row_id": digest(m.residual.row_id),
            "res_offset": digest(m.residual.row_nnz_offset),
            "res_col_id": digest(m.residual.col_id),
            "res_values": digest(m.residual.values),
        },
    }


def corpus_matrices():
    """name -> (recipe, CsrMatrix) for every corpus the digests cover."""
    out = {}
    for i, a in enumerate(corpus.small_corpus()):
        out[f"small{i:02d}"] = ({"kind": "small_corpus", "index": i}, a)
    for j, (nr, nc, nnz, skew, seed, _d) in enumerate(corpus.acceptance_cases()):
        if j % 4 == 0 or nr >= 2048:  # a quarter of the 200-matrix corpus plus all large ones
            out[f"accept{j:03d}"] = ({"kind": "power_law", "args": [nr, nc, nnz, skew, seed]},
                                     corpus.generate_power_law(nr, nc, nnz, skew, seed))
    for s in (12, 14, 16):
        out[f"rmat{s}"] = ({"kind": "rmat", "args": [s, 16, 0]}, synth.rmat(s, 16, 0))
    return out


def known_answers() -> list[dict]:
    cases = []

    def dense_case(name, dense, params, spmm_d=None, b_seed=0):
        a = core.CsrMatrix.from_dense(np.asarray(dense, dtype=np.float32))
        rec = {"name": name, "dense": np.asarray(dense, dtype=np.float32).tolist(), "params": params}
        rec.update(format_record(a, params))
        p = partition.PartitionParams(**params)
        plan = partition.split_long_work(a, partition.partition_rows(a, p), p)
        m = tile.build_rstile(a, plan)
        rec["plan_windows"] = [list(w) for w in plan.windows]
        rec["plan_residual"] = plan.residual_rows.tolist()
        rec["plan_split_map"] = {str(k): [list(s) for s in v] for k, v in plan.split_map.items()}
        rec["tc"] = {"row_window_id": m.tc.row_window_id.tolist(),
                     "row_window_offset": m.tc.row_window_offset.tolist(),
                     "bitmaps": [str(int(x)) for x in m.tc.bitmaps],
                     "col_id": m.tc.col_id.tolist(), "values": m.tc.values.tolist()}
        rec["residual_rows"] = m.residual.row_id.tolist()
        if spmm_d:
            b = np.random.default_rng(b_seed).uniform(-1, 1, (a.n_cols, spmm_d)).astype(np.float32)
            rec["b"] = b.tolist()
            rec["c_f32"] = rstile.hybrid_spmm(m, core.DenseMatrix.from_array(b)).data.tolist()
            rec["c_f64"] = rstile.hybrid_spmm(
                m, core.DenseMatrix.from_array(b), rstile.ExecConfig(accumulate_precision="f64")).data.tolist()
        cases.append(rec)

    one = np.zeros((1, 8)); one[0, 5] = 2.5
    dense_case("single_entry_block", one, {"tau_nnz": 0})
    dense_case("full_block", np.ones((8, 8)), {"tau_nnz": 0}, spmm_d=5)
    dense_case("diagonal_pair", [[3.0, 0.0], [0.0, 4.0]], {"tau_nnz": 0})
    dense_case("off_diagonal_order", [[0.0, 7.0], [5.0, 0.0]], {"tau_nnz": 0})
    pad = np.zeros((2, 16)); pad[0, [0, 4]] = 1.0; pad[1, 9] = 1.0
    dense_case("padding_slots", pad, {"tau_nnz": 0})
    comp = np.zeros((8, 64))
    for i, c in enumerate([3, 17, 40, 41, 42, 50, 61, 62, 63]):
        comp[i % 8, c] = float(i + 1)
    dense_case("compaction", comp, {"tau_nnz": 0}, spmm_d=7)
    wide = np.ones((1, 1037))
    dense_case("split_1037", wide, {"tau_nnz": 0, "max_blocks_per_item": 64}, spmm_d=3)
    dense_case("split_1037_unbounded", wide, {"tau_nnz": 0, "max_blocks_per_item": None}, spmm_d=3)
    dense_case("dense_20x16", np.ones((20, 16)), {}, spmm_d=4)
    thin = np.zeros((9, 16))
    for i in range(8):
        thin[i, [2 * i, 2 * i + 1]] = float(i + 1)
    thin[8, 0] = 99.0
    dense_case("thin_trailing_row", thin, {"tau_nnz": 2, "tau_inc": 2}, spmm_d=6)
    gaps = np.zeros((5, 6)); gaps[1, :3] = 1; gaps[4, 3:] = 1
    dense_case("empty_rows_skipped", gaps, {"tau_nnz": 0}, spmm_d=2)
    dense_case("identity16_residual", np.eye(16), {}, spmm_d=4)
    dense_case("identity16_window", np.eye(16), {"tau_nnz": 0}, spmm_d=4)
    unc = np.zeros((20, 16)); unc[:8] = 1.0; unc[19, 0] = 5.0
    dense_case("uncovered_rows_zero", unc, {}, spmm_d=3)
    dense_case("residual_only_4x4", np.diag([0, 0, 0, 2.0]), {}, spmm_d=2)
    dense_case("all_empty", np.zeros((10, 10)), {}, spmm_d=2)
    canc = np.zeros((1, 4)); canc[0] = [2.0 ** 24, 1.0, 1.0, -(2.0 ** 24)]
    a = core.CsrMatrix.from_dense(canc.astype(np.float32))
    m = tile.build_rstile(a, partition.partition_rows(a, partition.PartitionParams(tau_nnz=0)))
    ones = core.DenseMatrix.from_array(np.ones((4, 1), np.float32))
    cases.append({"name": "cancellation", "dense": canc.tolist(), "params": {"tau_nnz": 0},
                  "c_f64": rstile.hybrid_spmm(m, ones, rstile.ExecConfig(accumulate_precision="f64")).data.tolist(),
                  "c_f32": rstile.hybrid_spmm(m, ones).data.tolist()})
    # thresholds and column increments (test_partition.py:31-80)
    cases.append({"name": "thresholds", "cases": [[n, z, list(partition.estimate_thresholds(n, z))]
                                                  for n, z in ((10, 80), (10, 10), (10, 1000), (7, 70), (4, 36),
                                                               (1000, 9000), (3, 15))]})
    incs = []
    for sup, ncol, r, w in (([set(), {0, 1}], 2, 0, 8), ([{0, 3, 7}], 8, 0, 8), ([{1, 2}, {2, 3}, {3, 4}], 5, 0, 3),
                            ([{0, 1}, {0, 1, 2}], 3, 0, 2), ([{0, 1, 5}, {5}, set(), {1}], 6, 0, 8),
                            ([{0, 1, 5}, {5}, set(), {1}], 6, 0, 3)):
        d = np.zeros((len(sup), ncol), np.float32)
        for i, cs in enumerate(sup):
            d[i, list(cs)] = 1.0
        aa = core.CsrMatrix.from_dense(d)
        incs.append({"dense": d.tolist(), "r": r, "w": w, "delta": partition.column_increment(aa, r, w)})
    cases.append({"name": "column_increment", "cases": incs})
    return cases


def main() -> None:
    mats = corpus_matrices()
    formats = {"reference": f"rstile {rstile.__version__}", "param_sets": PARAM_SETS, "matrices": {}}
    for name, (recipe, a) in mats.items():
        ref_a = core.CsrMatrix(a.n_rows, a.n_cols, a.row_ptr, a.col_idx, a.values)
        entry = {"recipe": recipe, "input": csr_digest(ref_a), "nnz": ref_a.nnz, "formats": {}}
        sets = PARAM_SETS if name.startswith("small") else (
            {k: PARAM_SETS[k] for k in ("default", "bound2")} if ref_a.nnz < 300_000 else {"default": {}})
        for pname, params in sets.items():
            entry["formats"][pname] = format_record(ref_a, params)
        formats["matrices"][name] = entry
        print(name, ref_a.n_rows, ref_a.nnz, flush=True)
    with open(os.path.join(HERE, "formats.json"), "w") as fh:
        json.dump(formats, fh, indent=1, sort_keys=True)
    with open(os.path.join(HERE, "known_answers.json"), "w") as fh:
        json.dump(known_answers(), fh)
    spmm = {}
    for i, a in enumerate(corpus.small_corpus()):
        ref_a = core.CsrMatrix(a.n_rows, a.n_cols, a.row_ptr, a.col_idx, a.values)
        b = np.random.default_rng(a.nnz).uniform(-1, 1, (a.n_cols, 16)).astype(np.float32)
        spmm[f"c{i:02d}"] = core.oracle_spmm(ref_a, core.DenseMatrix.from_array(b)).data
    np.savez_compressed(os.path.join(HERE, "small_spmm.npz"), **spmm)


if __name__ == "__main__":
    main()
