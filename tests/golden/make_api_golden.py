"""Golden fixtures from the REFERENCE for the drop-in API functions added in round 2:
build_candidates (reorder.py:168-194), tile_density / threshold_sweep (metrics.py:28-78) and
oracle_spmm (core.py:380-395), over small seeded matrices.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_api_golden.py

Output: api_cases.json (+ api_oracle.npz: oracle_spmm outputs).  Only this script touches the
reference.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from rstile import metrics as M  # noqa: E402  (the reference)
from rstile import reorder as R  # noqa: E402
from rstile.core import CsrMatrix as RefCsr, DenseMatrix as RefDense, oracle_spmm  # noqa: E402
from rstile.partition import PartitionParams, partition_rows, split_long_work  # noqa: E402
from rstile.tile import build_rstile  # noqa: E402

from oracle import corpus  # noqa: E402
from paper_2603_08734_b200 import synth  # noqa: E402

CASES = [
    ("small3", {"kind": "small_corpus", "index": 3}),
    ("small8", {"kind": "small_corpus", "index": 8}),
    ("small14", {"kind": "small_corpus", "index": 14}),
    ("small20", {"kind": "small_corpus", "index": 20}),
    ("power200", {"kind": "power_law", "args": [200, 180, 1500, 1.4, 3]}),
    ("power400", {"kind": "power_law", "args": [400, 300, 3000, 1.6, 9]}),
    ("rmat9", {"kind": "rmat", "args": [9, 8, 0]}),
]


def matrix(recipe, small):
    if recipe["kind"] == "small_corpus":
        return small[recipe["index"]]
    if recipe["kind"] == "power_law":
        return corpus.generate_power_law(*recipe["args"])
    return synth.rmat(*recipe["args"])


def main():
    small = corpus.small_corpus()
    out, arrays = [], {}
    for name, recipe in CASES:
        a0 = matrix(recipe, small)
        a = RefCsr(a0.n_rows, a0.n_cols, np.asarray(a0.row_ptr), np.asarray(a0.col_idx), np.asarray(a0.values))
        case = {"name": name, "recipe": recipe}
        case["candidates"] = {str(mc): [c.tolist() for c in R.build_candidates(a, mc)] for mc in (256, 8)}
        p = PartitionParams()
        m = build_rstile(a, split_long_work(a, partition_rows(a, p), p))
        case["tile_density"] = M.tile_density(m).__dict__
        case["threshold_sweep"] = [[t, rep.__dict__] for t, rep in M.threshold_sweep(a, [0, 2, 4, 6])]
        case["sweep_csv"] = M.sweep_csv(M.threshold_sweep(a, [0, 4]))
        b = np.random.default_rng(len(name)).uniform(-1, 1, (a.n_cols, 24)).astype(np.float32)
        arrays[f"{name}_b"] = b
        arrays[f"{name}_c"] = oracle_spmm(a, RefDense.from_array(b)).data
        out.append(case)
    with open(os.path.join(HERE, "api_cases.json"), "w") as fh:
        json.dump(out, fh)
    np.savez_compressed(os.path.join(HERE, "api_oracle.npz"), **arrays)
    print(f"wrote {len(out)} cases")


if __name__ == "__main__":
    main()
