"""Golden reorder fixtures from the REFERENCE (reorder.py): column weights, the kNN graph, the
MST-stage order and objective, the 2-opt and pipeline objectives, and the objective of a seeded
random order, over small seeded matrices.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_reorder_golden.py

Output: reorder_cases.json.  Only this script touches the reference.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from rstile import reorder as R  # noqa: E402  (the reference)
from rstile.core import CsrMatrix as RefCsr  # noqa: E402

from paper_2603_08734_b200 import synth  # noqa: E402

from oracle import corpus  # noqa: E402

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
    out = []
    for name, recipe in CASES:
        a = matrix(recipe, small)
        ra = RefCsr(a.n_rows, a.n_cols, a.row_ptr, a.col_idx, a.values)
        p = R.ReorderParams()
        w = R.column_weights(ra, p.alpha)
        cand = R.build_candidates(ra, p.max_candidates)
        g = R.build_knn(ra, w, cand, p.k)
        mst = R.mst_order(g, ra, w)
        ref2 = R.refine_2opt(ra, w, mst, p.two_opt_window, p.two_opt_passes)
        iso = R.isolation_adjust(ra, w, ref2, p.iso_threshold)
        best, _ = R.reorder_pipeline(ra, p)
        rnd = np.random.default_rng(5).permutation(a.n_rows)
        out.append({
            "case": name, "recipe": recipe, "n_rows": a.n_rows,
            "weights": [float(x) for x in w.weights],
            "knn": [[[int(u), float(s)] for u, s in lst] for lst in g.neighbors],
            "max_candidates_hit": int(sum(len(c) >= p.max_candidates for c in cand)),
            "mst_order": [int(x) for x in mst.order], "mst_objective": mst.objective,
            "two_opt_order": [int(x) for x in ref2.order], "two_opt_objective": ref2.objective,
            "isolation_order": [int(x) for x in iso.order], "isolation_objective": iso.objective,
            "pipeline_objective": best.objective,
            "random_order": [int(x) for x in rnd], "random_objective": R.permutation_objective(ra, w, rnd),
        })
        print(name, a.n_rows, mst.objective, ref2.objective, best.objective)
    with open(os.path.join(HERE, "reorder_cases.json"), "w") as fh:
        json.dump(out, fh)


if __name__ == "__main__":
    main()
