"""Golden .rst files: run the REFERENCE's save_rstile / storage_report (tile.py:314-388,
410-440) over seeded matrices and record the SHA-256 of every file's bytes plus its storage
report.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_rst_golden.py

Output: rst_cases.json.  Only this script touches the reference.
"""

from __future__ import annotations

import dataclasses
import hashlib
import json
import os
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from rstile import partition, tile  # noqa: E402  (the reference)
from rstile.core import CsrMatrix as RefCsr  # noqa: E402

from paper_2603_08734_b200 import synth  # noqa: E402

from oracle import corpus  # noqa: E402

CASES = [
    ("small0", {"kind": "small_corpus", "index": 0}, {}),
    ("small5", {"kind": "small_corpus", "index": 5}, {}),
    ("small11_tc", {"kind": "small_corpus", "index": 11}, {"tau_nnz": 0}),
    ("small17_bound2", {"kind": "small_corpus", "index": 17}, {"max_blocks_per_item": 2}),
    ("small23_w5", {"kind": "small_corpus", "index": 23}, {"window_size": 5}),
    ("power300", {"kind": "power_law", "args": [300, 280, 4000, 1.4, 7]}, {}),
    ("power2k", {"kind": "power_law", "args": [2048, 1536, 30000, 1.5, 1]}, {}),
    ("rmat12", {"kind": "rmat", "args": [12, 16, 0]}, {}),
    ("rmat12_resid", {"kind": "rmat", "args": [12, 16, 0]}, {"tau_nnz": 10 ** 6, "tau_inc": 10 ** 6}),
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
    for name, recipe, params in CASES:
        a = matrix(recipe, small)
        ra = RefCsr(a.n_rows, a.n_cols, a.row_ptr, a.col_idx, a.values)
        p = partition.PartitionParams(**params)
        m = tile.build_rstile(ra, partition.split_long_work(ra, partition.partition_rows(ra, p), p))
        with tempfile.TemporaryDirectory() as d:
            path = os.path.join(d, "m.rst")
            tile.save_rstile(path, m)
            blob = open(path, "rb").read()
        out.append({"case": name, "recipe": recipe, "params": params, "bytes": len(blob),
                    "sha256": hashlib.sha256(blob).hexdigest(),
                    "storage": dataclasses.asdict(tile.storage_report(ra, m))})
    with open(os.path.join(HERE, "rst_cases.json"), "w") as fh:
        json.dump({"header_bytes": tile.HEADER_BYTES, "cases": out}, fh, indent=1)
    print(f"{len(out)} cases, header {tile.HEADER_BYTES} bytes")


if __name__ == "__main__":
    main()
