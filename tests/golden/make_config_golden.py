"""Full-size BASELINE configs pinned to the REFERENCE itself (rstile 0.1.0).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_config_golden.py [names...]

For each workload matrix (synth.workload_matrix; input digest recorded),
runs the reference's own partition_rows -> split_long_work -> build_rstile with default
parameters and writes SHA-256 digests of all nine format arrays (plus counts) to
tests/golden/config_formats.json.  tests/test_gpu_configs.py compares the DEVICE-built format
of the same matrix against these digests, so the full-size formats are pinned to the
reference and not only to the oracle restatement.  Only this script touches the reference.
"""

from __future__ import annotations

import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, HERE)

import rstile  # noqa: E402  (the reference; PYTHONPATH=/root/reference/pkg/src)
from rstile import core  # noqa: E402

from make_golden import csr_digest, format_record  # noqa: E402
from paper_2603_08734_b200 import synth  # noqa: E402

OUT = os.path.join(HERE, "config_formats.json")


def main(names) -> None:
    try:
        with open(OUT) as fh:
            rec = json.load(fh)
    except OSError:
        rec = {"reference": f"rstile {rstile.__version__}", "configs": {}}
    for name in names:
        a = synth.workload_matrix(name)
        t0 = time.time()
        ref_a = core.CsrMatrix(a.n_rows, a.n_cols, a.row_ptr, a.col_idx, a.values)
        entry = {"input": csr_digest(ref_a), "nnz": ref_a.nnz, "n_rows": ref_a.n_rows,
                 "format": format_record(ref_a, {})}
        entry["reference_build_s"] = round(time.time() - t0, 1)
        rec["configs"][name] = entry
        print(name, ref_a.nnz, entry["reference_build_s"], "s", flush=True)
        with open(OUT, "w") as fh:
            json.dump(rec, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["uniform4k", "rmat1m", "stencil2m"])
