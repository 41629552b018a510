"""Dump a BASELINE workload's col_idx (CSR order, int32) for tools/microbench/replay_gather.cu.

    python tools/replay_dump.py rmat1m /tmp/rmat1m.cols   -> prints "n_cols row_bytes"
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_08734_b200 import synth  # noqa: E402

name, path = sys.argv[1], sys.argv[2]
a = synth.workload_matrix(name)
w = synth.workload_spec(name)
np.ascontiguousarray(a.col_idx, np.int32).tofile(path)
print(a.n_cols, w.n_features * (2 if w.dtype == "bf16" else 4))
