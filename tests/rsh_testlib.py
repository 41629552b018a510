"""Helpers shared by the test modules (importable as a top-level module from tests/)."""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def corpus_matrix(recipe: dict, small=None):
    from paper_2603_08734_b200 import synth
    from oracle import corpus  # noqa: E402
    if recipe["kind"] == "small_corpus":
        return (small or corpus.small_corpus())[recipe["index"]]
    if recipe["kind"] == "power_law":
        return corpus.generate_power_law(*recipe["args"])
    if recipe["kind"] == "rmat":
        return synth.rmat(*recipe["args"])
    raise KeyError(recipe["kind"])


def gpu_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
