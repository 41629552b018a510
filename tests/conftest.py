"""Shared fixtures.  Tests marked ``gpu`` need a B200 (run through gpurun); everything else runs on
CPU.  The CPU oracle (oracle/, test infrastructure) is the checker for both."""

from __future__ import annotations

import json
import os

import pytest

from rsh_testlib import GOLDEN, corpus_matrix


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100a) device")
    config.addinivalue_line("markers", "slow: full-size configs (minutes)")


@pytest.fixture(scope="session")
def golden_formats():
    with open(os.path.join(GOLDEN, "formats.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def known_answers():
    with open(os.path.join(GOLDEN, "known_answers.json")) as fh:
        return {c["name"]: c for c in json.load(fh)}


@pytest.fixture(scope="session")
def small_corpus():
    from paper_2603_08734_b200 import synth
    from oracle import corpus  # noqa: E402
    return corpus.small_corpus()


@pytest.fixture(scope="session")
def golden_corpus(golden_formats, small_corpus):
    """name -> (CsrMatrix, golden entry) for every matrix the reference digests cover."""
    return {name: (corpus_matrix(e["recipe"], small_corpus), e)
            for name, e in golden_formats["matrices"].items()}
