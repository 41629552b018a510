"""CPU: the C-ABI library and the host-side mirror of the reference interface (no GPU compute).

* librsh.so loads and exports every entry point include/rsh.h declares, with the ctypes
  signatures the Python layer binds;
* the host types keep the reference's contracts (rstile core.py / partition.py / execute.py):
  validation errors, read-only arrays, threshold rounding, plan JSON round trip;
* compute entry points fail loudly without a CUDA device (no CPU fallback).
"""

from __future__ import annotations

import os
import re

import numpy as np
import pytest

import paper_2603_08734_b200 as P
from paper_2603_08734_b200 import _lib
from rsh_testlib import ROOT, gpu_available


def _header_symbols() -> list[str]:
    with open(os.path.join(ROOT, "include", "rsh.h")) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"\b(rsh_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    L = _lib.lib()
    syms = _header_symbols()
    assert len(syms) >= 14
    for name in syms:
        assert hasattr(L, name), name
        assert name in _lib.SIGNATURES, f"{name} has no ctypes signature"
    assert L.rsh_abi_version() == 1


def test_workspace_queries_are_pure_host_calls():
    L = _lib.lib()
    assert L.rsh_partition_workspace(1 << 20) > (1 << 20)
    assert L.rsh_plan_workspace(1000, 10000, 100) > 10000 * 4
    assert L.rsh_fill_workspace(10000, 500) > 10000 * 4
    a = L.rsh_schedule_bytes(1000, 100, 1000, 10)
    b = L.rsh_schedule_bytes(2000, 100, 1000, 10)
    assert b > a > 0
    # control block (4 words + one ticket per entry, 256-byte aligned) + the chunk partials
    assert L.rsh_partials_bytes(100, 10, 128, 0) == 512 + 10 * 8 * 128 * 4
    assert L.rsh_partials_bytes(100, 10, 128, 1) == 512 + 10 * 8 * 128 * 8
    assert L.rsh_partials_bytes(0, 10, 64, 0) == 256 + 10 * 8 * 64 * 4


def test_library_is_built_for_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


# ---------------------------------------------------------------------------------------------
# host types (rstile core.py:26-213)
# ---------------------------------------------------------------------------------------------

def test_csr_validation_matches_reference_errors():
    with pytest.raises(ValueError):
        P.CsrMatrix(2, 2, np.array([0, 1]), np.array([0]), np.array([1.0]))  # row_ptr length
    with pytest.raises(ValueError):
        P.CsrMatrix(1, 2, np.array([0, 2]), np.array([1, 0]), np.array([1.0, 2.0]))  # not increasing
    with pytest.raises(ValueError):
        P.CsrMatrix(1, 2, np.array([0, 1]), np.array([5]), np.array([1.0]))  # column range
    with pytest.raises(ValueError):
        P.CsrMatrix(2, 2, np.array([0, 2, 1]), np.array([0, 1]), np.array([1.0, 2.0]))
    a = P.CsrMatrix(2, 3, np.array([0, 2, 3]), np.array([0, 2, 1]), np.array([1.0, 2.0, 3.0]))
    assert a.row_ptr.dtype == np.int64 and a.col_idx.dtype == np.int32 and a.values.dtype == np.float32
    assert not a.values.flags.writeable
    assert np.array_equal(a.to_dense(), [[1, 0, 2], [0, 3, 0]])
    assert P.csr_equal(a, P.CsrMatrix.from_dense(a.to_dense()))


def test_dense_matrix_rejects_non_finite():
    with pytest.raises(ValueError):
        P.DenseMatrix.from_array(np.array([[1.0, np.inf]]))
    d = P.DenseMatrix.zeros(2, 3)
    assert d.data.shape == (2, 3) and not d.data.flags.writeable


@pytest.mark.parametrize("n,nnz,want", [(10, 80, 4), (10, 10, 2), (10, 1000, 6), (7, 70, 5), (4, 36, 4),
                                        (1000, 9000, 4), (3, 15, 2)])
def test_threshold_rounding_is_half_even(n, nnz, want, known_answers):
    assert P.estimate_thresholds(n, nnz) == (want, 2)
    ref = {(a, b): c for a, b, c in known_answers["thresholds"]["cases"]}
    assert list(P.estimate_thresholds(n, nnz)) == ref[(n, nnz)]


def test_partition_params_validation():
    for kw in ({"window_size": 0}, {"window_size": 9}, {"tau_nnz": -1}, {"tau_inc": -1},
               {"split_factor": 1.0}, {"max_blocks_per_item": 0}):
        with pytest.raises(ValueError):
            P.PartitionParams(**kw)


def test_plan_json_round_trip():
    plan = P.PartitionPlan(((0, 8), (8, 8)), np.array([17, 19]), {1: ((0, 64), (64, 70))})
    back = P.PartitionPlan.from_json_dict(plan.to_json_dict())
    assert back.windows == plan.windows and back.split_map == plan.split_map
    assert back.residual_rows.tolist() == [17, 19]


def test_exec_config_validation():
    with pytest.raises(ValueError):
        P.ExecConfig(num_workers=0)
    with pytest.raises(ValueError):
        P.ExecConfig(accumulate_precision="f16")
    with pytest.raises(ValueError):
        P.ExecConfig(math="int8")
    assert P.ExecConfig().dtype == np.float32
    assert P.ExecConfig(accumulate_precision="f64").dtype == np.float64


def test_max_relative_error_matches_reference_definition():
    c = np.array([[1.0, 2.0], [0.5, -3.0]])
    r = np.array([[1.0, 2.5], [0.0, -3.0]])
    assert P.max_relative_error(c, r) == pytest.approx(0.5 / 2.5 if 0.5 / 2.5 > 0.5 else 0.5)


@pytest.mark.skipif(gpu_available(), reason="checks the no-GPU behaviour")
def test_compute_fails_loudly_without_gpu():
    a = P.CsrMatrix.from_dense(np.eye(4, dtype=np.float32))
    b = P.DenseMatrix.from_array(np.ones((4, 2), np.float32))
    for fn in (lambda: P.partition_rows(a), lambda: P.oracle_spmm(a, b), lambda: P.build_candidates(a),
               lambda: P.threshold_sweep(a, [2])):
        with pytest.raises(RuntimeError, match="CUDA"):
            fn()


# names of the reference's public API (rstile __init__.py __all__) on the path SURVEY 8 scopes:
# the hot path (a1-a21), its drop-in types and the 8(f) rows; out of scope by SURVEY 2: CooMatrix,
# RowStats/row_stats, generate_power_law, Matrix Market / DMAT I/O, reorder_gain/ReorderGain
REFERENCE_NAMES = [
    "CsrMatrix", "DenseMatrix", "ExecConfig", "FormatError", "Fragment8x8", "KnnGraph", "PartitionParams",
    "PartitionPlan", "Permutation", "ReorderParams", "ResidualPart", "RsTileMatrix", "StorageReport", "TcPart",
    "TileDensityReport", "VerificationError", "build_candidates", "build_knn", "build_rstile", "column_weights",
    "csr_equal", "decode_rstile", "decode_tile", "estimate_thresholds", "exec_residual", "exec_tc_window",
    "hybrid_spmm", "isolation_adjust", "load_permutation", "load_rstile", "max_relative_error", "mst_order",
    "oracle_spmm", "partition_rows", "permutation_objective", "permute_rows", "refine_2opt", "reorder_pipeline",
    "save_permutation", "save_rstile", "split_long_work", "storage_report", "sweep_csv", "threshold_sweep",
    "tile_density", "validate_plan", "validate_rstile", "w_jaccard",
]


def test_public_api_keeps_reference_names():
    for name in REFERENCE_NAMES:
        assert hasattr(P, name), name
        assert name in P.__all__, name


def test_synthetic_config_counts_match_survey():
    """config 1 recipe."""
    from paper_2603_08734_b200 import synth
    a = synth.uniform_4096()
    assert a.nnz == 167_772 and a.n_rows == 4096
    b = synth.workload_b("uniform4k", 4096)
    assert b.shape == (4096, 32) and b.dtype == np.float32
    x = np.array([1.0, 1.00390625, 1.005859375, -3.14159], np.float32)
    r = synth.bf16_round(x)
    assert r[0] == 1.0 and r[1] == 1.0 and r[2] == np.float32(1.0078125)
