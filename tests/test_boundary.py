"""CPU checks of the drop-in boundary: the C-ABI library loads and exports every symbol
include/scrf.h declares; host-side API surface and input validation (no GPU compute)."""

from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    text = open(os.path.join(ROOT, "include", "scrf.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|void)\s+(scrf_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    from paper_2604_18780_b200 import _lib

    lib = ctypes.CDLL(_lib.LIB_PATH)
    names = header_functions()
    assert len(names) >= 9
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_lib.exported_symbols())


def test_default_delta_matches_reference_table():
    from paper_2604_18780_b200 import _lib
    from paper_2604_18780_b200.streaming import choose_checkpoint_interval

    lib = _lib.load(require_device=False)
    for T, K, want in [(100, 25, 50), (1, 1, 1), (1000, 8, 89), (100_000, 8, 894), (1_000_000, 200, 14_142), (4, 25, 4)]:
        assert lib.scrf_default_delta(T, K) == want
        assert choose_checkpoint_interval(T, K) == want


def test_abi_rejects_bad_arguments_without_a_gpu():
    from paper_2604_18780_b200 import _lib

    lib = _lib.load(require_device=False)
    p = _lib.ScrfProblem(None, None, None, None, None, None, 1, 1, 1, 1)
    n = ctypes.c_size_t(0)
    assert lib.scrf_checkpoint_bytes(ctypes.byref(p), 1, 0, ctypes.byref(n)) == -5
    p = _lib.ScrfProblem(8, 8, 8, 8, None, None, 0, 1, 1, 1)
    assert lib.scrf_checkpoint_bytes(ctypes.byref(p), 1, 0, ctypes.byref(n)) == -1
    p = _lib.ScrfProblem(8, 8, 8, 8, None, None, 2, 10, 3, 4)
    assert lib.scrf_checkpoint_bytes(ctypes.byref(p), 0, 0, ctypes.byref(n)) == -2
    assert lib.scrf_checkpoint_bytes(ctypes.byref(p), 5, 0, ctypes.byref(n)) == 0 and n.value > 0


def test_compute_fails_loudly_without_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    import paper_2604_18780_b200 as scrf
    from paper_2604_18780_b200._lib import NativeUnavailable

    _, params, cum = scrf.equivalence_instance(0, T=8, K=2, C=2, B=1)
    with pytest.raises(NativeUnavailable):
        scrf.forward_logZ(cum, params)


def test_api_surface_matches_reference_exports():
    import paper_2604_18780_b200 as scrf

    # hot-path names of streamcrf/__init__.py:18-97
    for name in ["BackendKind", "CenteredEmissions", "CenteringMode", "CheckpointSet", "ContractViolation",
                 "CumulativeScores", "EmissionBatch", "GradientSet", "MarginalSet", "MemoryLedger", "RunStats",
                 "Segmentation", "SemiCRFParams", "boundary_entropy", "build_scores", "center_emissions", "decode",
                 "dispatch", "forward_logZ", "nll", "posterior", "score_segmentation", "self_consistency_report",
                 "streaming_viterbi"]:
        assert hasattr(scrf, name), name


def test_input_stage_bit_identical_to_golden_digests():
    import golden_io

    n = sum(1 for _ in golden_io.small_cases())
    assert n >= 40
    for name in ["c1", "c1rp", "shmax", "c2", "c3s", "c4s", "c5s"]:
        golden_io.equiv_case(name)


def test_label_mismatch_message():
    import paper_2604_18780_b200 as scrf

    _, params, cum = scrf.equivalence_instance(0, T=8, K=2, C=3, B=1)
    bad = scrf.SemiCRFParams(np.zeros((2, 2)), np.zeros((2, 2)))
    with pytest.raises(ValueError, match="label count mismatch"):
        scrf.streaming_forward(cum, bad)
