"""ctypes binding of libscrf.so (C ABI declared in include/scrf.h).

The product path calls only this binding; there is no CPU fallback. If the
shared library is missing or no CUDA device is present, every compute entry
point raises `NativeUnavailable` (a RuntimeError) instead of silently running
something else.
"""

from __future__ import annotations

import ctypes
import os
import threading

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SCRF_LIB") or os.path.join(HERE, "libscrf.so")

SCRF_ERRORS = {
    -1: "dimension out of range",
    -2: "checkpoint interval must be >= 1",
    -3: "work buffer too small",
    -4: "no launch geometry fits shared memory",
    -5: "required pointer is NULL",
}


class NativeUnavailable(RuntimeError):
    """libscrf.so could not be loaded or no CUDA device is available."""


class ScrfProblem(ctypes.Structure):
    _fields_ = [
        ("S", ctypes.c_void_p),
        ("lengths", ctypes.c_void_p),
        ("transition", ctypes.c_void_p),
        ("duration_bias", ctypes.c_void_p),
        ("proj_start", ctypes.c_void_p),
        ("proj_end", ctypes.c_void_p),
        ("B", ctypes.c_int64),
        ("T", ctypes.c_int64),
        ("K", ctypes.c_int64),
        ("C", ctypes.c_int64),
    ]


_P = ctypes.POINTER(ScrfProblem)
_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_int = ctypes.c_int
_sz = ctypes.c_size_t
_psz = ctypes.POINTER(ctypes.c_size_t)

_SIGS = {
    "scrf_default_delta": (_i64, [_i64, _i64]),
    "scrf_checkpoint_bytes": (_int, [_P, _i64, _int, _psz]),
    "scrf_forward": (_int, [_P, _i64, _int, _vp, _vp, _vp, _vp, _sz, _vp]),
    "scrf_backward_work_bytes": (_int, [_P, _i64, _int, _psz]),
    "scrf_backward": (_int, [_P, _i64, _int, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "scrf_posterior": (_int, [_P, _i64, _int, _vp, _vp, _vp, _vp, _vp, _sz, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                               _vp, _sz, _vp]),
    "scrf_beta_logz": (_int, [_P, _int, _vp, _vp, _vp]),
    "scrf_backward_partials": (_int, [_P, _i64, _int, _vp, _vp, _vp, _vp]),
    "scrf_viterbi_work_bytes": (_int, [_P, _psz]),
    "scrf_viterbi": (_int, [_P, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "scrf_export_checkpoints": (_int, [_P, _i64, _int, _vp, _vp, _vp, _vp]),
    "scrf_clamp_events": (_int, [_P, _int, _vp, _vp, _vp, _vp]),
    "scrf_sparse_checkpoint_bytes": (_int, [_P, _i64, _int, _psz]),
    "scrf_sparse_backward_work_bytes": (_int, [_P, _i64, _int, _psz]),
    "scrf_forward_sparse": (_int, [_P, _i64, _int, _vp, _vp, _vp, _vp, _sz, _vp]),
    "scrf_backward_sparse": (_int, [_P, _i64, _int, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                    _vp, _sz, _vp]),
    "scrf_posterior_sparse": (_int, [_P, _i64, _int, _vp, _vp, _vp, _vp, _vp, _sz, _vp, _vp, _vp, _vp, _vp, _vp,
                                     _vp, _vp, _vp, _sz, _vp]),
    "scrf_backward_partials_sparse": (_int, [_P, _i64, _int, _vp, _vp, _vp, _vp]),
    "scrf_beta_logz_sparse": (_int, [_P, _i64, _int, _vp, _vp, _vp]),
    "scrf_clamp_events_sparse": (_int, [_P, _i64, _int, _vp, _vp, _vp, _vp]),
    "scrf_export_checkpoints_sparse": (_int, [_P, _i64, _int, _vp, _vp, _vp, _vp]),
    "scrf_recompute_alpha_work_bytes": (_int, [_P, _i64, _i64, _int, _psz]),
    "scrf_recompute_alpha": (_int, [_P, _int, _vp, _i64, _i64, _vp, _vp, _sz, _vp]),
    "scrf_reduce_partials": (_int, [_i64, _i64, _vp, _vp, _vp, _vp]),
    "scrf_last_launch_count": (_int, []),
    "scrf_profile_events": (None, [_vp, _vp]),
    "scrf_position_outputs_event": (None, [_vp]),
    "scrf_window_plan": (_int, [_P, _vp, _vp, _int]),
    "scrf_window_events": (None, [_vp, _int]),
    "scrf_input_gate": (_int, [_vp, _int, _int]),
    "scrf_gate_set": (_int, [_vp, _int, _vp]),
    "scrf_upload_rows": (_int, [_vp, _vp, _i64, _i64, _i64, _i64, _i64, _vp, _int, _vp]),
    "scrf_debug_trace": (None, [_vp]),
    "scrf_debug_hang": (_int, [_vp]),
}

_lock = threading.Lock()
_lib = None


def exported_symbols() -> list[str]:
    return list(_SIGS)


def load(require_device: bool = True):
    """Load libscrf.so (building nothing: build() in __graft_entry__ does that)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeUnavailable(
                    f"{LIB_PATH} is missing; build it with `python -m paper_2604_18780_b200.build_lib` "
                    "(nvcc, sm_100a). There is no CPU fallback."
                )
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    if require_device and not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device: the semi-CRF kernels run only on the GPU (sm_100a)")
    return _lib


def check(rc: int, what: str) -> None:
    if rc == 0:
        return
    if rc < 0:
        raise ValueError(f"{what}: {SCRF_ERRORS.get(rc, 'invalid argument')} (code {rc})")
    raise RuntimeError(f"{what}: CUDA error {rc} ({torch.cuda.get_device_name() if torch.cuda.is_available() else '?'})")


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def stream_handle() -> int:
    return torch.cuda.current_stream().cuda_stream


def launches() -> int:
    return int(load(require_device=False).scrf_last_launch_count())
