"""Drop-in streaming semi-CRF API backed by the sm_100a kernels in libscrf.so.

Mirror of `pkg/src/streamcrf/streaming.py` (streamcrf 0.1.0): same function
names, argument order, dataclasses and error messages. Every compute call goes
through the C ABI (include/scrf.h) on the current CUDA device and stream;
there is no CPU fallback and no multi-backend dispatch (`dispatch` always
answers `BackendKind.Streaming`, `backend=` is accepted and ignored).

Two layers:

* numpy layer (the reference's signatures): `streaming_forward`,
  `streaming_backward`, `streaming_viterbi`, `forward_logZ`, `posterior`,
  `decode`, `recompute_alpha` — host arrays in, host arrays out (H2D/D2H inside).
* torch layer (`DeviceProblem`, `device_forward`, `device_backward`,
  `device_viterbi`, `SemiCRFLogPartition`): device tensors in and out, no host
  round trip, usable inside autograd and CUDA graphs.
"""

from __future__ import annotations

import ctypes
import os
import enum
from dataclasses import dataclass, field
from math import sqrt

import numpy as np
import torch

from . import _lib
from ._numerics import CLAMP_LIMIT, LN2, NEG_INF, ClampSemanticsError, RunStats
from .accounting import MemoryLedger
from .diagnostics import GradientSet, MarginalSet
from .potentials import CumulativeScores, Segmentation, SemiCRFParams

_GUARD = NEG_INF + 1.0

PRECISIONS = {"fp32": 0, "fp64": 1}
_default_precision = "fp32"


def set_precision(name: str) -> None:
    """Working type of the log-semiring kernels: "fp32" (default) or "fp64" (validation)."""
    global _default_precision
    if name not in PRECISIONS:
        raise ValueError(f"precision must be one of {sorted(PRECISIONS)}")
    _default_precision = name


def get_precision() -> str:
    return _default_precision


class ContractViolation(RuntimeError):
    """An internal routing or sequencing contract was broken by the caller (streaming.py:39-40)."""


class BackendKind(enum.Enum):
    LinearK1 = "k1"
    NearLinearK2 = "k2"
    Streaming = "streaming"


@dataclass
class RingAudit:
    """API-compatible placeholder for the reference's ring hazard tracker (streaming.py:70-98).

    The device rings are checked by compute-sanitizer racecheck instead; this
    object records nothing.
    """

    slots: int
    reads: int = 0
    writes: int = 0
    violations: list = field(default_factory=list)


def choose_checkpoint_interval(T: int, K: int) -> int:
    """round(sqrt(T*K)) clamped to [1, T] (streaming.py:101-109)."""
    if T < 1:
        raise ValueError(f"sequence length must be positive, got {T}")
    return max(1, min(T, int(round(sqrt(T * K)))))


# ---------------------------------------------------------------------------
# device problem


def _dev() -> torch.device:
    _lib.load()
    return torch.device("cuda", torch.cuda.current_device())


@dataclass
class DeviceProblem:
    """Kernel operands resident in HBM (fp64 scores, int64 lengths)."""

    S: torch.Tensor  # (B, T+1, C)
    lengths: torch.Tensor  # (B,)
    transition: torch.Tensor  # (C, C)
    duration_bias: torch.Tensor  # (K, C)
    proj_start: torch.Tensor | None = None
    proj_end: torch.Tensor | None = None

    @property
    def B(self) -> int:
        return self.S.shape[0]

    @property
    def T(self) -> int:
        return self.S.shape[1] - 1

    @property
    def C(self) -> int:
        return self.S.shape[2]

    @property
    def K(self) -> int:
        return self.duration_bias.shape[0]

    @classmethod
    def from_host(cls, cum: CumulativeScores, params: SemiCRFParams, device=None, non_blocking=True,
                  defer_S: bool = False):
        """Copy the host problem to the device. Large arrays are staged through pinned memory
        (torch's caching host allocator keeps each staging block alive until its copy has run),
        which is ~2.5x faster than a pageable copy. defer_S: S is allocated but not copied (the
        caller streams it in behind the sweeps, _stream_S)."""
        dev = device or _dev()

        def put(a, dt=torch.float64):
            if a is None:
                return None
            t = torch.from_numpy(np.ascontiguousarray(a))
            if t.dtype != dt:
                t = t.to(dt)
            nbytes = t.numel() * t.element_size()
            if non_blocking and nbytes >= (16 << 20):
                out = torch.empty(t.shape, dtype=dt, device=dev)
                _fill_pinned(out, t)
                return out
            if non_blocking and nbytes >= (1 << 16):
                return t.pin_memory().to(device=dev, non_blocking=True)
            return t.to(device=dev)

        S = (torch.empty(np.shape(cum.S), dtype=torch.float64, device=dev) if defer_S else put(cum.S))
        return cls(S, put(np.asarray(cum.lengths, dtype=np.int64), torch.int64), put(params.transition),
                   put(params.duration_bias), put(cum.proj_start), put(cum.proj_end))

    def _signature(self):
        return tuple(None if t is None else (t.data_ptr(), t._version, tuple(t.shape), t.dtype)
                     for t in (self.S, self.lengths, self.transition, self.duration_bias, self.proj_start,
                               self.proj_end))

    def validate(self) -> None:
        """Shape / dtype / device contract of the C ABI (include/scrf.h): fp64 scores and
        parameters, int64 lengths with 1 <= L_b <= T (potentials.py:79-80; checked on the device
        without a host sync)."""
        S = self.S
        if S.dim() != 3:
            raise ValueError(f"S must be (B, T+1, C), got shape {tuple(S.shape)}")
        B, T1, C = S.shape
        K = self.duration_bias.shape[0] if self.duration_bias.dim() == 2 else -1
        want = {"S": (B, T1, C), "lengths": (B,), "transition": (C, C), "duration_bias": (K, C),
                "proj_start": (B, T1 - 1, C), "proj_end": (B, T1 - 1, C)}
        for name, shape in want.items():
            t = getattr(self, name)
            if t is None:
                continue
            if not t.is_cuda or not t.is_contiguous():
                raise ValueError(f"{name} must be a contiguous CUDA tensor")
            if t.device != S.device:
                raise ValueError(f"{name} is on {t.device}, S on {S.device}")
            dt = torch.int64 if name == "lengths" else torch.float64
            if t.dtype != dt:
                raise ValueError(f"{name} must be {dt}, got {t.dtype}")
            if tuple(t.shape) != shape or K < 1:
                raise ValueError(f"{name} must be shaped {shape}, got {tuple(t.shape)}")
        if T1 < 2:
            raise ValueError("S needs at least one position (T >= 1)")
        L = self.lengths
        torch._assert_async(((L >= 1) & (L <= T1 - 1)).all(), "lengths must lie in [1, T]")

    def c_struct(self) -> _lib.ScrfProblem:
        if getattr(self, "_checked", None) != self._signature():
            self.validate()
            self._checked = self._signature()
        return _lib.ScrfProblem(
            _lib.ptr(self.S), _lib.ptr(self.lengths), _lib.ptr(self.transition), _lib.ptr(self.duration_bias),
            _lib.ptr(self.proj_start), _lib.ptr(self.proj_end), self.B, self.T, self.K, self.C,
        )


MEMORY_MODES = ("full", "sublinear")


@dataclass
class DeviceForward:
    logZ: torch.Tensor  # (B,) fp64
    N: torch.Tensor  # (B, n_ckpt) fp64
    dead_at: torch.Tensor  # (B,) int32
    ckpt: torch.Tensor  # opaque uint8 buffer
    delta: int
    precision: str
    sparse: bool = False  # True: checkpoint rows only (sublinear memory), False: every position


def _check_delta(prob: DeviceProblem, delta) -> int:
    delta = choose_checkpoint_interval(prob.T, prob.K) if delta is None else int(delta)
    if delta < 1:
        raise ValueError(f"checkpoint interval must be >= 1, got {delta}")
    return delta


def _forward_buffers(prob: DeviceProblem, delta: int, prec: int, sparse: bool):
    lib = _lib.load()
    p = prob.c_struct()
    nbytes = ctypes_size()
    q = lib.scrf_sparse_checkpoint_bytes if sparse else lib.scrf_checkpoint_bytes
    _lib.check(q(p, delta, prec, nbytes), "checkpoint_bytes")
    dev = prob.S.device
    n_ckpt = -(-prob.T // delta)
    return (torch.empty(prob.B, dtype=torch.float64, device=dev),
            torch.empty((prob.B, n_ckpt), dtype=torch.float64, device=dev),
            torch.empty(prob.B, dtype=torch.int32, device=dev),
            torch.empty(nbytes.value, dtype=torch.uint8, device=dev))


def device_forward(prob: DeviceProblem, delta: int | None = None, precision: str | None = None,
                   sparse: bool = False) -> DeviceForward:
    """Forward pass on the current stream; no host synchronisation.

    sparse=False keeps every position's messages (fast backward, linear memory);
    sparse=True keeps only the checkpoint rows -- the reference's CheckpointSet
    (streaming.py:49-67) plus replay warm-up rows, O(sqrt(T K) C) -- and the backward
    recomputes alpha between checkpoints (streaming.py:232-261)."""
    lib = _lib.load()
    precision = precision or _default_precision
    prec = PRECISIONS[precision]
    delta = _check_delta(prob, delta)
    logZ, N, dead, ckpt = _forward_buffers(prob, delta, prec, sparse)
    fn = lib.scrf_forward_sparse if sparse else lib.scrf_forward
    rc = fn(prob.c_struct(), delta, prec, _lib.ptr(logZ), _lib.ptr(N), _lib.ptr(dead), _lib.ptr(ckpt), ckpt.numel(),
            _lib.stream_handle())
    _lib.check(rc, "scrf_forward")
    return DeviceForward(logZ, N, dead, ckpt, delta, precision, sparse)


def ctypes_size():
    return ctypes.c_size_t(0)


@dataclass
class DeviceBackward:
    grad_S: torch.Tensor
    grad_T: torch.Tensor
    grad_B: torch.Tensor
    grad_P_start: torch.Tensor | None
    grad_P_end: torch.Tensor | None
    position_marginals: torch.Tensor
    boundary_posterior: torch.Tensor
    expected_segment_count: torch.Tensor
    work: torch.Tensor
    sparse: bool = False
    delta: int = 0


def device_backward(prob: DeviceProblem, fwd: DeviceForward, upstream: torch.Tensor | None = None,
                    want_proj_grads: bool | None = None) -> DeviceBackward:
    """Backward from a device forward (its memory mode decides: a sparse forward is followed
    by the checkpoint-replay backward)."""
    lib = _lib.load()
    prec = PRECISIONS[fwd.precision]
    p = prob.c_struct()
    bw = _alloc_backward(prob, prec, fwd.delta, want_proj_grads, fwd.sparse)
    if upstream is not None:
        upstream = upstream.to(device=prob.S.device, dtype=torch.float64).contiguous()
    outs = (_lib.ptr(bw.grad_S), _lib.ptr(bw.grad_T), _lib.ptr(bw.grad_B), _lib.ptr(bw.grad_P_start),
            _lib.ptr(bw.grad_P_end), _lib.ptr(bw.position_marginals), _lib.ptr(bw.boundary_posterior),
            _lib.ptr(bw.expected_segment_count), _lib.ptr(bw.work), bw.work.numel(), _lib.stream_handle())
    if fwd.sparse:
        rc = lib.scrf_backward_sparse(p, fwd.delta, prec, _lib.ptr(fwd.logZ), _lib.ptr(fwd.N), _lib.ptr(fwd.ckpt),
                                      _lib.ptr(upstream), *outs)
    else:
        rc = lib.scrf_backward(p, fwd.delta, prec, _lib.ptr(fwd.logZ), _lib.ptr(fwd.ckpt), _lib.ptr(upstream), *outs)
    _lib.check(rc, "scrf_backward")
    return bw


def _alloc_backward(prob: DeviceProblem, prec: int, delta: int, want_proj_grads: bool | None, sparse: bool = False):
    lib = _lib.load()
    p = prob.c_struct()
    nbytes = ctypes_size()
    q = lib.scrf_sparse_backward_work_bytes if sparse else lib.scrf_backward_work_bytes
    _lib.check(q(p, delta, prec, nbytes), "backward_work_bytes")
    dev = prob.S.device
    B, T, K, C = prob.B, prob.T, prob.K, prob.C
    f64 = dict(dtype=torch.float64, device=dev)
    if want_proj_grads is None:
        want_proj_grads = prob.proj_start is not None or prob.proj_end is not None
    return DeviceBackward(
        grad_S=torch.empty((B, T + 1, C), **f64), grad_T=torch.empty((C, C), **f64),
        grad_B=torch.empty((K, C), **f64),
        grad_P_start=torch.empty((B, T, C), **f64) if want_proj_grads and prob.proj_start is not None else None,
        grad_P_end=torch.empty((B, T, C), **f64) if want_proj_grads and prob.proj_end is not None else None,
        position_marginals=torch.empty((B, T, C), **f64), boundary_posterior=torch.empty((B, T), **f64),
        expected_segment_count=torch.empty((B,), **f64),
        work=torch.empty(nbytes.value, dtype=torch.uint8, device=dev), sparse=sparse, delta=delta)


def device_posterior(prob: DeviceProblem, delta: int | None = None, upstream: torch.Tensor | None = None,
                     precision: str | None = None, want_proj_grads: bool | None = None, memory: str = "full"):
    """Forward + backward in one call (alpha and beta sweeps run concurrently); no host sync.

    memory="full": every position's messages are kept (fastest; O(T C) working memory).
    memory="sublinear": checkpoint rows only; alpha and beta are replayed window by window from
    them (streaming.py:232-261), O(sqrt(T K) C) working memory besides the
    O(T C) inputs and outputs."""
    if memory not in MEMORY_MODES:
        raise ValueError(f"memory must be one of {MEMORY_MODES}")
    sparse = memory == "sublinear"
    lib = _lib.load()
    precision = precision or _default_precision
    prec = PRECISIONS[precision]
    delta = _check_delta(prob, delta)
    p = prob.c_struct()
    dev = prob.S.device
    fwd = DeviceForward(*_forward_buffers(prob, delta, prec, sparse), delta, precision, sparse)
    bw = _alloc_backward(prob, prec, delta, want_proj_grads, sparse)
    if upstream is not None:
        upstream = upstream.to(device=dev, dtype=torch.float64).contiguous()
    fn = lib.scrf_posterior_sparse if sparse else lib.scrf_posterior
    rc = fn(p, delta, prec, _lib.ptr(upstream), _lib.ptr(fwd.logZ), _lib.ptr(fwd.N), _lib.ptr(fwd.dead_at),
            _lib.ptr(fwd.ckpt), fwd.ckpt.numel(), _lib.ptr(bw.grad_S), _lib.ptr(bw.grad_T), _lib.ptr(bw.grad_B),
            _lib.ptr(bw.grad_P_start), _lib.ptr(bw.grad_P_end), _lib.ptr(bw.position_marginals),
            _lib.ptr(bw.boundary_posterior), _lib.ptr(bw.expected_segment_count), _lib.ptr(bw.work),
            bw.work.numel(), _lib.stream_handle())
    _lib.check(rc, "scrf_posterior")
    return fwd, bw


def device_beta_logz(prob: DeviceProblem, fwd: DeviceForward, bw: DeviceBackward) -> torch.Tensor:
    """logZ recomputed from the beta sweep (consistency check of the two sweeps)."""
    lib = _lib.load()
    out = torch.empty(prob.B, dtype=torch.float64, device=prob.S.device)
    prec = PRECISIONS[fwd.precision]
    if bw.sparse:
        rc = lib.scrf_beta_logz_sparse(prob.c_struct(), bw.delta, prec, _lib.ptr(bw.work), _lib.ptr(out),
                                       _lib.stream_handle())
    else:
        rc = lib.scrf_beta_logz(prob.c_struct(), prec, _lib.ptr(bw.work), _lib.ptr(out), _lib.stream_handle())
    _lib.check(rc, "scrf_beta_logz")
    return out


def device_grad_partials(prob: DeviceProblem, fwd: DeviceForward, bwd: DeviceBackward):
    """Per-sequence (unreduced, upstream-unscaled) grad_T (B,C,C) and grad_B (B,K,C) partials."""
    lib = _lib.load()
    dev = prob.S.device
    gT = torch.empty((prob.B, prob.C, prob.C), dtype=torch.float64, device=dev)
    gB = torch.empty((prob.B, prob.K, prob.C), dtype=torch.float64, device=dev)
    fn = lib.scrf_backward_partials_sparse if bwd.sparse else lib.scrf_backward_partials
    rc = fn(prob.c_struct(), fwd.delta, PRECISIONS[fwd.precision], _lib.ptr(bwd.work), _lib.ptr(gT), _lib.ptr(gB),
            _lib.stream_handle())
    _lib.check(rc, "scrf_backward_partials")
    return gT, gB


def device_omega(prob: DeviceProblem, fwd: DeviceForward) -> torch.Tensor:
    """The reference-format checkpoint snapshots omega (B, n_ckpt, K, C), fp64, on the device."""
    lib = _lib.load()
    out = torch.empty((prob.B, fwd.N.shape[1], prob.K, prob.C), dtype=torch.float64, device=prob.S.device)
    fn = lib.scrf_export_checkpoints_sparse if fwd.sparse else lib.scrf_export_checkpoints
    rc = fn(prob.c_struct(), fwd.delta, PRECISIONS[fwd.precision], _lib.ptr(fwd.ckpt), _lib.ptr(fwd.N), _lib.ptr(out),
            _lib.stream_handle())
    _lib.check(rc, "scrf_export_checkpoints")
    return out


def device_recompute_alpha(prob: DeviceProblem, omega_i: torch.Tensor, t_start: int, t_end: int,
                           precision: str | None = None) -> torch.Tensor:
    """recompute_alpha on the device: (B, t_end - t_start + 1, C) fp64 in the snapshot frame."""
    lib = _lib.load()
    prec = PRECISIONS[precision or _default_precision]
    p = prob.c_struct()
    nbytes = ctypes_size()
    _lib.check(lib.scrf_recompute_alpha_work_bytes(p, t_start, t_end, prec, nbytes), "scrf_recompute_alpha_work_bytes")
    dev = prob.S.device
    work = torch.empty(nbytes.value, dtype=torch.uint8, device=dev)
    omega_i = omega_i.to(device=dev, dtype=torch.float64).contiguous()
    block = torch.empty((prob.B, t_end - t_start + 1, prob.C), dtype=torch.float64, device=dev)
    rc = lib.scrf_recompute_alpha(p, prec, _lib.ptr(omega_i), t_start, t_end, _lib.ptr(block), _lib.ptr(work),
                                  nbytes.value, _lib.stream_handle())
    _lib.check(rc, "scrf_recompute_alpha")
    return block


@dataclass
class DeviceViterbi:
    score: torch.Tensor  # (B,)
    seg_start: torch.Tensor  # (B, T) int32
    seg_end: torch.Tensor
    seg_label: torch.Tensor
    seg_count: torch.Tensor  # (B,)


def device_viterbi(prob: DeviceProblem) -> DeviceViterbi:
    lib = _lib.load()
    p = prob.c_struct()
    nbytes = ctypes_size()
    _lib.check(lib.scrf_viterbi_work_bytes(p, nbytes), "scrf_viterbi_work_bytes")
    dev = prob.S.device
    work = torch.empty(nbytes.value, dtype=torch.uint8, device=dev)
    score = torch.empty(prob.B, dtype=torch.float64, device=dev)
    i32 = dict(dtype=torch.int32, device=dev)
    st, en, lb = (torch.empty((prob.B, prob.T), **i32) for _ in range(3))
    cnt = torch.empty(prob.B, **i32)
    rc = lib.scrf_viterbi(p, _lib.ptr(score), _lib.ptr(st), _lib.ptr(en), _lib.ptr(lb), _lib.ptr(cnt),
                          _lib.ptr(work), nbytes.value, _lib.stream_handle())
    _lib.check(rc, "scrf_viterbi")
    return DeviceViterbi(score, st, en, lb, cnt)


# ---------------------------------------------------------------------------
# reference-shaped numpy API


class CheckpointSet:
    """Ring snapshots at every renormalisation boundary (streaming.py:49-67).

    Produced by `streaming_forward`, which keeps ONLY the checkpoint rows on the device (the
    last min(K+32, delta) alpha messages of every delta-period: the reference's snapshots
    plus the warm-up of a replay window) -- O(sqrt(T K) C) memory. `omega` (B, n_ckpt, K, C)
    and `N` (B, n_ckpt) are the reference-format views (materialised on first access);
    `streaming_backward` replays alpha between checkpoints from the device rows.
    """

    def __init__(self, prob: DeviceProblem, fwd: DeviceForward, cum=None, params=None):
        self._prob = prob
        self._fwd = fwd
        self._cum = cum
        self._params = params
        self.delta = fwd.delta
        self._omega = None
        self._N = None

    @property
    def n_checkpoints(self) -> int:
        return self._fwd.N.shape[1]

    @property
    def N(self) -> np.ndarray:
        if self._N is None:
            self._N = self._fwd.N.cpu().numpy()
        return self._N

    @property
    def omega(self) -> np.ndarray:
        if self._omega is None:
            self._omega = device_omega(self._prob, self._fwd).cpu().numpy()
        return self._omega

    def device_bytes(self) -> int:
        return int(self._fwd.ckpt.numel())


def _check_labels(cum: CumulativeScores, params: SemiCRFParams) -> None:
    if params.num_labels != cum.num_labels:
        raise ValueError(f"label count mismatch: scores have {cum.num_labels}, params {params.num_labels}")


def device_clamp_events(prob: DeviceProblem, fwd: DeviceForward, bw: "DeviceBackward | None" = None) -> torch.Tensor:
    """(B,) int32: positions where the reference would clip a message to +-CLAMP_LIMIT
    (alpha from the forward, plus beta when `bw` is given); no host sync."""
    lib = _lib.load()
    out = torch.empty(prob.B, dtype=torch.int32, device=prob.S.device)
    work = None if bw is None else _lib.ptr(bw.work)
    if fwd.sparse:
        rc = lib.scrf_clamp_events_sparse(prob.c_struct(), fwd.delta, PRECISIONS[fwd.precision], _lib.ptr(fwd.ckpt),
                                          work, _lib.ptr(out), _lib.stream_handle())
    else:
        rc = lib.scrf_clamp_events(prob.c_struct(), PRECISIONS[fwd.precision], _lib.ptr(fwd.ckpt), work,
                                   _lib.ptr(out), _lib.stream_handle())
    _lib.check(rc, "scrf_clamp_events")
    return out


def edge_score_bound(prob: DeviceProblem) -> torch.Tensor:
    """Device upper bound of |h| = |S[t]-S[t-k] + B[k-1] (+ Ps + Pe)| over unmasked terms
    (|S[t]-S[t-k]| <= k max|S[t]-S[t-1]|); the reference clips h beyond CLAMP_LIMIT."""
    K = prob.K
    S = prob.S
    step = (S[:, 1:] - S[:, :-1]).abs().amax() if S.shape[1] > 1 else S.new_zeros(())
    db = prob.duration_bias
    live = db > NEG_INF + 1.0
    bmax = torch.where(live, db.abs(), torch.zeros_like(db)).amax()
    bound = K * step + bmax
    for P in (prob.proj_start, prob.proj_end):
        if P is not None:
            bound = bound + P.abs().amax()
    return bound


def _check_clamp(prob: DeviceProblem, fwd: DeviceForward, bw=None, stats: RunStats | None = None) -> None:
    n = int(device_clamp_events(prob, fwd, bw).sum().item())
    if float(edge_score_bound(prob).item()) > CLAMP_LIMIT:
        n += 1
    if stats is not None:
        stats.clamp.add(n)
    if n:
        raise ClampSemanticsError(
            f"{n} position(s) would be clipped to +-{CLAMP_LIMIT:g} by the reference's clamp_log "
            "(_numerics.py:41-56); the device kernels carry exact normalisers and do not reproduce "
            "that clipping, so the results would differ -- use a smaller checkpoint interval or "
            "rescale the potentials"
        )


def _raise_if_dead(fwd: DeviceForward) -> None:
    dead = fwd.dead_at.cpu().numpy()
    bad = np.nonzero(dead >= 0)[0]
    if len(bad):
        b = int(bad[0])
        raise ValueError(
            f"sequence {b}: log-partition diverged to -inf; every duration/source "
            f"candidate fell below the guard first at t={int(dead[b])}"
        )


def streaming_forward(cum: CumulativeScores, params: SemiCRFParams, delta: int | None = None, *,
                      ledger: MemoryLedger | None = None, stats: RunStats | None = None,
                      audit: RingAudit | None = None):
    """(logZ (B,), CheckpointSet) — streaming.py:155-229."""
    _check_labels(cum, params)
    if delta is not None and int(delta) < 1:
        raise ValueError(f"checkpoint interval must be >= 1, got {int(delta)}")
    prob = DeviceProblem.from_host(cum, params)
    fwd = device_forward(prob, delta, sparse=True)
    _raise_if_dead(fwd)
    _check_clamp(prob, fwd, None, stats)
    if ledger is not None:
        ledger.record("checkpoints", fwd.ckpt)
    return fwd.logZ.cpu().numpy(), CheckpointSet(prob, fwd, cum, params)


def _same_problem(ckpts: CheckpointSet, cum: CumulativeScores, params: SemiCRFParams) -> bool:
    if ckpts._cum is cum and ckpts._params is params:
        return True
    pairs = [(cum.S, ckpts._cum.S), (cum.lengths, ckpts._cum.lengths), (cum.proj_start, ckpts._cum.proj_start),
             (cum.proj_end, ckpts._cum.proj_end), (params.transition, ckpts._params.transition),
             (params.duration_bias, ckpts._params.duration_bias)]
    for x, y in pairs:
        if (x is None) != (y is None):
            return False
        if x is not None and (x is not y) and not np.array_equal(np.asarray(x), np.asarray(y)):
            return False
    return True


def streaming_backward(cum: CumulativeScores, params: SemiCRFParams, logZ, ckpts, upstream=None, *,
                       ledger: MemoryLedger | None = None, stats: RunStats | None = None,
                       audit: RingAudit | None = None):
    """(GradientSet, MarginalSet) — streaming.py:264-408.

    `upstream` (B,) scales the gradients only; marginals are posteriors.
    """
    if not isinstance(ckpts, CheckpointSet):
        raise ContractViolation(
            "streaming_backward needs the CheckpointSet from streaming_forward; "
            f"got {type(ckpts).__name__}"
        )
    B, T = cum.batch_size, cum.max_length
    if ckpts.n_checkpoints != -(-T // ckpts.delta):
        raise ContractViolation(
            f"checkpoint set holds {ckpts.n_checkpoints} segments; T={T} with delta={ckpts.delta} "
            f"needs {-(-T // ckpts.delta)}"
        )
    _check_labels(cum, params)
    up = None
    if upstream is not None:
        up = np.asarray(upstream, dtype=np.float64)
        if up.shape != (B,):
            raise ValueError(f"upstream must be shaped ({B},), got {up.shape}")
    # the backward uses the cum / params it is given (as the reference does); the checkpoint rows
    # are the forward's, and alpha is replayed from them between checkpoints
    prob = ckpts._prob
    if ckpts._cum is not None and not _same_problem(ckpts, cum, params):
        prob = DeviceProblem.from_host(cum, params)
    fwd = ckpts._fwd
    logZ_t = torch.as_tensor(np.asarray(logZ, dtype=np.float64), device=prob.S.device)
    fwd_used = DeviceForward(logZ_t, fwd.N, fwd.dead_at, fwd.ckpt, fwd.delta, fwd.precision, fwd.sparse)
    up_t = None if up is None else torch.as_tensor(up, device=prob.S.device)
    bw = device_backward(prob, fwd_used, up_t)
    _check_clamp(prob, fwd, bw, stats)
    if ledger is not None:
        ledger.record("workspace", bw.work)
    return _grads_to_host(bw), _marg_to_host(bw, cum)


def _to_host(*tensors):
    """Device tensors -> numpy arrays backed by pinned host memory (torch's caching host
    allocator): all copies are queued non-blocking on the current stream, then one sync.
    A pageable .cpu() copy of a 154 MB array takes ~70 ms on this platform, a pinned one ~3 ms."""
    outs = []
    for t in tensors:
        if t is None:
            outs.append(None)
            continue
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        h.copy_(t, non_blocking=True)
        outs.append(h)
    torch.cuda.current_stream().synchronize()
    return [None if h is None else h.numpy() for h in outs]


_SIDE = {}


def _fill_pinned(out: torch.Tensor, t: torch.Tensor) -> None:
    """Host tensor -> existing contiguous device tensor through pinned memory in 8 chunks (the
    host copy of chunk i into pinned memory overlaps the DMA of chunk i-1)."""
    flat = t.reshape(-1)
    dst = out.view(-1)
    pin = torch.empty(flat.shape, dtype=flat.dtype, pin_memory=True)
    step = -(-flat.numel() // 8)
    for i0 in range(0, flat.numel(), step):
        pin[i0:i0 + step].copy_(flat[i0:i0 + step])
        dst[i0:i0 + step].copy_(pin[i0:i0 + step], non_blocking=True)


_GATE_SHIFT = 12  # 4096-row chunks of S
_EARLY_CHUNKS = int(os.environ.get("SCRF_EARLY_CHUNKS", "4"))  # chunks queued before the kernels are launched (two per sweep direction)
_PIN_KEEP = []    # pinned staging buffers of streamed uploads still in flight


def _gate_for(prob: DeviceProblem):
    n = -(-(prob.T + 1) // (1 << _GATE_SHIFT))
    return torch.zeros(n + 1, dtype=torch.int32, device=prob.S.device), _GATE_SHIFT


_PRIMED = set()


def _prime_streaming(dev) -> None:
    """First use, before any sweep waits on it: load gate_set_kernel (lazy module loading would
    otherwise load it on its first launch, behind the running sweep that waits for it), create
    the copy stream and run one pinned copy on it."""
    if dev in _PRIMED:
        return
    lib = _lib.load()
    g = torch.zeros(2, dtype=torch.int32, device=dev)
    h = torch.zeros(2, dtype=torch.int32, pin_memory=True)
    cs = _copy_stream()
    cs.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(cs):
        g.copy_(h, non_blocking=True)
        _lib.check(lib.scrf_gate_set(_lib.ptr(g), 0, _lib.stream_handle()), "scrf_gate_set")
    cs.synchronize()
    _PRIMED.add(dev)


def _stream_S(prob: DeviceProblem, S_host, gate: torch.Tensor, shift: int, gate_ready: torch.cuda.Event,
              pin: torch.Tensor, part: slice = slice(None), last: bool = True) -> None:
    """Copy S to prob.S chunk by chunk on the copy stream -- chunks from both ends inward, the
    order the alpha and beta sweeps consume them -- marking each chunk's gate after its copy.
    `part` selects a slice of that order (the first chunks are queued before the kernels are
    launched, the rest after); with `last` the current stream then waits for the last copy
    (later consumers of S)."""
    lib = _lib.load()
    Sh = np.asarray(S_host)
    if Sh.dtype != np.float64 or not Sh.flags.c_contiguous:
        Sh = np.ascontiguousarray(Sh, dtype=np.float64)
    B, T1, _ = Sh.shape
    R = 1 << shift
    n = gate.numel() - 1
    order = []
    lo, hi = 0, n - 1
    while lo <= hi:
        order.append(lo)
        if hi != lo:
            order.append(hi)
        lo, hi = lo + 1, hi - 1
    St = torch.from_numpy(Sh)  # no copy; torch's CPU copy into pinned memory is multi-threaded
    cs = _copy_stream()
    cs.wait_event(gate_ready)
    row_bytes = Sh.shape[2] * 8
    with torch.cuda.stream(cs):
        for j in order[part]:
            r0, r1 = j * R, min((j + 1) * R, T1)
            pin[:, r0:r1].copy_(St[:, r0:r1])
            # one 2-D copy of the chunk's rows of every sequence, then its gate
            _lib.check(lib.scrf_upload_rows(_lib.ptr(prob.S), _lib.ptr(pin), B, T1, row_bytes, r0, r1,
                                            _lib.ptr(gate), j, _lib.stream_handle()), "scrf_upload_rows")
    if not last:
        return
    # keep the pinned staging alive until its copies have run (torch's host allocator only
    # tracks copies it issued itself)
    done = torch.cuda.Event()
    done.record(cs)
    _PIN_KEEP.append((pin, done))
    while _PIN_KEEP and _PIN_KEEP[0][1].query():
        _PIN_KEEP.pop(0)
    torch.cuda.current_stream().wait_stream(cs)


_COPY = {}


def _copy_stream() -> torch.cuda.Stream:
    dev = torch.cuda.current_device()
    if dev not in _COPY:
        _COPY[dev] = torch.cuda.Stream()
    return _COPY[dev]


def _window_plan(prob: DeviceProblem) -> list[tuple[int, int]]:
    """Posterior-pass windows of a full-memory call, in completion order ([] = one pass)."""
    lib = _lib.load()
    cap = 4096
    w0 = (ctypes.c_int32 * cap)()
    w1 = (ctypes.c_int32 * cap)()
    n = lib.scrf_window_plan(prob.c_struct(), w0, w1, cap)
    return [(int(w0[i]), int(w1[i])) for i in range(max(n, 0))]


def _side_stream() -> torch.cuda.Stream:
    dev = torch.cuda.current_device()
    if dev not in _SIDE:
        _SIDE[dev] = torch.cuda.Stream()
    return _SIDE[dev]


def _to_host_async(*tensors):
    """Queue device->pinned-host copies on the current stream (no sync); returns the host
    tensors (None passes through)."""
    outs = []
    for t in tensors:
        if t is None:
            outs.append(None)
            continue
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        h.copy_(t, non_blocking=True)
        outs.append(h)
    return outs


def _grads_to_host(bw: DeviceBackward) -> GradientSet:
    gS, gT, gB, gPs, gPe = _to_host(bw.grad_S, bw.grad_T, bw.grad_B, bw.grad_P_start, bw.grad_P_end)
    return GradientSet(grad_S=gS, grad_T=gT, grad_B=gB, grad_P_start=gPs, grad_P_end=gPe)


def _marg_to_host(bw: DeviceBackward, cum: CumulativeScores) -> MarginalSet:
    pm, bp, ec = _to_host(bw.position_marginals, bw.boundary_posterior, bw.expected_segment_count)
    return MarginalSet(pm, bp, ec, np.asarray(cum.lengths))


def _segments_to_host(v: DeviceViterbi) -> list[Segmentation]:
    cnt = v.seg_count.cpu().numpy()
    st, en, lb = (x.cpu().numpy() for x in (v.seg_start, v.seg_end, v.seg_label))
    return [Segmentation(tuple(zip(st[b, : cnt[b]].tolist(), en[b, : cnt[b]].tolist(), lb[b, : cnt[b]].tolist())))
            for b in range(len(cnt))]


def streaming_viterbi(cum: CumulativeScores, params: SemiCRFParams, *, ledger: MemoryLedger | None = None):
    """(list[Segmentation], scores (B,)) — streaming.py:411-470, bit-identical paths and scores."""
    _check_labels(cum, params)
    prob = DeviceProblem.from_host(cum, params)
    v = device_viterbi(prob)
    return _segments_to_host(v), v.score.cpu().numpy()


def dispatch(params: SemiCRFParams, cum: CumulativeScores | None = None) -> BackendKind:
    """Always the generic streaming kernel (no multi-backend dispatch on B200)."""
    return BackendKind.Streaming


def forward_logZ(cum, params, delta=None, backend=None, *, ledger=None, stats=None) -> np.ndarray:
    """Per-sequence log-partition (streaming.py:707-722); `backend` is ignored."""
    return streaming_forward(cum, params, delta, ledger=ledger, stats=stats)[0]


def full_mode_bytes(prob: DeviceProblem, delta: int | None = None, precision: str | None = None) -> int:
    """Device working memory of the full-memory posterior (checkpoint + work buffers)."""
    lib = _lib.load()
    prec = PRECISIONS[precision or _default_precision]
    delta = _check_delta(prob, delta)
    p = prob.c_struct()
    a, b = ctypes_size(), ctypes_size()
    _lib.check(lib.scrf_checkpoint_bytes(p, delta, prec, a), "scrf_checkpoint_bytes")
    _lib.check(lib.scrf_backward_work_bytes(p, delta, prec, b), "scrf_backward_work_bytes")
    return a.value + b.value


def choose_memory_mode(prob: DeviceProblem, delta: int | None = None, memory: str = "auto") -> str:
    """"full" unless its working set would take more than half of the free device memory."""
    if memory != "auto":
        if memory not in MEMORY_MODES:
            raise ValueError(f"memory must be 'auto' or one of {MEMORY_MODES}")
        return memory
    free, _ = torch.cuda.mem_get_info(prob.S.device)
    return "full" if full_mode_bytes(prob, delta) <= free // 2 else "sublinear"


def posterior(cum, params, delta=None, upstream=None, *, ledger=None, stats=None, memory: str = "auto"):
    """(logZ, GradientSet, MarginalSet) — streaming.py:725-746.

    One fused device call: the alpha and beta sweeps run concurrently. `memory` selects the
    working-memory mode: "full" keeps every position's messages (fastest), "sublinear" keeps
    checkpoint rows only and replays alpha / beta between checkpoints, "auto" (default) takes
    "full" when it fits in half of the free device memory.
    """
    _check_labels(cum, params)
    if delta is not None and int(delta) < 1:
        raise ValueError(f"checkpoint interval must be >= 1, got {int(delta)}")
    B = cum.batch_size
    up_t = None
    if upstream is not None:
        up = np.asarray(upstream, dtype=np.float64)
        if up.shape != (B,):
            raise ValueError(f"upstream must be shaped ({B},), got {up.shape}")
        up_t = torch.as_tensor(up)
    # Full memory at long T: S is streamed in behind the sweeps (they start on its first row
    # chunks, scrf_input_gate) and the per-position outputs (the bulk of the device->host bytes)
    # are copied on a side stream window by window as the posterior passes that overlap the
    # sweeps finish them (scrf_window_plan); otherwise S is copied first and the outputs once they
    # are final (before the duration-gradient pass).
    lib = _lib.load()
    shape_only = DeviceProblem.from_host(cum, params, defer_S=True)
    mem = choose_memory_mode(shape_only, delta, memory)
    plan = _window_plan(shape_only) if mem == "full" else []
    streamed = (bool(plan) and np.asarray(cum.S).nbytes >= (32 << 20)
                and os.environ.get("SCRF_STREAM_INPUT", "1") != "0")
    if streamed:
        prob = shape_only
        _prime_streaming(prob.S.device)
        gate, shift = _gate_for(prob)
        _lib.check(lib.scrf_input_gate(_lib.ptr(gate), gate.numel() - 1, shift), "scrf_input_gate")
        gate_ready = torch.cuda.Event()
        gate_ready.record()  # the zeroed gate precedes every chunk mark
        # pinned staging allocated before the launch: nothing that could wait for the device
        # may run on this thread between the launch and the last chunk mark
        pin = torch.empty(prob.S.shape, dtype=torch.float64, pin_memory=True)
        # the first row chunks of both sweeps go out before the launch: the launch sequence of the
        # overlapped passes takes ~1 ms of host time, during which the sweeps would otherwise
        # wait on their first gates
        _stream_S(prob, cum.S, gate, shift, gate_ready, pin, part=slice(0, _EARLY_CHUNKS), last=False)
    else:
        prob = shape_only
        Sh = torch.from_numpy(np.ascontiguousarray(cum.S, dtype=np.float64))
        if Sh.numel() * 8 >= (16 << 20):
            _fill_pinned(prob.S, Sh)
        else:
            prob.S.copy_(Sh.pin_memory() if Sh.numel() * 8 >= (1 << 16) else Sh, non_blocking=True)
    ready = torch.cuda.Event()
    ready.record()  # torch creates the CUDA event lazily: make the handle real before passing it
    win_ev = [torch.cuda.Event() for _ in plan]
    for e in win_ev:
        e.record()
    handles = (ctypes.c_void_p * max(1, len(plan)))(*[e.cuda_event for e in win_ev])
    lib.scrf_position_outputs_event(ctypes.c_void_p(ready.cuda_event))
    if plan:
        lib.scrf_window_events(handles, len(plan))
    try:
        fwd, bw = device_posterior(prob, delta, None if up_t is None else up_t.to(prob.S.device), memory=mem)
    finally:
        lib.scrf_position_outputs_event(None)
        lib.scrf_window_events(None, 0)
        if streamed:
            lib.scrf_input_gate(None, 0, 0)
    if streamed:
        _stream_S(prob, cum.S, gate, shift, gate_ready, pin, part=slice(_EARLY_CHUNKS, None))
    side = _side_stream()
    dev_outs = (bw.grad_S, bw.grad_P_start, bw.grad_P_end, bw.position_marginals, bw.boundary_posterior)
    if plan:
        early = [None if t is None else torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in dev_outs]
        with torch.cuda.stream(side):
            for (w0, w1), ev in zip(plan, win_ev):
                side.wait_event(ev)
                for i, (t, h) in enumerate(zip(dev_outs, early)):
                    if t is None:
                        continue
                    # rows the pass over boundaries [w0, w1) finalises: grad_S (T + 1 rows) and
                    # grad_P_start / marginals / boundary (T rows) rows [w0, w1); grad_P_end row
                    # e - 1 belongs to boundary e, so rows [w0 - 1, w1 - 1)
                    lo, hi = (max(w0 - 1, 0), w1 - 1) if i == 2 else (w0, w1)
                    hi = min(hi, t.shape[1])
                    if hi <= lo:
                        continue
                    for b in range(t.shape[0]):  # contiguous per sequence: one async memcpy each
                        h[b, lo:hi].copy_(t[b, lo:hi], non_blocking=True)
    else:
        side.wait_event(ready)
        with torch.cuda.stream(side):
            early = _to_host_async(*dev_outs)
    _raise_if_dead(fwd)
    _check_clamp(prob, fwd, bw, stats)
    if ledger is not None:
        ledger.record("checkpoints", fwd.ckpt)
        ledger.record("workspace", bw.work)
    logZ, gT, gB, cnt = _to_host(fwd.logZ, bw.grad_T, bw.grad_B, bw.expected_segment_count)
    side.synchronize()
    if streamed and int(gate[-1].item()) != 0:
        raise RuntimeError("streamed input: a sweep timed out waiting for a row chunk of S")
    gS, gPs, gPe, pm, bp = (None if h is None else h.numpy() for h in early)
    return (logZ, GradientSet(grad_S=gS, grad_T=gT, grad_B=gB, grad_P_start=gPs, grad_P_end=gPe),
            MarginalSet(pm, bp, cnt, np.asarray(cum.lengths)))


def decode(cum, params, backend=None, *, ledger=None):
    """Best segmentations (streaming.py:749-762); `backend` is ignored."""
    return streaming_viterbi(cum, params, ledger=ledger)


# ---------------------------------------------------------------------------
# autograd


class SemiCRFLogPartition(torch.autograd.Function):
    """logZ = f(S, transition, duration_bias[, proj_start, proj_end]) with the device backward.

    Inputs are CUDA fp64 tensors; `lengths` is an int64 CUDA tensor. grad of each
    input is upstream-weighted exactly like the reference's `upstream` argument.
    """

    @staticmethod
    def forward(ctx, S, transition, duration_bias, lengths, proj_start=None, proj_end=None, delta=None):
        prob = DeviceProblem(S.detach().contiguous(), lengths.contiguous(), transition.detach().contiguous(),
                             duration_bias.detach().contiguous(),
                             None if proj_start is None else proj_start.detach().contiguous(),
                             None if proj_end is None else proj_end.detach().contiguous())
        fwd = device_forward(prob, delta)
        ctx.prob = prob
        ctx.fwd = fwd
        return fwd.logZ.clone()

    @staticmethod
    def backward(ctx, grad_out):
        bw = device_backward(ctx.prob, ctx.fwd, grad_out.detach().to(torch.float64))
        return bw.grad_S, bw.grad_T, bw.grad_B, None, bw.grad_P_start, bw.grad_P_end, None


def log_partition(S, transition, duration_bias, lengths, proj_start=None, proj_end=None, delta=None):
    return SemiCRFLogPartition.apply(S, transition, duration_bias, lengths, proj_start, proj_end, delta)


def recompute_alpha(omega_i, n_i, cum, params, t_start, t_end):
    """Replay forward messages t_start..t_end from one snapshot (streaming.py:232-261).

    Device replay (scrf_recompute_alpha): the snapshot's ring slots force the first
    positions of a sweep that then runs the recursion to t_end. Returns (B, t_end - t_start
    + 1, C) in the snapshot's frame (n_i is not re-applied), block[:, 0] straight from the
    snapshot slot, and past L_b the ring slot's held value, as the reference does.
    """
    if not 0 <= t_start <= t_end <= cum.max_length:
        raise ValueError(f"bad replay window [{t_start}, {t_end}] for T={cum.max_length}")
    _check_labels(cum, params)
    omega_i = np.asarray(omega_i, dtype=np.float64)
    B, K, C = cum.batch_size, params.max_duration, cum.num_labels
    if omega_i.shape != (B, K, C):
        raise ValueError(f"omega_i must be shaped ({B}, {K}, {C}), got {omega_i.shape}")
    del n_i  # kept in the signature so (omega, N) travel as a pair (streaming.py:250)
    prob = DeviceProblem.from_host(cum, params)
    block = device_recompute_alpha(prob, torch.as_tensor(omega_i), int(t_start), int(t_end))
    return block.cpu().numpy()
