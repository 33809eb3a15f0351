"""Log-domain constants and the instrumentation bundle of the streamcrf API.

Mirrors the public constants of the reference (`pkg/src/streamcrf/_numerics.py:16-23`)
so callers comparing against the sentinel keep working. The CUDA kernels do
not use the sentinel internally: they carry IEEE -inf for "no path" and map
it back to the reference's guard semantics (`max <= NEG_INF + 1` => dead) at
the boundary (`_numerics.py:59-75`, `streaming.py:194-225`).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

NEG_INF = -1.0e9
"""Reference sentinel for log(0) (`_numerics.py:18`)."""

CLAMP_LIMIT = 1.0e6
"""Reference clamp for finite intermediates (`_numerics.py:23`)."""

LOG2E = 1.4426950408889634
LN2 = 0.6931471805599453


@dataclass
class ClampStats:
    """Clamp-event counter (`_numerics.py:26-38`).

    The reference clips finite log-domain intermediates to +-CLAMP_LIMIT
    (`clamp_log`, `_numerics.py:41-56`), which changes its results once a message
    or a duration score leaves that range (e.g. alpha at T >~ 3e5 with
    delta = T, or a "soft mask" duration bias of -5e8). The device kernels carry
    exact fp64 normalisers instead and do NOT reproduce that clipping: they count
    the positions where the reference would clip (alpha: max message relative to
    the checkpoint normaliser; beta: the unnormalised max message; edge scores: a
    device bound on |S[t]-S[t-k] + B + P|) and the API raises `ClampSemanticsError`
    whenever that count is non-zero, instead of silently returning a different
    answer. On well-scaled inputs the count is 0, as in the reference.
    """

    events: int = 0

    def add(self, n: int) -> None:
        self.events += int(n)


@dataclass
class RunStats:
    """Per-call instrumentation bundle (`_numerics.py:104-112`)."""

    clamp: ClampStats = field(default_factory=ClampStats)

    @property
    def clamp_events(self) -> int:
        return self.clamp.events


class ClampSemanticsError(ValueError):
    """Raised when the reference would have clipped an intermediate to +-CLAMP_LIMIT."""


def logsumexp(a, axis, keepdims: bool = False):
    """Guarded host log-sum-exp with the reference's sentinel semantics (_numerics.py:59-75):
    a slice whose maximum is at or below NEG_INF + 1 reduces to NEG_INF. Host utility for
    callers of the numpy API (gold-path scoring, tests); the kernels never call it."""
    x = np.asarray(a, dtype=np.float64)
    top = np.max(x, axis=axis, keepdims=True)
    live = top > NEG_INF + 1.0
    ref = np.where(live, top, 0.0)
    with np.errstate(under="ignore", divide="ignore"):
        tot = np.sum(np.exp(x - ref), axis=axis, keepdims=True)
        val = np.where(live, ref + np.log(np.maximum(tot, 1e-300)), NEG_INF)
    return val if keepdims else np.squeeze(val, axis=axis)
