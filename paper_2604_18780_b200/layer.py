"""End-to-end differentiable semi-CRF layer on the device.

The input stage of the reference (potentials.build_scores: masked centering, prefix sum,
scalar-boundary fold; potentials.py:275-388) restated in torch ops so it runs on the GPU and
autograd carries the cumulative-score gradient back to the emissions (the suffix sum of
grad_S that validation.training_loss_and_grads derives by hand, validation.py:388-417). The
log-partition and its gradients come from the CUDA kernels (streaming.SemiCRFLogPartition);
the gold-path score (potentials.segment_path_score, potentials.py:420-459) is a gather on the
device. Torch ops here are prep and bookkeeping ("P0 prep, torch ops acceptable"),
not the hot path.
"""
from __future__ import annotations

import numpy as np
import torch

from ._numerics import NEG_INF
from .potentials import CenteringMode, Segmentation
from .streaming import log_partition


def center_emissions_t(emissions: torch.Tensor, lengths: torch.Tensor, mode: CenteringMode) -> torch.Tensor:
    """(B, T, C) emissions -> centered emissions, padding zeroed (potentials.py:275-310).

    MEAN subtracts the masked per-(b, c) mean over t < L_b; SHARED_MAX the per-position max
    over labels; NONE leaves the values. Non-finite valid entries raise like the reference.
    """
    B, T, C = emissions.shape
    valid = torch.arange(T, device=emissions.device)[None, :] < lengths[:, None]
    bad = ~torch.isfinite(emissions) & valid[:, :, None]
    if bool(bad.any()):
        b, t, c = (int(v) for v in torch.nonzero(bad)[0].tolist())
        raise ValueError(f"non-finite emission at valid position: b={b}, t={t}, c={c} "
                         f"(value {float(emissions[b, t, c])!r})")
    vm = valid[:, :, None].to(emissions.dtype)
    if mode is CenteringMode.MEAN:
        base = (emissions * vm).sum(dim=1) / lengths[:, None].to(emissions.dtype)
        centered = emissions - base[:, None, :]
    elif mode is CenteringMode.SHARED_MAX:
        rowmax = torch.where(valid[:, :, None], emissions, torch.full_like(emissions, NEG_INF)).amax(dim=2)
        centered = emissions - rowmax[:, :, None]
    elif mode is CenteringMode.NONE:
        centered = emissions
    else:  # pragma: no cover
        raise ValueError(f"unknown centering mode {mode!r}")
    return centered * vm


def build_scores_t(emissions: torch.Tensor, lengths: torch.Tensor, mode: CenteringMode = CenteringMode.NONE,
                   pi_start: torch.Tensor | None = None, pi_end: torch.Tensor | None = None) -> torch.Tensor:
    """center -> prefix sum -> fold scalar boundaries, as a differentiable (B, T+1, C) S
    (potentials.py:313-388; projections are not folded here: pass them to the layer)."""
    centered = center_emissions_t(emissions, lengths, mode)
    B, T, C = centered.shape
    S = torch.cat([torch.zeros(B, 1, C, dtype=centered.dtype, device=centered.device), centered.cumsum(dim=1)], dim=1)
    if pi_start is not None:
        S = S - torch.nn.functional.pad(pi_start[None, None, :].expand(B, 1, C), (0, 0, 0, T))
    if pi_end is not None:
        onehot = torch.zeros(B, T + 1, 1, dtype=S.dtype, device=S.device)
        onehot[torch.arange(B, device=S.device), lengths] = 1.0
        S = S + onehot * pi_end[None, None, :]
    return S


def gold_scores_t(S: torch.Tensor, transition: torch.Tensor, duration_bias: torch.Tensor,
                  golds: list[Segmentation], proj_start: torch.Tensor | None = None,
                  proj_end: torch.Tensor | None = None) -> torch.Tensor:
    """Log-score of each gold tiling, summed over the virtual source label
    (potentials.py:420-459): LSE_c0 (T[c0, first] + sum over segments of
    (S[e,c] - S[s,c]) + B[e-s-1, c] (+ Ps[s,c] + Pe[e-1,c]) + T[prev, c])."""
    dev = S.device
    bs, ss, es, cs, ps = [], [], [], [], []
    firsts = []
    for b, g in enumerate(golds):
        prev = -1
        for i, (s, e, c) in enumerate(g.segments):
            bs.append(b)
            ss.append(s)
            es.append(e)
            cs.append(c)
            ps.append(prev)
            prev = c
        firsts.append(g.segments[0][2])
    b_t = torch.tensor(bs, device=dev)
    s_t = torch.tensor(ss, device=dev)
    e_t = torch.tensor(es, device=dev)
    c_t = torch.tensor(cs, device=dev)
    p_t = torch.tensor(ps, device=dev)
    seg = (S[b_t, e_t, c_t] - S[b_t, s_t, c_t]) + duration_bias[e_t - s_t - 1, c_t]
    if proj_start is not None:
        seg = seg + proj_start[b_t, s_t, c_t]
    if proj_end is not None:
        seg = seg + proj_end[b_t, e_t - 1, c_t]
    has_prev = p_t >= 0
    trans = torch.where(has_prev, transition[p_t.clamp(min=0), c_t], torch.zeros_like(seg))
    total = torch.zeros(len(golds), dtype=S.dtype, device=dev).index_add(0, b_t, seg + trans)
    first = torch.tensor(firsts, device=dev)
    per_source = transition[:, first].T + total[:, None]  # (B, C)
    return torch.logsumexp(per_source, dim=1)


class SemiCRF(torch.nn.Module):
    """Semi-CRF layer with learnable transition (C, C) and duration bias (K, C) potentials.

    forward(emissions (B, T, C), lengths (B,)) -> log Z (B,); nll(...) -> mean gold NLL. Both
    are differentiable in the emissions and the potentials; the log-partition gradient is the
    device posterior (streaming.SemiCRFLogPartition).
    """

    def __init__(self, num_labels: int, max_duration: int, mode: CenteringMode = CenteringMode.NONE,
                 device=None, dtype=torch.float64):
        super().__init__()
        self.transition = torch.nn.Parameter(torch.zeros(num_labels, num_labels, device=device, dtype=dtype))
        self.duration_bias = torch.nn.Parameter(torch.zeros(max_duration, num_labels, device=device, dtype=dtype))
        self.mode = mode

    def scores(self, emissions: torch.Tensor, lengths: torch.Tensor) -> torch.Tensor:
        return build_scores_t(emissions.to(torch.float64), lengths, self.mode)

    def forward(self, emissions: torch.Tensor, lengths: torch.Tensor, proj_start=None, proj_end=None) -> torch.Tensor:
        S = self.scores(emissions, lengths)
        return log_partition(S, self.transition, self.duration_bias, lengths, proj_start, proj_end)

    def nll(self, emissions: torch.Tensor, lengths: torch.Tensor, golds: list[Segmentation]) -> torch.Tensor:
        """Mean over the batch of log Z - gold score (validation.training_loss_and_grads,
        validation.py:388-417, with its gradients obtained by autograd)."""
        for b, g in enumerate(golds):
            g.validate(int(lengths[b]), self.duration_bias.shape[0], self.transition.shape[0])
        S = self.scores(emissions, lengths)
        logZ = log_partition(S, self.transition, self.duration_bias, lengths)
        gold = gold_scores_t(S, self.transition, self.duration_bias, golds)
        return (logZ - gold).mean()


def training_loss_and_grads_device(emissions: np.ndarray, lengths: np.ndarray, transition: np.ndarray,
                                   duration_bias: np.ndarray, golds: list[Segmentation]):
    """numpy in / numpy out twin of validation.training_loss_and_grads (validation.py:388-417)
    computed on the device: (mean NLL, grad_emissions, grad_T, grad_B)."""
    dev = torch.device("cuda")
    e = torch.tensor(emissions, dtype=torch.float64, device=dev, requires_grad=True)
    L = torch.tensor(np.asarray(lengths, dtype=np.int64), device=dev)
    layer = SemiCRF(transition.shape[0], duration_bias.shape[0], CenteringMode.NONE, device=dev)
    with torch.no_grad():
        layer.transition.copy_(torch.as_tensor(transition))
        layer.duration_bias.copy_(torch.as_tensor(duration_bias))
    loss = layer.nll(e, L, golds)
    loss.backward()
    return (float(loss.detach()), e.grad.cpu().numpy(), layer.transition.grad.cpu().numpy(),
            layer.duration_bias.grad.cpu().numpy())
