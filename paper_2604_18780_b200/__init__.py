"""B200-native streaming semi-Markov CRF inference (capabilities of arXiv 2604.18780).

Drop-in for the hot path of the reference package `streamcrf` 0.1.0
(`pkg/src/streamcrf/__init__.py:18-97`, streaming/diagnostics/potentials
exports): build the prefix-sum scores with `build_scores`, then call
`forward_logZ`, `posterior` or `decode`. The compute runs in hand-written
sm_100a CUDA kernels (libscrf.so, C ABI in include/scrf.h); importing this
package does not need a GPU, calling a compute function does.
"""

from .accounting import MemoryLedger
from ._numerics import NEG_INF, RunStats
from .diagnostics import (
    GradientSet,
    MarginalSet,
    boundary_entropy,
    finalize_marginals,
    nll,
    position_marginals,
    self_consistency_report,
)
from .instances import CONFIGS, equivalence_instance
from .potentials import (
    CenteredEmissions,
    CenteringMode,
    CumulativeScores,
    EmissionBatch,
    Segmentation,
    SemiCRFParams,
    build_cumulative,
    build_scores,
    center_emissions,
    edge_potential,
    fold_scalar_boundaries,
    score_segmentation,
    segment_path_score,
)
from .streaming import (
    BackendKind,
    CheckpointSet,
    ContractViolation,
    DeviceProblem,
    RingAudit,
    choose_checkpoint_interval,
    decode,
    device_backward,
    device_forward,
    device_posterior,
    device_viterbi,
    dispatch,
    forward_logZ,
    log_partition,
    posterior,
    recompute_alpha,
    set_precision,
    streaming_backward,
    streaming_forward,
    streaming_viterbi,
)

from .layer import SemiCRF, build_scores_t, gold_scores_t, training_loss_and_grads_device

__version__ = "0.1.0"

__all__ = [
    "SemiCRF",
    "build_scores_t",
    "gold_scores_t",
    "training_loss_and_grads_device",
    "BackendKind", "CenteredEmissions", "CenteringMode", "CheckpointSet", "ContractViolation",
    "CumulativeScores", "DeviceProblem", "EmissionBatch", "GradientSet", "MarginalSet", "MemoryLedger",
    "NEG_INF", "RingAudit", "RunStats", "Segmentation", "SemiCRFParams", "CONFIGS", "boundary_entropy",
    "build_cumulative", "build_scores", "center_emissions", "choose_checkpoint_interval", "decode",
    "device_backward", "device_forward", "device_posterior", "device_viterbi", "dispatch", "edge_potential",
    "equivalence_instance", "finalize_marginals", "fold_scalar_boundaries", "forward_logZ", "log_partition",
    "nll", "position_marginals", "posterior", "recompute_alpha", "score_segmentation", "segment_path_score",
    "self_consistency_report", "set_precision", "streaming_backward", "streaming_forward",
    "streaming_viterbi", "__version__",
]
