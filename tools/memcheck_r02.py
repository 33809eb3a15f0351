"""Round-2 paths under compute-sanitizer: the overlapped windowed passes (two side streams,
progress waits), the streamed-input numpy posterior (gated MODE 3 sweep, window copies), the
sublinear replay path and the cut / prep / grad_B kernels. Smallest shapes that take each path."""
import os
import sys

sys.path.insert(0, os.environ.get("ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2604_18780_b200 as scrf  # noqa: E402
from paper_2604_18780_b200 import streaming as S  # noqa: E402

# windows need T + 1 >= 4 * 4096; K = 40 keeps the blocked tails; C = 6 keeps it small
_, params, cum = scrf.equivalence_instance(1, T=16400, K=40, C=6, B=2, mode=scrf.CenteringMode.MEAN, ragged=True,
                                           projections=True)
prob = S.DeviceProblem.from_host(cum, params)
fwd, bw = S.device_posterior(prob, memory="full")
torch.cuda.synchronize()
print("overlapped full posterior ok", float(fwd.logZ[0]), flush=True)
fwd2, bw2 = S.device_posterior(prob, memory="sublinear")
torch.cuda.synchronize()
print("sublinear posterior ok", float(fwd2.logZ[0]), flush=True)
os.environ["SCRF_STREAM_INPUT"] = "1"
S._window_plan(prob)
logZ, grads, marg = scrf.posterior(cum, params, memory="full")
print("numpy posterior ok", logZ[0], np.isfinite(grads.grad_S).all(), flush=True)
