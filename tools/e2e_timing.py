"""posterior() wall time at config 4 with and without streamed input (SCRF_STREAM_INPUT)."""
import os
import sys
import time

ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2604_18780_b200 as scrf  # noqa: E402
from paper_2604_18780_b200.instances import CONFIGS  # noqa: E402

c = CONFIGS["c4"]
_, params, cum = scrf.equivalence_instance(0, T=c["T"], K=c["K"], C=c["C"], B=c["B"], mode=scrf.CenteringMode.MEAN)
torch.set_num_threads(int(sys.argv[1]) if len(sys.argv) > 1 else torch.get_num_threads())
print("threads", torch.get_num_threads())
for mode in ("1", "0", "1", "0"):
    os.environ["SCRF_STREAM_INPUT"] = mode
    res = scrf.posterior(cum, params)
    res = scrf.posterior(cum, params)
    del res
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    n = 4
    for _ in range(n):
        out = scrf.posterior(cum, params)
    dt = (time.perf_counter() - t0) / n
    print("stream", mode, f"{dt * 1e3:.2f} ms/step", f"{c['B'] * c['T'] / dt / 1e6:.2f} M pos/s", flush=True)
