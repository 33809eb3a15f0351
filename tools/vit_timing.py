"""Device time of Viterbi at a config for several library builds: python tools/vit_timing.py c4 lib1.so lib2.so ..."""
import os
import subprocess
import sys

ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 3 or (len(sys.argv) == 3 and not os.environ.get("SCRF_LIB")):
    for lib in sys.argv[2:]:
        env = dict(os.environ, SCRF_LIB=os.path.join(ROOT, lib))
        out = subprocess.run([sys.executable, __file__, sys.argv[1]], env=env, capture_output=True, text=True)
        print(lib, out.stdout.strip() or out.stderr[-500:])
    sys.exit(0)
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2604_18780_b200 as scrf  # noqa: E402
from paper_2604_18780_b200 import streaming as S  # noqa: E402
from paper_2604_18780_b200.instances import CONFIGS  # noqa: E402

c = CONFIGS[sys.argv[1]]
_, params, cum = scrf.equivalence_instance(0, T=c["T"], K=c["K"], C=c["C"], B=c["B"], mode=scrf.CenteringMode.MEAN)
prob = S.DeviceProblem.from_host(cum, params)
for _ in range(2):
    S.device_viterbi(prob)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5):
    r = S.device_viterbi(prob)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / 5
print(f"{ms:.2f} ms  {c['B'] * c['T'] / ms / 1e3:.2f} M pos/s")
