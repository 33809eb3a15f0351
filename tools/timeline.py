"""Device timeline of one full-memory posterior at a config (CUPTI kernel records via
torch.profiler): which posterior-pass kernels run while the sweep kernel is still running.

    python tools/timeline.py c4 out.txt
"""
import collections
import json
import os
import sys
import tempfile

ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2604_18780_b200 as scrf  # noqa: E402
from paper_2604_18780_b200 import streaming as S  # noqa: E402
from paper_2604_18780_b200.instances import CONFIGS  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
out = sys.argv[2] if len(sys.argv) > 2 else None
cfg = dict(CONFIGS[name])
_, params, cum = scrf.equivalence_instance(0, T=cfg["T"], K=cfg["K"], C=cfg["C"], B=cfg["B"], mode=scrf.CenteringMode.MEAN)
prob = S.DeviceProblem.from_host(cum, params)
for _ in range(2):
    S.device_posterior(prob, memory="full")
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    S.device_posterior(prob, memory="full")
    torch.cuda.synchronize()
path = os.path.join(tempfile.mkdtemp(), "trace.json")
prof.export_chrome_trace(path)
ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel"]
ev.sort(key=lambda e: e["ts"])
t0 = ev[0]["ts"]
sw = [e for e in ev if "sweep_kernel" in e["name"]]
s0, s1 = sw[0]["ts"], max(e["ts"] + e["dur"] for e in sw)
lines = [f"{name}: one full-memory posterior (device_posterior), CUPTI kernel records (torch.profiler), times in us from the first kernel",
         f"sweep kernel(s): start {s0 - t0:.1f}, end {s1 - t0:.1f} ({(s1 - s0) / 1e3:.2f} ms)"]
agg = collections.OrderedDict()
for e in ev:
    if "sweep_kernel" in e["name"]:
        continue
    k = e["name"].replace("(anonymous namespace)::", "").split("<")[0].split("(")[0].replace("void ", "").split("::")[-1]
    a = agg.setdefault(k, [0, 0.0, 0.0, None, 0])
    a[0] += 1
    a[1] += e["dur"]
    ov = max(0.0, min(e["ts"] + e["dur"], s1) - max(e["ts"], s0))
    a[2] += ov
    a[3] = e.get("args", {}).get("stream")
    a[4] += 1 if e["ts"] < s1 else 0
tot = sum(a[1] for k, a in agg.items() if k != "prog_wait_kernel")  # the spin-wait gates are not work
tov = sum(a[2] for k, a in agg.items() if k != "prog_wait_kernel")
lines.append(f"{'kernel':28s} {'launches':>8s} {'busy us':>10s} {'under sweep us':>15s} {'started under sweep':>20s}")
for k, a in agg.items():
    lines.append(f"{k:28s} {a[0]:8d} {a[1]:10.1f} {a[2]:15.1f} {a[4]:20d}")
end = max(e["ts"] + e["dur"] for e in ev)
lines.append(f"pass kernels: {tot / 1e3:.2f} ms busy in total, {tov / 1e3:.2f} ms of it while the sweep runs "
             f"({100 * tov / max(tot, 1):.0f} %); last kernel ends {(end - s1) / 1e3:.2f} ms after the sweep")
lines.append(f"step span (first kernel start -> last kernel end): {(end - t0) / 1e3:.2f} ms")
print("\n".join(lines))
if out:
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")
        f.write("\nfirst 40 and last 40 kernel records (start us, dur us, stream, name):\n")
        for e in ev[:40] + ev[-40:]:
            f.write(f"{e['ts'] - t0:10.1f} {e['dur']:9.1f} {e.get('args', {}).get('stream')} {e['name'][:90]}\n")
