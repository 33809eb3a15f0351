"""Where the numpy posterior() spends its wall time at config 4: host wall per call, and the
device clock from call start (an event recorded on entry) to the sweep's start / end events."""
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
lib = scrf._lib.load()
for _ in range(2):
    scrf.posterior(cum, params)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
for e in ev:
    e.record()
torch.cuda.synchronize()
for rep in range(4):
    ev[0].record()
    t0 = time.perf_counter()
    lib.scrf_profile_events(ev[1].cuda_event, ev[2].cuda_event)
    out = scrf.posterior(cum, params)
    t1 = time.perf_counter()
    lib.scrf_profile_events(None, None)
    torch.cuda.synchronize()
    print(f"wall {1e3 * (t1 - t0):.2f} ms | entry->sweep start {ev[0].elapsed_time(ev[1]):.2f} | sweep "
          f"{ev[1].elapsed_time(ev[2]):.2f} | entry->sweep end {ev[0].elapsed_time(ev[2]):.2f} ms", flush=True)

# MODE 3 sweep with every chunk already marked (gate overhead without waiting) vs MODE 0
from paper_2604_18780_b200 import streaming as S  # noqa: E402

prob = S.DeviceProblem.from_host(cum, params)
gate, shift = S._gate_for(prob)
gate[:-1] = 1
for label, use_gate in (("mode0", False), ("mode3-open", True), ("mode0", False), ("mode3-open", True)):
    if use_gate:
        lib.scrf_input_gate(scrf._lib.ptr(gate), gate.numel() - 1, shift)
    for _ in range(2):
        S.device_posterior(prob, memory="full")
    torch.cuda.synchronize()
    ms = []
    for _ in range(3):
        lib.scrf_profile_events(ev[1].cuda_event, ev[2].cuda_event)
        S.device_posterior(prob, memory="full")
        lib.scrf_profile_events(None, None)
        torch.cuda.synchronize()
        ms.append(ev[1].elapsed_time(ev[2]))
    lib.scrf_input_gate(None, 0, 0)
    print(label, "sweep ms", [f"{x:.2f}" for x in ms], flush=True)
