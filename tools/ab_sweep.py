"""A/B device time of scrf_posterior (full mode) between two builds of libscrf.so at a config.

    python tools/ab_sweep.py c4 paper_2604_18780_b200/libscrf.so tools/r1_libscrf.so
"""
import ctypes
import os
import sys

ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2604_18780_b200 as scrf  # noqa: E402
from paper_2604_18780_b200 import _lib  # noqa: E402
from paper_2604_18780_b200 import streaming as S  # noqa: E402
from paper_2604_18780_b200.instances import CONFIGS  # noqa: E402

cfg = dict(CONFIGS[sys.argv[1]])
_, params, cum = scrf.equivalence_instance(0, T=cfg["T"], K=cfg["K"], C=cfg["C"], B=cfg["B"], mode=scrf.CenteringMode.MEAN)
prob = S.DeviceProblem.from_host(cum, params)
p = prob.c_struct()
delta = S.choose_checkpoint_interval(prob.T, prob.K)
vp, sz = ctypes.c_void_p, ctypes.c_size_t
for path in sys.argv[2:]:
    lib = ctypes.CDLL(os.path.join(ROOT, path))
    for n in ("scrf_checkpoint_bytes", "scrf_backward_work_bytes"):
        getattr(lib, n).argtypes = [ctypes.POINTER(_lib.ScrfProblem), ctypes.c_int64, ctypes.c_int, ctypes.POINTER(sz)]
    lib.scrf_posterior.argtypes = [ctypes.POINTER(_lib.ScrfProblem), ctypes.c_int64, ctypes.c_int] + [vp] * 5 + [sz] + [vp] * 9 + [sz, vp]
    lib.scrf_profile_events.argtypes = [vp, vp]
    a, b = sz(0), sz(0)
    lib.scrf_checkpoint_bytes(p, delta, 0, a)
    lib.scrf_backward_work_bytes(p, delta, 0, b)
    dev = prob.S.device
    B, T, K, C = prob.B, prob.T, prob.K, prob.C
    f64 = dict(dtype=torch.float64, device=dev)
    ck = torch.empty(a.value, dtype=torch.uint8, device=dev)
    wk = torch.empty(b.value, dtype=torch.uint8, device=dev)
    logZ, N, dead = torch.empty(B, **f64), torch.empty((B, -(-T // delta)), **f64), torch.empty(B, dtype=torch.int32, device=dev)
    gS, gT, gB = torch.empty((B, T + 1, C), **f64), torch.empty((C, C), **f64), torch.empty((K, C), **f64)
    pm, bp, cnt = torch.empty((B, T, C), **f64), torch.empty((B, T), **f64), torch.empty(B, **f64)
    ptr = lambda t: t.data_ptr()  # noqa: E731
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    for e in ev:
        e.record()
    torch.cuda.synchronize()
    res = []
    for it in range(4):
        lib.scrf_profile_events(ev[0].cuda_event, ev[1].cuda_event)
        ev[2].record()
        rc = lib.scrf_posterior(p, delta, 0, None, ptr(logZ), ptr(N), ptr(dead), ptr(ck), a.value, ptr(gS), ptr(gT), ptr(gB),
                                None, None, ptr(pm), ptr(bp), ptr(cnt), ptr(wk), b.value, torch.cuda.current_stream().cuda_stream)
        ev[3].record()
        lib.scrf_profile_events(None, None)
        torch.cuda.synchronize()
        assert rc == 0, rc
        res.append((ev[0].elapsed_time(ev[1]), ev[2].elapsed_time(ev[3])))
    print(path, "sweep ms / step ms:", [f"{x:.2f}/{y:.2f}" for x, y in res[1:]], "logZ", logZ[:2].tolist(), flush=True)
