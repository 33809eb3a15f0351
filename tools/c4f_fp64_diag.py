"""fp64 at full config 4 (T = 1e5) against the reference fixture: error profile along the sequence,
with and without the cut normalisers (SCRF_CUT_D=0), full memory single pass vs windows."""
import os
import sys

ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import golden_io  # noqa: E402
import paper_2604_18780_b200 as scrf  # noqa: E402
from paper_2604_18780_b200 import streaming as S  # noqa: E402
from paper_2604_18780_b200.potentials import CenteringMode  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4f"
z = golden_io.load(name)
_, params, cum = scrf.equivalence_instance(int(z["seed"]), T=int(z["T"]), K=int(z["K"]), C=int(z["C"]),
                                           B=int(z["B"]), mode=CenteringMode(str(z["mode"])))
rows = z["rows_p"]
S.set_precision("fp64")
for label, env in (("windows", {}), ("single-pass", {"SCRF_OVERLAP": "-1"}), ("no-cuts", {"SCRF_CUT_D": "0", "SCRF_OVERLAP": "-1"})):
    for k in ("SCRF_OVERLAP", "SCRF_CUT_D"):
        os.environ.pop(k, None)
    os.environ.update(env)
    logZ, grads, marg = scrf.posterior(cum, params, memory="full")
    for arr, ref, nm in ((marg.boundary_posterior[:1][:, rows], z["boundary_posterior"], "bnd"),
                         (marg.position_marginals[:1][:, rows], z["position_marginals"], "pos"),
                         (grads.grad_S[:1][:, z["rows_s"]], z["grad_S"], "gS")):
        d = np.abs(arr - ref).reshape(arr.shape[0], arr.shape[1], -1).max(axis=(0, 2))
        r = rows if nm != "gS" else z["rows_s"]
        bins = np.linspace(0, int(z["T"]) + 1, 11).astype(int)
        prof = [float(d[(r >= bins[i]) & (r < bins[i + 1])].max()) if ((r >= bins[i]) & (r < bins[i + 1])).any() else 0
                for i in range(10)]
        print(label, nm, f"max {d.max():.2e} at row {int(r[d.argmax()])}", " ".join(f"{x:.1e}" for x in prof), flush=True)
    print(label, "logZ", float(abs(logZ[0] - z["logZ"][0])), "grad_T", float(np.abs(grads.grad_T - z["grad_T"]).max()))
