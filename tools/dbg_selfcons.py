import os, sys, json
ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2604_18780_b200 as scrf
from paper_2604_18780_b200 import streaming as S
from paper_2604_18780_b200.diagnostics import self_consistency_report
_, params, cum = scrf.equivalence_instance(4, T=300, K=8, C=8, B=1)
for prec in ("fp32", "fp64"):
    S.set_precision(prec)
    logZ, grads, marg = scrf.posterior(cum, params)
    rep = self_consistency_report(marg)
    print(prec, logZ, json.dumps(rep, default=str)[:800])
    print(marg.position_marginals.sum(-1)[0, :10], marg.boundary_posterior[0, :10])
