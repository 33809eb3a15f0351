import os, sys
sys.path.insert(0, os.environ["ROOT"])
import torch
import paper_2604_18780_b200 as scrf
from paper_2604_18780_b200 import streaming as S
for (C, K, B, T) in [(24, 100, 1, 300), (9, 16, 2, 60), (36, 100, 1, 200), (40, 64, 1, 150)]:
    _, params, cum = scrf.equivalence_instance(0, T=T, K=K, C=C, B=B, mode=scrf.CenteringMode.MEAN)
    prob = S.DeviceProblem.from_host(cum, params)
    S.device_posterior(prob)
    S.device_viterbi(prob)
    torch.cuda.synchronize()
    print("done", C, K, B, T, flush=True)
