import sys, os, json
sys.path.insert(0, "/root/repo")
import paper_1712_09999_b200.solver as S
if len(sys.argv) > 1:
    S.LIB_PATH = sys.argv[1]
import torch
import paper_1712_09999_b200 as pb
from paper_1712_09999_b200.api import PasdConfig
from paper_1712_09999_b200.workloads import WORKLOADS, generate_gpu
w = WORKLOADS["c5"]
T = generate_gpu(w)
cfg = PasdConfig(lambdas=w.lambdas(), ranks=list(w.ranks), maxiter=20)
s = pb.Solver(w.dims, cfg, fixed_iters=True)
s.load(T.data_ptr(), t_is_device=True)
s.run(2)
p = s.profile(2)
print(sys.argv[1:] , {k: round(v["ms"] / max(1, v["launches"]), 3) for k, v in p.items()})
