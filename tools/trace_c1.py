import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, oracle, paper_1712_09999_b200 as pb
from paper_1712_09999_b200.api import PasdConfig
dims=(100,100,100)
L0=oracle.gen_tucker(dims,[10]*3,seed=0); T=oracle.corrupt_sparse(L0,0.10,seed=0)
cfg=PasdConfig(lambdas=oracle.default_lambdas(dims), ranks=[10]*3, eps=1e-7)
for i in range(3):
    t0=time.perf_counter(); r=pb.pasd_recover(T,cfg); print("call", i, time.perf_counter()-t0, r.iters, flush=True)
