"""Full-size CPU timing of the reference restatement at C5 (1000^3, R = 50):
the measurement the bench's bounded cpu_baseline extrapolates from a
1000 x 1000 x 50 slab.  Run on the GPU box's host (196 GB RAM):

    python tools/cpu_fullsize.py [iters] > gpurun_out/cpu_fullsize_c5.json

Per-iteration time = gaps between observer callbacks (iteration 1 includes
the setup, reference timing pattern bench.cpp:274-286), 1 thread (linops.cpp:17-23).
"""
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_1712_09999_b200 import _abi  # noqa: E402
from paper_1712_09999_b200.api import PasdConfig  # noqa: E402
from paper_1712_09999_b200.workloads import WORKLOADS  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 3
w = WORKLOADS["c5"]
out = {"workload": w.name, "dims": list(w.dims), "ranks": list(w.ranks), "threads": 1, "iters": iters}
t0 = time.perf_counter()
L0 = oracle.gen_tucker(w.dims, w.tucker, seed=0)
T = oracle.corrupt_sparse(L0, w.rho, seed=0, lo=w.noise[0], hi=w.noise[1])
del L0
out["generate_s"] = round(time.perf_counter() - t0, 1)
S = int(np.prod(w.dims))
lam = [math.sqrt(float(max(d, S // d))) / 3.0 for d in w.dims]
stamps = []
cb = _abi.PasdObserverFn(lambda v, u: stamps.append(time.perf_counter()))
cfg = PasdConfig(lambdas=lam, ranks=list(w.ranks), maxiter=iters, eps=w.eps)
t0 = time.perf_counter()
res = oracle.pasd_recover(T, cfg, observer=cb, fixed_iters=True, threads=1, want_z=False, want_y=False)
t1 = time.perf_counter()
gaps = [b - a for a, b in zip(stamps[:-1], stamps[1:])]
out.update({
    "solve_s": round(t1 - t0, 2), "first_iteration_s": round(stamps[0] - t0, 2),
    "iteration_gaps_s": [round(g, 2) for g in gaps],
    "per_iteration_s": float(np.median(gaps)) if gaps else None,
    "iter_per_s": 1.0 / float(np.median(gaps)) if gaps else None,
    "residual_history": list(res.residual_history),
    "nproc": os.cpu_count(),
})
print(json.dumps(out), flush=True)
