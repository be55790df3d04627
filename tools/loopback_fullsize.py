"""The sharded code path at a BASELINE size on one GPU: C3 (400^3, R = 40) split
into 2 and 3 mode-3 slabs run through the loopback group (pasd_comm.cuh), 40
fixed iterations (the V = 0 phase: every quantity is exact) and then to 100
(through the phase exit at iteration 93), against the unsharded solver.

    python tools/loopback_fullsize.py > gpurun_out/loopback_c3.json
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1712_09999_b200 as pb  # noqa: E402
from paper_1712_09999_b200 import synth  # noqa: E402
from paper_1712_09999_b200.api import PasdConfig  # noqa: E402
from paper_1712_09999_b200.sharding import run_loopback  # noqa: E402
from paper_1712_09999_b200.workloads import WORKLOADS  # noqa: E402

def rel(a, b):
    n = float(np.linalg.norm(b))
    d = float(np.linalg.norm(a - b))
    return d / n if n > 0 else d


w = WORKLOADS["c3"]
T, _, _ = synth.generate(synth.workload_spec(w, seed=0))
out = {"workload": w.name, "dims": list(w.dims), "ranks": list(w.ranks), "runs": []}
for iters in (40, 100):
    cfg = PasdConfig(lambdas=w.lambdas(), ranks=list(w.ranks), maxiter=iters)
    t0 = time.perf_counter()
    r0 = pb.pasd_recover(T, cfg, fixed_iters=True, want_z=False, want_y=False)
    t_un = time.perf_counter() - t0
    for nranks in (2, 3):
        t0 = time.perf_counter()
        it, conv, parts, slabs = run_loopback(T, cfg, nranks, iters)
        t_lb = time.perf_counter() - t0
        x = np.empty(T.shape)
        e = np.empty(T.shape)
        for p, (b, en) in zip(parts, slabs):
            x[:, :, b:en] = p.x
            e[:, :, b:en] = p.e
        row = {"iters": iters, "nranks": nranks, "slabs": [list(s) for s in slabs],
               "e_bit_identical": bool(np.array_equal(e, r0.e)),
               "x_rel": rel(x, r0.x),
               "e_rel": rel(e, r0.e),
               "e_nonzeros": int(np.count_nonzero(r0.e)),
               "support_flips": int(np.count_nonzero((e != 0) != (r0.e != 0))),
               "residual_history_equal": parts[0].residual_history == r0.residual_history,
               "objective": [parts[0].objective, r0.objective],
               "seconds_unsharded": round(t_un, 2), "seconds_loopback": round(t_lb, 2)}
        out["runs"].append(row)
        print(json.dumps(row), flush=True)
print(json.dumps(out))
