"""PASD vs the SNN full-SVT baseline per iteration (the paper's
complexity claim, sec. 4.1: PASD O(N R I^N) per iteration vs SNN O(N I^(N+1))),
GPU and CPU restatement, 3 modes, I in {40, 60, 80, 100}, Tucker rank 4, R = 12
(SPEC's setting), 10% corruption.  GPU rows: marginal time per iteration,
(t(220 iterations) - t(20 iterations)) / 200 of whole calls, so allocation and
graph capture cancel; CPU rows: 30 fixed iterations of the restatement on 1 thread.

    python tools/snn_vs_pasd.py > gpurun_out/snn_vs_pasd.json
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_1712_09999_b200 as pb  # noqa: E402
from paper_1712_09999_b200.api import PasdConfig, SnnConfig  # noqa: E402

ITERS = 30
rows = []
for I in (40, 60, 80, 100):
    dims = (I, I, I)
    L0 = oracle.gen_tucker(dims, [4, 4, 4], seed=0)
    T = oracle.corrupt_sparse(L0, 0.10, seed=0)
    lam = oracle.default_lambdas(dims)
    pc = PasdConfig(lambdas=lam, ranks=[12, 12, 12], maxiter=ITERS)
    sc = SnnConfig(lambdas=lam, maxiter=ITERS)
    row = {"I": I}

    def timed(fn, cfg):
        t0 = time.perf_counter()
        fn(T, cfg, fixed_iters=True, want_z=False, want_y=False)
        return time.perf_counter() - t0

    for name, fn, mk in (("pasd_gpu", pb.pasd_recover, lambda n: PasdConfig(lambdas=lam, ranks=[12] * 3, maxiter=n)),
                         ("snn_gpu", pb.snn_recover, lambda n: SnnConfig(lambdas=lam, maxiter=n))):
        timed(fn, mk(20))  # warm-up
        t20 = min(timed(fn, mk(20)) for _ in range(2))
        t220 = min(timed(fn, mk(220)) for _ in range(2))
        row[name + "_ms_per_iter"] = round((t220 - t20) / 200 * 1e3, 4)
    for name, fn, cfg in (("pasd_cpu", oracle.pasd_recover, pc), ("snn_cpu", oracle.snn_recover, sc)):
        row[name + "_ms_per_iter"] = round(timed(fn, cfg) / ITERS * 1e3, 4)
    rows.append(row)
    print(json.dumps(row), flush=True)
# log-log slopes (PASD slope <= SNN slope - 0.7 on the CPU)
x = np.log([r["I"] for r in rows])
out = {"rows": rows, "note": "GPU: marginal ms per iteration of whole calls (setup cancels); CPU: whole call / 30"}
for k in ("pasd_gpu", "snn_gpu", "pasd_cpu", "snn_cpu"):
    out[k + "_loglog_slope"] = float(np.polyfit(x, np.log([r[k + "_ms_per_iter"] for r in rows]), 1)[0])
print(json.dumps(out), flush=True)
