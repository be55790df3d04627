"""GPU-vs-oracle distances on the parity-floor cases (companion of parity_floor.py).

For every case of tools/parity_floor.py it runs the CUDA path (C-ABI) and the
oracle (dgesdd, 16 threads -- the "thr16" build of the floor) on the same
seeded input and records the same quantities as the floor (iterations, x / e /
y relative distance, E-support flips), so each GPU distance can be read next
to the reference's own spread in profiles/r02_parity_floor.json.

    python tools/parity_gpu.py [--cases ...] -> profiles/r02_parity_gpu.json
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

from parity_floor import CASES, instance, rel  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default=",".join(CASES))
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_parity_gpu.json"))
    a = ap.parse_args()
    import oracle
    import paper_1712_09999_b200 as pb
    from paper_1712_09999_b200.api import PasdConfig

    out = {}
    if os.path.exists(a.out):
        out = json.load(open(a.out)).get("cases", {})
    for case in [c for c in a.cases.split(",") if c]:
        dims, r, R, rho, maxiter, eps, fixed = CASES[case]
        L0, T = instance(dims, r, rho)
        cfg = PasdConfig(lambdas=oracle.default_lambdas(dims), ranks=[R] * len(dims), eps=eps, maxiter=maxiter)
        t0 = time.time()
        ro = oracle.pasd_recover(T, cfg, fixed_iters=fixed, threads=16)
        t1 = time.time()
        rg = pb.pasd_recover(T, cfg, fixed_iters=fixed)
        t2 = time.time()
        hist_o, hist_g = ro.residual_history, rg.residual_history
        k = min(len(hist_o), len(hist_g))
        out[case] = {
            "iters": {"oracle_thr16": ro.iters, "gpu": rg.iters},
            "converged": {"oracle_thr16": ro.converged, "gpu": rg.converged},
            "d_iters": abs(ro.iters - rg.iters),
            "x_rel": rel(rg.x, ro.x), "e_rel": rel(rg.e, ro.e),
            "y_rel": rel(np.stack(rg.y), np.stack(ro.y)),
            "support_flips": int(np.count_nonzero((rg.e != 0) != (ro.e != 0))),
            "first_history_divergence_iter": next((i + 1 for i in range(k) if hist_o[i] != hist_g[i]), None),
            "rse": {"oracle_thr16": rel(ro.x, L0), "gpu": rel(rg.x, L0)},
            "objective": {"oracle_thr16": ro.objective, "gpu": rg.objective},
            "seconds": {"oracle_thr16": t1 - t0, "gpu": t2 - t1},
        }
        print(case, json.dumps(out[case]), flush=True)
    json.dump({"meta": {"generated_by": "tools/parity_gpu.py", "oracle": "dgesdd, 16 threads"}, "cases": out},
              open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
