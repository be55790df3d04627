"""Intrinsic parity floor of the reference itself (VERDICT r01 "Next" #1).

The reference's Procrustes step takes U = u v^T from dgesdd(W) (linops.cpp:93-104).
Whenever V_n has rank k < R_n (every transition iteration, pasd.cpp:187-188) the
last R_n - k columns of u are LAPACK rounding noise, so two equally valid builds
of the reference disagree there.  This script measures how far apart they land,
using the CPU restatement (oracle/, test infrastructure) in three builds:

  ref         dgesdd, 1 thread         (the reference: linops.cpp:17-23, 62)
  gesvd       dgesvd, 1 thread         (another LAPACK driver for the same SVD)
  thr16       dgesdd, 16 BLAS threads  (OpenBLAS threading changes GEMM order)
  thr4        dgesdd, 4 BLAS threads
  gesvd_thr8  dgesvd, 8 BLAS threads

on BASELINE configs[0] (C1, 100^3 r=R=10, 10%: 100 fixed iterations and run to
eps=1e-7) and configs[1] (C2, 200^3 r=R=20, 20%: 200 fixed and run to 1e-7),
plus the two small regression cases of r01_parity_debug.txt.  For every pair
it records x / e / y relative Frobenius distance, E-support flips and
iteration counts; the floor of a case is the maximum over the pairs.

    python tools/parity_floor.py [--cases c1_fixed,c2_conv,...] [--jobs 3]
        -> profiles/r02_parity_floor.json

The GPU tests (tests/test_gpu_parity.py) read that file for the tolerances
they cannot meet below the floor.  Inputs: the oracle's restatement of the
reference generator (gen_lowrank_tucker + corrupt_sparse, synth.cpp:71-121),
master seed 0 (cli.cpp:164).
"""
from __future__ import annotations

import argparse
import itertools
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CASES = {
    # name: (dims, r, R, rho, maxiter, eps, fixed)
    "c1_fixed100": ((100, 100, 100), 10, 10, 0.10, 100, 1e-7, True),
    "c1_conv": ((100, 100, 100), 10, 10, 0.10, 1000, 1e-7, False),
    "c2_fixed200": ((200, 200, 200), 20, 20, 0.20, 200, 1e-7, True),
    "c2_conv": ((200, 200, 200), 20, 20, 0.20, 1000, 1e-7, False),
    "s1_20x22x24_r2R2": ((20, 22, 24), 2, 2, 0.05, 1000, 1e-5, False),
    "s2_20cube_r2R3": ((20, 20, 20), 2, 3, 0.0, 1000, 1e-5, False),
    "smoke_24x20x16": ((24, 20, 16), 2, 2, 0.05, 300, 1e-6, False),
}
VARIANTS = {"ref": (0, 1), "gesvd": (1, 1), "thr16": (0, 16), "thr4": (0, 4), "gesvd_thr8": (1, 8)}
TMP = os.environ.get("PARITY_FLOOR_TMP", "/tmp/parity_floor")


def instance(dims, r, rho, seed=0):
    import oracle
    L0 = oracle.gen_tucker(dims, [r] * len(dims), seed=seed)
    return L0, oracle.corrupt_sparse(L0, rho, seed=seed)


def run_one(case: str, variant: str) -> str:
    """One oracle solve; writes TMP/<case>.<variant>.npz and returns the path."""
    import oracle
    from paper_1712_09999_b200.api import PasdConfig
    dims, r, R, rho, maxiter, eps, fixed = CASES[case]
    svd_variant, threads = VARIANTS[variant]
    L0, T = instance(dims, r, rho)
    cfg = PasdConfig(lambdas=oracle.default_lambdas(dims), ranks=[R] * len(dims), eps=eps, maxiter=maxiter)
    keep = []

    def obs(v):  # rank of each V_n per iteration (the phase trace)
        keep.append([int(np.linalg.matrix_rank(x)) if x.any() else 0 for x in v.v])

    t0 = time.time()
    res = oracle.pasd_recover(T, cfg, observer=obs if np.prod(dims) <= 2e5 else None, svd_variant=svd_variant,
                              threads=threads, fixed_iters=fixed)
    dt = time.time() - t0
    os.makedirs(TMP, exist_ok=True)
    path = os.path.join(TMP, f"{case}.{variant}.npz")
    np.savez(path, x=res.x, e=res.e, y=np.stack(res.y), iters=res.iters, converged=res.converged,
             hist=np.asarray(res.residual_history), objective=res.objective, seconds=dt,
             rse=np.linalg.norm(res.x - L0) / np.linalg.norm(L0), keep=np.asarray(keep))
    return path


def rel(a, b):
    n = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / n) if n > 0 else float(np.linalg.norm(a - b))


def compare(a, b) -> dict:
    ea, eb = a["e"], b["e"]
    ha, hb = a["hist"], b["hist"]
    k = min(len(ha), len(hb))
    div = next((i + 1 for i in range(k) if ha[i] != hb[i]), None)
    return {
        "iters": [int(a["iters"]), int(b["iters"])],
        "d_iters": abs(int(a["iters"]) - int(b["iters"])),
        "x_rel": rel(a["x"], b["x"]),
        "e_rel": rel(ea, eb),
        "y_rel": rel(a["y"], b["y"]),
        "support_flips": int(np.count_nonzero((ea != 0) != (eb != 0))),
        "first_history_divergence_iter": div,
    }


def aggregate(cases) -> dict:
    out = {}
    for case in cases:
        runs = {v: np.load(os.path.join(TMP, f"{case}.{v}.npz")) for v in VARIANTS}
        dims, r, R, rho, maxiter, eps, fixed = CASES[case]
        pairs = {f"{a}_vs_{b}": compare(runs[a], runs[b]) for a, b in itertools.combinations(VARIANTS, 2)}
        floor = {k: max(p[k] for p in pairs.values()) for k in ("d_iters", "x_rel", "e_rel", "y_rel", "support_flips")}
        out[case] = {
            "dims": list(dims), "r": r, "R": R, "rho": rho, "maxiter": maxiter, "eps": eps, "fixed": fixed,
            "runs": {v: {"iters": int(x["iters"]), "converged": bool(x["converged"]), "rse": float(x["rse"]),
                         "objective": float(x["objective"]), "seconds": float(x["seconds"]),
                         "first_full_rank_iter": _first_full(x, R)} for v, x in runs.items()},
            "pairs": pairs,
            "floor": floor,
        }
    return out


def _first_full(x, R):
    keep = x["keep"]
    if keep.size == 0:
        return None
    idx = [i + 1 for i, k in enumerate(keep.tolist()) if all(v == R for v in k)]
    return idx[0] if idx else None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default=",".join(CASES))
    ap.add_argument("--jobs", type=int, default=3)
    ap.add_argument("--one", nargs=2, metavar=("CASE", "VARIANT"), help=argparse.SUPPRESS)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_parity_floor.json"))
    ap.add_argument("--aggregate-only", action="store_true")
    a = ap.parse_args()
    if a.one:
        print(run_one(*a.one))
        return
    cases = [c for c in a.cases.split(",") if c]
    if not a.aggregate_only:
        todo = [(c, v) for c in cases for v in VARIANTS if not os.path.exists(os.path.join(TMP, f"{c}.{v}.npz"))]
        procs = []
        while todo or procs:
            while todo and len(procs) < a.jobs:
                c, v = todo.pop(0)
                procs.append(subprocess.Popen([sys.executable, __file__, "--one", c, v]))
            procs[0].wait()
            if procs[0].returncode != 0:
                raise SystemExit(f"oracle run failed: {procs[0].args}")
            procs.pop(0)
    res = aggregate(cases)
    host = {"nproc": os.cpu_count(), "generated_by": "tools/parity_floor.py",
            "variants": {k: {"svd": ["dgesdd", "dgesvd"][s], "threads": t} for k, (s, t) in VARIANTS.items()}}
    old = {}
    if os.path.exists(a.out):
        old = json.load(open(a.out)).get("cases", {})
    old.update(res)
    json.dump({"meta": host, "cases": old}, open(a.out, "w"), indent=1)
    for c, v in res.items():
        print(c, json.dumps(v["floor"]), {k: r["iters"] for k, r in v["runs"].items()})


if __name__ == "__main__":
    main()
