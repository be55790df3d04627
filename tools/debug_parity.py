"""Quick GPU-vs-oracle diagnostics (development aid)."""
import sys, time
import numpy as np
sys.path.insert(0, "/root/repo")
import oracle
import paper_1712_09999_b200 as pb
from paper_1712_09999_b200.api import PasdConfig


def rel(a, b):
    d = np.linalg.norm(a - b); n = np.linalg.norm(b)
    return d / n if n > 0 else d


def case(dims, r, R, rho, maxiter, eps=1e-7, fixed=False, seed=0):
    L0 = oracle.gen_tucker(dims, [r] * len(dims), seed=seed)
    T = oracle.corrupt_sparse(L0, rho, seed=seed)
    lam = oracle.default_lambdas(dims)
    cfg = PasdConfig(lambdas=lam, ranks=[R] * len(dims), eps=eps, maxiter=maxiter)
    t = time.time(); ro = oracle.pasd_recover(T, cfg, fixed_iters=fixed, threads=16); to = time.time() - t
    t = time.time(); rg = pb.pasd_recover(T, cfg, fixed_iters=fixed); tg = time.time() - t
    print(f"dims={dims} r={r} R={R} rho={rho} maxiter={maxiter} fixed={fixed}: iters oracle={ro.iters} gpu={rg.iters} "
          f"conv={ro.converged}/{rg.converged} t_or={to:.2f}s t_gpu={tg:.2f}s")
    print(f"   x rel={rel(rg.x, ro.x):.3e} e rel={rel(rg.e, ro.e):.3e} e bitexact={np.array_equal(rg.e, ro.e)} "
          f"y0 bitexact={np.array_equal(rg.y[0], ro.y[0])} supp flips={int(np.sum((rg.e!=0)!=(ro.e!=0)))} "
          f"rse gpu={rel(rg.x, L0):.3e} oracle={rel(ro.x, L0):.3e}")
    print(f"   obj {ro.objective:.12e} {rg.objective:.12e}; hist last {ro.residual_history[-1]:.6e} {rg.residual_history[-1]:.6e}")
    k = min(len(ro.residual_history), len(rg.residual_history))
    hd = [abs(a - b) / max(abs(a), 1e-300) for a, b in zip(ro.residual_history[:k], rg.residual_history[:k])]
    first = next((i for i, h in enumerate(hd) if h > 1e-12), None)
    print(f"   first history divergence at iter {first}")
    if ro.certificate and rg.certificate:
        print(f"   cert oracle={ro.certificate} gpu={rg.certificate}")


case([20, 20, 20], 2, 3, 0.0, 1000, eps=1e-5)
case([20, 22, 24], 2, 2, 0.05, 1000, eps=1e-5)
case([100, 100, 100], 10, 10, 0.10, 90, fixed=True)
case([100, 100, 100], 10, 10, 0.10, 100, fixed=True)
case([100, 100, 100], 10, 10, 0.10, 1000, eps=1e-7)
