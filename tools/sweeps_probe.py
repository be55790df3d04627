"""Jacobi sweep counts per small solve in steady state (build with
-DPASD_DEBUG_SWEEPS, select with PASD_B200_LIB): python tools/sweeps_probe.py c3 150"""
import sys

sys.path.insert(0, ".")
import paper_1712_09999_b200 as pb  # noqa: E402
from paper_1712_09999_b200.api import PasdConfig  # noqa: E402
from paper_1712_09999_b200.workloads import WORKLOADS, generate_gpu  # noqa: E402

w = WORKLOADS[sys.argv[1]]
k = int(sys.argv[2])
T = generate_gpu(w, seed=0)
cfg = PasdConfig(lambdas=w.lambdas(), ranks=list(w.ranks), maxiter=k + 10)
s = pb.Solver(w.dims, cfg, fixed_iters=True, poll_every=1)
s.load(T.data_ptr(), t_is_device=True)
for it in range(k + 3):
    if it >= k:
        print(f"--- iteration {it + 1}", flush=True)
    s.run(1)
