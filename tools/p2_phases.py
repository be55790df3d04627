"""Per-phase cycle split of k_pass2_fused from a PASD_P2_TIMING probe build
(tools/build_variant.sh p2t -DPASD_P2_TIMING=1; PASD_B200_LIB=build/p2t.so):
runs a few pass-2 launches of a workload through the solver's eager profile and
prints warp 0's cycles per phase (summed over CTAs) as shares and cycles/step.

    PASD_B200_LIB=build/p2t.so python tools/p2_phases.py [c5]
"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1712_09999_b200 as pb  # noqa: E402
from paper_1712_09999_b200.api import PasdConfig  # noqa: E402
from paper_1712_09999_b200.workloads import WORKLOADS  # noqa: E402

NAMES = ["loop top", "load issue + staging wait", "barrier A", "Z products", "barrier B", "elementwise",
         "barrier C", "Wt_1 + Wt_3", "barrier D", "staging issue", "Wt_2 + exchange", "pencil end"]
if os.environ.get("P2_NAMES"):
    NAMES = os.environ["P2_NAMES"].split(",")
w = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c5"]
T = bench.generate_input(w)
cfg = PasdConfig(lambdas=w.lambdas(), ranks=list(w.ranks), maxiter=40)
sol = pb.Solver(w.dims, cfg, fixed_iters=True)
sol.load(T.data_ptr(), t_is_device=True)
sol.run(3)
L = pb.lib()
L.pasd_b200_debug_p2_phases.restype = C.c_int
out = (C.c_double * 12)()
L.pasd_b200_debug_p2_phases(out)  # reset
prof = sol.profile(2)
L.pasd_b200_debug_p2_phases(out)
cyc = np.array(out[:])
brick = 512.0 if max(w.ranks) <= 24 else 1024.0  # k_pass2_m8: 8x8x8 bricks
steps = 2 * w.size / brick
print(f"{w.name}: pass 2 {prof['update']['ms'] / 2:.3f} ms/launch; warp-0 cycles per {int(brick)}-element step:")
for n, c in zip(NAMES, cyc):
    print(f"  {n:28s} {c / cyc.sum() * 100:5.1f}%  {c / steps:8.0f} cyc/step")
print(f"  {'total':28s}        {cyc.sum() / steps:8.0f} cyc/step (summed over CTAs / steps)")
