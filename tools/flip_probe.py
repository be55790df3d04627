"""E-support flips between the CUDA path and the oracle at C2 (200^3, R=20, 200
fixed iterations): how far from the shrink threshold 1/(mu N) the flipped
entries are, for both pass-2 variants (k_pass2_m8 default at R=20, and the
16x8x8 k_pass2_fused forced with PASD_PASS2_M16), and how the multiplier sums
sum_n Y_n compare.  Development probe (prints JSON lines)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_1712_09999_b200 as pb  # noqa: E402
from paper_1712_09999_b200.api import PasdConfig  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


dims, r, rho, K = (200, 200, 200), 20, 0.2, int(os.environ.get("FLIP_K", "200"))
L0 = oracle.gen_tucker(dims, [r] * 3, seed=0)
T = oracle.corrupt_sparse(L0, rho, seed=0)
cfg = PasdConfig(lambdas=oracle.default_lambdas(dims), ranks=[r] * 3, eps=1e-7, maxiter=K)
ro = oracle.pasd_recover(T, cfg, fixed_iters=True, threads=16)
ro2 = oracle.pasd_recover(T, cfg, fixed_iters=True, threads=16, svd_variant=1)
print(json.dumps({"oracle_dgesdd_vs_dgesvd": {"flips": int(np.count_nonzero((ro.e != 0) != (ro2.e != 0))),
                                                "sumY_rel": rel(sum(ro2.y), sum(ro.y)), "x_rel": rel(ro2.x, ro.x)}}),
      flush=True)
mu = cfg.mu0 * cfg.rho ** (K - 1)
tau = 1.0 / (mu * 3)
runs = {"m8": {}, "m16": {"PASD_PASS2_M16": "1"}}
for name, env in runs.items():
    os.environ.pop("PASD_PASS2_M16", None)
    os.environ.update(env)
    rg = pb.pasd_recover(T, cfg, fixed_iters=True)
    egf, eof = np.ravel(rg.e, order="F"), np.ravel(ro.e, order="F")
    fl = np.flatnonzero((egf != 0) != (eof != 0))
    eg, eo = egf[fl], eof[fl]
    mag = np.maximum(np.abs(eg), np.abs(eo))  # the nonzero side: |x| - tau
    sy_g = sum(rg.y)
    sy_o = sum(ro.y)
    print(json.dumps({
        "variant": name, "iters": K, "tau_E": tau, "flips": int(fl.size),
        "flip_nonzero_mag_max": float(mag.max()) if fl.size else None,
        "flip_nonzero_mag_median": float(np.median(mag)) if fl.size else None,
        "flip_gpu_side_nonzero": int(np.count_nonzero(eg)), "flip_oracle_side_nonzero": int(np.count_nonzero(eo)),
        "flip_mag_over_tau_max": float(mag.max() / tau) if fl.size else None,
        "x_rel": rel(rg.x, ro.x), "e_rel": rel(rg.e, ro.e), "sumY_rel": rel(sy_g, sy_o),
        "e_support_gpu": int(np.count_nonzero(rg.e)), "e_support_oracle": int(np.count_nonzero(ro.e)),
    }), flush=True)
