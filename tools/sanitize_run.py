"""Small solves that touch every kernel of the library, for memory checking.

compute-sanitizer is closed on this GPU pool (runs under it left GPUs needing
a reset), so the check is the library's own guard-band mode:

    PASD_B200_GUARD=1 python tools/sanitize_run.py

(every device buffer gets 64 KB canary bands of NaN bytes, verified on free;
the run fails if any band was written, and a stray read of a band poisons the
result with NaN, which the NaN guard and the parity tests catch).  Under a
working compute-sanitizer the same script serves memcheck / racecheck.

Covers k_pass2_fused (16x8x8, RP 40 and 56 with ragged bricks), k_pass2_m8
(8x8x8), k_pass1 (both tile shapes), the Gram kernels, the cluster small
solves (k_polar, k_svt) through the V = 0 phase, the rank-deficient transition
and the full-rank phase, the generic order-4 path, the spec-shaped helpers,
the device generator and the sharded (one-rank NCCL) path.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1712_09999_b200 as pb  # noqa: E402
from paper_1712_09999_b200 import synth  # noqa: E402
from paper_1712_09999_b200.api import PasdConfig, PasdState  # noqa: E402


def instance(dims, r, rho, seed=0):
    spec = synth.SynthSpec(tuple(dims), (r,) * len(dims), rho, seed)
    T, _, _ = synth.generate(spec)
    return T


def run(dims, r, R, iters, env=None):
    for k in ("PASD_PASS2_M8", "PASD_PASS2_M16"):
        os.environ.pop(k, None)
    os.environ.update(env or {})
    T = instance(dims, r, 0.05)
    cfg = PasdConfig(lambdas=pb.default_lambdas(dims), ranks=[R] * len(dims), eps=1e-9, maxiter=iters)
    res = pb.pasd_recover(T, cfg, fixed_iters=True)
    print(dims, R, env, "iters", res.iters, "resid", res.residual_history[-1], flush=True)


run((37, 30, 29), 3, 3, 160)                                   # m8, through the transition to full rank
run((50, 44, 41), 6, 40, 12, {"PASD_PASS2_M16": "1"})          # fused 16x8x8, RP 40, ragged
run((66, 60, 57), 6, 50, 8, {"PASD_PASS2_M16": "1"})           # fused, RP 56
run((12, 11, 10, 9), 2, 2, 60)                                 # generic order-4 kernels
# spec helpers + certificate
T = instance((14, 12, 10), 2, 0.05, seed=2)
cfg = PasdConfig(lambdas=pb.default_lambdas(T.shape), ranks=[2, 2, 2], eps=1e-6)
res = pb.pasd_recover(T, cfg)
st = PasdState(u=[np.linalg.qr(np.random.default_rng(n).standard_normal((d, 2)))[0] for n, d in enumerate(T.shape)],
               v=[np.random.default_rng(5 + n).standard_normal((2, T.size // d)) for n, d in enumerate(T.shape)],
               e=res.e, y=res.y, mu=1.0)
for mode in (1, 2, 3):
    pb.pasd_g_matrix(T, res.e, res.y[mode - 1], 1.0, mode)
    pb.update_u(st, T, mode)
    pb.update_v(st, T, mode, 0.5)
pb.update_e(st, T)
if res.converged:
    pb.suboptimality_certificate(res, T, cfg)
# C4-style generator recipe
synth.generate(synth.SynthSpec((64, 48, 12), (6, 6, 3), 0.05, 0, 1, 2, 0.0, 1.0, 16, 5))
# sharded code path with a one-rank communicator
from paper_1712_09999_b200.sharding import Shard  # noqa: E402
s = pb.Solver(T.shape, cfg, shard=Shard(0, 1, (0, T.shape[2]), None))
s.load(T)
s.run(50)
s.finalize()
s.close()
# SNN baseline kernels and the loopback (nranks = 3) sharded path
from paper_1712_09999_b200.api import SnnConfig  # noqa: E402
from paper_1712_09999_b200.sharding import run_loopback  # noqa: E402

# fp32 mode: both pass-2 kernels (m8 at R = 3, the fused one at RP 40) on float32 storage
T32 = instance((37, 30, 29), 3, 0.05)
pb.pasd_recover(T32, PasdConfig(lambdas=pb.default_lambdas(T32.shape), ranks=[3, 3, 3], maxiter=160),
                fixed_iters=True, fp32=True)
T32 = instance((50, 44, 41), 6, 0.05)
pb.pasd_recover(T32, PasdConfig(lambdas=pb.default_lambdas(T32.shape), ranks=[40, 40, 40], maxiter=12),
                fixed_iters=True, fp32=True)
Ts = instance((20, 18, 16), 2, 0.05, seed=4)
pb.snn_recover(Ts, SnnConfig(lambdas=pb.default_lambdas(Ts.shape), maxiter=30), fixed_iters=True)
Tl = instance((26, 24, 29), 3, 0.05, seed=2)
run_loopback(Tl, PasdConfig(lambdas=pb.default_lambdas(Tl.shape), ranks=[3, 3, 3], maxiter=60), 3, 60)
import ctypes as C  # noqa: E402

L = pb.lib()
L.pasd_b200_guard_report.restype = C.c_int64
L.pasd_b200_guard_report.argtypes = [C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
pb.release_cache()
import gc  # noqa: E402

gc.collect()
checked, live = C.c_int64(0), C.c_int64(0)
viol = L.pasd_b200_guard_report(C.byref(checked), C.byref(live))
print(f"guard bands: mode={'on' if os.environ.get('PASD_B200_GUARD') == '1' else 'off'} buffers checked={checked.value} "
      f"still live={live.value} violations={viol}", flush=True)
assert viol == 0, "guard band overwritten"
print("sanitize_run done", flush=True)
