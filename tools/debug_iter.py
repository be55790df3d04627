import sys
import numpy as np
sys.path.insert(0, "/root/repo")
import oracle
import paper_1712_09999_b200 as pb
from paper_1712_09999_b200.api import PasdConfig
dims = [20, 20, 20]
L0 = oracle.gen_tucker(dims, [2, 2, 2], seed=0)
T = L0
lam = oracle.default_lambdas(dims)
cfg = PasdConfig(lambdas=lam, ranks=[3, 3, 3], eps=1e-5, maxiter=110)
logs = {}
def mk(name):
    logs[name] = []
    def f(v):
        if v.iter < 88: return
        logs[name].append((v.iter, [np.linalg.svd(x, compute_uv=False)[:3].round(6).tolist() for x in v.v],
                           [float(np.abs(u.T @ u - np.eye(u.shape[1])).max()) for u in v.u],
                           max(v.residual_inf), float(np.linalg.norm(v.e)), [float(np.linalg.norm(z)) for z in v.z],
                           v.u[0][:4, :].round(4).tolist()))
    return f
oracle.pasd_recover(T, cfg, observer=mk("oracle"), fixed_iters=True)
pb.pasd_recover(T, cfg, observer=mk("gpu"), fixed_iters=True)
for a, b in zip(logs["oracle"], logs["gpu"]):
    print("iter", a[0], "\n  O sv", a[1], "orth", a[2], "res", a[3], "|e|", a[4], "|z|", a[5], "\n  G sv", b[1], "orth", b[2], "res", b[3], "|e|", b[4], "|z|", b[5])
    if a[0] in (96, 97, 98): print("  O u0", a[6], "\n  G u0", b[6])
