import sys
import numpy as np
sys.path.insert(0, "/root/repo")
import oracle
from paper_1712_09999_b200 import solver as S
rng = np.random.default_rng(0)
for (r, c, tau) in [(3, 8, 0.5), (10, 200, 5.0), (20, 1000, 10.0), (50, 3000, 30.0), (7, 7, 1.0)]:
    m = rng.standard_normal((r, c))
    vo = oracle.svt(m, tau); vg, kept = S.svt(m, tau)
    print("svt", r, c, tau, "kept", kept, "rel", np.linalg.norm(vo - vg) / max(np.linalg.norm(vo), 1e-300))
for (I, P, R, rk) in [(20, 50, 3, 3), (20, 50, 3, 1), (100, 400, 10, 10), (100, 400, 10, 4), (200, 900, 20, 0), (1000, 300, 50, 50), (1000, 300, 50, 17)]:
    g = rng.standard_normal((I, P))
    v = rng.standard_normal((R, P))
    if rk < R:
        # rank-deficient v: rk nonzero directions
        q, _ = np.linalg.qr(rng.standard_normal((R, R)))
        d = np.zeros(R); d[:rk] = rng.uniform(0.5, 2, rk)
        v = q @ np.diag(d) @ q.T @ v
    uo = oracle.procrustes(g, v); ug, rank = S.procrustes(g, v)
    if ug is None or uo is None:
        print("proc", I, P, R, rk, "degenerate", uo is None, ug is None); continue
    orth = np.abs(ug.T @ ug - np.eye(R)).max()
    fo = np.linalg.norm(uo @ v - g); fg = np.linalg.norm(ug @ v - g)
    print("proc", I, P, R, rk, "rank", rank, "rel", np.linalg.norm(uo - ug) / np.linalg.norm(uo), "orth", orth,
          "obj oracle", fo, "gpu", fg)
