import sys, ctypes as C
import numpy as np
sys.path.insert(0, "/root/repo")
from paper_1712_09999_b200 import solver as S
S.LIB_PATH = "/root/repo/tools/libpasd_dbg.so"
rng = np.random.default_rng(0)
g = rng.standard_normal((6, 5)); v = rng.standard_normal((2, 5))
w = g @ v.T
print("W", w)
u, s, vt = np.linalg.svd(w, full_matrices=False)
print("ref polar", u @ vt)
print("eig WtW", np.linalg.eigh(w.T @ w))
ug, rank = S.procrustes(g, v)
print("gpu", ug, rank)
