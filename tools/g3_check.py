import sys, json, os
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_1712_09999_b200 as pb
from paper_1712_09999_b200.api import PasdConfig
from paper_1712_09999_b200.tnsr import read_tensor
d = "/root/repo/tests/golden/g3_24x20x16_r3_R4"
meta = json.load(open(d + "/meta.json"))
T = read_tensor(d + "/t.tnsr"); L0 = read_tensor(d + "/l0.tnsr")
cfg = PasdConfig(lambdas=meta["lambdas"], ranks=meta["ranks"], eps=meta["eps"])
r = pb.pasd_recover(T, cfg)
print(os.environ.get("PASD_PASS2_M16"), r.iters, r.converged, np.linalg.norm(r.x - L0) / np.linalg.norm(L0), r.residual_history[-3:], "oracle iters", meta["iters"])
