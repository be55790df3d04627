"""Bounded CPU samples of C5 against the measured full-size iteration
(profiles/r02_cpu_fullsize_c5.json: 91.2 s/iter on 1 thread): which sample,
scaled per element, predicts the full-size per-iteration time.

    python tools/cpu_samples.py > gpurun_out/cpu_samples.json
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_1712_09999_b200.workloads import WORKLOADS  # noqa: E402

w = WORKLOADS["c5"]
out = {}
for name, dims, tucker in (("slab_1000x1000x50", (1000, 1000, 50), (50, 50, 50)),
                           ("half_cube_500", (500, 500, 500), (50, 50, 50)),
                           ("cube_400", (400, 400, 400), (50, 50, 50))):
    cb = bench.cpu_baseline(w, 1, iters=3, sample=(dims, tucker, (50, 50, 50)))
    out[name] = {k: cb[k] for k in ("value", "elem_iters_per_s", "sample_dims")}
    out[name]["predicted_full_s_per_iter"] = 1.0 / cb["value"]
    print(json.dumps({name: out[name]}), flush=True)
