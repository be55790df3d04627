"""BASELINE.json workloads (configs C1-C5) and a seeded GPU input generator.

Inputs come from the reference generator (proj/src/synth.cpp:71-121) with the
reference's random streams, run on the device by synth.py (pasd_b200_synth);
the oracle restates the same generator for the parity tests.  Outputs are
torch tensors of shape (I_N, ..., I_1) in C order, i.e. the reference's
first-index-fastest layout (tensor.hpp:23-24) of a tensor with dims
(I_1, ..., I_N).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Tuple


@dataclass(frozen=True)
class Workload:
    name: str
    dims: Tuple[int, ...]
    tucker: Tuple[int, ...]
    ranks: Tuple[int, ...]
    rho: float
    noise: Tuple[float, float]
    iters: int
    kind: str = "haar"          # "haar" (reference recipe) or "nonneg" (C4 video-like)
    mode: str = "add"           # corruption: "add" (additive) or "replace"
    eps: float = 1e-7

    @property
    def size(self) -> int:
        return int(math.prod(self.dims))

    def lambdas(self) -> List[float]:
        """PasdConfig::default_lambdas (pasd.cpp:51-60) == alpha_n/lambda_n of
        BASELINE's HoRPCA parameterisation (SURVEY 8(d) lambda mapping)."""
        total = self.size
        n = float(len(self.dims))
        return [math.sqrt(float(max(d, total // d))) / n for d in self.dims]


# BASELINE.json "configs" (index = list position).
WORKLOADS = {
    "c1": Workload("c1_100cube_r10", (100, 100, 100), (10, 10, 10), (10, 10, 10), 0.10, (-1.0, 1.0), 100),
    "c2": Workload("c2_200cube_r20", (200, 200, 200), (20, 20, 20), (20, 20, 20), 0.20, (-1.0, 1.0), 200),
    "c3": Workload("c3_400cube_r40", (400, 400, 400), (40, 40, 40), (40, 40, 40), 0.10, (-5.0, 5.0), 100),
    "c4": Workload("c4_video_256x256x1024", (256, 256, 1024), (30, 30, 15), (30, 30, 15), 0.05, (0.0, 1.0), 100,
                   kind="nonneg", mode="replace"),
    "c5": Workload("c5_1000cube_r50", (1000, 1000, 1000), (50, 50, 50), (50, 50, 50), 0.10, (-1.0, 1.0), 50),
}


def generate_gpu(w: Workload, seed: int = 0, device: str = "cuda:0"):
    """Seeded observation T = L0 + E0 of workload w from the reference
    generator on the device (synth.py: synth.cpp:71-121 with the reference's
    RNG streams).  Returns a contiguous torch tensor of shape reversed(dims)
    (first index of the reference tensor fastest)."""
    from . import synth

    dev = int(str(device).split(":")[1]) if ":" in str(device) else 0
    T, _, _ = synth.generate(synth.workload_spec(w, seed=seed), device=dev, out="torch")
    return T
