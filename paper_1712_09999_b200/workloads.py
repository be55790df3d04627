"""BASELINE.json workloads (configs C1-C5) and a seeded GPU input generator.

The reference generator (proj/src/synth.cpp:71-121) is reproduced bit-for-bit
by the oracle (oracle/pasd_oracle.cpp) for parity tests at small sizes.  For
benchmark-scale inputs (C3-C5: up to 8 GB per tensor) this module draws the
same distributions on the GPU with torch (plumbing, outside the timed hot
path): Gaussian Tucker core, Haar (QR-of-Gaussian, sign-fixed) factors,
i.i.d. Bernoulli(rho) support with uniform values.  Outputs are torch tensors
of shape (I_N, ..., I_1) in C order, i.e. the reference's first-index-fastest
layout (tensor.hpp:23-24) of a tensor with dims (I_1, ..., I_N).
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
    """Seeded synthetic observation T = L0 + E0 on the GPU (fp64).

    Returns a contiguous torch tensor of shape reversed(dims) (first index of
    the reference tensor fastest)."""
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(seed)
    dt = torch.float64
    core = torch.randn(*reversed(w.tucker), generator=g, device=device, dtype=dt)  # (r3, r2, r1)
    if w.kind == "nonneg":
        core = core.abs()
    facs = []
    for d, r in zip(w.dims, w.tucker):
        a = torch.randn(d, r, generator=g, device=device, dtype=dt)
        if w.kind == "nonneg":
            a = a.abs()
            a = a / a.norm(dim=0, keepdim=True)
        else:
            q, rr = torch.linalg.qr(a)
            q = q * torch.sign(torch.diagonal(rr)).where(torch.diagonal(rr) != 0, torch.ones((), device=device, dtype=dt))
            a = q
        facs.append(a)
    if len(w.dims) != 3:
        raise ValueError("generate_gpu: order-3 workloads only")
    u1, u2, u3 = facs
    # core is (r3, r2, r1); L[k, j, i] = sum core[c, b, a] u1[i,a] u2[j,b] u3[k,c]
    t1 = torch.einsum("cba,kc->kba", core, u3)
    t2 = torch.einsum("kba,jb->kja", t1, u2)
    L = torch.matmul(t2, u1.T).contiguous()  # (I3, I2, I1)
    del t1, t2
    if w.kind == "nonneg":
        L /= L.max()
    lo, hi = w.noise
    flat = L.view(-1)
    chunk = 1 << 27
    if w.name.startswith("c4"):
        _blocks_gpu(L, g, lo, hi)
    else:
        for s in range(0, flat.numel(), chunk):
            part = flat[s:s + chunk]
            mask = torch.rand(part.numel(), generator=g, device=device, dtype=dt) < w.rho
            vals = lo + (hi - lo) * torch.rand(part.numel(), generator=g, device=device, dtype=dt)
            if w.mode == "add":
                part.add_(torch.where(mask, vals, torch.zeros((), device=device, dtype=dt)))
            else:
                part.copy_(torch.where(mask, vals, part))
    return L


def _blocks_gpu(L, g, lo, hi, block: int = 16, cells: int = 13):
    """C4 foreground: per frame, `cells` of the aligned 16x16 cells of the
    (mode-1 x mode-2) plane replaced by U[lo,hi] (~5.08% of entries)."""
    import torch

    I3, I2, I1 = L.shape
    c1, c2 = I1 // block, I2 // block
    dev = L.device
    scores = torch.rand(I3, c2 * c1, generator=g, device=dev)
    chosen = scores.argsort(dim=1)[:, :cells]  # cells per frame without replacement
    mask = torch.zeros(I3, c2 * c1, dtype=torch.bool, device=dev)
    mask.scatter_(1, chosen, True)
    mask = mask.view(I3, c2, 1, c1, 1).expand(I3, c2, block, c1, block).reshape(I3, I2, I1)
    vals = lo + (hi - lo) * torch.rand(L.shape, generator=g, device=dev, dtype=L.dtype)
    L.copy_(torch.where(mask, vals, L))
