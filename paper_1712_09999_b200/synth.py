"""The reference's synthetic instance generator on the B200 (pasd_b200_synth).

Mirrors ``tenrec::gen_lowrank_tucker`` + ``tenrec::corrupt_sparse``
(proj/src/synth.cpp:71-121) with the reference's random streams
(proj/include/tenrec/rng.hpp:17-79): every draw -- core and factor Gaussians,
the partial Fisher-Yates support, the noise values -- is the reference's; the
tensor work (mode products, scatter in sorted-index order) runs on the device.
BASELINE configs[2..3] extensions (C3's U[-5,5] noise, C4's non-negative
factors and 16x16 block foreground) follow the oracle's documented recipe.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence, Tuple

import numpy as np

from . import _abi
from .api import raise_for_status
from .solver import _err, lib


class SynthSpecC(C.Structure):
    _fields_ = [
        ("order", C.c_int32),
        ("dims", _abi.c_int64_p),
        ("ranks", _abi.c_int64_p),
        ("seed", C.c_uint64),
        ("factor_kind", C.c_int32),
        ("corrupt_mode", C.c_int32),
        ("corruption", C.c_double),
        ("lo", C.c_double),
        ("hi", C.c_double),
        ("block", C.c_int64),
        ("cells", C.c_int64),
        ("device", C.c_int32),
    ]


@dataclass
class SynthSpec:
    """tenrec::SynthSpec (synth.hpp) plus the corruption recipe."""

    dims: Tuple[int, ...]
    ranks: Tuple[int, ...]
    corruption: float = 0.05
    seed: int = 0
    factor_kind: int = 0        # 0 Haar (reference), 1 non-negative (C4)
    corrupt_mode: int = 0       # 0 additive, 1 replace, 2 C4 blocks
    lo: float = -1.0
    hi: float = 1.0
    block: int = 16
    cells: int = 13


def workload_spec(w, seed: int = 0) -> SynthSpec:
    """The SynthSpec of a BASELINE workload (paper_1712_09999_b200.workloads)."""
    if w.kind == "nonneg":
        return SynthSpec(tuple(w.dims), tuple(w.tucker), w.rho, seed, 1, 2, w.noise[0], w.noise[1], 16, 13)
    return SynthSpec(tuple(w.dims), tuple(w.tucker), w.rho, seed, 0, 0 if w.mode == "add" else 1, w.noise[0],
                     w.noise[1])


def _cspec(s: SynthSpec, device: int):
    d = np.ascontiguousarray(np.asarray(s.dims, dtype=np.int64))
    r = np.ascontiguousarray(np.asarray(s.ranks, dtype=np.int64))
    c = SynthSpecC(len(s.dims), d.ctypes.data_as(_abi.c_int64_p), r.ctypes.data_as(_abi.c_int64_p), s.seed,
                   s.factor_kind, s.corrupt_mode, s.corruption, s.lo, s.hi, s.block, s.cells, device)
    return c, (d, r)


def generate(spec: SynthSpec, *, device: int = 0, out: str = "numpy", want_l0: bool = False,
             want_support: bool = False):
    """Observed tensor T (and optionally L0 and the sorted support).

    out="numpy": Fortran-ordered host arrays of shape dims.  out="torch": a
    CUDA tensor of shape reversed(dims) (C order = the reference's first-index-
    fastest layout).  Returns (T, L0 or None, support or None)."""
    cs, keep = _cspec(spec, device)
    S = int(np.prod(spec.dims))
    L = lib()
    L.pasd_b200_synth.restype = C.c_int
    sup = np.empty(S if want_support else 1, dtype=np.int64)
    cnt = C.c_int64(0)
    err = _err()
    if out == "torch":
        import torch

        dev = torch.device("cuda", device)
        T = torch.empty(tuple(reversed(spec.dims)), dtype=torch.float64, device=dev)
        L0 = torch.empty_like(T) if want_l0 else None
        rc = L.pasd_b200_synth(C.byref(cs), C.cast(C.c_void_p(T.data_ptr()), _abi.c_double_p), 1,
                               C.cast(C.c_void_p(L0.data_ptr()), _abi.c_double_p) if want_l0 else None, 1,
                               sup.ctypes.data_as(_abi.c_int64_p) if want_support else None, C.byref(cnt), err,
                               C.c_size_t(len(err)))
    else:
        T = np.empty(spec.dims, order="F")
        L0 = np.empty(spec.dims, order="F") if want_l0 else None
        rc = L.pasd_b200_synth(C.byref(cs), T.ctypes.data_as(_abi.c_double_p), 0,
                               L0.ctypes.data_as(_abi.c_double_p) if want_l0 else None, 0,
                               sup.ctypes.data_as(_abi.c_int64_p) if want_support else None, C.byref(cnt), err,
                               C.c_size_t(len(err)))
    raise_for_status(rc, err)
    return T, L0, (sup[: cnt.value].copy() if want_support else None)


def factor(rows: int, cols: int, seed: int, mode: int, kind: int = 0) -> np.ndarray:
    """Host-side factor of 1-based `mode` (no device needed)."""
    out = np.empty((rows, cols), order="F")
    err = _err()
    f = lib().pasd_b200_synth_factor
    f.restype = C.c_int
    rc = f(C.c_int64(rows), C.c_int64(cols), C.c_uint64(seed), C.c_int32(mode), C.c_int32(kind),
           out.ctypes.data_as(_abi.c_double_p), err, C.c_size_t(len(err)))
    raise_for_status(rc, err)
    return out


def support_draw_order(total: int, rho: float, seed: int) -> np.ndarray:
    """The partial Fisher-Yates selection of corrupt_sparse in draw order (host)."""
    out = np.empty(int(rho * total) + 2, dtype=np.int64)  # >= llround(rho * total)
    cnt = C.c_int64(0)
    err = _err()
    f = lib().pasd_b200_synth_support
    f.restype = C.c_int
    rc = f(C.c_int64(total), C.c_double(rho), C.c_uint64(seed), out.ctypes.data_as(_abi.c_int64_p), C.byref(cnt),
           err, C.c_size_t(len(err)))
    raise_for_status(rc, err)
    return out[: cnt.value]
