"""ctypes wrapper of the CPU restatement (``oracle/liboracle.so``).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
CPU-baseline legs of bench.py — never by the product package.  See the header
of pasd_oracle.cpp for what it restates and how parity is pinned.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_1712_09999_b200 import _abi
from paper_1712_09999_b200.api import (ArgumentError, PasdConfig, raise_for_status, run_recover,
                                       as_tensor)

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def build() -> str:
    """Compile liboracle.so with the committed Makefile (gcc, no GPU)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return os.path.join(_HERE, "liboracle.so")


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        L.oracle_pasd_recover.restype = C.c_int
        L.oracle_pasd_recover.argtypes = [
            _abi.c_double_p, C.POINTER(_abi.PasdOptions), C.POINTER(_abi.PasdOutputs), _abi.PasdObserverFn,
            C.c_void_p, C.c_int, C.c_int, C.c_char_p, C.c_size_t]
        L.oracle_snn_recover.restype = C.c_int
        L.oracle_snn_recover.argtypes = L.oracle_pasd_recover.argtypes
        _LIB = L
    return _LIB


def _err():
    return C.create_string_buffer(1024)


def pasd_recover(t, config: PasdConfig, observer=None, *, svd_variant: int = 0, threads: int = 1,
                 fixed_iters: bool = False, want_z: bool = True, want_y: bool = True):
    """Reference-restated pasd_recover (pasd.cpp:132-275)."""
    flags = _abi.PASD_FLAG_FIXED_ITERS if fixed_iters else 0
    return run_recover(lib().oracle_pasd_recover, t, config, observer, flags=flags, want_z=want_z,
                       want_y=want_y, extra_args=(C.c_int(svd_variant), C.c_int(threads)))


def snn_recover(t, config, observer=None, *, svd_variant: int = 0, threads: int = 1, fixed_iters: bool = False,
                want_z: bool = True, want_y: bool = True):
    """Reference-restated snn_recover (baselines.cpp:37-143); config: api.SnnConfig."""
    flags = _abi.PASD_FLAG_FIXED_ITERS if fixed_iters else 0
    return run_recover(lib().oracle_snn_recover, t, config, observer, flags=flags, want_z=want_z,
                       want_y=want_y, extra_args=(C.c_int(svd_variant), C.c_int(threads)))


def gen_tucker(dims, ranks, seed: int = 0, kind: int = 0) -> np.ndarray:
    """gen_lowrank_tucker (synth.cpp:71-89), kind 1 = non-negative C4 recipe."""
    dims = [int(d) for d in dims]
    out = np.empty(int(np.prod(dims)))
    d = np.asarray(dims, dtype=np.int64)
    r = np.asarray(ranks, dtype=np.int64)
    err = _err()
    rc = lib().oracle_gen_tucker(C.c_int(len(dims)), d.ctypes.data_as(_abi.c_int64_p),
                                 r.ctypes.data_as(_abi.c_int64_p), C.c_uint64(seed), C.c_int(kind),
                                 _abi.dptr(out), err, C.c_size_t(len(err)))
    raise_for_status(rc, err)
    return out.reshape(dims, order="F")


def corrupt_sparse(t, rho: float, seed: int = 0, mode: int = 0, lo: float = -1.0, hi: float = 1.0):
    """corrupt_sparse (synth.cpp:91-121); mode 0 additive U[lo,hi], 1 replace."""
    t = as_tensor(t)
    flat = np.ravel(t, order="F")
    out = np.empty_like(flat)
    cnt = C.c_int64(0)
    err = _err()
    rc = lib().oracle_corrupt_sparse(_abi.dptr(flat), C.c_int64(flat.size), C.c_double(rho), C.c_uint64(seed),
                                     C.c_int(mode), C.c_double(lo), C.c_double(hi), _abi.dptr(out),
                                     C.byref(cnt), err, C.c_size_t(len(err)))
    raise_for_status(rc, err)
    return out.reshape(t.shape, order="F")


def corrupt_blocks(t, block: int, cells: int, seed: int = 0, lo: float = 0.0, hi: float = 1.0):
    t = as_tensor(t)
    flat = np.ravel(t, order="F")
    out = np.empty_like(flat)
    d = np.asarray(t.shape, dtype=np.int64)
    err = _err()
    rc = lib().oracle_corrupt_blocks(_abi.dptr(flat), C.c_int(t.ndim), d.ctypes.data_as(_abi.c_int64_p),
                                     C.c_int64(block), C.c_int64(cells), C.c_uint64(seed), C.c_double(lo),
                                     C.c_double(hi), _abi.dptr(out), err, C.c_size_t(len(err)))
    raise_for_status(rc, err)
    return out.reshape(t.shape, order="F")


def unfold(t, mode: int) -> np.ndarray:
    t = as_tensor(t)
    d = np.asarray(t.shape, dtype=np.int64)
    rows = t.shape[mode - 1] if 1 <= mode <= t.ndim else 1
    out = np.empty(t.size)
    err = _err()
    rc = lib().oracle_unfold(_abi.dptr(np.ravel(t, order="F")), C.c_int(t.ndim), d.ctypes.data_as(_abi.c_int64_p),
                             C.c_int(mode), _abi.dptr(out), err, C.c_size_t(len(err)))
    raise_for_status(rc, err)
    return out.reshape((rows, t.size // rows), order="F")


def fold(m, mode: int, dims) -> np.ndarray:
    m = np.asfortranarray(np.asarray(m, dtype=np.float64))
    d = np.asarray(dims, dtype=np.int64)
    out = np.empty(int(np.prod(dims)))
    err = _err()
    rc = lib().oracle_fold(_abi.dptr(np.ravel(m, order="F")), C.c_int(len(dims)), d.ctypes.data_as(_abi.c_int64_p),
                           C.c_int(mode), _abi.dptr(out), err, C.c_size_t(len(err)))
    raise_for_status(rc, err)
    return out.reshape(tuple(dims), order="F")


def thin_svd(m):
    m = np.asfortranarray(np.asarray(m, dtype=np.float64))
    rows, cols = m.shape
    k = min(rows, cols)
    u = np.empty((rows, k), order="F")
    s = np.empty(k)
    v = np.empty((cols, k), order="F")
    err = _err()
    rc = lib().oracle_thin_svd(_abi.dptr(np.ravel(m, order="F")), C.c_int64(rows), C.c_int64(cols),
                               u.ctypes.data_as(_abi.c_double_p), _abi.dptr(s), v.ctypes.data_as(_abi.c_double_p),
                               err, C.c_size_t(len(err)))
    raise_for_status(rc, err)
    return u, s, v


def svt(m, tau: float):
    m = np.asfortranarray(np.asarray(m, dtype=np.float64))
    out = np.empty(m.shape, order="F")
    err = _err()
    rc = lib().oracle_svt(_abi.dptr(np.ravel(m, order="F")), C.c_int64(m.shape[0]), C.c_int64(m.shape[1]),
                          C.c_double(tau), out.ctypes.data_as(_abi.c_double_p), err, C.c_size_t(len(err)))
    raise_for_status(rc, err)
    return out


def procrustes(g, v):
    """Returns U, or None for the degenerate case (linops.cpp:93-104)."""
    g = np.asfortranarray(np.asarray(g, dtype=np.float64))
    v = np.asfortranarray(np.asarray(v, dtype=np.float64))
    out = np.empty((g.shape[0], v.shape[0]), order="F")
    deg = C.c_int(0)
    err = _err()
    rc = lib().oracle_procrustes(_abi.dptr(np.ravel(g, order="F")), C.c_int64(g.shape[0]), C.c_int64(g.shape[1]),
                                 _abi.dptr(np.ravel(v, order="F")), C.c_int64(v.shape[0]),
                                 C.c_int64(v.shape[1]), out.ctypes.data_as(_abi.c_double_p), C.byref(deg), err, C.c_size_t(len(err)))
    raise_for_status(rc, err)
    return None if deg.value else out


def soft_threshold(x: float, tau: float) -> float:
    f = lib().oracle_soft_threshold
    f.restype = C.c_double
    f.argtypes = [C.c_double, C.c_double]
    return f(x, tau)


def default_lambdas(dims):
    """PasdConfig::default_lambdas restated in Python (pasd.cpp:51-60)."""
    import math
    total = int(np.prod([int(d) for d in dims]))
    n = float(len(dims))
    return [math.sqrt(float(max(int(d), total // int(d)))) / n for d in dims]


def pasd_v0_phase(t, config: PasdConfig, iters: int, *, threads: int = 1, fixed_iters: bool = True,
                  e_out=None, y_out=None):
    """pasd_recover restricted to the V = 0 phase (pasd_oracle.cpp v0_phase).

    Returns (e, y, history, final_residuals, min_margin, left_at, iters_done):
    left_at is the first iteration whose SVT would keep a singular value (the
    phase ends there and the run stops before it), 0 if the phase lasted.
    e_out / y_out may be preallocated Fortran-ordered float64 tensors."""
    from paper_1712_09999_b200.api import build_options
    t = as_tensor(t)
    dims = t.shape
    opt, _keep = build_options(dims, config, flags=_abi.PASD_FLAG_FIXED_ITERS if fixed_iters else 0)
    S = t.size
    e = e_out if e_out is not None else np.empty(dims, order="F")
    ys = y_out if y_out is not None else [np.empty(dims, order="F") for _ in dims]
    for a in [e] + list(ys):
        assert a.flags.f_contiguous and a.dtype == np.float64 and a.shape == dims
    yp = (_abi.c_double_p * len(dims))(*[_abi.dptr(np.ravel(y, order="K")) for y in ys])
    hist = np.zeros(max(1, iters))
    resid = np.zeros(len(dims))
    margin = C.c_double(0.0)
    left = C.c_int(0)
    done = C.c_int(0)
    err = _err()
    f = lib().oracle_pasd_v0_phase
    f.restype = C.c_int
    rc = f(_abi.dptr(np.ravel(t, order="K")), C.byref(opt), C.c_int(iters), C.c_int(threads),
           _abi.dptr(np.ravel(e, order="K")), yp, _abi.dptr(hist), _abi.dptr(resid), C.byref(margin),
           C.byref(left), C.byref(done), err, C.c_size_t(len(err)))
    raise_for_status(rc, err)
    assert e.size == S
    return e, ys, hist[:done.value].tolist(), resid, margin.value, left.value, done.value


def factor(rows: int, cols: int, seed: int, mode: int, kind: int = 0) -> np.ndarray:
    """Factor matrix of gen_lowrank_tucker for 1-based `mode` (synth.cpp:40-53, 80-83)."""
    out = np.empty((rows, cols), order="F")
    err = _err()
    f = lib().oracle_factor
    f.restype = C.c_int
    rc = f(C.c_int64(rows), C.c_int64(cols), C.c_uint64(seed), C.c_int(mode), C.c_int(kind),
           out.ctypes.data_as(_abi.c_double_p), err, C.c_size_t(len(err)))
    raise_for_status(rc, err)
    return out
