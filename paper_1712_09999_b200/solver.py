"""Host-side mirror of the reference entry point over the C-ABI library.

``pasd_recover`` is the drop-in for ``tenrec::pasd_recover``
(proj/include/tenrec/pasd.hpp:65-66): it hands the host tensor to
``pasd_b200_recover`` (include/pasd_b200.h), which runs every per-iteration
step as sm_100a kernels.  There is no CPU fallback: if ``libpasd_b200.so`` is
missing or no CUDA device is present the call raises.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

import numpy as np

from . import _abi
from .api import (ArgumentError, DeviceError, PasdConfig, RecoveryResult, as_tensor, build_options,
                  count_checks, raise_for_status, run_recover)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PASD_B200_LIB") or os.path.join(_HERE, "libpasd_b200.so")
_LIB = None


def lib():
    """Load libpasd_b200.so (raises if it was not built)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise DeviceError(f"{LIB_PATH} not built: run __graft_entry__.build() (make -C csrc)")
        L = C.CDLL(LIB_PATH)
        L.pasd_b200_recover.restype = C.c_int
        L.pasd_b200_recover.argtypes = [_abi.c_double_p, C.POINTER(_abi.PasdOptions), C.POINTER(_abi.PasdOutputs),
                                        _abi.PasdObserverFn, C.c_void_p, C.c_char_p, C.c_size_t]
        L.pasd_b200_release_cache.restype = None
        L.pasd_b200_release_cache.argtypes = []
        L.pasd_b200_validate.restype = C.c_int
        L.pasd_b200_validate.argtypes = [C.POINTER(_abi.PasdOptions), C.c_char_p, C.c_size_t]
        L.pasd_b200_default_lambdas.restype = C.c_int
        L.pasd_b200_default_lambdas.argtypes = [C.c_int32, _abi.c_int64_p, _abi.c_double_p, C.c_char_p, C.c_size_t]
        L.pasd_b200_default_rank_bound.restype = C.c_int
        L.pasd_b200_default_rank_bound.argtypes = [C.c_int64, _abi.c_int64_p, C.c_char_p, C.c_size_t]
        L.pasd_b200_solver_create.restype = C.c_int
        L.pasd_b200_solver_create.argtypes = [C.POINTER(_abi.PasdOptions), C.POINTER(_abi.PasdShard),
                                              C.POINTER(C.c_void_p), C.c_char_p, C.c_size_t]
        L.pasd_b200_solver_load.restype = C.c_int
        L.pasd_b200_solver_load.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_char_p, C.c_size_t]
        L.pasd_b200_solver_reset.restype = C.c_int
        L.pasd_b200_solver_reset.argtypes = [C.c_void_p, C.c_char_p, C.c_size_t]
        L.pasd_b200_solver_run.restype = C.c_int
        L.pasd_b200_solver_run.argtypes = [C.c_void_p, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                           C.c_char_p, C.c_size_t]
        L.pasd_b200_solver_finalize.restype = C.c_int
        L.pasd_b200_solver_finalize.argtypes = [C.c_void_p, C.POINTER(_abi.PasdOutputs), C.c_char_p, C.c_size_t]
        L.pasd_b200_solver_device_e.restype = C.c_void_p
        L.pasd_b200_solver_device_e.argtypes = [C.c_void_p]
        L.pasd_b200_solver_stream.restype = C.c_void_p
        L.pasd_b200_solver_stream.argtypes = [C.c_void_p]
        L.pasd_b200_solver_launches.restype = C.c_int64
        L.pasd_b200_solver_launches.argtypes = [C.c_void_p]
        L.pasd_b200_solver_destroy.restype = None
        L.pasd_b200_solver_destroy.argtypes = [C.c_void_p]
        L.pasd_b200_abi_version.restype = C.c_int
        L.pasd_b200_build_info.restype = C.c_char_p
        _LIB = L
    return _LIB


def _err():
    return C.create_string_buffer(1024)


def release_cache() -> None:
    """Free the solver pasd_recover keeps between calls of the same shape."""
    lib().pasd_b200_release_cache()


def validate_config(config: PasdConfig, dims: Sequence[int]) -> None:
    """PasdConfig::validate (pasd.cpp:12-49) through the C-ABI."""
    dims = [int(d) for d in dims]
    count_checks(dims, config)
    opt, keep = build_options(dims, config)
    err = _err()
    raise_for_status(lib().pasd_b200_validate(C.byref(opt), err, len(err)), err)


def default_lambdas(dims: Sequence[int]):
    d = np.asarray([int(x) for x in dims], dtype=np.int64)
    out = np.zeros(len(d))
    err = _err()
    rc = lib().pasd_b200_default_lambdas(len(d), d.ctypes.data_as(_abi.c_int64_p), _abi.dptr(out), err, len(err))
    raise_for_status(rc, err)
    return [float(x) for x in out]


def default_rank_bound(target_rank: int) -> int:
    out = C.c_int64(0)
    err = _err()
    rc = lib().pasd_b200_default_rank_bound(int(target_rank), C.byref(out), err, len(err))
    raise_for_status(rc, err)
    return int(out.value)


def pasd_recover(t, config: PasdConfig, observer=None, *, device: int = 0, fixed_iters: bool = False,
                 want_z: bool = True, want_y: bool = True, poll_every: int = 0,
                 reuse_solver: bool = False, fp32: bool = False) -> RecoveryResult:
    """Drop-in for tenrec::pasd_recover (pasd.hpp:65-66) on a B200.

    reuse_solver: keep the device solver for the next call with identical
    options (PASD_FLAG_REUSE_SOLVER; frees with release_cache()).
    fp32: float32 storage of the element tensors (PASD_FLAG_FP32)."""
    flags = (_abi.PASD_FLAG_FIXED_ITERS if fixed_iters else 0) | (_abi.PASD_FLAG_REUSE_SOLVER if reuse_solver else 0)
    flags |= _abi.PASD_FLAG_FP32 if fp32 else 0
    return run_recover(lib().pasd_b200_recover, t, config, observer, flags=flags, want_z=want_z, want_y=want_y,
                       device=device, poll_every=poll_every)


def snn_recover(t, config, observer=None, *, device: int = 0, fixed_iters: bool = False, want_z: bool = True,
                want_y: bool = True, poll_every: int = 0) -> RecoveryResult:
    """Drop-in for tenrec::snn_recover (baselines.hpp:39-40, baselines.cpp:37-143),
    the full-SVT ADMM baseline, on a B200 (pasd_b200_snn_recover).  `config`
    is an api.SnnConfig; y_hat and the certificate stay empty as in the
    reference."""
    L = lib()
    L.pasd_b200_snn_recover.restype = C.c_int
    flags = _abi.PASD_FLAG_FIXED_ITERS if fixed_iters else 0
    return run_recover(L.pasd_b200_snn_recover, t, config, observer, flags=flags, want_z=want_z, want_y=want_y,
                       device=device, poll_every=poll_every)


class Solver:
    """Device-resident solver handle (``pasd_b200_solver_*``) for benchmarks
    and sharded runs.  ``t`` may be a host numpy array or, with
    ``t_is_device``, an integer device pointer (e.g. ``torch_tensor.data_ptr()``)."""

    def __init__(self, dims: Sequence[int], config: PasdConfig, *, device: int = 0, fixed_iters: bool = False,
                 poll_every: int = 0, shard: Optional[_abi.PasdShard] = None, flags: int = 0, fp32: bool = False):
        self.dims = [int(d) for d in dims]
        self.local_dims = list(self.dims)
        sh = getattr(shard, "struct", shard)
        if sh is not None:
            self.local_dims[-1] = int(sh.slab_end - sh.slab_begin)
        self.config = config
        count_checks(self.dims, config)
        flags = int(flags) | (_abi.PASD_FLAG_FIXED_ITERS if fixed_iters else 0) | (_abi.PASD_FLAG_FP32 if fp32 else 0)
        self._opt, self._keep = build_options(self.dims, config, device=device, flags=flags, poll_every=poll_every)
        self._h = C.c_void_p()
        err = _err()
        self._shard = shard
        sh = getattr(shard, "struct", shard)
        rc = lib().pasd_b200_solver_create(C.byref(self._opt), C.byref(sh) if sh is not None else None,
                                           C.byref(self._h), err, len(err))
        raise_for_status(rc, err)

    def load(self, t, t_is_device: bool = False) -> None:
        err = _err()
        if t_is_device:
            ptr = C.c_void_p(int(t))
            self._t_keep = None
        else:
            flat = np.ravel(as_tensor(t), order="F")
            self._t_keep = flat
            ptr = C.c_void_p(flat.ctypes.data)
        rc = lib().pasd_b200_solver_load(self._h, ptr, 1 if t_is_device else 0, err, len(err))
        raise_for_status(rc, err)

    def reset(self) -> None:
        err = _err()
        raise_for_status(lib().pasd_b200_solver_reset(self._h, err, len(err)), err)

    def run(self, iters: int):
        done = C.c_int32(0)
        conv = C.c_int32(0)
        err = _err()
        rc = lib().pasd_b200_solver_run(self._h, int(iters), C.byref(done), C.byref(conv), err, len(err))
        raise_for_status(rc, err)
        return int(done.value), bool(conv.value)

    @property
    def stream(self) -> int:
        return int(lib().pasd_b200_solver_stream(self._h) or 0)

    @property
    def launches(self) -> int:
        return int(lib().pasd_b200_solver_launches(self._h))

    def ranks(self):
        """(svt_keep, polar_rank) per mode of the current iterate (pasd_b200_solver_ranks)."""
        n = len(self.dims)
        keep = (C.c_int32 * n)()
        prank = (C.c_int32 * n)()
        err = _err()
        L = lib()
        L.pasd_b200_solver_ranks.restype = C.c_int
        L.pasd_b200_solver_ranks.argtypes = [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.c_char_p,
                                             C.c_size_t]
        raise_for_status(L.pasd_b200_solver_ranks(self._h, keep, prank, err, len(err)), err)
        return list(keep), list(prank)

    def finalize(self, want_x=True, want_e=True, want_z=False, want_y=False, out_x=None, out_e=None,
                 want_y_hat=None):
        """Finalise into new arrays, or into `out_x` / `out_e` (contiguous float64
        buffers of the local slab's size, e.g. views of pinned host memory).
        Y-hat is returned with Y unless want_y_hat says otherwise."""
        if want_y_hat is None:
            want_y_hat = want_y
        n = len(self.dims)
        total = int(np.prod(self.local_dims))

        def dest(buf, want):
            if buf is None:
                return np.empty(total) if want else None
            buf = np.asarray(buf)
            if buf.dtype != np.float64 or buf.size != total or not buf.flags.c_contiguous:
                raise ValueError("finalize: output buffers must be contiguous float64 of the slab's size")
            return buf.reshape(-1)
        x = dest(out_x, want_x)
        e = dest(out_e, want_e)
        z = [np.empty(total) for _ in range(n)] if want_z else None
        y = [np.empty(total) for _ in range(n)] if want_y else None
        yh = [np.empty(total) for _ in range(n)] if want_y_hat else None
        hist = np.zeros(max(1, int(self.config.maxiter)))
        fres = np.zeros(n)
        out = _abi.PasdOutputs()
        out.x, out.e = _abi.dptr(x), _abi.dptr(e)
        zp, yp, yhp = _abi.ptr_array(z), _abi.ptr_array(y), _abi.ptr_array(yh)
        out.z, out.y, out.y_hat = zp, yp, yhp
        out.residual_history = _abi.dptr(hist)
        out.final_residuals = _abi.dptr(fres)
        err = _err()
        raise_for_status(lib().pasd_b200_solver_finalize(self._h, C.byref(out), err, len(err)), err)
        shape = tuple(self.local_dims)

        def rs(a):
            return None if a is None else a.reshape(shape, order="F")

        from .api import Certificate
        return RecoveryResult(
            x=rs(x), e=rs(e), z=[rs(a) for a in z] if z else None, iters=int(out.iters),
            converged=bool(out.converged), residual_history=[float(h) for h in hist[: out.iters]],
            final_residuals=[float(r) for r in fres], objective=float(out.objective),
            certificate=Certificate(out.cert_epsilon_hat, out.cert_c, out.cert_bound) if out.has_certificate else None,
            y=[rs(a) for a in y] if y else None, y_hat=[rs(a) for a in yh] if yh else None)

    def close(self) -> None:
        if getattr(self, "_h", None) and self._h.value:
            lib().pasd_b200_solver_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def svt(m, tau: float, *, device: int = 0):
    """SVT_tau(m) on the device (linops.cpp:78-91); returns (V, kept)."""
    m = np.asfortranarray(np.asarray(m, dtype=np.float64))
    if m.ndim != 2:
        raise ArgumentError("svt: expected a matrix")
    out = np.empty(m.shape, order="F")
    kept = C.c_int32(0)
    err = _err()
    L = lib()
    L.pasd_b200_svt.restype = C.c_int
    rc = L.pasd_b200_svt(_abi.dptr(np.ravel(m, order="F")), C.c_int64(m.shape[0]), C.c_int64(m.shape[1]),
                         C.c_double(tau), out.ctypes.data_as(_abi.c_double_p), C.byref(kept), C.c_int32(device),
                         err, C.c_size_t(len(err)))
    raise_for_status(rc, err)
    return out, int(kept.value)


def procrustes(g, v, u_prev=None, *, device: int = 0):
    """polar(g v^T) on the device (linops.cpp:93-104).

    Returns (U or None for the degenerate case, numerical rank of g v^T)."""
    g = np.asfortranarray(np.asarray(g, dtype=np.float64))
    v = np.asfortranarray(np.asarray(v, dtype=np.float64))
    if g.ndim != 2 or v.ndim != 2:
        raise ArgumentError("procrustes: expected matrices")
    if g.shape[1] != v.shape[1]:
        raise ArgumentError("procrustes: g and v must have the same number of columns")
    out = np.empty((g.shape[0], v.shape[0]), order="F")
    up = None if u_prev is None else np.ravel(np.asfortranarray(np.asarray(u_prev, dtype=np.float64)), order="F")
    deg = C.c_int32(0)
    rank = C.c_int32(0)
    err = _err()
    L = lib()
    L.pasd_b200_procrustes.restype = C.c_int
    rc = L.pasd_b200_procrustes(_abi.dptr(np.ravel(g, order="F")), C.c_int64(g.shape[0]), C.c_int64(g.shape[1]),
                                _abi.dptr(np.ravel(v, order="F")), C.c_int64(v.shape[0]), _abi.dptr(up),
                                out.ctypes.data_as(_abi.c_double_p), C.byref(deg), C.byref(rank), C.c_int32(device),
                                err, C.c_size_t(len(err)))
    raise_for_status(rc, err)
    return (None if deg.value else out), int(rank.value)


def _solver_profile(self, iters: int):
    """Eager run of `iters` iterations with CUDA events around every kernel
    (pasd_b200_solver_profile).  Returns {class: {ms, launches, bytes, flops}}."""
    K = len(_abi.PASD_KERNEL_CLASSES)
    ms = (C.c_double * K)()
    cnt = (C.c_int64 * K)()
    by = (C.c_double * K)()
    fl = (C.c_double * K)()
    err = _err()
    L = lib()
    L.pasd_b200_solver_profile.restype = C.c_int
    L.pasd_b200_solver_profile.argtypes = [C.c_void_p, C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_int64),
                                           C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_char_p, C.c_size_t]
    rc = L.pasd_b200_solver_profile(self._h, int(iters), ms, cnt, by, fl, err, len(err))
    raise_for_status(rc, err)
    return {name: {"ms": ms[k], "launches": int(cnt[k]), "bytes": by[k], "flops": fl[k]}
            for k, name in enumerate(_abi.PASD_KERNEL_CLASSES)}


Solver.profile = _solver_profile


def _solver_set_state(self, e, y, u, v, mu: float, iteration: int) -> None:
    """Inject a reference iterate (PasdState, pasd.hpp:33-41); see
    pasd_b200_solver_set_state.  e, y[n]: tensors; u[n]: I_n x R_n; v[n]:
    R_n x J_n in the unfolding layout."""
    n = len(self.dims)
    ef = np.ravel(np.asarray(e, dtype=np.float64), order="F")
    yf = [np.ravel(np.asarray(a, dtype=np.float64), order="F") for a in y]
    uf = [np.ravel(np.asfortranarray(np.asarray(a, dtype=np.float64)), order="F") for a in u]
    vf = [np.ravel(np.asfortranarray(np.asarray(a, dtype=np.float64)), order="F") for a in v]
    if len(yf) != n or len(uf) != n or len(vf) != n:
        raise ArgumentError("set_state: expected one y/u/v per mode")
    err = _err()
    L = lib()
    L.pasd_b200_solver_set_state.restype = C.c_int
    L.pasd_b200_solver_set_state.argtypes = [C.c_void_p, _abi.c_double_p, C.POINTER(_abi.c_double_p),
                                             C.POINTER(_abi.c_double_p), C.POINTER(_abi.c_double_p), C.c_double,
                                             C.c_int32, C.c_char_p, C.c_size_t]
    rc = L.pasd_b200_solver_set_state(self._h, _abi.dptr(ef), _abi.ptr_array(yf), _abi.ptr_array(uf),
                                      _abi.ptr_array(vf), C.c_double(mu), C.c_int32(iteration), err, len(err))
    raise_for_status(rc, err)


Solver.set_state = _solver_set_state


# ---- spec-shaped single-step API (pasd.hpp:43-58, 68-70) -------------------
def _f64(a):
    return np.ravel(np.asfortranarray(np.asarray(a, dtype=np.float64)), order="F")


def _dims_arg(t):
    d = np.ascontiguousarray(np.asarray(t.shape, dtype=np.int64))
    return d, d.ctypes.data_as(_abi.c_int64_p)


def pasd_g_matrix(t, e, y, mu: float, mode: int, *, device: int = 0) -> np.ndarray:
    """G_n = unfold_n(T - E + Y / mu) (pasd.cpp:82-97), on the device; mode 1-based."""
    t = as_tensor(t)
    if np.shape(e) != t.shape or np.shape(y) != t.shape:
        raise ArgumentError("g_matrix: dimension mismatch")  # pasd.cpp:84-85
    d, dp = _dims_arg(t)
    rows = t.shape[mode - 1] if 1 <= mode <= t.ndim else 1
    g = np.empty((rows, t.size // rows), order="F")
    err = _err()
    L = lib()
    L.pasd_b200_g_matrix.restype = C.c_int
    rc = L.pasd_b200_g_matrix(C.c_int32(t.ndim), dp, _abi.dptr(_f64(t)), _abi.dptr(_f64(e)), _abi.dptr(_f64(y)),
                              C.c_double(mu), C.c_int32(mode), g.ctypes.data_as(_abi.c_double_p), C.c_int32(device),
                              err, C.c_size_t(len(err)))
    raise_for_status(rc, err)
    return g


def update_u(state, t, mode: int, *, device: int = 0) -> np.ndarray:
    """Basis update (pasd.cpp:99-103): polar(G_n V_n^T), or the previous basis
    when the product is numerically zero."""
    t = as_tensor(t)
    n = mode - 1
    d, dp = _dims_arg(t)
    u_prev = _f64(state.u[n]) if 0 <= n < t.ndim else np.zeros(1)
    v = _f64(state.v[n]) if 0 <= n < t.ndim else np.zeros(1)
    rank = np.asarray(state.u[n]).shape[1] if 0 <= n < t.ndim else 1
    rows = t.shape[n] if 0 <= n < t.ndim else 1
    out = np.empty((rows, rank), order="F")
    deg = C.c_int32(0)
    err = _err()
    L = lib()
    L.pasd_b200_update_u.restype = C.c_int
    y = state.y[n] if 0 <= n < t.ndim else t
    rc = L.pasd_b200_update_u(C.c_int32(t.ndim), dp, _abi.dptr(_f64(t)), _abi.dptr(_f64(state.e)),
                              _abi.dptr(_f64(y)), C.c_double(state.mu), C.c_int32(mode), C.c_int64(rank),
                              _abi.dptr(u_prev), _abi.dptr(v), out.ctypes.data_as(_abi.c_double_p), C.byref(deg),
                              C.c_int32(device), err, C.c_size_t(len(err)))
    raise_for_status(rc, err)
    return out


def update_v(state, t, mode: int, lam: float, *, device: int = 0) -> np.ndarray:
    """Coefficient update (pasd.cpp:105-109): SVT_{lambda/mu}(U_n^T G_n)."""
    t = as_tensor(t)
    n = mode - 1
    d, dp = _dims_arg(t)
    ok = 0 <= n < t.ndim
    rank = np.asarray(state.u[n]).shape[1] if ok else 1
    cols = t.size // t.shape[n] if ok else 1
    out = np.empty((rank, cols), order="F")
    kept = C.c_int32(0)
    err = _err()
    L = lib()
    L.pasd_b200_update_v.restype = C.c_int
    rc = L.pasd_b200_update_v(C.c_int32(t.ndim), dp, _abi.dptr(_f64(t)), _abi.dptr(_f64(state.e)),
                              _abi.dptr(_f64(state.y[n] if ok else t)), C.c_double(state.mu), C.c_int32(mode),
                              C.c_int64(rank), _abi.dptr(_f64(state.u[n] if ok else np.zeros(1))), C.c_double(lam),
                              out.ctypes.data_as(_abi.c_double_p), C.byref(kept), C.c_int32(device), err,
                              C.c_size_t(len(err)))
    raise_for_status(rc, err)
    return out


def update_e(state, t, *, device: int = 0) -> np.ndarray:
    """Sparse update (pasd.cpp:111-130): shrink(mean_n(T - fold_n(U_n V_n) + Y_n / mu), 1 / (mu N))."""
    t = as_tensor(t)
    n = t.ndim
    d, dp = _dims_arg(t)
    if len(state.u) != n or len(state.v) != n or len(state.y) != n:
        raise ArgumentError("update_e: expected one u/v/y per mode")
    ranks = np.ascontiguousarray(np.asarray([np.asarray(u).shape[1] for u in state.u], dtype=np.int64))
    uf = [_f64(u) for u in state.u]
    vf = [_f64(v) for v in state.v]
    yf = [_f64(y) for y in state.y]
    out = np.empty(t.shape, order="F")
    err = _err()
    L = lib()
    L.pasd_b200_update_e.restype = C.c_int
    rc = L.pasd_b200_update_e(C.c_int32(n), dp, ranks.ctypes.data_as(_abi.c_int64_p), _abi.dptr(_f64(t)),
                              _abi.ptr_array(uf), _abi.ptr_array(vf), _abi.ptr_array(yf), C.c_double(state.mu),
                              out.ctypes.data_as(_abi.c_double_p), C.c_int32(device), err, C.c_size_t(len(err)))
    raise_for_status(rc, err)
    return out


def suboptimality_certificate(result: RecoveryResult, t, config: PasdConfig, *, device: int = 0):
    """Certificate of a converged run (pasd.cpp:277-309); StateError otherwise."""
    from .api import Certificate, StateError

    t = as_tensor(t)
    count_checks(list(t.shape), config)
    if not result.converged:
        raise StateError("certificate requires a converged result")
    if not result.y or not result.y_hat or len(result.y) != t.ndim or len(result.y_hat) != t.ndim:
        raise StateError("certificate requires the final multipliers")
    opt, keep = build_options(list(t.shape), config, device=device)
    yf = [_f64(a) for a in result.y]
    hf = [_f64(a) for a in result.y_hat]
    eh, c, b = C.c_double(0), C.c_double(0), C.c_double(0)
    err = _err()
    L = lib()
    L.pasd_b200_certificate.restype = C.c_int
    rc = L.pasd_b200_certificate(_abi.dptr(_f64(t)), C.byref(opt), C.c_int32(result.iters),
                                 C.c_int32(1 if result.converged else 0), _abi.ptr_array(yf), _abi.ptr_array(hf),
                                 C.byref(eh), C.byref(c), C.byref(b), err, C.c_size_t(len(err)))
    raise_for_status(rc, err)
    return Certificate(eh.value, c.value, b.value)
