"""Python mirror of the reference solver interface (``proj/include/tenrec``).

* ``PasdConfig``      — ``tenrec::PasdConfig``      (pasd.hpp:8-27)
* ``Certificate``     — ``tenrec::Certificate``     (recovery.hpp:14-18)
* ``RecoveryResult``  — ``tenrec::RecoveryResult``  (recovery.hpp:20-34)
* ``IterationView``   — ``tenrec::IterationView``   (recovery.hpp:38-48)
* ``PasdState``       — ``tenrec::PasdState``       (pasd.hpp:33-41)
* ``ArgumentError`` / ``IoError`` / ``NumericalError`` / ``StateError``
  — the exception taxonomy of errors.hpp:9-30.

Tensors are numpy float64 arrays of shape ``dims`` in Fortran order (first
index fastest), the reference's storage order (tensor.hpp:23-24).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

import numpy as np

from . import _abi


class TenrecError(Exception):
    """Base of the reference exception taxonomy."""


class ArgumentError(TenrecError, ValueError):
    """tenrec::ArgumentError (errors.hpp:9-12)."""


class IoError(TenrecError, OSError):
    """tenrec::IoError (errors.hpp:15-18)."""


class NumericalError(TenrecError, RuntimeError):
    """tenrec::NumericalError (errors.hpp:21-24)."""


class StateError(TenrecError, RuntimeError):
    """tenrec::StateError (errors.hpp:27-30)."""


class DeviceError(TenrecError, RuntimeError):
    """CUDA / NCCL failure (no reference analogue)."""


_ERR = {
    _abi.PASD_ERR_ARGUMENT: ArgumentError,
    _abi.PASD_ERR_IO: IoError,
    _abi.PASD_ERR_NUMERICAL: NumericalError,
    _abi.PASD_ERR_STATE: StateError,
    _abi.PASD_ERR_CUDA: DeviceError,
}


def raise_for_status(rc: int, errbuf) -> None:
    if rc == _abi.PASD_OK:
        return
    msg = errbuf.value.decode(errors="replace") if errbuf is not None else ""
    raise _ERR.get(rc, TenrecError)(msg)


@dataclass
class PasdConfig:
    """Hyperparameters of the factored ADMM solver (pasd.hpp:8-27)."""

    lambdas: List[float]
    ranks: List[int]
    mu0: float = 1e-4
    mu_max: float = 1e10
    rho: float = 1.1
    eps: float = 1e-5
    maxiter: int = 1000
    output_weights: List[float] = field(default_factory=list)

    def alphas(self) -> List[float]:
        """output_weights, or lambdas when empty (pasd.hpp:26)."""
        return list(self.output_weights) if self.output_weights else list(self.lambdas)

    def validate(self, dims: Sequence[int]) -> None:
        """PasdConfig::validate (pasd.cpp:12-49): same checks and messages."""
        from .solver import validate_config

        validate_config(self, dims)

    @staticmethod
    def default_lambdas(dims: Sequence[int]) -> List[float]:
        """lambda_n = sqrt(max(I_n, prod_{j!=n} I_j)) / N (pasd.cpp:51-60)."""
        from .solver import default_lambdas

        return default_lambdas(dims)

    @staticmethod
    def default_rank_bound(target_rank: int) -> int:
        """floor(1.2 r) in exact integer arithmetic (pasd.cpp:62-66)."""
        from .solver import default_rank_bound

        return default_rank_bound(target_rank)


@dataclass
class SnnConfig:
    """Hyperparameters of the full-SVT ADMM baseline (tenrec::SnnConfig,
    baselines.hpp:9-20): one nuclear-norm term per unfolding, no ranks."""

    lambdas: List[float]
    mu0: float = 1e-4
    mu_max: float = 1e10
    rho: float = 1.1
    eps: float = 1e-5
    maxiter: int = 1000
    output_weights: List[float] = field(default_factory=list)

    @property
    def ranks(self) -> List[int]:  # the C-ABI options struct carries ranks; SNN ignores them
        return [1] * len(self.lambdas)

    def alphas(self) -> List[float]:
        return list(self.output_weights) if self.output_weights else list(self.lambdas)


@dataclass
class Certificate:
    epsilon_hat: float = 0.0
    c: float = 0.0
    bound: float = 0.0


@dataclass
class RecoveryResult:
    x: Optional[np.ndarray]
    e: Optional[np.ndarray]
    z: Optional[List[np.ndarray]]
    iters: int
    converged: bool
    residual_history: List[float]
    final_residuals: List[float]
    objective: float
    certificate: Optional[Certificate]
    y: Optional[List[np.ndarray]] = None
    y_hat: Optional[List[np.ndarray]] = None


@dataclass
class IterationView:
    """Per-iteration snapshot (recovery.hpp:38-48); arrays are copies."""

    iter: int
    mu_used: float
    mu_next: float
    residual_inf: List[float]
    e: np.ndarray
    z: List[np.ndarray]
    y: List[np.ndarray]
    u: List[np.ndarray]
    v: List[np.ndarray]


IterationObserver = Callable[[IterationView], None]


@dataclass
class PasdState:
    """Solver iterate (tenrec::PasdState, pasd.hpp:33-41): u[n] (I_n x R_n),
    v[n] (R_n x J_n, unfolding column order), e, y[n], y_hat[n], mu, iter."""

    u: List[np.ndarray]
    v: List[np.ndarray]
    e: np.ndarray
    y: List[np.ndarray]
    y_hat: List[np.ndarray] = field(default_factory=list)
    mu: float = 0.0
    iter: int = 0


def as_tensor(t) -> np.ndarray:
    """Fortran-ordered contiguous float64 copy/view of t (first index fastest)."""
    a = np.asarray(t, dtype=np.float64)
    if a.ndim == 0:
        raise ArgumentError("tensor order must be at least 1")
    return np.asfortranarray(a)


def build_options(dims: Sequence[int], config: PasdConfig, device: int = 0, flags: int = 0,
                  poll_every: int = 0):
    """PasdOptions plus the numpy arrays that keep its pointers alive."""
    n = len(dims)

    def padded(vals, dtype):
        v = list(vals)[:n] + [0] * max(0, n - len(vals))
        return np.ascontiguousarray(np.asarray(v, dtype=dtype))

    d = np.ascontiguousarray(np.asarray(dims, dtype=np.int64))
    r = padded(config.ranks, np.int64)
    lam = padded(config.lambdas, np.float64)
    w = padded(config.output_weights, np.float64) if config.output_weights else None
    opt = _abi.PasdOptions()
    opt.order = n
    opt.dims = d.ctypes.data_as(_abi.c_int64_p)
    opt.ranks = r.ctypes.data_as(_abi.c_int64_p)
    opt.lambdas = lam.ctypes.data_as(_abi.c_double_p)
    opt.output_weights = _abi.dptr(w)
    opt.mu0 = config.mu0
    opt.mu_max = config.mu_max
    opt.rho = config.rho
    opt.eps = config.eps
    opt.maxiter = int(config.maxiter)
    opt.device = int(device)
    opt.flags = int(flags)
    opt.poll_every = int(poll_every)
    keep = (d, r, lam, w)
    # Length checks the C side cannot see (it trusts order): mirror the
    # reference's count messages (pasd.cpp:15-17, 21-23, 42-43).
    return opt, keep


def count_checks(dims: Sequence[int], config: PasdConfig) -> None:
    n = len(dims)
    if len(config.lambdas) != n:
        raise ArgumentError(f"config: expected {n} lambdas, got {len(config.lambdas)}")
    if isinstance(config, SnnConfig):  # SnnConfig::validate (baselines.cpp:12-29)
        if config.output_weights and len(config.output_weights) != n:
            raise ArgumentError(f"config: expected {n} output weights")
        return
    if len(config.ranks) != n:
        raise ArgumentError(f"config: expected {n} ranks, got {len(config.ranks)}")
    if config.output_weights and len(config.output_weights) != n:
        raise ArgumentError(f"config: expected {n} output weights")


def make_observer(dims: Sequence[int], ranks: Sequence[int], user_fn: Optional[IterationObserver]):
    """Wrap a Python observer as a pasd_observer_fn (copies the host view)."""
    if user_fn is None:
        return _abi.PasdObserverFn()
    snn_view = ranks is None  # SNN views carry no u / v (baselines.cpp:124-125)
    if isinstance(user_fn, _abi.PasdObserverFn):  # raw C callback, passed through
        return user_fn
    dims = [int(x) for x in dims]
    total = int(np.prod(dims))
    n = len(dims)

    def cb(view_p, _user):
        v = view_p.contents

        def arr(p, count, shape=None):
            a = np.ctypeslib.as_array(p, shape=(count,)).copy()
            return a.reshape(shape, order="F") if shape is not None else a

        view = IterationView(
            iter=int(v.iter), mu_used=float(v.mu_used), mu_next=float(v.mu_next),
            residual_inf=[float(v.residual_inf[i]) for i in range(n)],
            e=arr(v.e, total, dims),
            z=[arr(v.z[i], total, dims) for i in range(n)],
            y=[arr(v.y[i], total, dims) for i in range(n)],
            u=[] if snn_view else [arr(v.u[i], dims[i] * ranks[i], (dims[i], ranks[i])) for i in range(n)],
            v=[] if snn_view else [arr(v.v[i], ranks[i] * (total // dims[i]), (ranks[i], total // dims[i]))
                                   for i in range(n)],
        )
        user_fn(view)

    return _abi.PasdObserverFn(cb)


def run_recover(fn, t, config: PasdConfig, observer=None, *, flags=0, want_z=True, want_y=True,
                device=0, poll_every=0, extra_args=()):
    """Shared driver for any library exporting the pasd_b200_recover signature."""
    t = as_tensor(t)
    dims = list(t.shape)
    count_checks(dims, config)
    total = int(t.size)
    n = len(dims)
    opt, keep = build_options(dims, config, device=device, flags=flags, poll_every=poll_every)
    flat_t = np.ravel(t, order="F")
    x = np.empty(total)
    e = np.empty(total)
    z = [np.empty(total) for _ in range(n)] if want_z else None
    y = [np.empty(total) for _ in range(n)] if want_y else None
    yh = [np.empty(total) for _ in range(n)] if want_y and not isinstance(config, SnnConfig) else None
    hist = np.zeros(max(1, int(config.maxiter)))
    fres = np.zeros(n)
    out = _abi.PasdOutputs()
    out.x = _abi.dptr(x)
    out.e = _abi.dptr(e)
    zp, yp, yhp = _abi.ptr_array(z), _abi.ptr_array(y), _abi.ptr_array(yh)
    out.z, out.y, out.y_hat = zp, yp, yhp
    out.residual_history = _abi.dptr(hist)
    out.final_residuals = _abi.dptr(fres)
    obs = make_observer(dims, None if isinstance(config, SnnConfig) else config.ranks, observer)
    err = C.create_string_buffer(1024)
    rc = fn(flat_t.ctypes.data_as(_abi.c_double_p), C.byref(opt), C.byref(out), obs, None, *extra_args,
            err, C.c_size_t(len(err)))
    raise_for_status(rc, err)
    shape = tuple(dims)

    def rs(a):
        return a.reshape(shape, order="F")

    cert = None
    if out.has_certificate:
        cert = Certificate(out.cert_epsilon_hat, out.cert_c, out.cert_bound)
    return RecoveryResult(
        x=rs(x), e=rs(e), z=[rs(a) for a in z] if z is not None else None,
        iters=int(out.iters), converged=bool(out.converged),
        residual_history=[float(h) for h in hist[: out.iters]],
        final_residuals=[float(r) for r in fres], objective=float(out.objective), certificate=cert,
        y=[rs(a) for a in y] if y is not None else None,
        y_hat=[rs(a) for a in yh] if yh is not None else None,
    )
