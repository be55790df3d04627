"""ctypes mirror of ``include/pasd_b200.h`` (the C-ABI structs and entry points).

Shared by the product wrapper (``paper_1712_09999_b200.solver``) and by the
test-only oracle wrapper (``oracle/__init__.py``), which binds the same struct
layout to the CPU restatement.
"""
from __future__ import annotations

import ctypes as C

PASD_OK = 0
PASD_ERR_ARGUMENT = 1
PASD_ERR_IO = 2
PASD_ERR_NUMERICAL = 3
PASD_ERR_STATE = 4
PASD_ERR_CUDA = 5

PASD_FLAG_NONE = 0
PASD_FLAG_NO_CERTIFICATE = 1 << 0
PASD_FLAG_FIXED_ITERS = 1 << 1
PASD_FLAG_REUSE_SOLVER = 1 << 2
PASD_FLAG_CHECK_REPLICAS = 1 << 3
PASD_FLAG_FP32 = 1 << 4

PASD_KERNEL_CLASSES = ("polar", "contract_A", "gram", "svt", "update", "finish", "contract_W")

c_double_p = C.POINTER(C.c_double)
c_int64_p = C.POINTER(C.c_int64)


class PasdOptions(C.Structure):
    _fields_ = [
        ("order", C.c_int32),
        ("dims", c_int64_p),
        ("ranks", c_int64_p),
        ("lambdas", c_double_p),
        ("output_weights", c_double_p),
        ("mu0", C.c_double),
        ("mu_max", C.c_double),
        ("rho", C.c_double),
        ("eps", C.c_double),
        ("maxiter", C.c_int32),
        ("device", C.c_int32),
        ("flags", C.c_uint32),
        ("poll_every", C.c_int32),
    ]


class PasdShard(C.Structure):
    _fields_ = [
        ("rank", C.c_int32),
        ("nranks", C.c_int32),
        ("nccl_unique_id", C.c_void_p),
        ("slab_begin", C.c_int64),
        ("slab_end", C.c_int64),
        ("loopback", C.c_void_p),
    ]


class PasdIterationView(C.Structure):
    _fields_ = [
        ("iter", C.c_int32),
        ("mu_used", C.c_double),
        ("mu_next", C.c_double),
        ("residual_inf", c_double_p),
        ("e", c_double_p),
        ("z", C.POINTER(c_double_p)),
        ("y", C.POINTER(c_double_p)),
        ("u", C.POINTER(c_double_p)),
        ("v", C.POINTER(c_double_p)),
    ]


PasdObserverFn = C.CFUNCTYPE(None, C.POINTER(PasdIterationView), C.c_void_p)


class PasdOutputs(C.Structure):
    _fields_ = [
        ("x", c_double_p),
        ("e", c_double_p),
        ("z", C.POINTER(c_double_p)),
        ("y", C.POINTER(c_double_p)),
        ("y_hat", C.POINTER(c_double_p)),
        ("residual_history", c_double_p),
        ("final_residuals", c_double_p),
        ("iters", C.c_int32),
        ("converged", C.c_int32),
        ("objective", C.c_double),
        ("has_certificate", C.c_int32),
        ("cert_epsilon_hat", C.c_double),
        ("cert_c", C.c_double),
        ("cert_bound", C.c_double),
    ]


# Every symbol include/pasd_b200.h declares (checked by tests/test_abi.py).
HEADER_SYMBOLS = (
    "pasd_b200_recover",
    "pasd_b200_release_cache",
    "pasd_b200_solver_create",
    "pasd_b200_solver_load",
    "pasd_b200_solver_reset",
    "pasd_b200_solver_set_state",
    "pasd_b200_solver_run",
    "pasd_b200_solver_finalize",
    "pasd_b200_solver_device_e",
    "pasd_b200_solver_stream",
    "pasd_b200_solver_launches",
    "pasd_b200_solver_ranks",
    "pasd_b200_solver_profile",
    "pasd_b200_solver_destroy",
    "pasd_b200_default_lambdas",
    "pasd_b200_default_rank_bound",
    "pasd_b200_validate",
    "pasd_b200_svt",
    "pasd_b200_procrustes",
    "pasd_b200_g_matrix",
    "pasd_b200_update_u",
    "pasd_b200_update_v",
    "pasd_b200_update_e",
    "pasd_b200_certificate",
    "pasd_b200_nuclear_norm_unfold",
    "pasd_b200_synth",
    "pasd_b200_synth_factor",
    "pasd_b200_synth_support",
    "pasd_b200_nccl_unique_id",
    "pasd_b200_loopback_create",
    "pasd_b200_snn_recover",
    "pasd_b200_guard_report",
    "pasd_b200_loopback_destroy",
    "pasd_b200_abi_version",
    "pasd_b200_build_info",
)


def dptr(arr) -> "c_double_p":
    """Pointer to a contiguous float64 numpy buffer (or NULL for None)."""
    if arr is None:
        return c_double_p()
    return arr.ctypes.data_as(c_double_p)


def ptr_array(arrs):
    """double*[N] from a list of numpy buffers (or NULL for None)."""
    if arrs is None:
        return C.POINTER(c_double_p)()
    return (c_double_p * len(arrs))(*[dptr(a) for a in arrs])
