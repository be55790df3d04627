"""B200-native PASD (arXiv 1712.09999) ADMM hot path.

Public API mirrors ``proj/include/tenrec`` of the reference:
``PasdConfig``, ``pasd_recover``, ``RecoveryResult``, ``Certificate``,
``IterationView`` and the error taxonomy.  Compute runs in
``libpasd_b200.so`` (sm_100a CUDA, C-ABI in include/pasd_b200.h).
"""
from .api import (ArgumentError, Certificate, DeviceError, IoError, IterationView, NumericalError, PasdConfig,
                  PasdState, SnnConfig, RecoveryResult, StateError, TenrecError)
from .solver import (Solver, default_lambdas, default_rank_bound, lib, pasd_g_matrix, pasd_recover, release_cache,
                     snn_recover, suboptimality_certificate, update_e, update_u, update_v, validate_config)

__all__ = [
    "ArgumentError", "Certificate", "DeviceError", "IoError", "IterationView", "NumericalError", "PasdConfig",
    "RecoveryResult", "StateError", "TenrecError", "Solver", "default_lambdas", "default_rank_bound", "lib",
    "pasd_recover", "release_cache", "validate_config", "PasdState", "pasd_g_matrix", "update_u", "update_v",
    "update_e", "suboptimality_certificate", "SnnConfig", "snn_recover",
]
