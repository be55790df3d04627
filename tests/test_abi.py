"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/pasd_b200.h declares, and its host-side logic (validation,
defaults) mirrors the reference.  The product path must fail loudly (no CPU
fallback) when no CUDA device is present."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_1712_09999_b200 as pb
from paper_1712_09999_b200 import _abi
from paper_1712_09999_b200.api import ArgumentError, DeviceError, PasdConfig

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "pasd_b200.h")).read()
    return sorted(set(re.findall(r"\b(pasd_b200_[a-z_]+)\s*\(", src)))


def test_header_symbols_exported():
    lib = pb.lib()
    names = header_functions()
    assert set(names) == set(_abi.HEADER_SYMBOLS)
    for name in names:
        assert hasattr(lib, name), name  # dlsym succeeds
    assert lib.pasd_b200_abi_version() == 2


def test_header_compiles_as_c():
    import subprocess
    import tempfile

    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "t.c")
        with open(src, "w") as f:
            f.write('#include "pasd_b200.h"\nint main(void){pasd_options o; (void)o; return PASD_OK;}\n')
        subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), "-c", src,
                        "-o", os.path.join(d, "t.o")], check=True)


def test_defaults_match_reference_formulas():
    assert pb.default_lambdas([100, 100, 100]) == [100 / 3] * 3
    assert pb.default_lambdas([256, 256, 1024]) == pytest.approx([512 / 3, 512 / 3, 256 / 3])
    assert pb.default_rank_bound(10) == 12
    assert pb.default_rank_bound(4) == 4
    with pytest.raises(ArgumentError, match="target rank must be positive"):
        pb.default_rank_bound(0)
    assert PasdConfig.default_lambdas([20, 30]) == pb.default_lambdas([20, 30])


def test_validate_matches_oracle_messages(oracle_mod):
    dims = (4, 3, 2)
    lam = [1.0, 1.0, 1.0]
    bad = [
        PasdConfig(lambdas=lam, ranks=[2, 2, 3]),
        PasdConfig(lambdas=[1.0, float("nan"), 1.0], ranks=[1, 1, 1]),
        PasdConfig(lambdas=lam, ranks=[1, 0, 1]),
        PasdConfig(lambdas=lam, ranks=[1, 1, 1], mu0=-1.0),
        PasdConfig(lambdas=lam, ranks=[1, 1, 1], mu_max=1e-6),
        PasdConfig(lambdas=lam, ranks=[1, 1, 1], rho=0.5),
        PasdConfig(lambdas=lam, ranks=[1, 1, 1], eps=-1.0),
        PasdConfig(lambdas=lam, ranks=[1, 1, 1], maxiter=-3),
        PasdConfig(lambdas=lam, ranks=[1, 1, 1], output_weights=[1.0, 1.0, -2.0]),
        PasdConfig(lambdas=lam, ranks=[1, 1]),
    ]
    for cfg in bad:
        with pytest.raises(ArgumentError) as ours:
            cfg.validate(dims)
        with pytest.raises(ArgumentError) as ref:
            oracle_mod.pasd_recover(np.zeros(dims), cfg)
        assert str(ours.value) == str(ref.value)
    PasdConfig(lambdas=lam, ranks=[1, 1, 1]).validate(dims)  # valid config passes


def test_kernel_limits_are_argument_errors():
    with pytest.raises(ArgumentError, match="exceeds the supported maximum 64"):
        PasdConfig(lambdas=[1.0, 1.0], ranks=[65, 1]).validate([100, 100])


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present; the no-device failure mode is exercised on CPU hosts")
    cfg = PasdConfig(lambdas=[1.0, 1.0, 1.0], ranks=[1, 1, 1])
    with pytest.raises(DeviceError, match="cuda"):
        pb.pasd_recover(np.ones((3, 3, 3)), cfg)


def test_snn_validate_matches_oracle_messages(oracle_mod):
    """pasd_b200_snn_recover validates like SnnConfig::validate (baselines.cpp:12-29)
    before touching the device: same messages as the oracle's snn_recover."""
    from paper_1712_09999_b200.api import SnnConfig

    dims = (4, 3, 2)
    lam = [1.0, 1.0, 1.0]
    bad = [
        SnnConfig(lambdas=[1.0, 0.0, 1.0]),
        SnnConfig(lambdas=lam, mu0=-1.0),
        SnnConfig(lambdas=lam, mu_max=1e-6),
        SnnConfig(lambdas=lam, rho=1.0),
        SnnConfig(lambdas=lam, eps=0.0),
        SnnConfig(lambdas=lam, maxiter=0),
        SnnConfig(lambdas=lam, output_weights=[1.0, 0.0, 1.0]),
        SnnConfig(lambdas=[1.0, 1.0]),
    ]
    for cfg in bad:
        with pytest.raises(ArgumentError) as ours:
            pb.snn_recover(np.zeros(dims), cfg)
        with pytest.raises(ArgumentError) as ref:
            oracle_mod.snn_recover(np.zeros(dims), cfg)
        assert str(ours.value) == str(ref.value)
    t = np.zeros(dims)
    t[1, 1, 1] = np.inf
    for f in (pb.snn_recover, oracle_mod.snn_recover):
        with pytest.raises(ArgumentError, match="snn: input tensor contains non-finite entries"):
            f(t, SnnConfig(lambdas=lam))
    with pytest.raises(ArgumentError, match="snn supports unfoldings"):
        pb.snn_recover(np.zeros((120, 120, 2)), SnnConfig(lambdas=lam))


def test_oracle_snn_recovers_desk_case(oracle_mod):
    """SPEC.md desk case (30^3, r = 3, 5% corruption): the restated SNN baseline
    recovers L0 (RSE <= 1e-4) and leaves y_hat / the certificate empty."""
    from paper_1712_09999_b200.api import SnnConfig

    dims = (30, 30, 30)
    L0 = oracle_mod.gen_tucker(dims, [3, 3, 3], seed=0)
    T = oracle_mod.corrupt_sparse(L0, 0.05, seed=0)
    r = oracle_mod.snn_recover(T, SnnConfig(lambdas=oracle_mod.default_lambdas(dims)))
    assert r.converged and r.certificate is None and r.y_hat is None
    assert np.linalg.norm(r.x - L0) / np.linalg.norm(L0) <= 1e-4
