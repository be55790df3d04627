"""GPU SNN baseline (pasd_b200_snn_recover, pasd_snn.cuh) against the oracle's
restatement of tenrec::snn_recover (baselines.cpp:37-143) on the same seeded
inputs.  The full SVT of every unfolding runs as Gram + Jacobi on the device
and as dgesdd in the oracle, so iterates agree to rounding, not bitwise; the
elementwise E / Y arithmetic is the reference's operation order."""
import numpy as np
import pytest

from paper_1712_09999_b200.api import SnnConfig

pytestmark = pytest.mark.gpu


def rel(a, b):
    n = np.linalg.norm(b)
    return np.linalg.norm(a - b) / n if n > 0 else np.linalg.norm(a - b)


def instance(oracle_mod, dims, r, rho, seed=0):
    L0 = oracle_mod.gen_tucker(dims, [r] * len(dims), seed=seed)
    return L0, oracle_mod.corrupt_sparse(L0, rho, seed=seed)


@pytest.mark.parametrize("dims,r,rho", [((30, 30, 30), 3, 0.05), ((20, 24, 18), 2, 0.1), ((12, 12, 12, 12), 2, 0.05)])
def test_snn_fixed_iterations_match_oracle(gpu, oracle_mod, dims, r, rho):
    L0, T = instance(oracle_mod, dims, r, rho)
    cfg = SnnConfig(lambdas=oracle_mod.default_lambdas(dims), maxiter=40)
    rg = gpu.snn_recover(T, cfg, fixed_iters=True)
    ro = oracle_mod.snn_recover(T, cfg, fixed_iters=True)
    assert rg.iters == ro.iters == 40
    assert rel(rg.x, ro.x) <= 1e-9, rel(rg.x, ro.x)
    assert rel(rg.e, ro.e) <= 1e-9, rel(rg.e, ro.e)
    for zg, zo in zip(rg.z, ro.z):
        assert rel(zg, zo) <= 1e-9
    np.testing.assert_allclose(rg.residual_history, ro.residual_history, rtol=1e-7)
    assert rg.y_hat is None and rg.certificate is None


@pytest.mark.parametrize("dims,r,rho", [((30, 30, 30), 3, 0.05), ((40, 36, 44), 4, 0.1)])
def test_snn_convergence_matches_oracle(gpu, oracle_mod, dims, r, rho):
    L0, T = instance(oracle_mod, dims, r, rho, seed=1)
    cfg = SnnConfig(lambdas=oracle_mod.default_lambdas(dims), eps=1e-7)
    rg = gpu.snn_recover(T, cfg)
    ro = oracle_mod.snn_recover(T, cfg)
    assert rg.converged and ro.converged
    assert abs(rg.iters - ro.iters) <= 1, (rg.iters, ro.iters)
    assert rel(rg.x, ro.x) <= 1e-8, rel(rg.x, ro.x)
    assert rel(rg.e, ro.e) <= 1e-8, rel(rg.e, ro.e)
    assert np.array_equal(rg.e != 0, ro.e != 0)
    assert abs(rg.objective - ro.objective) <= 1e-8 * abs(ro.objective)
    assert rel(rg.x, L0) <= 1e-4


def test_snn_c1_scale(gpu, oracle_mod):
    """BASELINE configs[0] shape (100^3, Tucker rank 10, 10% corruption): the
    paper's PASD-vs-SNN comparison instance, 30 fixed iterations."""
    L0, T = instance(oracle_mod, (100, 100, 100), 10, 0.10)
    cfg = SnnConfig(lambdas=oracle_mod.default_lambdas(T.shape), maxiter=30)
    rg = gpu.snn_recover(T, cfg, fixed_iters=True, want_z=False, want_y=False)
    ro = oracle_mod.snn_recover(T, cfg, fixed_iters=True, threads=16, want_z=False, want_y=False)
    assert rel(rg.x, ro.x) <= 1e-9, rel(rg.x, ro.x)
    assert rel(rg.e, ro.e) <= 1e-9, rel(rg.e, ro.e)


def test_snn_observer_sequence(gpu, oracle_mod):
    L0, T = instance(oracle_mod, (16, 14, 12), 2, 0.05)
    cfg = SnnConfig(lambdas=oracle_mod.default_lambdas(T.shape), maxiter=5)
    seen = []
    gpu.snn_recover(T, cfg, observer=lambda v: seen.append((v.iter, v.mu_used, v.mu_next, len(v.z), v.u)),
                    fixed_iters=True)
    assert [s[0] for s in seen] == [1, 2, 3, 4, 5]
    assert seen[0][1] == cfg.mu0 and seen[0][2] == pytest.approx(cfg.mu0 * cfg.rho)
    assert all(s[3] == 3 and s[4] == [] for s in seen)
