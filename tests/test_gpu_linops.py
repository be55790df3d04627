"""Device SVT / Procrustes (the solver's own small-solve kernels) against the
oracle's LAPACK-based linops (linops.cpp:78-104)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_svt_matches_oracle(gpu, oracle_mod):
    from paper_1712_09999_b200.solver import svt

    rng = np.random.default_rng(0)
    for (r, c, tau) in [(3, 8, 0.5), (10, 200, 5.0), (20, 1000, 10.0), (50, 3000, 30.0), (64, 700, 20.0), (7, 7, 1.0)]:
        m = rng.standard_normal((r, c))
        vo = oracle_mod.svt(m, tau)
        vg, kept = svt(m, tau)
        assert kept == int((np.linalg.svd(m, compute_uv=False) > tau).sum())
        assert np.linalg.norm(vg - vo) <= 1e-12 * max(1.0, np.linalg.norm(vo))
    m = rng.standard_normal((4, 9))
    np.testing.assert_array_equal(svt(m, 0.0)[0], m)
    np.testing.assert_allclose(svt(np.diag([3.0, 1.0]), 2.0)[0], np.diag([1.0, 0.0]), atol=1e-15)


@pytest.mark.parametrize("r,c", [(8, 2000), (12, 5000), (50, 3000)])
def test_svt_ill_conditioned_tiny_threshold(gpu, oracle_mod, r, c):
    """The late-iteration regime (tau = lambda/mu with mu -> mu_max): singular
    values spread over 1 .. 1e-10 sigma_1 and tau = 1e-9 sigma_1.  eig(A A^T)
    alone cannot resolve sigma_i < ~1e-8 sigma_1 (absolute error eps sigma_1^2
    in sigma^2); the device SVT refines them from A (svt_refine_small) and must
    keep exactly the oracle's set sigma > tau (linops.cpp:84-86) and match its
    result far below the smallest kept contribution sigma - tau."""
    from paper_1712_09999_b200.solver import svt

    rng = np.random.default_rng(r)
    qu, _ = np.linalg.qr(rng.standard_normal((r, r)))
    qv, _ = np.linalg.qr(rng.standard_normal((c, r)))
    sig = np.logspace(0, -10, r)  # 1 ... 1e-10
    sig[-2] = 5e-9  # just above tau, the hardest kept value
    m = (qu * sig) @ qv.T
    tau = 1e-9
    vo = oracle_mod.svt(m, tau)
    vg, kept = svt(m, tau)
    assert kept == int((sig > tau).sum())
    # rounding level of an R x J product (the kept sigma - tau >= 4e-9 is far above it)
    assert np.linalg.norm(vg - vo) <= 5e-12 * np.linalg.norm(vo), np.linalg.norm(vg - vo) / np.linalg.norm(vo)


def test_procrustes_full_rank_matches_oracle(gpu, oracle_mod):
    from paper_1712_09999_b200.solver import procrustes

    rng = np.random.default_rng(1)
    for (I, P, R) in [(20, 50, 3), (100, 400, 10), (1000, 300, 50), (64, 64, 64), (9, 5, 1)]:
        g = rng.standard_normal((I, P))
        v = rng.standard_normal((R, P))
        uo = oracle_mod.procrustes(g, v)
        ug, rank = procrustes(g, v)
        assert rank == R
        assert np.linalg.norm(ug - uo) <= 1e-11 * np.sqrt(R)


def test_procrustes_rank_deficient_is_a_valid_polar_factor(gpu, oracle_mod):
    """Rank-deficient g v^T: the polar factor is non-unique (the reference's
    completion is dgesdd rounding noise).  Ours must be orthonormal, optimal
    (same ||U v - g||), agree on range(g v^T), and complete deterministically."""
    from paper_1712_09999_b200.solver import procrustes

    rng = np.random.default_rng(2)
    for (I, P, R, k) in [(20, 50, 3, 1), (100, 400, 10, 4), (1000, 300, 50, 17)]:
        g = rng.standard_normal((I, P))
        q, _ = np.linalg.qr(rng.standard_normal((R, R)))
        d = np.zeros(R)
        d[:k] = rng.uniform(0.5, 2, k)
        v = q @ np.diag(d) @ q.T @ rng.standard_normal((R, P))
        uo = oracle_mod.procrustes(g, v)
        ug, rank = procrustes(g, v)
        assert rank == k
        assert np.abs(ug.T @ ug - np.eye(R)).max() <= 1e-12
        assert abs(np.linalg.norm(ug @ v - g) - np.linalg.norm(uo @ v - g)) <= 1e-10 * np.linalg.norm(g)
        w = g @ v.T
        np.testing.assert_allclose(ug @ (ug.T @ w), w, atol=1e-10 * np.linalg.norm(w))
        ug2, _ = procrustes(g, v)
        np.testing.assert_array_equal(ug, ug2)  # deterministic


def test_procrustes_degenerate(gpu):
    from paper_1712_09999_b200.solver import procrustes

    u, rank = procrustes(np.random.default_rng(3).standard_normal((8, 5)), np.zeros((2, 5)))
    assert u is None and rank == 0
