"""Pin the CPU restatement (oracle/) against the reference's own known-answer
examples and invariants (SPEC.md; the reference ships no test suite,
proj/tests/CMakeLists.txt:1).  CPU only."""
import itertools
import math

import numpy as np
import pytest

from paper_1712_09999_b200.api import ArgumentError, PasdConfig


def brute_unfold(t, mode):
    """Index map of SPEC.md:47-49 / tensor.cpp:106-107 by brute force."""
    dims = t.shape
    n = mode - 1
    cols = t.size // dims[n]
    out = np.zeros((dims[n], cols))
    for idx in itertools.product(*[range(d) for d in dims]):
        col, stride = 0, 1
        for m in range(len(dims)):
            if m == n:
                continue
            col += idx[m] * stride
            stride *= dims[m]
        out[idx[n], col] = t[idx]
    return out


def test_unfold_spec_example(oracle_mod):
    # t[i,j,k] = (i-1) + 2(j-1) + 4(k-1); mode-1 row i = [i-1, i+1, i+3, i+5]
    t = np.zeros((2, 2, 2), order="F")
    for i, j, k in itertools.product(range(2), repeat=3):
        t[i, j, k] = i + 2 * j + 4 * k
    m = oracle_mod.unfold(t, 1)
    assert m.shape == (2, 4)
    for i in range(2):
        assert list(m[i]) == [i, i + 2, i + 4, i + 6]
    np.testing.assert_array_equal(oracle_mod.fold(m, 1, (2, 2, 2)), t)


def test_unfold_degenerate_dims(oracle_mod):
    t = np.arange(3.0).reshape((3, 1, 1), order="F")
    m = oracle_mod.unfold(t, 1)
    assert m.shape == (3, 1)
    np.testing.assert_array_equal(m[:, 0], [0.0, 1.0, 2.0])


def test_fold_unfold_roundtrip_random_shapes(oracle_mod):
    # acceptance criterion 5: bitwise round trips on 50 random shapes up to order 4
    rng = np.random.default_rng(7)
    for _ in range(50):
        order = int(rng.integers(1, 5))
        dims = tuple(int(d) for d in rng.integers(1, 6, size=order))
        t = np.asfortranarray(rng.standard_normal(dims))
        for mode in range(1, order + 1):
            m = oracle_mod.unfold(t, mode)
            if t.size <= 200:
                np.testing.assert_array_equal(m, brute_unfold(t, mode))
            np.testing.assert_array_equal(oracle_mod.fold(m, mode, dims), t)


def test_unfold_mode_out_of_range(oracle_mod):
    with pytest.raises(ArgumentError, match="mode 4 out of range 1..3"):
        oracle_mod.unfold(np.zeros((2, 2, 2)), 4)


def test_thin_svd_examples(oracle_mod):
    u, s, v = oracle_mod.thin_svd(np.eye(3))
    np.testing.assert_allclose(s, [1, 1, 1], atol=1e-15)
    u, s, v = oracle_mod.thin_svd(np.diag([3.0, 1.0]))
    np.testing.assert_allclose(s, [3, 1], atol=1e-15)
    rng = np.random.default_rng(1)
    m = rng.standard_normal((4, 6))
    u, s, v = oracle_mod.thin_svd(m)
    np.testing.assert_allclose(u @ np.diag(s) @ v.T, m, atol=1e-10 * np.linalg.norm(m))
    lam = np.sort(np.linalg.eigvalsh(m @ m.T))[::-1]  # SPEC.md:131 Gram eigen-oracle
    np.testing.assert_allclose(s, np.sqrt(lam), rtol=1e-10)
    for j in range(u.shape[1]):  # sign convention (linops.cpp:25-41)
        piv = int(np.argmax(np.abs(u[:, j])))
        assert u[piv, j] >= 0


def test_svt_examples(oracle_mod):
    np.testing.assert_allclose(oracle_mod.svt(np.diag([3.0, 1.0]), 2.0), np.diag([1.0, 0.0]), atol=1e-15)
    rng = np.random.default_rng(2)
    m = rng.standard_normal((5, 7))
    np.testing.assert_array_equal(oracle_mod.svt(m, 0.0), m)  # tau == 0 returns input
    s1 = np.linalg.svd(m, compute_uv=False)[0]
    np.testing.assert_array_equal(oracle_mod.svt(m, s1 * 1.0001), np.zeros_like(m))
    with pytest.raises(ArgumentError, match="svt: threshold must be a nonnegative finite number"):
        oracle_mod.svt(m, -1.0)
    # acceptance criterion 5: explicit definition on random 5x5..20x20
    for _ in range(20):
        r, c = rng.integers(5, 21, size=2)
        m = rng.standard_normal((r, c))
        tau = float(rng.uniform(0.1, 2.0))
        u, s, vt = np.linalg.svd(m, full_matrices=False)
        ref = u @ np.diag(np.maximum(s - tau, 0)) @ vt
        np.testing.assert_allclose(oracle_mod.svt(m, tau), ref, atol=1e-10 * max(1, np.linalg.norm(m)))


def test_shrink_examples(oracle_mod):
    assert oracle_mod.soft_threshold(1.2, 0.5) == pytest.approx(0.7, abs=1e-15)
    assert oracle_mod.soft_threshold(-0.3, 0.5) == 0.0
    assert oracle_mod.soft_threshold(-1.5, 0.5) == -1.0
    assert oracle_mod.soft_threshold(0.5, 0.5) == 0.0  # strict comparison


def test_procrustes_examples(oracle_mod):
    rng = np.random.default_rng(3)
    q, _ = np.linalg.qr(rng.standard_normal((6, 3)))
    np.testing.assert_allclose(oracle_mod.procrustes(q, np.eye(3)), q, atol=1e-12)
    g = np.array([[0.0, 1.0], [1.0, 0.0]])
    np.testing.assert_allclose(oracle_mod.procrustes(g, np.eye(2)), g, atol=1e-14)
    assert oracle_mod.procrustes(rng.standard_normal((6, 10)), np.zeros((3, 10))) is None  # degenerate
    # optimality vs random orthonormal candidates (acceptance criterion 5)
    for _ in range(5):
        g = rng.standard_normal((6, 10))
        v = rng.standard_normal((3, 10))
        u = oracle_mod.procrustes(g, v)
        best = np.linalg.norm(u @ v - g)
        for _ in range(200):
            c, _ = np.linalg.qr(rng.standard_normal((6, 3)))
            assert np.linalg.norm(c @ v - g) >= best - 1e-12
    with pytest.raises(ArgumentError, match="same number of columns"):
        oracle_mod.procrustes(np.zeros((4, 3)), np.zeros((2, 5)))


def test_default_lambdas_and_rank_bound(oracle_mod, ):
    lam = oracle_mod.default_lambdas([100, 100, 100])
    assert lam == [math.sqrt(10000) / 3] * 3
    lam4 = oracle_mod.default_lambdas([256, 256, 1024])
    assert lam4 == pytest.approx([512 / 3, 512 / 3, 256 / 3])


def small_instance(oracle_mod, dims=(12, 10, 8), r=2, rho=0.05, seed=0):
    L0 = oracle_mod.gen_tucker(dims, [r] * len(dims), seed=seed)
    T = oracle_mod.corrupt_sparse(L0, rho, seed=seed)
    return L0, T


def test_zero_tensor_converges_in_one_iteration(oracle_mod):
    # T == 0 -> X == 0, E == 0, converged at iteration 1, eps_hat == 0
    T = np.zeros((5, 4, 3))
    cfg = PasdConfig(lambdas=oracle_mod.default_lambdas(T.shape), ranks=[2, 2, 2])
    r = oracle_mod.pasd_recover(T, cfg)
    assert r.converged and r.iters == 1
    assert not r.x.any() and not r.e.any()
    assert r.certificate is not None and r.certificate.epsilon_hat == 0.0


def test_pasd_invariants(oracle_mod):
    """SPEC.md:255-259 invariant suite on a converged desk run."""
    L0, T = small_instance(oracle_mod, dims=(16, 14, 12), r=2, rho=0.05)
    cfg = PasdConfig(lambdas=oracle_mod.default_lambdas(T.shape), ranks=[2, 2, 2], eps=1e-6)
    lam_sum = sum(cfg.lambdas)
    seen = []

    def obs(v):
        ysum = sum(v.y)
        assert np.abs(ysum).max() <= 1 + 1e-8  # Appendix A boundedness
        assert v.mu_next == min(cfg.rho * v.mu_used, cfg.mu_max)  # exact mu schedule
        for u in v.u:
            if np.count_nonzero(u - np.eye(*u.shape)):
                assert np.abs(u.T @ u - np.eye(u.shape[1])).max() <= 1e-8
        seen.append(v.iter)

    r = oracle_mod.pasd_recover(T, cfg, observer=obs)
    assert seen == list(range(1, r.iters + 1))
    assert r.converged
    assert all(x < cfg.eps for x in r.final_residuals)
    assert r.certificate.epsilon_hat <= 1 + lam_sum  # Eq. (19) bound
    assert np.isfinite(r.certificate.c) and r.certificate.c >= 0 and r.certificate.bound >= 0


def test_validate_messages(oracle_mod):
    T = np.zeros((4, 3, 2))
    lam = [1.0, 1.0, 1.0]
    cases = [
        (PasdConfig(lambdas=lam, ranks=[2, 2, 3]), "config: rank 3 exceeds dimension 2 in mode 3"),
        (PasdConfig(lambdas=[1.0, -1.0, 1.0], ranks=[1, 1, 1]), "config: lambda of mode 2 must be positive"),
        (PasdConfig(lambdas=lam, ranks=[1, 0, 1]), "config: rank of mode 2 must be positive"),
        (PasdConfig(lambdas=lam, ranks=[1, 1, 1], mu0=0.0), "config: mu0 must be positive"),
        (PasdConfig(lambdas=lam, ranks=[1, 1, 1], mu_max=1e-5), "config: mu_max must be at least mu0"),
        (PasdConfig(lambdas=lam, ranks=[1, 1, 1], rho=1.0), "config: rho must exceed 1"),
        (PasdConfig(lambdas=lam, ranks=[1, 1, 1], eps=0.0), "config: eps must be positive"),
        (PasdConfig(lambdas=lam, ranks=[1, 1, 1], maxiter=0), "config: maxiter must be positive"),
        (PasdConfig(lambdas=lam, ranks=[1, 1, 1], output_weights=[1.0, 0.0, 1.0]),
         "config: output weight of mode 2 must be positive"),
        (PasdConfig(lambdas=[1.0, 1.0], ranks=[1, 1, 1]), "config: expected 3 lambdas, got 2"),
    ]
    for cfg, msg in cases:
        with pytest.raises(ArgumentError) as ei:
            oracle_mod.pasd_recover(T, cfg)
        assert str(ei.value) == msg


def test_generator_reference_recipe(oracle_mod):
    dims, r = (9, 8, 7), 2
    L0 = oracle_mod.gen_tucker(dims, [r] * 3, seed=5)
    np.testing.assert_array_equal(L0, oracle_mod.gen_tucker(dims, [r] * 3, seed=5))  # deterministic per seed
    assert not np.array_equal(L0, oracle_mod.gen_tucker(dims, [r] * 3, seed=6))
    for mode in (1, 2, 3):  # exact Tucker rank (synth.cpp:55-67)
        s = np.linalg.svd(oracle_mod.unfold(L0, mode), compute_uv=False)
        assert s[r - 1] >= 1e-8 * s[0] and s[r] <= 1e-10 * s[0]
    T = oracle_mod.corrupt_sparse(L0, 0.1, seed=5)
    diff = T != L0
    assert int(diff.sum()) == round(0.1 * L0.size)  # exactly round(rho*size) entries
    assert np.abs(T - L0).max() <= 1.0
