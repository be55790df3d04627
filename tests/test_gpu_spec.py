"""The spec-shaped half of the reference header (pasd.hpp:43-58, 68-70) on the
device, against the oracle's restatement on the same state:
pasd_g_matrix, update_u, update_v, update_e, suboptimality_certificate, and the
finalisation (Y-hat, objective, certificate) on a shared final iterate."""
import numpy as np
import pytest

import paper_1712_09999_b200 as pb
from paper_1712_09999_b200.api import ArgumentError, PasdConfig, PasdState, StateError

pytestmark = pytest.mark.gpu


def rel(a, b):
    n = np.linalg.norm(b)
    return np.linalg.norm(a - b) / n if n > 0 else np.linalg.norm(a - b)


def _snapshots(oracle_mod, dims, r, rho, seed, eps, want):
    L0 = oracle_mod.gen_tucker(dims, [r] * len(dims), seed=seed)
    T = oracle_mod.corrupt_sparse(L0, rho, seed=seed)
    cfg = PasdConfig(lambdas=oracle_mod.default_lambdas(dims), ranks=[r] * len(dims), eps=eps)
    snaps = {}

    def obs(v):
        if want(v.iter):
            snaps[v.iter] = v

    res = oracle_mod.pasd_recover(T, cfg, observer=obs)
    return T, cfg, res, snaps


def _state(view):
    return PasdState(u=list(view.u), v=list(view.v), e=view.e, y=list(view.y), mu=view.mu_next, iter=view.iter)


@pytest.mark.parametrize("dims", [(14, 11, 9), (7, 6, 5, 4)])
def test_g_matrix_bit_exact(gpu, oracle_mod, dims):
    rng = np.random.default_rng(1)
    T, E, Y = (rng.standard_normal(dims) for _ in range(3))
    mu = 0.37
    for mode in range(1, len(dims) + 1):
        g = pb.pasd_g_matrix(T, E, Y, mu, mode)
        ref = oracle_mod.unfold((T - E) + Y * (1.0 / mu), mode)  # pasd.cpp:91-96
        np.testing.assert_array_equal(g, ref)
    N = len(dims)
    with pytest.raises(ArgumentError, match=f"mode {N + 1} out of range 1..{N}"):  # tensor.cpp:133-137
        pb.pasd_g_matrix(T, E, Y, mu, N + 1)


def test_update_u_v_e_match_oracle(gpu, oracle_mod):
    """One mode sweep of the reference (pasd.cpp:175-209) through the spec API,
    from the oracle's full-rank iterate k, against the oracle's own update_u_from
    (procrustes), update_v_from (svt) and update_e restated in numpy."""
    T, cfg, res, snaps = _snapshots(oracle_mod, (26, 24, 22), 3, 0.05, 6, 1e-9, lambda k: k in (150,))
    st = _state(snaps[150])
    for n in range(3):
        assert np.linalg.matrix_rank(st.v[n]) == 3
    mu = st.mu
    for mode in (1, 2, 3):
        n = mode - 1
        G = oracle_mod.unfold((T - st.e) + st.y[n] * (1.0 / mu), mode)
        u_ref = oracle_mod.procrustes(G, st.v[n])
        u = pb.update_u(st, T, mode)
        assert np.abs(u - u_ref).max() <= 1e-10
        st.u[n] = u_ref
        v_ref = oracle_mod.svt(u_ref.T @ G, cfg.lambdas[n] / mu)
        v = pb.update_v(st, T, mode, cfg.lambdas[n])
        assert rel(v, v_ref) <= 1e-10
        st.v[n] = v_ref
    # update_e (pasd.cpp:111-130) restated: acc from 0 in mode order, shrink at 1/(mu N)
    acc = np.zeros(T.shape)
    for n in range(3):
        z = oracle_mod.fold(st.u[n] @ st.v[n], n + 1, T.shape)
        acc = acc + ((T - z) + st.y[n] * (1.0 / mu))
    x = acc * (1.0 / 3)
    tau = 1.0 / (mu * 3)
    e_ref = np.where(x > tau, x - tau, np.where(x < -tau, x + tau, 0.0))
    e = pb.update_e(st, T)
    assert rel(e, e_ref) <= 1e-12
    assert np.count_nonzero((e != 0) != (e_ref != 0)) <= 2


def test_update_u_degenerate_keeps_basis(gpu):
    """V = 0 (the first iteration, pasd.cpp:152-153): W = 0 -> keep U (linops.cpp:99-101)."""
    rng = np.random.default_rng(3)
    dims = (9, 8, 7)
    T = rng.standard_normal(dims)
    u0 = np.linalg.qr(rng.standard_normal((9, 2)))[0]
    st = PasdState(u=[u0, np.eye(8, 2), np.eye(7, 2)], v=[np.zeros((2, 56)), np.zeros((2, 63)), np.zeros((2, 72))],
                   e=np.zeros(dims), y=[np.zeros(dims)] * 3, mu=1e-4)
    np.testing.assert_array_equal(pb.update_u(st, T, 1), u0)


def test_certificate_matches_oracle(gpu, oracle_mod):
    T, cfg, res, _ = _snapshots(oracle_mod, (20, 18, 16), 2, 0.05, 9, 1e-6, lambda k: False)
    assert res.converged and res.certificate is not None
    c = pb.suboptimality_certificate(res, T, cfg)
    assert c.epsilon_hat == res.certificate.epsilon_hat  # same mode-order accumulation, exact max
    assert c.c == pytest.approx(res.certificate.c, rel=1e-13)
    assert c.bound == pytest.approx(res.certificate.bound, rel=1e-12)
    res.converged = False
    with pytest.raises(StateError, match="certificate requires a converged result"):
        pb.suboptimality_certificate(res, T, cfg)
    res.converged = True
    res.y_hat = None
    with pytest.raises(StateError, match="certificate requires the final multipliers"):
        pb.suboptimality_certificate(res, T, cfg)


def test_finalisation_on_a_shared_final_iterate(gpu, oracle_mod):
    """Y-hat, objective and certificate (pasd.cpp:246-274, 277-309) computed by
    the GPU finalisation and by the oracle from the same last step: inject the
    oracle's iterate K*-1 of a converged run, run the final iteration on the
    GPU, finalise, compare with the oracle's result."""
    T, cfg, res, snaps = _snapshots(oracle_mod, (24, 22, 20), 2, 0.05, 12, 1e-7, lambda k: True)
    K = res.iters
    assert res.converged and K - 1 in snaps
    a = snaps[K - 1]
    s = pb.Solver(T.shape, cfg)
    s.load(T)
    s.set_state(a.e, a.y, a.u, a.v, a.mu_next, a.iter)
    s.run(1)
    r = s.finalize(want_z=True, want_y=True)
    s.close()
    assert r.iters == K and r.converged
    assert rel(r.e, res.e) <= 1e-10
    for n in range(3):
        assert rel(r.y_hat[n], res.y_hat[n]) <= 1e-9
    assert r.objective == pytest.approx(res.objective, rel=1e-10)
    assert r.certificate is not None
    # eps_hat = |sum_n (Y_n - Yhat_n)|_inf = mu N |E - E_prev|_inf: rounding of E scaled by mu
    assert r.certificate.epsilon_hat == pytest.approx(res.certificate.epsilon_hat, rel=1e-6)
    assert r.certificate.c == pytest.approx(res.certificate.c, rel=1e-13)
    assert r.certificate.bound == pytest.approx(res.certificate.bound, rel=1e-6)
