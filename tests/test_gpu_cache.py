"""The one-shot drop-in can keep its solver between identical calls
(pasd_b200_recover with PASD_FLAG_REUSE_SOLVER); results must not depend on it."""
import numpy as np
import pytest

import paper_1712_09999_b200 as pb
from paper_1712_09999_b200.api import PasdConfig

pytestmark = pytest.mark.gpu


def _problem(seed):
    rng = np.random.default_rng(seed)
    dims = (18, 14, 12)
    L = np.einsum("abc,ia,jb,kc->ijk", rng.standard_normal((3, 3, 3)),
                  *(np.linalg.qr(rng.standard_normal((d, 3)))[0] for d in dims))
    E = np.where(rng.random(dims) < 0.1, rng.uniform(-1, 1, dims), 0.0)
    return L + E


def test_repeated_calls_match_fresh_solver():
    cfg = PasdConfig(lambdas=[1.0, 1.0, 1.0], ranks=[3, 3, 3], maxiter=60)
    pb.release_cache()
    X1, X2 = _problem(1), _problem(2)
    first = pb.pasd_recover(X1, cfg, reuse_solver=True)       # fresh solver, then cached
    second = pb.pasd_recover(X2, cfg, reuse_solver=True)      # reuses the cached solver
    again = pb.pasd_recover(X1, cfg, reuse_solver=True)       # reuses it again
    pb.release_cache()
    fresh2 = pb.pasd_recover(X2, cfg, reuse_solver=True)      # fresh solver for X2
    pb.release_cache()
    assert np.array_equal(first.x, again.x)
    assert np.array_equal(first.e, again.e)
    assert first.iters == again.iters
    assert np.array_equal(second.x, fresh2.x)
    assert np.array_equal(second.e, fresh2.e)
    assert second.iters == fresh2.iters


def test_changed_options_do_not_reuse():
    X = _problem(3)
    a = pb.pasd_recover(X, PasdConfig(lambdas=[1.0, 1.0, 1.0], ranks=[3, 3, 3], maxiter=40), reuse_solver=True)
    b = pb.pasd_recover(X, PasdConfig(lambdas=[1.0, 1.0, 1.0], ranks=[3, 3, 3], maxiter=40, rho=1.2), reuse_solver=True)
    pb.release_cache()
    c = pb.pasd_recover(X, PasdConfig(lambdas=[1.0, 1.0, 1.0], ranks=[3, 3, 3], maxiter=40, rho=1.2), reuse_solver=True)
    pb.release_cache()
    assert np.array_equal(b.x, c.x)
    assert a.iters >= 1


def test_solvers_of_different_rank_coexist():
    """Small-solve shared-memory caps are per (kernel, device) and process-wide:
    a solver built later with a small rank must not break an earlier large-rank
    one (it used to lower cudaFuncAttributeMaxDynamicSharedMemorySize)."""
    rng = np.random.default_rng(4)
    Xb = rng.standard_normal((60, 56, 52))
    big = pb.Solver(Xb.shape, PasdConfig(lambdas=[1.0] * 3, ranks=[50, 50, 50], maxiter=20), fixed_iters=True)
    small = pb.Solver((8, 8, 8), PasdConfig(lambdas=[1.0] * 3, ranks=[2, 2, 2], maxiter=20), fixed_iters=True)
    big.load(Xb)
    small.load(rng.standard_normal((8, 8, 8)))
    small.run(5)
    big.run(20)  # first graph capture of the large-rank solver after the small one was built
    r = big.finalize()
    assert r.iters == 20
    ref = pb.pasd_recover(Xb, PasdConfig(lambdas=[1.0] * 3, ranks=[50, 50, 50], maxiter=20), fixed_iters=True)
    np.testing.assert_array_equal(r.e, ref.e)
    big.close()
    small.close()


def test_no_solver_kept_without_the_flag():
    """Without PASD_FLAG_REUSE_SOLVER the library keeps no device memory."""
    import torch

    pb.release_cache()
    X = _problem(5)
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    for _ in range(3):
        pb.pasd_recover(X, PasdConfig(lambdas=[1.0, 1.0, 1.0], ranks=[3, 3, 3], maxiter=10))
    torch.cuda.synchronize()
    assert torch.cuda.mem_get_info()[0] >= free0 - (8 << 20)
