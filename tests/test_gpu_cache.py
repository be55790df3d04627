"""The one-shot drop-in keeps its solver between identical calls
(pasd_b200_recover's cache); results must not depend on it."""
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
    first = pb.pasd_recover(X1, cfg)       # fresh solver, then cached
    second = pb.pasd_recover(X2, cfg)      # reuses the cached solver
    again = pb.pasd_recover(X1, cfg)       # reuses it again
    pb.release_cache()
    fresh2 = pb.pasd_recover(X2, cfg)      # fresh solver for X2
    pb.release_cache()
    assert np.array_equal(first.x, again.x)
    assert np.array_equal(first.e, again.e)
    assert first.iters == again.iters
    assert np.array_equal(second.x, fresh2.x)
    assert np.array_equal(second.e, fresh2.e)
    assert second.iters == fresh2.iters


def test_changed_options_do_not_reuse():
    X = _problem(3)
    a = pb.pasd_recover(X, PasdConfig(lambdas=[1.0, 1.0, 1.0], ranks=[3, 3, 3], maxiter=40))
    b = pb.pasd_recover(X, PasdConfig(lambdas=[1.0, 1.0, 1.0], ranks=[3, 3, 3], maxiter=40, rho=1.2))
    pb.release_cache()
    c = pb.pasd_recover(X, PasdConfig(lambdas=[1.0, 1.0, 1.0], ranks=[3, 3, 3], maxiter=40, rho=1.2))
    pb.release_cache()
    assert np.array_equal(b.x, c.x)
    assert a.iters >= 1
