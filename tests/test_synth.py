"""The device generator (pasd_b200_synth, paper_1712_09999_b200/synth.py)
against the oracle's restatement of the reference generator (synth.cpp:40-121,
rng.hpp:17-79) on the same seeds: the random streams, the partial
Fisher-Yates support and the noise values are integer / RNG work and must be
identical; L0 differs by rounding only (Householder vs LAPACK dgeqrf/dorgqr,
fma order of the mode products)."""
import numpy as np
import pytest

from paper_1712_09999_b200 import synth


@pytest.mark.parametrize("rows,cols,mode,kind", [(100, 10, 1, 0), (37, 37, 2, 0), (256, 30, 3, 1), (9, 1, 1, 0)])
def test_factor_matches_oracle(oracle_mod, rows, cols, mode, kind):
    q = synth.factor(rows, cols, seed=0, mode=mode, kind=kind)
    qo = oracle_mod.factor(rows, cols, 0, mode, kind)
    assert np.abs(q - qo).max() <= 1e-13
    if kind == 0:
        assert np.abs(q.T @ q - np.eye(cols)).max() <= 1e-13


@pytest.mark.parametrize("total,rho,seed", [(1000, 0.1, 0), (24 * 20 * 16, 0.05, 3), (50000, 0.2, 7), (10, 1.0, 1),
                                            (7, 0.0, 0)])
def test_support_matches_oracle(oracle_mod, total, rho, seed):
    pos = synth.support_draw_order(total, rho, seed)
    # oracle corrupt_sparse of a zero tensor: nonzeros are exactly the selected positions
    out = oracle_mod.corrupt_sparse(np.zeros(total), rho, seed=seed)
    ref = np.flatnonzero(out)
    assert pos.size == int(np.floor(rho * total + 0.5))
    assert len(set(pos.tolist())) == pos.size  # without replacement
    np.testing.assert_array_equal(np.sort(pos), ref)


@pytest.mark.gpu
@pytest.mark.parametrize("dims,r,rho,mode,kind,lohi", [
    ((24, 20, 16), 2, 0.05, 0, 0, (-1.0, 1.0)),
    ((40, 36, 30), 4, 0.2, 0, 0, (-5.0, 5.0)),
    ((13, 12, 11, 10), 2, 0.1, 1, 0, (0.0, 255.0)),
    ((100, 100, 100), 10, 0.1, 0, 0, (-1.0, 1.0)),
])
def test_generate_matches_oracle(gpu, oracle_mod, dims, r, rho, mode, kind, lohi):
    spec = synth.SynthSpec(dims, (r,) * len(dims), rho, 0, kind, mode, *lohi)
    T, L0, sup = synth.generate(spec, want_l0=True, want_support=True)
    Lo = oracle_mod.gen_tucker(dims, [r] * len(dims), seed=0, kind=kind)
    To = oracle_mod.corrupt_sparse(Lo, rho, seed=0, mode=mode, lo=lohi[0], hi=lohi[1])
    assert np.linalg.norm(L0 - Lo) <= 1e-13 * np.linalg.norm(Lo)
    ref_sup = np.flatnonzero(np.ravel(To - Lo, order="F") != 0) if mode == 0 else None
    if mode == 0:
        np.testing.assert_array_equal(sup, ref_sup)
        # noise values: exact draws, added to L0 (which differs by rounding)
        np.testing.assert_allclose(np.ravel(T - L0, order="F")[sup], np.ravel(To - Lo, order="F")[sup],
                                   rtol=0, atol=1e-12)
    else:
        np.testing.assert_array_equal(np.ravel(T, order="F")[sup], np.ravel(To, order="F")[sup])
    off = np.ones(T.size, dtype=bool)
    off[sup] = False
    np.testing.assert_array_equal(np.ravel(T, order="F")[off], np.ravel(L0, order="F")[off])


@pytest.mark.gpu
def test_generate_c4_recipe_matches_oracle(gpu, oracle_mod):
    dims = (64, 48, 20)
    spec = synth.SynthSpec(dims, (6, 6, 3), 0.05, 0, 1, 2, 0.0, 1.0, 16, 5)
    T, L0, sup = synth.generate(spec, want_l0=True, want_support=True)
    Lo = oracle_mod.gen_tucker(dims, [6, 6, 3], seed=0, kind=1)
    To = oracle_mod.corrupt_blocks(Lo, 16, 5, seed=0, lo=0.0, hi=1.0)
    assert np.linalg.norm(L0 - Lo) <= 1e-13 * np.linalg.norm(Lo)
    assert L0.max() == 1.0 and L0.min() >= 0.0
    assert sup.size == 20 * 5 * 256
    np.testing.assert_array_equal(np.ravel(T, order="F")[sup], np.ravel(To, order="F")[sup])


@pytest.mark.gpu
def test_generate_torch_output_matches_numpy(gpu):
    from paper_1712_09999_b200.workloads import WORKLOADS

    w = WORKLOADS["c1"]
    spec = synth.workload_spec(w)
    Tn, _, _ = synth.generate(spec)
    Tt, _, _ = synth.generate(spec, out="torch")
    np.testing.assert_array_equal(Tt.cpu().numpy().reshape(-1), np.ravel(Tn, order="F"))
