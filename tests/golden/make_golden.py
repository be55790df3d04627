"""Regenerate the golden fixtures from the oracle (the reference restatement).

    python tests/golden/make_golden.py

Each fixture = input tensor (TNSR, the reference's file format) + oracle
outputs X, E (TNSR) + scalars (JSON).  The reference itself is unbuildable in
this image (no Eigen / lapacke.h), so these pin the restatement over time and
feed the GPU parity tests; the restatement itself is pinned against SPEC.md's
known-answer examples in tests/test_oracle_kat.py.
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402
from paper_1712_09999_b200.api import PasdConfig  # noqa: E402
from paper_1712_09999_b200.tnsr import write_tensor  # noqa: E402

CASES = {
    "g1_12x10x8_r2": dict(dims=(12, 10, 8), r=2, R=2, rho=0.05, eps=1e-6, seed=1),
    "g2_6x5x4x3_r2": dict(dims=(6, 5, 4, 3), r=2, R=2, rho=0.05, eps=1e-6, seed=2),
    "g3_24x20x16_r3_R4": dict(dims=(24, 20, 16), r=3, R=4, rho=0.10, eps=1e-6, seed=3),
}


def make(name, dims, r, R, rho, eps, seed):
    L0 = oracle.gen_tucker(dims, [r] * len(dims), seed=seed)
    T = oracle.corrupt_sparse(L0, rho, seed=seed)
    cfg = PasdConfig(lambdas=oracle.default_lambdas(dims), ranks=[R] * len(dims), eps=eps)
    res = oracle.pasd_recover(T, cfg)
    d = os.path.join(HERE, name)
    os.makedirs(d, exist_ok=True)
    write_tensor(T, os.path.join(d, "t.tnsr"))
    write_tensor(L0, os.path.join(d, "l0.tnsr"))
    write_tensor(res.x, os.path.join(d, "x.tnsr"))
    write_tensor(res.e, os.path.join(d, "e.tnsr"))
    meta = dict(dims=list(dims), tucker_rank=r, ranks=[R] * len(dims), rho=rho, eps=eps, seed=seed,
                lambdas=cfg.lambdas, iters=res.iters, converged=res.converged,
                residual_history=res.residual_history, final_residuals=res.final_residuals,
                objective=res.objective,
                certificate=None if res.certificate is None else vars(res.certificate))
    with open(os.path.join(d, "meta.json"), "w") as f:
        json.dump(meta, f, indent=1)


if __name__ == "__main__":
    for k, v in CASES.items():
        make(k, **v)
        print("wrote", k)
