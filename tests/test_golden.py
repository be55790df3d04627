"""Golden fixtures (tests/golden/*, made by make_golden.py from the oracle).

CPU: the oracle reproduces its committed outputs bit-for-bit (pins the
restatement across rebuilds) and TNSR round-trips are exact."""
import json
import os

import numpy as np
import pytest

from paper_1712_09999_b200.api import IoError, PasdConfig
from paper_1712_09999_b200.tnsr import read_tensor, write_tensor

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASES = sorted(d for d in os.listdir(GOLD) if os.path.isdir(os.path.join(GOLD, d)))


def load(name):
    d = os.path.join(GOLD, name)
    meta = json.load(open(os.path.join(d, "meta.json")))
    return meta, {k: read_tensor(os.path.join(d, k + ".tnsr")) for k in ("t", "l0", "x", "e")}


@pytest.mark.parametrize("name", CASES)
def test_oracle_reproduces_golden(oracle_mod, name):
    meta, g = load(name)
    cfg = PasdConfig(lambdas=meta["lambdas"], ranks=meta["ranks"], eps=meta["eps"])
    r = oracle_mod.pasd_recover(g["t"], cfg)
    assert r.iters == meta["iters"] and r.converged == meta["converged"]
    np.testing.assert_array_equal(r.x, g["x"])
    np.testing.assert_array_equal(r.e, g["e"])
    assert r.residual_history == meta["residual_history"]


def test_tnsr_roundtrip_and_errors(tmp_path):
    rng = np.random.default_rng(0)
    for shape in [(3, 4, 2), (7,), (2, 1, 3, 2)]:
        t = np.asfortranarray(rng.standard_normal(shape))
        p = tmp_path / "a.tnsr"
        write_tensor(t, p)
        np.testing.assert_array_equal(read_tensor(p), t)
    write_tensor(np.zeros((2, 2, 2)), tmp_path / "h.tnsr")
    assert os.path.getsize(tmp_path / "h.tnsr") == 32 + 64  # header 4+2+2+24 (SPEC.md io_cli)
    raw = (tmp_path / "h.tnsr").read_bytes()
    (tmp_path / "bad.tnsr").write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(IoError, match="bad magic at byte offset 0"):
        read_tensor(tmp_path / "bad.tnsr")
    (tmp_path / "trunc.tnsr").write_bytes(raw[:-8])
    with pytest.raises(IoError, match="truncated payload at byte offset 88"):
        read_tensor(tmp_path / "trunc.tnsr")
    (tmp_path / "trail.tnsr").write_bytes(raw + b"\0")
    with pytest.raises(IoError, match="trailing bytes after payload"):
        read_tensor(tmp_path / "trail.tnsr")
