"""The C++ drop-in (include/tenrec_b200/pasd.hpp) through tools/tenrec_recover.cpp,
the minimal `recover` front end (reference: proj/tools/cli.cpp:244-354):
TNSR in, X/E TNSR out, exit codes of cli.hpp:9-14.

CPU: the client compiles against the header + libpasd_b200.so and maps a
missing input to IoError (exit 2) before touching the device.  GPU: on a
golden fixture it returns what the Python binding returns, bit for bit."""
import json
import os
import subprocess

import numpy as np
import pytest

from paper_1712_09999_b200.api import PasdConfig
from paper_1712_09999_b200.tnsr import read_tensor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1712_09999_b200")


@pytest.fixture(scope="module")
def client(tmp_path_factory):
    if not os.path.exists(os.path.join(LIBDIR, "libpasd_b200.so")):
        pytest.fail("libpasd_b200.so not built (run __graft_entry__.build())")
    exe = str(tmp_path_factory.mktemp("cli") / "tenrec_recover")
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tools", "tenrec_recover.cpp"), "-L", LIBDIR, "-lpasd_b200",
                    "-Wl,-rpath," + LIBDIR, "-o", exe], check=True)
    return exe


def test_client_builds_and_reports_io_errors(client, tmp_path):
    p = subprocess.run([client, str(tmp_path / "missing.tnsr"), "2", str(tmp_path / "out")],
                       capture_output=True, text=True)
    assert p.returncode == 2
    assert "cannot open" in p.stderr
    bad = tmp_path / "bad.tnsr"
    bad.write_bytes(b"XXXX0000")
    p = subprocess.run([client, str(bad), "2", str(tmp_path / "out")], capture_output=True, text=True)
    assert p.returncode == 2 and "bad magic" in p.stderr
    p = subprocess.run([client], capture_output=True, text=True)
    assert p.returncode == 1


@pytest.mark.gpu
def test_client_matches_python_binding(client, gpu, tmp_path):
    src = os.path.join(ROOT, "tests", "golden", "g3_24x20x16_r3_R4", "t.tnsr")
    p = subprocess.run([client, src, "3", str(tmp_path / "out"), "1e-6", "500"], capture_output=True, text=True)
    assert p.returncode == 0, p.stderr
    summary = json.loads(p.stdout.strip().splitlines()[-1])
    T = read_tensor(src)
    dims = T.shape
    R = int(np.floor(1.2 * 3))  # PasdConfig::default_rank_bound (pasd.cpp:62-66), as the client uses
    from oracle import default_lambdas

    cfg = PasdConfig(lambdas=default_lambdas(dims), ranks=[R] * 3, eps=1e-6, maxiter=500)
    r = gpu.pasd_recover(T, cfg)
    assert summary["iters"] == r.iters and summary["converged"] == r.converged
    np.testing.assert_array_equal(read_tensor(str(tmp_path / "out_x.tnsr")), r.x)
    np.testing.assert_array_equal(read_tensor(str(tmp_path / "out_e.tnsr")), r.e)
