"""The C++ drop-in (include/tenrec_b200/pasd.hpp) through tools/tenrec_b200_cli.cpp,
the reference's `tenrec` front end for synth / recover / certify / defaults
(proj/tools/cli.cpp:158-208, 244-354, 457-567): TNSR in and out, key = value
manifests, the exit codes of cli.hpp:9-14.

CPU: the client compiles against the header + libpasd_b200.so, prints the
defaults, and maps usage / I/O errors to exit 1 / 2 before touching the device.
GPU: synth -> recover -> certify on the device (SPEC.md:529's chain), recover
bit-equal to the Python binding, --strict -> 4, --no-z, --from-manifest."""
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
    exe = str(tmp_path_factory.mktemp("cli") / "tenrec_b200")
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tools", "tenrec_b200_cli.cpp"), "-L", LIBDIR, "-lpasd_b200",
                    "-Wl,-rpath," + LIBDIR, "-o", exe], check=True)
    return exe


def run(client, *args):
    return subprocess.run([client, *map(str, args)], capture_output=True, text=True)


def manifest(path):
    out = {}
    for line in open(path):
        k, v = line.split("=", 1)
        out[k.strip()] = v.strip()
    return out


def test_client_builds_and_reports_errors(client, tmp_path):
    p = run(client, "defaults")
    assert p.returncode == 0 and "mu0 = 0.0001" in p.stdout and "maxiter = 1000" in p.stdout  # cli.cpp:557-567
    p = run(client, "recover", "--input", tmp_path / "missing.tnsr", "--out-prefix", tmp_path / "o", "--target-rank", 2)
    assert p.returncode == 2 and "cannot open" in p.stderr
    bad = tmp_path / "bad.tnsr"
    bad.write_bytes(b"XXXX0000")
    p = run(client, "recover", "--input", bad, "--out-prefix", tmp_path / "o", "--target-rank", 2)
    assert p.returncode == 2 and "bad magic" in p.stderr
    assert run(client).returncode == 1
    assert run(client, "recover", "--bogus", "1").returncode == 1
    p = run(client, "recover", "--out-prefix", tmp_path / "o")
    assert p.returncode == 1 and "recover needs --input" in p.stderr


@pytest.mark.gpu
def test_synth_recover_certify_chain(client, gpu, tmp_path):
    pre = tmp_path / "inst"
    p = run(client, "synth", "--dims", "24,20,16", "--rank", 2, "--corruption", 0.05, "--seed", 0, "--out-prefix", pre)
    assert p.returncode == 0, p.stderr
    syn = manifest(str(pre) + "_synth.manifest")
    assert syn["corrupted_entries"] == str(round(0.05 * 24 * 20 * 16))
    obs, truth = str(pre) + "_observed.tnsr", str(pre) + "_truth.tnsr"
    # the device generator is the oracle's generator (support and noise exact, L0 to rounding)
    import oracle

    L0 = oracle.gen_tucker((24, 20, 16), [2, 2, 2], seed=0)
    np.testing.assert_allclose(read_tensor(truth), L0, rtol=0, atol=1e-13)
    out = tmp_path / "rec"
    p = run(client, "recover", "--input", obs, "--truth", truth, "--out-prefix", out, "--ranks", "2,2,2",
            "--eps", "1e-7")
    assert p.returncode == 0, p.stderr
    man = manifest(str(out) + ".manifest")
    assert man["converged"] == "true" and float(man["rse"]) < 1e-4
    assert len(man["z_out"].split(",")) == 3 and "cert_epsilon_hat" in man
    T = read_tensor(obs)
    cfg = PasdConfig(lambdas=[float(v) for v in man["lambdas"].split(",")], ranks=[2, 2, 2], eps=1e-7)
    r = gpu.pasd_recover(T, cfg)
    assert int(man["iters"]) == r.iters
    np.testing.assert_array_equal(read_tensor(str(out) + "_x.tnsr"), r.x)
    np.testing.assert_array_equal(read_tensor(str(out) + "_e.tnsr"), r.e)
    np.testing.assert_array_equal(read_tensor(str(out) + "_z2.tnsr"), r.z[1])
    c = run(client, "certify", "--manifest", str(out) + ".manifest")
    assert c.returncode == 0, c.stdout + c.stderr
    for check in ("feasibility", "objective", "constant_c", "bound", "epsilon_hat", "gap_bound"):
        assert f"[ OK ] {check}" in c.stdout, c.stdout
    # --from-manifest re-runs the same configuration (cli.cpp:225-242)
    p = run(client, "recover", "--from-manifest", str(out) + ".manifest", "--out-prefix", tmp_path / "again", "--no-z")
    assert p.returncode == 0, p.stderr
    again = manifest(str(tmp_path / "again") + ".manifest")
    assert again["iters"] == man["iters"] and "z_out" not in again
    np.testing.assert_array_equal(read_tensor(str(tmp_path / "again") + "_x.tnsr"), r.x)
    # a tampered input fails the checksum (cli.cpp:465-466)
    T2 = T.copy()
    T2[0, 0, 0] += 1.0
    from paper_1712_09999_b200.tnsr import write_tensor
    write_tensor(T2, obs)
    c = run(client, "certify", "--manifest", str(out) + ".manifest")
    assert c.returncode == 2 and "checksum" in c.stderr


@pytest.mark.gpu
def test_strict_non_convergence_exits_4(client, gpu, tmp_path):
    src = os.path.join(ROOT, "tests", "golden", "g3_24x20x16_r3_R4", "t.tnsr")
    p = run(client, "recover", "--input", src, "--out-prefix", tmp_path / "s", "--target-rank", 3, "--maxiter", 5,
            "--strict")
    assert p.returncode == 4, p.stderr  # cli.cpp:351-352
    assert manifest(str(tmp_path / "s") + ".manifest")["converged"] == "false"
    p = run(client, "recover", "--input", src, "--out-prefix", tmp_path / "s", "--target-rank", 3, "--maxiter", 5)
    assert p.returncode == 0
    p = run(client, "recover", "--input", src, "--out-prefix", tmp_path / "s", "--ranks", "9,9,9,9")
    assert p.returncode == 1 and "expected 3 ranks" in p.stderr


@pytest.mark.gpu
def test_recover_snn_solver(client, gpu, tmp_path):
    """`recover --solver snn` (cli.cpp:278-282) runs the device SNN baseline through the
    C++ drop-in tenrec_b200::snn_recover: same X / E as the Python binding, no
    certificate in the manifest; rpca stays outside this build."""
    src = os.path.join(ROOT, "tests", "golden", "g3_24x20x16_r3_R4", "t.tnsr")
    out = tmp_path / "snn"
    p = run(client, "recover", "--input", src, "--out-prefix", out, "--solver", "snn", "--maxiter", 60)
    assert p.returncode == 0, p.stderr
    man = manifest(str(out) + ".manifest")
    assert man["solver"] == "snn" and "ranks" not in man and "cert_epsilon_hat" not in man
    from paper_1712_09999_b200.api import SnnConfig
    T = read_tensor(src)
    r = gpu.snn_recover(T, SnnConfig(lambdas=[float(v) for v in man["lambdas"].split(",")], maxiter=60))
    assert int(man["iters"]) == r.iters
    np.testing.assert_array_equal(read_tensor(str(out) + "_x.tnsr"), r.x)
    np.testing.assert_array_equal(read_tensor(str(out) + "_e.tnsr"), r.e)
    p = run(client, "recover", "--input", src, "--out-prefix", out, "--solver", "rpca")
    assert p.returncode == 1 and "rpca" in p.stderr
