"""Memory check of every kernel (compute-sanitizer is closed on this GPU pool):
tools/sanitize_run.py -- both pass-2 variants on ragged bricks, the generic
order-4 kernels, the cluster small solves through the rank transition, the spec
helpers, the generator, the SNN baseline, the loopback sharded path and the fp32
mode -- under the library's guard-band mode (PASD_B200_GUARD=1: 64 KB canary
bands of NaN bytes around every device buffer, verified when it is freed)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_guard_bands_intact(gpu):
    env = dict(os.environ, PASD_B200_GUARD="1")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_run.py")], env=env,
                       capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-2000:]
    line = [l for l in p.stdout.splitlines() if l.startswith("guard bands:")]
    assert line and "mode=on" in line[0] and line[0].endswith("violations=0"), p.stdout[-2000:]
    checked = int(line[0].split("buffers checked=")[1].split()[0])
    assert checked > 500
