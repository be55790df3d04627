"""Time consecutive pasd_b200_recover calls (C-ABI, host buffers) per phase."""
import ctypes as C
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1712_09999_b200 import _abi, solver as S  # noqa: E402
from paper_1712_09999_b200.api import PasdConfig, build_options, raise_for_status  # noqa: E402
from paper_1712_09999_b200.workloads import WORKLOADS, generate_gpu  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c1"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
w = WORKLOADS[cfgname]
T = generate_gpu(w, seed=0)
Th = torch.empty(T.numel(), dtype=torch.float64, pin_memory=True)
Th.copy_(T.view(-1))
xh = torch.empty_like(Th)
eh = torch.empty_like(Th)
cfg = PasdConfig(lambdas=w.lambdas(), ranks=list(w.ranks), eps=w.eps, maxiter=steps)
opt, keep = build_options(list(w.dims), cfg, flags=_abi.PASD_FLAG_FIXED_ITERS, poll_every=steps)
out = _abi.PasdOutputs()
out.x = C.cast(C.c_void_p(xh.data_ptr()), _abi.c_double_p)
out.e = C.cast(C.c_void_p(eh.data_ptr()), _abi.c_double_p)
err = C.create_string_buffer(1024)
tptr = C.cast(C.c_void_p(Th.data_ptr()), _abi.c_double_p)
for k in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rc = S.lib().pasd_b200_recover(tptr, C.byref(opt), C.byref(out), _abi.PasdObserverFn(), None, err, len(err))
    t1 = time.perf_counter()
    raise_for_status(rc, err)
    print(f"{cfgname} call {k}: {1e3 * (t1 - t0):.2f} ms for {steps} iterations", flush=True)
