"""Slab sharding of the last mode across ranks (one process per GPU).

The reference has no distributed code ("Distributed comm backend:
absent"); the B200 build shards the PASD iteration as SURVEY 8(e) plans:
rank k owns T[:, :, b_k:e_k] (a contiguous byte range in first-index-fastest
layout) and the per-iteration exchanges are NCCL all-reduces inside the
library (pasd_solver.cu): A_3 partials (SUM), Gram_1/Gram_2 partials (SUM),
Wt_1/Wt_2 partials and the zero-padded own rows of Wt_3 (SUM), ||G_n||^2
(SUM), residual maxima and the NaN flag (MAX).  U_n, M_n and the small solves
are replicated (every rank reduces the same bytes, so no broadcast).
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Tuple

from . import _abi
from .api import raise_for_status


def slab_bounds(n: int, nranks: int, rank: int) -> Tuple[int, int]:
    """Contiguous, balanced partition of range(n) into nranks slabs."""
    if nranks < 1 or not (0 <= rank < nranks):
        raise ValueError("invalid rank/nranks")
    if n < nranks:
        raise ValueError(f"cannot split {n} slices over {nranks} ranks")
    base, extra = divmod(n, nranks)
    b = rank * base + min(rank, extra)
    return b, b + base + (1 if rank < extra else 0)


def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId from the library (rank 0)."""
    from .solver import lib

    buf = C.create_string_buffer(128)
    err = C.create_string_buffer(1024)
    L = lib()
    L.pasd_b200_nccl_unique_id.restype = C.c_int
    L.pasd_b200_nccl_unique_id.argtypes = [C.c_void_p, C.c_char_p, C.c_size_t]
    raise_for_status(L.pasd_b200_nccl_unique_id(buf, err, len(err)), err)
    return bytes(buf.raw[:128])


class Shard:
    """pasd_shard plus the buffers its pointers refer to."""

    def __init__(self, rank: int, nranks: int, slab: Tuple[int, int], uid: Optional[bytes],
                 loopback: Optional["LoopbackGroup"] = None):
        self._uid = C.create_string_buffer(uid, 128) if uid is not None else None
        self.struct = _abi.PasdShard()
        self.struct.rank = rank
        self.struct.nranks = nranks
        self.struct.nccl_unique_id = C.cast(self._uid, C.c_void_p) if self._uid is not None else None
        self.struct.slab_begin, self.struct.slab_end = int(slab[0]), int(slab[1])
        self._loopback = loopback  # keeps the group alive while the shard exists
        self.struct.loopback = loopback.handle if loopback is not None else None


class LoopbackGroup:
    """pasd_b200_loopback_create: nranks sharded solvers sharing ONE device in
    this process, one host thread per rank.  The library's own sharded path
    (slab partials, the same all-reduce sequence, replicated small solves) runs
    with its collectives done by host rendezvous + a rank-ordered reduce kernel
    instead of NCCL.  For testing nranks > 1 on one GPU; not a speed-up."""

    def __init__(self, nranks: int):
        from .solver import lib

        L = lib()
        L.pasd_b200_loopback_create.restype = C.c_int
        L.pasd_b200_loopback_create.argtypes = [C.c_int32, C.POINTER(C.c_void_p), C.c_char_p, C.c_size_t]
        L.pasd_b200_loopback_destroy.restype = None
        L.pasd_b200_loopback_destroy.argtypes = [C.c_void_p]
        self._lib = L
        self.nranks = int(nranks)
        h = C.c_void_p()
        err = C.create_string_buffer(1024)
        raise_for_status(L.pasd_b200_loopback_create(self.nranks, C.byref(h), err, len(err)), err)
        self.handle = h

    def close(self):
        if self.handle:
            self._lib.pasd_b200_loopback_destroy(self.handle)
            self.handle = None


def run_loopback(t, config, nranks: int, iters: int, *, fixed_iters: bool = True, slabs=None,
                 check_replicas: bool = True, device: int = 0, poll_every: int = 0, want_z: bool = False,
                 want_y: bool = False, fp32: bool = False):
    """Solve `t` (I_1 x I_2 x I_3) as `nranks` mode-3 slabs through the library's
    sharded path on one device (LoopbackGroup).  Returns (iters, converged,
    per-rank finalize() results, slabs)."""
    import threading

    import numpy as np

    from . import _abi as A
    from .solver import Solver

    t = np.asarray(t, dtype=np.float64)
    dims = list(t.shape)
    if slabs is None:
        slabs = [slab_bounds(dims[-1], nranks, r) for r in range(nranks)]
    group = LoopbackGroup(nranks)
    flags = A.PASD_FLAG_CHECK_REPLICAS if check_replicas else 0
    results = [None] * nranks
    errors = [None] * nranks
    ready = threading.Barrier(nranks)  # no rank enters a collective unless every rank was built

    def rank_main(r):
        sol = None
        try:
            try:
                shard = Shard(r, nranks, slabs[r], None, loopback=group)
                sol = Solver(dims, config, device=device, fixed_iters=fixed_iters, poll_every=poll_every,
                             shard=shard, flags=flags, fp32=fp32)
                sol.load(np.asfortranarray(t[:, :, slabs[r][0]:slabs[r][1]]))
            except BaseException:
                ready.abort()
                raise
            ready.wait()
            done, conv = sol.run(iters)
            results[r] = (done, conv, sol.finalize(want_x=True, want_e=True, want_z=want_z, want_y=want_y))
        except BaseException as exc:  # re-raised on the caller's thread
            errors[r] = exc
        finally:
            if sol is not None:
                sol.close()

    threads = [threading.Thread(target=rank_main, args=(r,)) for r in range(nranks)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    group.close()
    real = [e for e in errors if e is not None and not isinstance(e, threading.BrokenBarrierError)]
    if real or any(e is not None for e in errors):
        raise (real or [e for e in errors if e is not None])[0]
    done = {r[0] for r in results}
    conv = {r[1] for r in results}
    if len(done) != 1 or len(conv) != 1:
        raise RuntimeError(f"loopback ranks disagree: iterations {done}, converged {conv}")
    return done.pop(), conv.pop(), [r[2] for r in results], slabs
