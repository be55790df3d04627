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

    def __init__(self, rank: int, nranks: int, slab: Tuple[int, int], uid: Optional[bytes]):
        self._uid = C.create_string_buffer(uid, 128) if uid is not None else None
        self.struct = _abi.PasdShard()
        self.struct.rank = rank
        self.struct.nranks = nranks
        self.struct.nccl_unique_id = C.cast(self._uid, C.c_void_p) if self._uid is not None else None
        self.struct.slab_begin, self.struct.slab_end = int(slab[0]), int(slab[1])
