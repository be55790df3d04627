"""Host-side logic of the slab-sharded (multi-GPU) path, on CPU with gloo.

World size 2.  Each rank owns T[:, :, b:e] (sharding.slab_bounds) and forms
exactly the partial quantities the library reduces with NCCL
(pasd_solver.cu, launch_iteration_marked): A_3 partials, Gram_1/Gram_2
partials, Wt_1/Wt_2 partials, zero-padded own rows of Wt_3, ||G||^2 (SUM)
and residual maxima (MAX).  After the all-reduces every rank must hold the
unsharded values (computed here with numpy from the full tensor)."""
import os
import socket

import numpy as np
import pytest

from paper_1712_09999_b200.sharding import slab_bounds


def unfold(t, mode):
    return np.reshape(np.moveaxis(t, mode, 0), (t.shape[mode], -1), order="F")


def quantities(G, Gn, U, A_prev):
    """Per-mode pass-1 / pass-2 reduction quantities of one PASD iteration."""
    out = {}
    for n in range(3):
        Gu = unfold(G, n)
        out[f"A{n}"] = U[n].T @ Gu                      # A_n = U_n^T G_(n)
        out[f"gram{n}"] = out[f"A{n}"] @ out[f"A{n}"].T
        out[f"W{n}"] = unfold(Gn, n) @ A_prev[n].T      # Wt_n = G^{next}_(n) A_n^T
        out[f"g2{n}"] = float(np.sum(Gn * Gn))
    return out


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(0)
        I1, I2, I3, R = 6, 5, 7, 3
        G = rng.standard_normal((I1, I2, I3))
        Gn = rng.standard_normal((I1, I2, I3))
        U = [np.linalg.qr(rng.standard_normal((I, R)))[0] for I in (I1, I2, I3)]
        full = quantities(G, Gn, U, [rng.standard_normal((R, G.size // I)) for I in (I1, I2, I3)])
        rng = np.random.default_rng(0)  # same draws for A_prev on every rank
        rng.standard_normal((I1, I2, I3)); rng.standard_normal((I1, I2, I3))
        [np.linalg.qr(rng.standard_normal((I, R)))[0] for I in (I1, I2, I3)]
        A_prev = [rng.standard_normal((R, G.size // I)) for I in (I1, I2, I3)]
        b, e = slab_bounds(I3, world, rank)
        Gs, Gns = G[:, :, b:e], Gn[:, :, b:e]

        def allreduce(a, op=dist.ReduceOp.SUM):
            t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
            dist.all_reduce(t, op=op)
            return t.numpy()

        errs = {}
        # mode 3: partial over the local i3 range, rows of U_3 restricted to the slab
        A3 = allreduce(U[2][b:e].T @ unfold(Gs, 2))
        errs["A2"] = np.abs(A3 - full["A2"]).max()
        errs["gram2"] = np.abs(A3 @ A3.T - full["gram2"]).max()  # replicated from the reduced A_3
        # modes 1, 2: A_n columns are local (complete); Grams are partial
        for n in (0, 1):
            An = U[n].T @ unfold(Gs, n)
            cols = full[f"A{n}"].reshape(U[n].shape[1], -1, order="F")
            ref_cols = full[f"A{n}"][:, [c for c in range(full[f"A{n}"].shape[1]) if b <= (c // (G.size // I3 // G.shape[n]))
                                         and (c // (G.size // I3 // G.shape[n])) < e]]
            errs[f"A{n}"] = np.abs(An - ref_cols).max()
            errs[f"gram{n}"] = np.abs(allreduce(An @ An.T) - full[f"gram{n}"]).max()
            # Wt_n partial: local columns of G^{next} against the matching columns of A_n^{prev}
            Ap = A_prev[n]
            sel = [c for c in range(Ap.shape[1]) if b <= c // (G.size // I3 // G.shape[n]) < e]
            errs[f"W{n}"] = np.abs(allreduce(unfold(Gns, n) @ Ap[:, sel].T) - full[f"W{n}"]).max()
        # mode 3 Wt: own rows complete, zero-padded then summed (acts as an allgather)
        W3 = np.zeros_like(full["W2"])
        W3[b:e] = unfold(Gns, 2) @ A_prev[2].T
        errs["W2"] = np.abs(allreduce(W3) - full["W2"]).max()
        g2 = allreduce(np.array([np.sum(Gns * Gns)]))[0]
        errs["g2"] = abs(g2 - full["g20"])
        rmax = allreduce(np.array([np.abs(Gs).max()]), op=dist.ReduceOp.MAX)[0]
        errs["rmax"] = abs(rmax - np.abs(G).max())
        q.put((rank, {k: float(v) for k, v in errs.items()}, (b, e)))
    finally:
        dist.destroy_process_group()


def test_slab_bounds_partition():
    for n in (1, 7, 400, 1000, 1024):
        for world in (1, 2, 3, 4, 8):
            if n < world:
                with pytest.raises(ValueError):
                    slab_bounds(n, world, 0)
                continue
            parts = [slab_bounds(n, world, r) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))
            assert max(e - b for b, e in parts) - min(e - b for b, e in parts) <= 1


def test_two_rank_reductions_match_unsharded():
    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    [p.start() for p in procs]
    res = [q.get(timeout=120) for _ in procs]
    [p.join(timeout=60) for p in procs]
    assert sorted(r for r, _, _ in res) == [0, 1]
    slabs = sorted(s for _, _, s in res)
    assert slabs[0][0] == 0 and slabs[0][1] == slabs[1][0] and slabs[1][1] == 7
    for _, errs, _ in res:
        for k, v in errs.items():
            assert v <= 1e-12, (k, v)


def test_loopback_group_rejects_bad_sizes():
    """pasd_b200_loopback_create validates its size before any device work."""
    import paper_1712_09999_b200  # noqa: F401
    from paper_1712_09999_b200.api import ArgumentError
    from paper_1712_09999_b200.sharding import LoopbackGroup

    for n in (0, 9):
        with pytest.raises(ArgumentError, match="loopback groups hold 1..8 ranks"):
            LoopbackGroup(n)
    g = LoopbackGroup(3)
    assert g.handle
    g.close()
