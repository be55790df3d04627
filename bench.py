#!/usr/bin/env python
"""PASD ADMM iteration throughput on B200 (BASELINE.json metric).

One "step" = one PASD ADMM iteration (Algorithm 1, proj/src/pasd.cpp:168-244)
over the resident state of the configured workload.  Default workload: C5,
1000^3 fp64, Tucker/solver rank 50, 10% corruption (BASELINE configs[4], the
largest config of the 1/2/4/8-GPU sweep).

  python bench.py [--gpus N --steps K --warmup W --config c5 --impl ours|reference]

Prints ONE JSON line (rank 0).  `value` = iterations/s with the state resident
in HBM (CUDA events on the solver's stream, max over ranks); `e2e` = the same
metric through the C-ABI drop-in pasd_b200_recover with host buffers (H2D of
T, the loop, finalisation, D2H of X and E inside the timed region);
`roofline` = the dominant kernel's achieved throughput from CUDA events around
each kernel; `cpu_baseline` = the reference restatement (oracle/) on the host.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=os.environ.get("PASD_BENCH_CONFIG", "c5"))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--dtype", default="f64", choices=["f64", "f32"],
                    help="f32: the optional fp32 mode (float32 element storage, fp64 arithmetic)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--profile-iters", type=int, default=3)
    ap.add_argument("--steady-after", type=int, default=140,
                    help="N=1: also time 10 iterations after this many (the full-rank phase), 0 = skip")
    return ap.parse_args()


def load_peaks():
    peaks = {"hbm_gbs": 6538.9, "source_hbm": "fallback"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        peaks["hbm_gbs"] = float(d["hbm_gbs"])
        peaks["source_hbm"] = "measured (MEASURED_PEAKS.json)"
    except Exception:
        pass
    # FP64 tensor pipe: measured on this pool with tools/fp64_peak.sh (profiles/r02_fp64_peak.txt):
    # DMMA m16n8k4 37.0 TF/s burst, 36.9 sustained over 5 s at 1965 MHz (no throttle reason);
    # DFMA 34.1.  The burst figure is the (larger, so stricter) denominator.
    peaks["fp64_tflops"] = 37.0
    peaks["source_fp64"] = "measured DMMA burst 37.0 (36.9 sustained), profiles/r02_fp64_peak.txt"
    return peaks


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            time.sleep(0.25)
        except Exception:
            self.proc = None

    def stop(self):
        out = {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        if self.proc is None:
            return out
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 7:
                    continue
                try:
                    sm.append(float(parts[0]))
                    mx.append(float(parts[1]))
                except ValueError:
                    continue
                for nm, v in zip(names, parts[3:7]):
                    if v.lower().startswith("active"):
                        reasons.add(nm)
        os.unlink(self.path)
        if sm:
            out = {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                   "samples": len(sm)}
        return out


def cpu_sample_dims(w):
    """Bounded CPU sample of workload w: the full config up to 7e7 elements
    (C1-C4), else the same-shaped tensor scaled to ~6.4e7 elements with the
    same Tucker and solver ranks (C5: 400^3, R = 50; ~8 s per CPU iteration).
    Calibrated against a measured full-size C5 run (profiles/r02_cpu_fullsize_c5.json:
    the 400^3 sample predicts 117 s/iter, the full run took 91 s/iter; a
    1000x1000x50 slab predicted 216 s/iter)."""
    if w.size <= 70_000_000:
        return tuple(w.dims), tuple(w.tucker), tuple(w.ranks)
    f = (64_000_000 / w.size) ** (1.0 / len(w.dims))
    dims = tuple(max(r, int(round(d * f))) for d, r in zip(w.dims, w.ranks))
    return dims, tuple(min(t, d) for t, d in zip(w.tucker, dims)), tuple(min(r, d) for r, d in zip(w.ranks, dims))


def full_size_cpu(w):
    """The committed full-size CPU measurement of this workload, if any."""
    path = os.path.join(ROOT, "profiles", "r02_cpu_fullsize_c5.json")
    if w.name != "c5_1000cube_r50" or not os.path.exists(path):
        return None
    with open(path) as f:
        d = json.load(f)
    return {"value": d["iter_per_s"], "s_per_iter": d["per_iteration_s"], "threads": d["threads"],
            "iters": d["iters"], "source": "profiles/r02_cpu_fullsize_c5.json (tools/cpu_fullsize.py on a GPU-box host)"}


def cpu_baseline(w, threads: int, iters: int = 3, sample=None):
    """Time the oracle (reference restatement) per iteration on a bounded sample.

    Per-iteration time = median gap between observer callbacks after the first
    iteration (reference timing pattern: warm-up excluded, bench.cpp:274-286)."""
    import oracle
    from paper_1712_09999_b200 import _abi
    from paper_1712_09999_b200.api import PasdConfig

    dims, tucker, ranks = sample if sample is not None else cpu_sample_dims(w)
    L0 = oracle.gen_tucker(dims, tucker, seed=0, kind=1 if w.kind == "nonneg" else 0)
    T = oracle.corrupt_sparse(L0, w.rho, seed=0, mode=0 if w.mode == "add" else 1, lo=w.noise[0], hi=w.noise[1])
    total = int(np.prod(dims))
    n = float(len(dims))
    lam = [math.sqrt(float(max(d, total // d))) / n for d in dims]
    stamps = []
    cb = _abi.PasdObserverFn(lambda v, u: stamps.append(time.perf_counter()))
    cfg = PasdConfig(lambdas=lam, ranks=list(ranks), maxiter=iters, eps=w.eps)
    oracle.pasd_recover(T, cfg, observer=cb, fixed_iters=True, threads=threads, want_z=False, want_y=False)
    gaps = [b - a for a, b in zip(stamps[:-1], stamps[1:])]
    per_iter = statistics.median(gaps)
    elem_rate = total / per_iter
    extrapolated = total != w.size
    return {
        "value": elem_rate / w.size,
        "unit": "iter/s",
        "cores": threads,
        "kind": "port",
        "extrapolated": extrapolated,
        "sample_dims": list(dims),
        "elem_iters_per_s": elem_rate,
        "full_size_measured": full_size_cpu(w) if extrapolated else None,
        "sample": f"oracle/ (C++ restatement of proj/src/pasd.cpp, OpenBLAS dgesdd/dgemm) on dims {list(dims)} "
                  f"ranks {list(ranks)}, {iters} fixed iterations, per-iteration time = median gap between "
                  f"iterations 2..{iters}; value = sample elem*iters/s / S({w.name}) = {per_iter:.3f} s/iter "
                  f"on {total} elements",
    }


def generate_input(w):
    """The workload's observed tensor from the reference generator on the device
    (paper_1712_09999_b200/synth.py: synth.cpp:71-121 with the reference's RNG
    streams, seed 0), as a CUDA tensor of shape reversed(dims)."""
    from paper_1712_09999_b200 import synth

    T, _, _ = synth.generate(synth.workload_spec(w, seed=0), out="torch")
    return T


def e2e_recover(w, T_dev, steps: int, fp32: bool = False):
    """Whole-solve throughput through the C-ABI drop-in with host buffers."""
    import torch
    from paper_1712_09999_b200 import _abi, solver as S
    from paper_1712_09999_b200.api import PasdConfig, build_options, raise_for_status

    total = w.size
    Th = torch.empty(total, dtype=torch.float64, pin_memory=True)
    Th.copy_(T_dev.view(-1))
    xh = torch.empty(total, dtype=torch.float64, pin_memory=True)
    eh = torch.empty(total, dtype=torch.float64, pin_memory=True)
    cfg = PasdConfig(lambdas=w.lambdas(), ranks=list(w.ranks), eps=w.eps, maxiter=steps)
    flags = _abi.PASD_FLAG_FIXED_ITERS | _abi.PASD_FLAG_REUSE_SOLVER | (_abi.PASD_FLAG_FP32 if fp32 else 0)
    opt, keep = build_options(list(w.dims), cfg, flags=flags, poll_every=steps)
    out = _abi.PasdOutputs()
    out.x = C.cast(C.c_void_p(xh.data_ptr()), _abi.c_double_p)
    out.e = C.cast(C.c_void_p(eh.data_ptr()), _abi.c_double_p)
    hist = np.zeros(steps)
    fres = np.zeros(len(w.dims))
    out.residual_history = _abi.dptr(hist)
    out.final_residuals = _abi.dptr(fres)
    err = C.create_string_buffer(1024)
    tptr = C.cast(C.c_void_p(Th.data_ptr()), _abi.c_double_p)
    # one cold call (solver allocation + graph capture, kept by the opt-in
    # PASD_FLAG_REUSE_SOLVER), reported separately, then the median of timed calls
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rc = S.lib().pasd_b200_recover(tptr, C.byref(opt), C.byref(out), _abi.PasdObserverFn(), None, err, len(err))
    cold = time.perf_counter() - t0
    raise_for_status(rc, err)
    times = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rc = S.lib().pasd_b200_recover(tptr, C.byref(opt), C.byref(out), _abi.PasdObserverFn(), None, err, len(err))
        t1 = time.perf_counter()
        raise_for_status(rc, err)
        times.append(t1 - t0)
    S.lib().pasd_b200_release_cache()
    sec = float(np.median(times))
    return {
        "value": steps / sec,
        "unit": "iter/s",
        "h2d_bytes_per_step": 8 * total / steps,
        "d2h_bytes_per_step": (16 * total + 8 * steps) / steps,
        "seconds": sec,
        "iters": int(out.iters),
        "cold_call_seconds": cold,
        "cold_value": steps / cold,
        "note": "pasd_b200_recover (C-ABI, PASD_FLAG_REUSE_SOLVER) on pinned host buffers, median of 3 calls "
                f"after one cold call (allocation + graph capture, reported as cold_*): H2D of T, {steps} fixed "
                "iterations, finalisation, D2H of X and E; bytes amortised per iteration",
    }


def e2e_sharded(w, steps, shard, dist):
    """Per-rank end-to-end run from pinned host slabs (H2D of the slab, the
    loop with its NCCL exchanges, finalisation, D2H of the slab's X and E);
    wall time max over ranks."""
    import torch
    import paper_1712_09999_b200 as pb
    from paper_1712_09999_b200.api import PasdConfig
    from paper_1712_09999_b200.sharding import Shard, nccl_unique_id

    b, e = shard.struct.slab_begin, shard.struct.slab_end
    rank = shard.struct.rank
    uid = [nccl_unique_id() if rank == 0 else None]  # a unique id serves one communicator
    dist.broadcast_object_list(uid, src=0)
    shard = Shard(rank, shard.struct.nranks, (b, e), uid[0])
    T = generate_input(w)
    Th = torch.empty(T[b:e].numel(), dtype=torch.float64, pin_memory=True)
    Th.copy_(T[b:e].reshape(-1))
    del T
    torch.cuda.empty_cache()
    cfg = PasdConfig(lambdas=w.lambdas(), ranks=list(w.ranks), eps=w.eps, maxiter=steps)
    xh = torch.empty_like(Th, pin_memory=True)
    eh = torch.empty_like(Th, pin_memory=True)
    # the solver (buffers, graph, NCCL communicator) is built once, like the one-shot
    # entry point's cached solver; each timed solve resets it, uploads the slab,
    # iterates and downloads X and E into pinned buffers
    sol = pb.Solver(w.dims, cfg, fixed_iters=True, poll_every=steps, shard=shard)
    times = []
    for rep in range(4):
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sol.reset()
        sol.load(Th.numpy().reshape(list(w.dims[:-1]) + [e - b], order="F"))
        sol.run(steps)
        sol.finalize(want_x=True, want_e=True, out_x=xh.numpy(), out_e=eh.numpy())
        if rep:
            times.append(time.perf_counter() - t0)
    sol.close()
    sec = float(np.median(times))
    t = torch.tensor([sec], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    sec = float(t.item())
    slab_elems = Th.numel()
    return {"value": steps / sec, "unit": "iter/s", "h2d_bytes_per_step": 8 * slab_elems / steps,
            "d2h_bytes_per_step": 16 * slab_elems / steps, "seconds": sec,
            "note": "per rank, median of 3 solves after a warm-up: reset + H2D of its pinned slab + fixed "
                    "iterations with the NCCL exchanges + finalise + D2H of its X/E slab into pinned buffers; "
                    "max over ranks; bytes per rank amortised per iteration"}


def roofline_from_profile(prof, peaks, iters, workload):
    # Dominant kernel = largest share of device time.
    name = max(prof, key=lambda k: prof[k]["ms"])
    p = prof[name]
    per_launch_ms = p["ms"] / max(1, p["launches"])
    launches_per_iter = p["launches"] / max(1, iters)
    bytes_per_launch = p["bytes"] / max(1.0, launches_per_iter)
    flops_per_launch = p["flops"] / max(1.0, launches_per_iter)
    gbs = bytes_per_launch / (per_launch_ms * 1e-3) / 1e9
    tfs = flops_per_launch / (per_launch_ms * 1e-3) / 1e12
    hbm_frac = gbs / peaks["hbm_gbs"]
    fp_frac = tfs / peaks["fp64_tflops"]
    intensity = flops_per_launch / max(1.0, bytes_per_launch)
    ridge = peaks["fp64_tflops"] * 1e12 / (peaks["hbm_gbs"] * 1e9)
    traffic = None  # DRAM bytes per launch from an ncu --set full capture of THIS workload, else null
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as f:
                traffic = json.load(f).get(workload, {}).get(name)
        except Exception:
            traffic = None
    total_ms = sum(v["ms"] for v in prof.values())
    shares = {k: round(v["ms"] / total_ms, 4) for k, v in prof.items()}
    if intensity > ridge:
        # FP64 tensor-core (DMMA) bound: "tensor" in the contract's vocabulary
        r = {"bound": "tensor", "pipe": "fp64 DMMA", "achieved": round(tfs, 3), "peak": peaks["fp64_tflops"],
             "unit": "TFLOP/s",
             "frac": round(fp_frac, 4), "peak_source": peaks["source_fp64"]}
    else:
        r = {"bound": "hbm", "achieved": round(gbs, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
             "frac": round(hbm_frac, 4), "peak_source": peaks["source_hbm"]}
    r.update({"kernel": name, "traffic": traffic, "algorithmic_bytes_per_launch": bytes_per_launch,
              "algorithmic_flops_per_launch": flops_per_launch, "ms_per_launch": round(per_launch_ms, 4),
              "hbm_gbs": round(gbs, 1), "fp64_tflops": round(tfs, 3), "kernel_time_shares": shares})
    # Every kernel class with algorithmic work: the same achieved / bound computation.
    per = {}
    for k, v in prof.items():
        if v["ms"] <= 0 or (v["bytes"] <= 0 and v["flops"] <= 0):
            continue
        lpi = v["launches"] / max(1, iters)
        ms_l = v["ms"] / max(1, v["launches"])
        b_l, f_l = v["bytes"] / max(1.0, lpi), v["flops"] / max(1.0, lpi)
        g = b_l / (ms_l * 1e-3) / 1e9
        t = f_l / (ms_l * 1e-3) / 1e12
        fp = f_l / max(1.0, b_l) > ridge
        per[k] = {"ms_per_launch": round(ms_l, 4), "hbm_gbs": round(g, 1), "fp64_tflops": round(t, 3),
                  "bound": "tensor" if fp else "hbm",
                  "frac": round(t / peaks["fp64_tflops"] if fp else g / peaks["hbm_gbs"], 4)}
    r["per_kernel"] = per
    return r


def main():
    args = parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    from paper_1712_09999_b200.workloads import WORKLOADS

    w = WORKLOADS[args.config]

    if args.impl == "reference":
        if rank != 0:
            return 0
        # The reference runs single-threaded: Eigen without OpenMP and OpenBLAS
        # pinned to one thread (linops.cpp:17-23), so its stock setting -- the
        # line's value -- is 1 thread; the restatement on every host thread is
        # reported beside it.
        cb = cpu_baseline(w, 1, iters=max(3, min(args.steps, 6)))
        threads = os.cpu_count() or 1
        try:
            cb_all = cpu_baseline(w, threads, iters=max(3, min(args.steps, 6)))
            all_threads = {k: cb_all[k] for k in ("value", "unit", "cores", "extrapolated", "sample")}
        except Exception as exc:  # reported, never fatal
            all_threads = {"error": str(exc)}
        line = {
            "impl": "reference", "metric": "PASD ADMM iters/s", "value": cb["value"], "unit": "iter/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": w.name, "dims": list(w.dims), "ranks": list(w.ranks)},
            "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "extrapolated", "sample_dims",
                                                 "full_size_measured", "sample")},
            "e2e": {"value": cb["value"], "unit": "iter/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "elem_iters_per_s": cb["elem_iters_per_s"],
            "all_threads": all_threads,
        }
        print(json.dumps(line), flush=True)
        return 0

    import torch
    import paper_1712_09999_b200 as pb
    from paper_1712_09999_b200.api import PasdConfig
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local_rank)
    dist = None
    shard = None
    if world > 1 or os.environ.get("PASD_BENCH_FORCE_SHARD") == "1":  # the latter: exercise the path on 1 GPU
        import torch.distributed as dist
        from paper_1712_09999_b200.sharding import Shard, nccl_unique_id, slab_bounds

        for k, v in (("RANK", "0"), ("WORLD_SIZE", "1"), ("MASTER_ADDR", "127.0.0.1"), ("MASTER_PORT", "29517")):
            os.environ.setdefault(k, v)  # PASD_BENCH_FORCE_SHARD=1 without torchrun: a one-rank group
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        uid = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        slab = slab_bounds(w.dims[-1], world, rank)
        shard = Shard(rank, world, slab, uid[0])
    peaks = load_peaks()
    K, W = args.steps, max(3, args.warmup)
    T = generate_input(w)  # identical on every rank (same seed); rank keeps its slab
    T_loc = T[shard.struct.slab_begin:shard.struct.slab_end].contiguous() if shard else T
    if shard:
        del T
    steady_after = args.steady_after if world == 1 else 0
    steady_start = max(steady_after, W + K + args.profile_iters) if steady_after else 0
    cfg = PasdConfig(lambdas=w.lambdas(), ranks=list(w.ranks), eps=w.eps,
                     maxiter=max(W + K + args.profile_iters + 1, steady_start + 13))
    f32 = args.dtype == "f32"
    sol = pb.Solver(w.dims, cfg, fixed_iters=True, poll_every=K, shard=shard, fp32=f32)
    sol.load(T_loc.data_ptr(), t_is_device=True)
    sol.run(W)
    stream = torch.cuda.ExternalStream(sol.stream)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    clk = ClockSampler(local_rank)
    clk.start()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ev0.record(stream)
    done, _ = sol.run(K)
    ev1.record(stream)
    ev1.synchronize()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clocks = clk.stop()
    ms = ev0.elapsed_time(ev1)
    if dist:  # device time, max over ranks
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    launches = sol.launches
    prof = sol.profile(args.profile_iters)
    steady = None
    if steady_after:
        # The fixed-count BASELINE runs of C3-C5 stay in the V_n = 0 phase; this
        # times the same solver later, with every V_n at full rank (non-degenerate
        # Procrustes, longer Jacobi solves), as a representative steady state.
        done_iters = W + K + args.profile_iters
        if steady_after > done_iters:
            sol.run(steady_after - done_iters)
        keep, prank = sol.ranks()
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s0.record(stream)
        sol.run(10)
        s1.record(stream)
        s1.synchronize()
        sms = s0.elapsed_time(s1) / 10
        sprof = sol.profile(2)
        steady = {"after_iters": max(steady_after, done_iters), "ms_per_step": round(sms, 4),
                  "value": round(1e3 / sms, 4), "unit": "iter/s", "svt_keep": keep, "polar_rank": prank,
                  "kernel_ms_per_iter": {k: round(v["ms"] / 2, 4) for k, v in sprof.items() if v["ms"] > 0}}
    sol.close()
    del sol
    value = K / (ms * 1e-3)
    roof = roofline_from_profile(prof, peaks, args.profile_iters, w.name)
    # Whole-iteration roofline against the canonical fused-schedule work.
    S = w.size
    N = len(w.dims)
    RJ = sum(r * (S // d) for r, d in zip(w.ranks, w.dims))
    es = 4.0 if f32 else 8.0  # element-tensor bytes (fp32 mode: float32 storage)
    B_iter = (es * (3 * N + 4) * S + 8.0 * 2 * RJ) / world
    F_iter = 6.0 * S * sum(w.ranks) / world
    t_roof = max(B_iter / (peaks["hbm_gbs"] * 1e9), F_iter / (peaks["fp64_tflops"] * 1e12))
    iteration_roofline = {"B_iter_per_gpu": B_iter, "F_iter_per_gpu": F_iter, "t_roof_ms": t_roof * 1e3,
                          "t_measured_ms": ms / K, "frac": round(t_roof / (ms / K * 1e-3), 4)}
    line = {
        "metric": "PASD ADMM iters/s", "value": round(value, 4), "unit": "iter/s", "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": round(ms / K, 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32-storage/f64-arith" if f32 else "f64",
        "data": "synthetic",
        "config": {"workload": w.name, "dims": list(w.dims), "ranks": list(w.ranks), "rho": w.rho,
                   "noise": list(w.noise), "iters_fixed": True,
                   "input": "reference generator (synth.cpp:71-121, rng.hpp streams, seed 0) on the device", "l2": (f"inputs larger than L2 (T, E x2, D, Y x3: 7 x {S * es / 1e9:.3g} GB resident, re-streamed "
                          "every iteration)")
                   if 7 * S * es > 126e6 else
                   f"working set 7 x {S * es / 1e6:.3g} MB fits the 126 MB L2 (an iterative solve re-reads it every step)"},
        "elem_iters_per_s": value * S,
        "gpu_launches": int(launches),
        "clocks": clocks,
        "roofline": roof,
        "iteration_roofline": iteration_roofline,
    }
    if steady:
        line["steady_state"] = steady
    del T_loc
    torch.cuda.empty_cache()
    if not args.no_e2e and shard is None:
        Tg = generate_input(w)
        line["e2e"] = e2e_recover(w, Tg, K, fp32=f32)
        del Tg
        torch.cuda.empty_cache()
    elif not args.no_e2e:
        line["e2e"] = e2e_sharded(w, K, shard, dist)
    if dist:
        line["config"]["parallelism"] = f"slab{world} (mode-3 slabs, NCCL all-reduce of A_3/Gram/Wt partials)"
    if rank != 0:
        dist.destroy_process_group()
        return 0
    if not args.no_cpu_baseline and shard is None:
        try:
            line["cpu_baseline"] = cpu_baseline(w, threads=1)
        except Exception as exc:  # reported, never fatal
            line["cpu_baseline"] = {"error": str(exc)}
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
