#!/usr/bin/env python
"""Benchmark of the B200 M-step solver (BASELINE.json metric: solver
voxel-iterations/s at 512^3, time-to-tolerance, % HBM roofline per iteration).

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]

A step = one m_step solve of --iters ISTA iterations (the reference's default
semantics: lipschitz step, per-inner reweighting, monotone audit every
iteration) over the resident 512^3 synthetic problem (synth.py).
value = N^3 * iters * steps / device time (CUDA events), inputs resident in HBM.
e2e   = the same through the C ABI call cm_m_step with pinned HOST buffers
        (full-grid fp64 accumulator + volume H2D, result D2H inside the timing).
Under torchrun (--mode auto) the same 512^3 solve is z-slab decomposed over the
ranks (NCCL all-to-all transposes + one-plane halos; strong
scaling); --mode replicas runs independent replicas instead (config 5).
Every line also carries "big": the 1024^3 z-slab solve (device-rendered timing
problem) on the same ranks, so the 1024^3 scaling can be
read across the N=1,2,4,8 lines.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

HBM_FALLBACK_GBS = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--iters", type=int, default=100, help="ISTA iterations per step")
    ap.add_argument("--precision", type=int, default=32)
    ap.add_argument("--cpu-n", type=int, default=512, help="CPU reference sample side")
    ap.add_argument("--cpu-iters", type=int, default=1, help="iterations per reference call")
    ap.add_argument("--cpu-threads", type=int, default=1,
                    help="FFT threads under the reference (1: the reference as written)")
    ap.add_argument("--ref-all-cores", type=int, default=0,
                    help="reference arm: also time a labelled all-cores-FFT variant")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--ttt", type=int, default=1, help="measure time-to-tolerance (0/1)")
    ap.add_argument("--ttt-max-iters", type=int, default=6000)
    ap.add_argument("--mode", default="auto", choices=["auto", "single", "slab", "replicas"],
                    help="auto: one context at N=1, z-slab decomposition under torchrun")
    ap.add_argument("--big-n", type=int, default=1024,
                    help="side of the device-rendered z-slab scaling run (0: skip)")
    ap.add_argument("--big-iters", type=int, default=20)
    ap.add_argument("--em", type=int, default=1, help="time the EM-block extras (V, FSC)")
    ap.add_argument("--prec64", type=int, default=1, help="also time the fp64 parity mode")
    ap.add_argument("--configs", type=int, default=1,
                    help="also time BASELINE configs 1, 2 and one config-5 replica (0/1)")
    return ap.parse_args()


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d.get("hbm_gbs", HBM_FALLBACK_GBS)), "measured"
    return HBM_FALLBACK_GBS, "fallback"


# ---------------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [q.strip() for q in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------------
def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def allreduce_max(v: float, world: int) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist

    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def load_problem(n: int, rank: int, world: int):
    """Rank 0 generates (synth.py); other ranks memory-map the same bytes."""
    from paper_1905_13408_b200 import synth

    if world == 1:
        return synth.synthetic_problem(n)
    cache = Path(f"/tmp/cm_bench_problem_{n}")
    if rank == 0:
        p = synth.synthetic_problem(n)
        cache.mkdir(exist_ok=True)
        for k in ("truth", "weight", "numerator", "x0"):
            np.save(cache / f"{k}.npy", getattr(p, k))
        (cache / "meta.json").write_text(json.dumps({"eps": p.eps, "eps_prime": p.eps_prime}))
    barrier(world)
    if rank != 0:
        meta = json.loads((cache / "meta.json").read_text())
        arr = {k: np.load(cache / f"{k}.npy") for k in ("truth", "weight", "numerator", "x0")}
        p = synth.Problem(n, arr["truth"], arr["weight"], arr["numerator"], arr["x0"],
                          meta["eps"], meta["eps_prime"])
    return p


# ---- algorithmic bytes per launch ------------------------------
KERNELS = ("z_pass", "y_inverse", "x_c2r", "stencil", "finalize", "x_r2c", "y_forward")


def iteration_bytes_s8d(n: int, rsize: int = 4, audit_prev: bool = True) -> float:
    """SURVEY §8(d)'s ALGORITHMIC bytes of one ISTA iteration: the canonical fused
    4-kernel schedule (K1 = x C2R + sweep + x R2C, K2 y forward, K3 z pass with
    the W / Yh multiply, K4 y inverse), B_iter = 76 H + 12 L (fp32; H =
    n^2 (n/2 + 1), L = n^3), + 4 L when the lagged audit reads x_{i-1}. Scaled by
    rsize / 4 for the fp64 mode."""
    H = n * n * (n // 2 + 1)
    L = n ** 3
    return (76 * H + 12 * L + (4 * L if audit_prev else 0)) * rsize / 4


def kernel_bytes(n: int, rsize: int, audit_prev: bool):
    """IMPLEMENTATION bytes per launch of each per-iteration kernel of this
    build's schedule (the x transforms run as separate kernels: g is written and
    read back and x_{i+1} re-read, 12 L more than SURVEY §8(d)'s fused K1, see
    iteration_bytes_s8d). Packed half spectrum: H' = n^2 * n/2 complex (+ the
    n^2 Nyquist planes of W and Yh); real volumes: L = n^3. Per kernel these are
    what the kernel must move; roofline.iteration.frac is quoted against the
    §8(d) algorithmic total."""
    L = n ** 3
    c = 2 * rsize
    Hp = n * n * (n // 2)
    nyq = n * n
    return {
        "z_pass": Hp * c * 2 + (Hp + nyq) * rsize + (Hp + nyq) * c,  # S r/w, W, Yh
        "y_inverse": Hp * c * 2,
        "x_c2r": Hp * c + L * rsize,                                  # S in, g out
        "stencil": L * rsize * (5 if audit_prev else 4),              # g, x, anchor, (x_prev) in; x out
        "finalize": 0,
        "x_r2c": L * rsize + Hp * c,
        "y_forward": Hp * c * 2,
    }


def ncu_traffic(n: int):
    p = ROOT / "profiles" / "ncu_traffic.json"
    if not p.exists():
        return {}
    d = json.loads(p.read_text())
    return d.get(str(n), {})


# ---------------------------------------------------------------------------------
_CPU_PROBLEM = {}


def reference_sample(args, threads: int, prefer_reference=True, problem=None) -> dict:
    """One m_step call of the reference solver on the host (BASELINE config 3's
    workload: args.cpu_n^3 synthetic blob phantom, lipschitz step with the
    monotone audit, per_inner reweighting — the same RegConfig semantics as the
    GPU arm), timed with std::chrono around m_step inside oracle/_ref (inputs
    already in the reference's host types). The FFT under it is the FFTW3-API
    shim over oneMKL DFTI with `threads` threads (the reference itself is
    single-threaded: threads=1 is the unmodified baseline)."""
    sys.path.insert(0, str(ROOT / "tests"))
    from oracle_lib import REF_DIR, Oracle, Reference
    from paper_1905_13408_b200 import synth

    kind = "reference" if (prefer_reference and (REF_DIR / "libcryomap_ref.so").exists()) else "port"
    os.environ["CM_REF_FFT_THREADS"] = str(threads)
    lib = Reference() if kind == "reference" else Oracle()
    n = args.cpu_n
    if _CPU_PROBLEM.get("n") != n:
        _CPU_PROBLEM.clear()
        p = problem if (problem is not None and problem.n == n) else synth.synthetic_problem(n)
        rc, sy, sn = lib.scale_data(p.weight, p.numerator)
        rc, cfg = lib.derive_config(sy, sn, p.eps, p.eps_prime)
        _CPU_PROBLEM.update(n=n, p=p, cfg=cfg)
    p, cfg = _CPU_PROBLEM["p"], _CPU_PROBLEM["cfg"]
    cfg.inner_iters = args.cpu_iters
    t0 = time.perf_counter()
    rc, x, tr = lib.m_step(p.weight, p.numerator, p.x0, p.x0, cfg, trace=False)
    wall = time.perf_counter() - t0
    assert rc == 0, rc
    secs = lib.last_seconds if kind == "reference" else wall
    fft = ("FFTW3-API shim over oneMKL DFTI (libtorch_cpu.so), "
           f"{threads} FFT thread(s)") if kind == "reference" else "oracle/fftc.c"
    src = ("unmodified reference sources (oracle/_ref/libcryomap_ref.so)" if kind == "reference"
           else "oracle C restatement")
    return {
        "value": n ** 3 * args.cpu_iters / secs, "unit": "voxel-iterations/s", "cores": threads,
        "kind": kind, "seconds": secs, "voxel_iterations": n ** 3 * args.cpu_iters,
        "sample": f"{src} + {fft}; one m_step call on the {n}^3 synthetic blob phantom "
                  f"(BASELINE config 3 inputs), {args.cpu_iters} iteration(s), lipschitz step "
                  f"with audit, per_inner reweighting; m_step wall {secs:.2f} s (std::chrono "
                  f"around the call, inputs resident in host memory); host nproc={os.cpu_count()}",
    }


def cpu_baseline(args, problem=None):
    """The reference on ONE host core (m_step and its FFTW calls are
    single-threaded as written), bounded sample: one call of one
    iteration (about 95 s at 512^3: the reference's non-FFT passes over its
    fp64 full-grid temporaries dominate, not its FFTs)."""
    cb = reference_sample(args, 1, problem=problem)
    cb.pop("seconds", None)
    cb.pop("voxel_iterations", None)
    return cb


def run_reference(args):
    """--impl reference: the unmodified reference m_step on the host cores, the
    same workload (512^3, reference semantics) as the GPU arm; rank 0 only.
    Each step = one m_step call of args.cpu_iters iteration(s) (about 95 s at
    512^3 on one core), so K and W are capped to keep the run to a few minutes:
    one step and no warm-up at 512^3 (the call allocates and faults in its own
    temporaries every time, warm or not)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    big = args.cpu_n >= 512
    steps = 1 if big else max(1, min(args.steps, 2))
    warm = 0 if big else min(args.warmup, 1)
    secs, work = 0.0, 0
    cb = None
    for s in range(warm + steps):
        cb = reference_sample(args, args.cpu_threads)
        if s >= warm:
            secs += cb["seconds"]
            work += cb["voxel_iterations"]
    v = work / secs
    secondary = None
    if args.ref_all_cores and args.cpu_threads == 1 and (os.cpu_count() or 1) > 1:
        # labelled modified baseline: the same call with the FFT shim on all cores
        mt = reference_sample(args, os.cpu_count())
        secondary = {"value": mt["value"], "unit": mt["unit"], "cores": mt["cores"],
                     "note": "MODIFIED baseline: reference m_step with its FFTs multi-threaded "
                             "(the reference never calls fftw_init_threads)",
                     "sample": mt["sample"]}
    line = {
        "metric": "solver voxel-iterations/s (512^3 m_step, ISTA, per-inner reweighting, audit)",
        "value": v, "unit": "voxel-iterations/s", "impl": "reference", "n_gpus": args.gpus,
        "steps": steps, "warmup": warm, "ms_per_step": 1e3 * secs / steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"m_step {args.cpu_n}^3 synthetic blob phantom (BASELINE config 3),"
                               f" {args.cpu_iters} ISTA iteration(s) per step",
                   "side": args.cpu_n, "iters_per_step": args.cpu_iters, "step_rule": "lipschitz",
                   "refresh": "per_inner", "audit": True},
        "cpu_baseline": {k: cb[k] for k in ("kind", "cores", "sample")} | {"value": v,
                                                                           "unit": cb["unit"]},
        "e2e": {"value": v, "unit": "voxel-iterations/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "secondary_all_cores": secondary,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------
def broadcast_nccl_id(world, rank):
    if world == 1:
        return None
    import torch.distributed as dist
    from paper_1905_13408_b200.slab import nccl_unique_id

    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def time_slab_solves(sc, cfg, steps, warmup, world):
    import torch

    for _ in range(warmup):
        sc.solve(cfg)
    barrier(world)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    dev_ms, launches, st = 0.0, 0, None
    e0.record()
    for _ in range(steps):
        st = sc.solve(cfg)
        dev_ms += st.solve_ms
        launches += st.kernel_launches
    e1.record()
    torch.cuda.synchronize()
    barrier(world)
    return allreduce_max(e0.elapsed_time(e1), world), allreduce_max(dev_ms, world), launches, st


def big_slab(args, world, rank, local):
    """1024^3 z-slab solve on a device-rendered problem (timing only)."""
    import paper_1905_13408_b200 as cm
    from paper_1905_13408_b200.slab import SlabContext, SlabPlan

    n = args.big_n
    plan = SlabPlan(n, world)
    if not plan.supported():
        return {"n": n, "skipped": f"{world} ranks do not tile {n}^3 into 64-plane slabs"}
    sc = SlabContext(n, world, rank, local, broadcast_nccl_id(world, rank))
    try:
        sy = sc.set_synthetic(7)
        cfg = cm.derive_config(sy, 1.5, 0.1, 0.1 / 3)
        cfg.inner_iters = args.big_iters
        t_ms, dev_ms, launches, st = time_slab_solves(sc, cfg, 2, 1, world)
    finally:
        sc.close()
    ms_iter = t_ms / (2 * args.big_iters)
    L = float(n) ** 3
    hbm, _ = peaks()
    iter_bytes = iteration_bytes_s8d(n, 4) / world
    return {"n": n, "ranks": world, "iters_per_step": args.big_iters, "steps": 2,
            "value": L * args.big_iters * 2 / (t_ms / 1e3), "unit": "voxel-iterations/s",
            "ms_per_iter": ms_iter, "stop_reason": st.stop_reason,
            "hbm_frac_per_gpu": iter_bytes / (ms_iter / 1e3) / 1e9 / hbm,
            "exchange_bytes_per_rank_per_iter": plan.exchange_bytes_per_iteration(),
            "model_per_p": slab_model(n, ms_iter * world),
            "data": "device-rendered blob lattice + random symmetric weight (timing only)"}


def slab_model(n, compute_ms_1, link_gbs=900.0):
    """Modelled split of one z-slab iteration at P ranks: compute = the measured
    one-GPU-equivalent iteration time / P; comm = the bytes each rank sends
    (SlabPlan.exchange_bytes_per_iteration) at the nominal NVLink 5 rate per
    direction; 'serial' if no exchange overlaps compute, 'overlapped' if all of it
    does. Also the accumulator upload per rank (rows + mirrors) against the full
    grid's 24 n^3 bytes."""
    from paper_1905_13408_b200.slab import SlabPlan

    out = {}
    for P in (1, 2, 4, 8):
        pl = SlabPlan(n, P)
        if not pl.supported():
            continue
        comp = compute_ms_1 / P
        comm = 0.0 if P == 1 else pl.exchange_bytes_per_iteration() / (link_gbs * 1e9) * 1e3
        out[str(P)] = {"compute_ms": round(comp, 3), "comm_ms": round(comm, 3),
                       "serial_ms": round(comp + comm, 3), "overlapped_ms": round(max(comp, comm), 3),
                       "acc_upload_gb_per_rank": round(pl.acc_upload_bytes(0) / 1e9, 3),
                       "acc_full_grid_gb": round(24 * n ** 3 / 1e9, 3)}
    return out


def run_slab(args, world, rank, local):
    """The 512^3 solve z-slab decomposed over the torchrun ranks (strong scaling)."""
    import torch

    import paper_1905_13408_b200 as cm
    from paper_1905_13408_b200.slab import SlabContext, SlabPlan

    n, iters = args.n, args.iters
    t0 = time.time()
    p = load_problem(n, rank, world)
    gen_s = time.time() - t0
    acc = cm.AccumulatorPair(n, p.numerator, p.weight, True)
    s = cm.scale_data(acc, precision=32)
    cfg = cm.derive_config(s.s_y, s.s_n, p.eps, p.eps_prime)
    cfg.inner_iters = iters
    plan = SlabPlan(n, world)
    sc = SlabContext(n, world, rank, local, broadcast_nccl_id(world, rank))
    sc.set_accumulator(acc)
    sc.set_volumes(p.x0)
    with ClockSampler(local) as clk:
        t_ms, dev_ms, launches, st = time_slab_solves(sc, cfg, args.steps, args.warmup, world)
    clocks = clk.summary()
    value = float(n) ** 3 * iters * args.steps / (t_ms / 1e3)
    ms_iter = t_ms / (args.steps * iters)
    hbm, peak_kind = peaks()
    iter_bytes = iteration_bytes_s8d(n, 4) / world
    xb = plan.exchange_bytes_per_iteration()
    roofline = {
        "bound": "hbm", "kernel": "iteration (per GPU, z-slab)", "achieved":
            iter_bytes / (ms_iter / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
            "frac": iter_bytes / (ms_iter / 1e3) / 1e9 / hbm, "traffic": None,
            "peak_kind": peak_kind, "algorithmic_bytes_per_iter_per_gpu": iter_bytes,
            "exchange_bytes_per_iter_per_gpu": xb,
            "exchange_GBps_per_gpu": xb / (ms_iter / 1e3) / 1e9}
    # end to end through the C ABI: host accumulator + volume in, this rank's planes out
    e2e = None
    if not args.no_e2e:
        L = n ** 3
        pin_w = torch.empty(L, dtype=torch.float64, pin_memory=True).numpy().reshape(n, n, n)
        pin_y = torch.empty(2 * L, dtype=torch.float64, pin_memory=True).numpy()
        pin_x = torch.empty(L, dtype=torch.float64, pin_memory=True).numpy().reshape(n, n, n)
        pin_o = torch.empty(L, dtype=torch.float64, pin_memory=True).numpy().reshape(n, n, n)
        pin_w[...] = p.weight
        pin_y[...] = p.numerator.view(np.float64).reshape(-1)
        pin_x[...] = p.x0
        pacc = cm.AccumulatorPair(n, pin_y.view(np.complex128).reshape(n, n, n), pin_w, True)

        def one():
            sc.set_accumulator(pacc)
            sc.set_volumes(pin_x)
            sc.solve(cfg)
            sc.get_volume(pin_o)

        one()
        barrier(world)
        torch.cuda.synchronize()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record()
        for _ in range(args.e2e_steps):
            one()
        f1.record()
        torch.cuda.synchronize()
        e_ms = allreduce_max(f0.elapsed_time(f1), world)
        e2e = {"value": float(n) ** 3 * iters * args.e2e_steps / (e_ms / 1e3),
               "unit": "voxel-iterations/s", "h2d_bytes_per_step": 32 * L * world,
               "d2h_bytes_per_step": 8 * L, "steps": args.e2e_steps,
               "ms_per_step": e_ms / args.e2e_steps,
               "api": "cm_dctx_set_accumulator/set_volumes/solve/get_volume (every rank uploads "
                      "the full accumulator, downloads its planes)"}
    ttt = None
    if args.ttt:
        tc = cm.RegConfig(**{**cfg.__dict__, "inner_iters": args.ttt_max_iters,
                             "refresh": cm.Refresh.per_m_step, "momentum": 1, "tol_kind": 2,
                             "tol": 0.03})
        sc.set_accumulator(acc)
        sc.set_volumes(p.x0)
        barrier(world)
        tst = sc.solve(tc)
        ttt = {"fista": {"iterations": tst.iterations,
                         "seconds": allreduce_max(tst.solve_ms, world) / 1e3,
                         "stop_reason": tst.stop_reason,
                         "criterion": "step norm < 3% of the largest step"}}
    sc.close()
    del p, acc
    big = big_slab(args, world, rank, local) if args.big_n else None
    if rank == 0:
        line = {
            "metric": "solver voxel-iterations/s (512^3 m_step, ISTA, per-inner reweighting, audit)",
            "value": value, "unit": "voxel-iterations/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"m_step {n}^3 synthetic blob phantom, {iters} ISTA iterations "
                                   f"per step, z-slab decomposed over {world} GPUs",
                       "side": n, "iters_per_step": iters, "step_rule": "lipschitz",
                       "refresh": "per_inner", "audit": True,
                       "l2": "working set larger than the 126 MB L2; no flush needed",
                       "parallelism": f"zslab{world}"},
            "device_ms_solver_stream": dev_ms, "gen_seconds": gen_s,
            "roofline": roofline, "cpu_baseline": None, "e2e": e2e, "clocks": clocks,
            "gpu_launches": launches, "time_to_tolerance": ttt, "big": big,
        }
        print(json.dumps(line), flush=True)


def run_ours(args):
    import torch

    world, rank, local = dist_setup()
    torch.cuda.set_device(local)
    import paper_1905_13408_b200 as cm

    mode = args.mode if args.mode != "auto" else ("single" if world == 1 else "slab")
    if mode == "slab":
        run_slab(args, world, rank, local)
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()
        return

    n, iters = args.n, args.iters
    t0 = time.time()
    p = load_problem(n, rank, world)
    gen_s = time.time() - t0
    acc = cm.AccumulatorPair(n, p.numerator, p.weight, True)
    ctx = cm.Context(n, args.precision, device=local)
    ctx.set_accumulator(acc)
    s = ctx.scale_data()
    cfg = cm.derive_config(s.s_y, s.s_n, p.eps, p.eps_prime)
    cfg.inner_iters = iters  # reference semantics: lipschitz + per_inner + audit
    ctx.set_volumes(p.x0, p.x0)

    for _ in range(args.warmup):
        ctx.solve(cfg)
    barrier(world)
    torch.cuda.synchronize()
    launches = 0
    dev_ms = 0.0
    with ClockSampler(local) as clk:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            st = ctx.solve(cfg)
            launches += st.kernel_launches
            dev_ms += st.solve_ms
        e1.record()
        torch.cuda.synchronize()
    barrier(world)
    t_ms = e0.elapsed_time(e1)
    t_ms = allreduce_max(t_ms, world)
    clocks = clk.summary()
    total_vox_iters = float(n) ** 3 * iters * args.steps * world
    value = total_vox_iters / (t_ms / 1e3)

    # ---- per-kernel profile pass (events around every launch, same stream) --------
    ctx.set_profiling(True)
    prof_iters = min(iters, 30)
    pcfg = cm.RegConfig(**{**cfg.__dict__, "inner_iters": prof_iters})
    ctx.solve(pcfg)
    ms5, it = ctx.get_profile()
    ctx.set_profiling(False)
    names = list(KERNELS)
    avg = {k: ms5[q] / it for q, k in enumerate(names)}
    rsize = 4 if args.precision == 32 else 8
    kb = kernel_bytes(n, rsize, audit_prev=True)
    hbm, peak_kind = peaks()
    dom = max(names, key=lambda k: avg[k])
    achieved = kb[dom] / (avg[dom] / 1e3) / 1e9
    traffic = ncu_traffic(n).get(dom)
    iter_bytes = sum(kb.values())
    ms_iter = t_ms / (args.steps * iters)
    roofline = {
        "bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm, "unit": "GB/s",
        "frac": achieved / hbm, "traffic": traffic, "peak_kind": peak_kind,
        "algorithmic_bytes_per_launch": kb[dom], "avg_launch_ms": avg[dom],
        "per_kernel_ms": avg,
        "per_kernel_frac": {k: (kb[k] / (avg[k] / 1e3) / 1e9 / hbm if kb[k] else None)
                            for k in names},
        "iteration": {"algorithmic_bytes_s8d": iteration_bytes_s8d(n, rsize),
                      "implementation_bytes": iter_bytes, "ms": ms_iter,
                      "achieved": iteration_bytes_s8d(n, rsize) / (ms_iter / 1e3) / 1e9,
                      "frac": iteration_bytes_s8d(n, rsize) / (ms_iter / 1e3) / 1e9 / hbm,
                      "implementation_frac": iter_bytes / (ms_iter / 1e3) / 1e9 / hbm,
                      "note": "frac: SURVEY 8(d) algorithmic bytes (76H + 12L + 4L audit) / "
                              "device time of the graph-replayed iteration; implementation_frac: "
                              "the bytes this schedule moves (separate x transforms)"},
    }

    # ---- end to end through the C ABI -----------------------------------------------
    # e2e: PAGEABLE numpy buffers, what the drop-in receives (std::vector storage
    # behind regularizer.hpp's AccumulatorPair / Volume3D; the library streams them
    # through its pinned chunk ring); e2e_pinned: the same from page-locked buffers
    e2e = e2e_pinned = None
    if not args.no_e2e:
        L = n ** 3
        out_pg = np.empty((n, n, n))
        ctx.m_step_host(acc, p.x0, p.x0, cfg, out_pg)  # warm
        torch.cuda.synchronize()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record()
        for _ in range(args.e2e_steps):
            ctx.m_step_host(acc, p.x0, p.x0, cfg, out_pg)
        f1.record()
        torch.cuda.synchronize()
        e_ms = allreduce_max(f0.elapsed_time(f1), world)
        e2e = {"value": float(n) ** 3 * iters * args.e2e_steps * world / (e_ms / 1e3),
               "unit": "voxel-iterations/s", "h2d_bytes_per_step": 32 * L,
               "d2h_bytes_per_step": 8 * L, "steps": args.e2e_steps,
               "ms_per_step": e_ms / args.e2e_steps, "host_buffers": "pageable (numpy)",
               "api": "cm_m_step: fp64 full-grid W, Y, x_init (= anchor) in, x out"}
    if not args.no_e2e:
        L = n ** 3
        pin_w = torch.empty(L, dtype=torch.float64, pin_memory=True).numpy().reshape(n, n, n)
        pin_y = torch.empty(2 * L, dtype=torch.float64, pin_memory=True).numpy()
        pin_x = torch.empty(L, dtype=torch.float64, pin_memory=True).numpy().reshape(n, n, n)
        pin_o = torch.empty(L, dtype=torch.float64, pin_memory=True).numpy().reshape(n, n, n)
        pin_w[...] = p.weight
        pin_y[...] = p.numerator.view(np.float64).reshape(-1)
        pin_x[...] = p.x0
        pacc = cm.AccumulatorPair(n, pin_y.view(np.complex128).reshape(n, n, n), pin_w, True)
        ctx.m_step_host(pacc, pin_x, pin_x, cfg, pin_o)  # warm
        barrier(world)
        torch.cuda.synchronize()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record()
        for _ in range(args.e2e_steps):
            ctx.m_step_host(pacc, pin_x, pin_x, cfg, pin_o)
        f1.record()
        torch.cuda.synchronize()
        e_ms = allreduce_max(f0.elapsed_time(f1), world)
        e2e_pinned = {"value": float(n) ** 3 * iters * args.e2e_steps * world / (e_ms / 1e3),
                      "unit": "voxel-iterations/s", "h2d_bytes_per_step": 32 * L,
                      "d2h_bytes_per_step": 8 * L, "steps": args.e2e_steps,
                      "ms_per_step": e_ms / args.e2e_steps, "host_buffers": "page-locked"}

    # ---- time to tolerance ----------------------------------------------------------------
    # "Medium accuracy" = relative error <= 1e-2 against a converged
    # solution (profiles/r1_convergence_512.json: a 20000-iteration FISTA run with
    # frozen weights). Stopping rules calibrated there: FISTA stops on the step norm
    # falling below 3% of the largest step (0.50% error); the reference's ISTA needs
    # a 3e-7 frozen-weight surrogate decrease to get to 0.99%.
    ttt = None
    if args.ttt:
        ttt = {"definition": "rel. L2 error <= 1e-2 vs the converged solution of the same "
                             "subproblem (BASELINE.md section 4; calibration profiles/r2_ttt.json)"}
        for name, extra in (("fista", dict(momentum=1, tol_kind=2, tol=0.03,
                                           refresh=cm.Refresh.per_m_step)),
                            ("fista_restart", dict(momentum=2, tol_kind=2, tol=0.03,
                                                   refresh=cm.Refresh.per_m_step)),
                            ("ista", dict(momentum=0, tol_kind=1, tol=3e-7,
                                          refresh=cm.Refresh.per_m_step)),
                            ("ista_per_inner", dict(momentum=0, tol_kind=1, tol=1e-7,
                                                    refresh=cm.Refresh.per_inner))):
            tc = cm.RegConfig(**{**cfg.__dict__, "inner_iters": args.ttt_max_iters, **extra})
            torch.cuda.synchronize()
            st = ctx.solve(tc)
            ttt[name] = {"iterations": st.iterations, "seconds": st.solve_ms / 1e3,
                         "stop_reason": st.stop_reason, "last_rel": st.last_rel,
                         "criterion": ("step norm < 3% of the largest step" if name.startswith("fista")
                                       else f"surrogate relative decrease < {extra['tol']:g}"),
                         "refresh": ("per_inner (the reference's semantics)"
                                     if name == "ista_per_inner" else "per_m_step")}
            if e2e is not None and name == "fista":
                # the same solve through cm_m_step on pinned host buffers: fp64 full-grid
                # accumulator + volume H2D, result D2H ("including H2D")
                torch.cuda.synchronize()
                g0 = torch.cuda.Event(enable_timing=True)
                g1 = torch.cuda.Event(enable_timing=True)
                g0.record()
                ctx.m_step_host(pacc, pin_x, pin_x, tc, pin_o)
                g1.record()
                torch.cuda.synchronize()
                ttt[name]["seconds_incl_transfers"] = g0.elapsed_time(g1) / 1e3

    # ---- EM M-step block extras: V = fft3_centered of the
    # resident result and the FSC of two resident half-map results, on the device
    em = None
    if args.em and world == 1:
        ctx.solve(cfg)
        ctx2 = cm.Context(n, args.precision, device=local)
        ctx2.set_accumulator(acc)
        ctx2.set_volumes(p.x0 * 0.98, p.x0 * 0.98)
        ctx2.solve(cm.RegConfig(**{**cfg.__dict__, "inner_iters": 10}))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        V = ctx.get_spectrum(centered=True)
        t_spec = time.perf_counter() - t0
        t0 = time.perf_counter()
        curve = ctx.fsc(ctx2)
        t_fsc = time.perf_counter() - t0
        em = {"n": n, "spectrum_centered_s": t_spec, "fsc_s": t_fsc,
              "spectrum_bytes_to_host": int(V.nbytes), "fsc_shells": int(curve.size),
              "note": "fft3_centered of the resident m_step result (full complex128 grid to "
                      "the host) and the FSC of two resident results; the reference does both "
                      "on the host (full-grid FFTW transforms + shell loop, refine.cpp:182,194)"}
        del V, ctx2
        try:
            em["iteration_128"] = em_iteration(local)
        except Exception as e:  # reported, never fatal to the headline line
            em["iteration_128"] = {"error": str(e)[:200]}

    # ---- the fp64 parity mode (the C++ adapter's default precision): same solve
    p64 = None
    if args.prec64 and world == 1 and args.precision == 32:
        c64 = cm.Context(n, 64, device=local)
        c64.set_accumulator(acc)
        c64.set_volumes(p.x0, p.x0)
        k64 = cm.RegConfig(**{**cfg.__dict__, "inner_iters": 20})
        c64.solve(k64)
        torch.cuda.synchronize()
        h0 = torch.cuda.Event(enable_timing=True)
        h1 = torch.cuda.Event(enable_timing=True)
        h0.record()
        for _ in range(3):
            c64.solve(k64)
        h1.record()
        torch.cuda.synchronize()
        ms64 = h0.elapsed_time(h1) / (3 * 20)
        p64 = {"dtype": "f64", "iters_per_step": 20, "steps": 3, "ms_per_iter": ms64,
               "value": float(n) ** 3 / (ms64 / 1e3), "unit": "voxel-iterations/s",
               "note": "same 512^3 solve in the fp64 parity mode (cm_ctx_create precision 64, "
                       "the C++ adapter's default): every device array twice the bytes"}
        c64.close()
        del c64

    oc = None
    if args.configs and world == 1 and args.precision == 32:
        try:
            oc = other_configs(local, with_reference=not args.no_cpu_baseline)
        except Exception as e:  # reported, never fatal to the headline line
            oc = {"error": str(e)[:300]}

    big = None
    if args.big_n:
        del ctx
        big = big_slab(args, world, rank, local)

    cb = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cb = cpu_baseline(args, problem=p)
        except Exception as e:  # noqa: BLE001
            cb = {"value": None, "error": str(e)[:200]}

    if rank == 0:
        line = {
            "metric": "solver voxel-iterations/s (512^3 m_step, ISTA, per-inner reweighting, audit)",
            "value": value, "unit": "voxel-iterations/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None,
            "dtype": "f32" if args.precision == 32 else "f64", "data": "synthetic",
            "config": {"workload": f"m_step {n}^3 synthetic blob phantom (BASELINE config 3), "
                                   f"{iters} ISTA iterations per step" +
                                   (f", {world} independent replicas" if world > 1 else ""),
                       "side": n, "iters_per_step": iters, "step_rule": "lipschitz",
                       "refresh": "per_inner", "audit": True,
                       "l2": "working set (>2 GB) larger than the 126 MB L2; no flush needed",
                       "parallelism": f"replicas{world}"},
            "device_ms_solver_stream": dev_ms, "gen_seconds": gen_s,
            "roofline": roofline, "cpu_baseline": cb, "e2e": e2e, "e2e_pinned": e2e_pinned,
            "clocks": clocks,
            "gpu_launches": launches, "time_to_tolerance": ttt, "big": big, "em_block": em,
            "precision64": p64, "other_configs": oc,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def other_configs(device: int = 0, with_reference: bool = True) -> dict:
    """The BASELINE configs other than the headline (one GPU each; the driver's
    multi-GPU runs cover config 4's scaling):
      config1: 64^3 blob phantom, 100 iterations, single reweighting pass
        (per_m_step weights), lipschitz + audit — launch-bound; the solve on the
        device (graph), end to end through cm_m_step from pageable buffers, and
        the unmodified reference (oracle/_ref, one core) on the same call;
      config2: 256^3 bond-like phantom, 3 reweighting loops (per_m_step,
        x_init <- previous output) each to tolerance (ISTA surrogate 1e-6; FISTA
        step 3%, opt-in);
      config5: one 384^3 replica of the 8-volume batch (100 ISTA iterations,
        reference semantics); `bench.py --gpus N --mode replicas` runs N."""
    import torch

    import paper_1905_13408_b200 as cm
    from paper_1905_13408_b200 import synth

    out = {}
    # ---- config 1
    n = 64
    p = synth.synthetic_problem(n)
    acc = cm.AccumulatorPair(n, p.numerator, p.weight, True)
    ctx = cm.Context(n, 32, device=device)
    ctx.set_accumulator(acc)
    s = ctx.scale_data()
    cfg = cm.derive_config(s.s_y, s.s_n, p.eps, p.eps_prime)
    cfg = cm.RegConfig(**{**cfg.__dict__, "inner_iters": 100, "refresh": cm.Refresh.per_m_step})
    ctx.set_volumes(p.x0, p.x0)
    ctx.solve(cfg)
    reps = 20
    dev = sorted(ctx.solve(cfg).solve_ms for _ in range(reps))[reps // 2]
    o64 = np.empty((n, n, n))
    ctx.m_step_host(acc, p.x0, p.x0, cfg, o64)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        ctx.m_step_host(acc, p.x0, p.x0, cfg, o64)
    e2e_ms = (time.perf_counter() - t0) / reps * 1e3
    c1 = {"side": n, "iterations": 100, "refresh": "per_m_step", "solve_ms_device": dev,
          "value": n ** 3 * 100 / (dev / 1e3), "unit": "voxel-iterations/s",
          "e2e_ms_pageable": e2e_ms, "e2e_value": n ** 3 * 100 / (e2e_ms / 1e3),
          "ms_per_iteration": dev / 100,
          "note": "launch-bound: one CUDA graph of 100 iterations x 7 kernels"}
    if with_reference:
        try:
            sys.path.insert(0, str(ROOT / "tests"))
            from oracle_lib import REF_DIR, Reference, make_cfg

            if (REF_DIR / "libcryomap_ref.so").exists():
                os.environ["CM_REF_FFT_THREADS"] = "1"
                R = Reference()
                rcfg = make_cfg(alpha=cfg.alpha, beta=cfg.beta, gamma=cfg.gamma, eps=cfg.eps,
                                eps_prime=cfg.eps_prime, mu=cfg.mu, inner_iters=100, refresh=1)
                rc, xr, _ = R.m_step(p.weight, p.numerator, p.x0, p.x0, rcfg, trace=False)
                assert rc == 0
                c1["reference_seconds_1core"] = R.last_seconds
                c1["reference_value"] = n ** 3 * 100 / R.last_seconds
                c1["rel_l2_vs_reference"] = float(np.linalg.norm(o64 - xr) / np.linalg.norm(xr))
        except Exception as e:  # reported, never fatal
            c1["reference_error"] = str(e)[:200]
    out["config1_64"] = c1
    ctx.close()
    # ---- config 2
    n = 256
    p = synth.synthetic_problem(n, kind="bonds")
    acc = cm.AccumulatorPair(n, p.numerator, p.weight, True)
    ctx = cm.Context(n, 32, device=device)
    ctx.set_accumulator(acc)
    s = ctx.scale_data()
    base = cm.derive_config(s.s_y, s.s_n, p.eps, p.eps_prime)
    c2 = {"side": n, "phantom": "bond-like chains", "loops": 3}
    for name, extra in (("ista_surrogate_1e-6", dict(tol_kind=1, tol=1e-6)),
                        ("fista_step_3pct", dict(momentum=1, tol_kind=2, tol=0.03))):
        cfg = cm.RegConfig(**{**base.__dict__, "inner_iters": 20000,
                              "refresh": cm.Refresh.per_m_step, **extra})
        x, its, secs = p.x0, [], 0.0
        for _ in range(3):
            ctx.set_volumes(x, p.x0)
            st = ctx.solve(cfg)
            x = ctx.get_volume()
            its.append(st.iterations)
            secs += st.solve_ms / 1e3
        c2[name] = {"iterations": its, "seconds": secs,
                    "rel_err_vs_truth": float(np.linalg.norm(x - p.truth) / np.linalg.norm(p.truth))}
    out["config2_256"] = c2
    ctx.close()
    # ---- config 5 (one replica)
    n = 384
    p = synth.synthetic_problem(n)
    acc = cm.AccumulatorPair(n, p.numerator, p.weight, True)
    ctx = cm.Context(n, 32, device=device)
    ctx.set_accumulator(acc)
    s = ctx.scale_data()
    cfg = cm.derive_config(s.s_y, s.s_n, p.eps, p.eps_prime)
    cfg.inner_iters = 100
    ctx.set_volumes(p.x0, p.x0)
    ctx.solve(cfg)
    ms = sorted(ctx.solve(cfg).solve_ms for _ in range(5))[2]
    out["config5_384_replica"] = {"side": n, "iterations": 100, "solve_ms_device": ms,
                                  "ms_per_iteration": ms / 100,
                                  "value": n ** 3 * 100 / (ms / 1e3), "unit": "voxel-iterations/s",
                                  "note": "per-GPU work of the 8 x 384^3 batch"}
    ctx.close()
    return out


def em_iteration(device: int = 0, n: int = 128, m: int = 1000, n_poses: int = 200,
                 iters: int = 50, rounds: int = 3) -> dict:
    """One device-resident EM iteration of em_refine (refine.cpp:150-183) on a
    synthetic particle set: M-step (the solver) -> E-step with V from the
    resident result -> backprojection into the resident accumulator, images
    uploaded once (cm_set_particles). Per-stage seconds (host clock around
    synchronised calls; the posteriors cross to the host as sparse PosteriorRow
    lists (cm_estep_sparse) and back as entry lists, everything else stays on
    the device)."""
    import torch

    import paper_1905_13408_b200 as cm
    from paper_1905_13408_b200 import synth
    inp = synth.synthetic_backprojection(n, m, n_poses=n_poses, trans_radius=2,
                                         entries_per_image=3, seed=11)
    sigma2 = np.ones(n // 2 + 1)  # the data's per-shell |X|^2 / 2 (init_noise_from_data)
    ctx = cm.Context(n, 32, device=device)
    cm.set_particles(ctx, inp)
    cm.backproject_into(ctx, inp, download=False, resident_images=True)
    s = ctx.scale_data()
    cfg = cm.derive_config(s.s_y, s.s_n, 1e-3, 1e-3)
    cfg.inner_iters = iters
    x = np.zeros((n, n, n))
    ctx.set_volumes(x)
    out = {"n": n, "particles": m, "poses": n_poses, "shifts": int(inp.shifts.shape[0]),
           "m_step_iters": iters, "rounds": []}
    for _ in range(rounds):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx.solve(cfg)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        rows = cm.e_step(ctx, inp, sigma2, resident_images=True, sparse=True)
        t2 = time.perf_counter()
        inp.entry_particle, inp.entry_candidate, inp.entry_posterior = cm.sparse_entries(*rows)
        cm.backproject_into(ctx, inp, download=False, resident_images=True)
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        ctx.set_volumes(ctx.get_volume())  # the next M-step starts from this one's result
        out["rounds"].append({"m_step_s": t1 - t0, "e_step_s": t2 - t1, "backproject_s": t3 - t2,
                              "entries": int(inp.entry_posterior.size)})
    ctx.close()
    best = min(out["rounds"], key=lambda r: r["m_step_s"] + r["e_step_s"] + r["backproject_s"])
    out["iteration_s"] = best["m_step_s"] + best["e_step_s"] + best["backproject_s"]
    out["note"] = ("device-resident EM iteration; reference per-stage CPU rates on the same "
                   "shapes are in profiles/r1_estep_128.json and r1_backproject_128.json")
    return out


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
