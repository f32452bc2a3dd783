#!/usr/bin/env python3
"""Benchmark of the FTCS hot path (BASELINE.json metric: FP64 lattice updates/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Workload (BASELINE.json configs[2], "cfg3"): N = 2^30 FP64 points per GPU,
r = from_r(0.4), Dirichlet(0,0), sine initial profile, 10^4 FTCS time steps.
One bench STEP = 1000 FTCS time steps over the whole field, so the default
--steps 10 is exactly the cfg3 run.  For N > 1 GPUs (torchrun, one rank per
GPU) each rank owns a 2^30-point slab of a G*2^30 domain (weak scaling; at
G = 8 the total is cfg4's 2^33); the timed run is K5 with q = 1 (the exact
synchronous scheme) whose slab-boundary tiles store their edge values
straight into the neighbours' receive rings over NVLink (one seeded run, one
launch per rank, no collective inside).

Arms
  b200       the sm_100a kernels (libheat_b200.so) -- value is device-timed
             with inputs resident in HBM; e2e is timed through the C-ABI:
             one heat_sync_run call per e2e step running the whole K x 1000
             steps (cfg3: 10^4) from pinned host buffers, copies included
             (also with pageable buffers, and with 1000-step calls).
  reference  the reference's own CPU executor (exec_run Barriered, all host
             threads) from oracle/_ref (compiled from /root/reference), or the
             C port when that library is absent; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FP64 lattice updates/s (GLUPS) at 1/2/4/8 B200, % HBM roofline, async vs sync"
UNIT = "GLUPS"
N_PER_GPU = 1 << 30
R = 0.4
STEPS_PER_BENCH_STEP = 1000
STEPS_PER_PASS = 32  # fallback; the library reports its kernel's (heat_sync_kernel_info)
BYTES_PER_UPDATE = 16  # one FP64 read + one FP64 write per point per step
FP64_OPS_PER_UPDATE = 4  # 2 DMUL + 2 DADD with the shared r*u products


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic_per_launch():
    """dram bytes per launch of the dominant kernel from the committed ncu capture."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        key = "sync_col_kernel" if sync_kernel_info()["exact"] > 2000 else "sync_tb_kernel"
        return d.get(key, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


class ClockSampler:
    """Samples SM clocks and throttle reasons during the timed region (NVML)."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, device: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


_CPU_FIELDS = {}
REF_SAMPLE_STEPS = 16  # FTCS steps per CPU sample at N = 2^30 (~2.6 s on 16 host threads)


def _cpu_field(n):
    from oracle import oracle as O
    u0 = _CPU_FIELDS.get(n)
    if u0 is None:  # 8 GiB at N = 2^30: built once per process, reused by every sample
        u0 = O.port().sine_init(n)
        u0[0] = 0.0
        u0[-1] = 0.0
        _CPU_FIELDS[n] = u0
    return u0


def cpu_info():
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


def cpu_exec_samples(n, steps, reps, mode=0):
    """The reference's exec_run (oracle/_ref; the C port's threaded executor when
    the reference library is absent) on all host threads, `reps` calls on one
    field.  Returns (list of GLUPS per call, workers, kind)."""
    from oracle import oracle as O
    u0 = _cpu_field(n)
    kind = "reference" if O.Ref.available() else "port"
    eng = O.ref() if kind == "reference" else O.port()
    hw = (eng.hardware_concurrency() if kind == "reference" else 0) or os.cpu_count() or 1
    workers = 1
    while workers * 2 <= hw and n % (workers * 2) == 0:
        workers *= 2
    if kind == "reference":
        durs, _ = eng.exec_run_reps(u0, R, O.DIRICHLET, 0.0, 0.0, n // workers, workers, steps,
                                    mode, reps)
    else:
        durs = [eng.exec_run(u0, R, O.DIRICHLET, 0.0, 0.0, n // workers, workers, steps,
                             O.BARRIERED if mode == 0 else O.BARRIER_FREE)[1]
                for _ in range(reps)]
    return [n * steps / (d * 1e-9) / 1e9 for d in durs], workers, kind


def cpu_baseline_b200_arm(n):
    """BASELINE.md §3 on the GPU box's host: exec_run(Barriered) on all host
    threads (the value, median of 3), exec_run(BarrierFree) (median of 3), and
    the single-core detail::sync_step_into loop."""
    from oracle import oracle as O
    vals, workers, kind = cpu_exec_samples(n, REF_SAMPLE_STEPS, 3, 0)
    free, _, _ = cpu_exec_samples(n, REF_SAMPLE_STEPS, 3, 1)
    one = None
    if kind == "reference":
        k1 = 2
        _, ns = O.ref().sync_step_into_loop(_cpu_field(n), R, O.DIRICHLET, 0.0, 0.0, k1)
        one = round(n * k1 / (ns * 1e-9) / 1e9, 4)
    return {
        "value": round(statistics.median(vals), 4), "unit": UNIT, "cores": workers, "kind": kind,
        "sample": (f"N=2^{n.bit_length() - 1} FP64, {REF_SAMPLE_STEPS} FTCS steps per sample, "
                   f"exec_run(Barriered) with P={workers} threads, median of 3 samples "
                   f"{[round(v, 3) for v in vals]}; time = exec_run's own duration (thread "
                   f"spawn..join, async_exec.cpp:101-106)"),
        "barrier_free": {"value": round(statistics.median(free), 4), "unit": UNIT,
                         "cores": workers, "samples": [round(v, 3) for v in free],
                         "what": "exec_run(BarrierFree), same N/P/steps (async_exec.cpp:156-259)"},
        "sync_step_into_1core": {"value": one, "unit": UNIT, "cores": 1,
                                 "what": f"detail::sync_step_into loop, 2 steps at N=2^{n.bit_length() - 1} "
                                         "(sync_solver.hpp:26-39)"},
        **cpu_info(),
    }


def run_reference(args, rank, world):
    """The reference arm: the reference's own exec_run(Barriered) (oracle/_ref,
    compiled from /root/reference) on all host threads, rank 0 only.  One
    bench step = one exec_run call of REF_SAMPLE_STEPS FTCS steps at N = 2^30,
    timed by the reference's own duration; ms_per_step is that measured time.
    One untimed warm-up call (page first touch) stands in for --warmup: the CPU
    path has no clocks or caches to warm beyond it."""
    if rank != 0:
        return 0
    n = N_PER_GPU
    warm = min(1, args.warmup)
    vals, workers, kind = cpu_exec_samples(n, REF_SAMPLE_STEPS, warm + args.steps, 0)
    vals = vals[warm:]
    v = statistics.median(vals)
    ms = n * REF_SAMPLE_STEPS / (v * 1e9) * 1e3
    cfg = config_dict(world, impl="reference", steps=args.steps)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(v, 4), "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (sine IC)",
        "config": cfg,
        "cpu_baseline": {"value": round(v, 4), "unit": UNIT, "cores": workers, "kind": kind,
                         "sample": (f"N=2^30 FP64, {REF_SAMPLE_STEPS} FTCS steps per bench step, "
                                    f"exec_run(Barriered) with P={workers} threads; time = "
                                    f"exec_run's own duration; median of {args.steps} measured "
                                    f"calls after {warm} warm-up call"),
                         **cpu_info()},
        "e2e": {"value": round(v, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def sync_kernel_info():
    """The f64 pass kernel the library selected (heat_sync_kernel_info)."""
    import ctypes
    from paper_1510_08982_b200 import _lib
    v, nb, out, sp = ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    _lib.lib().heat_sync_kernel_info(ctypes.byref(v), ctypes.byref(nb), ctypes.byref(out),
                                     ctypes.byref(sp))
    return {"V": v.value, "buffers": nb.value, "exact": out.value, "steps_per_pass": sp.value}


def sync_kernel_name():
    try:
        k = sync_kernel_info()
        V, H = k['V'], k['steps_per_pass']
        if k['exact'] > 32 * V:  # K1s: `exact` is a chunk's outputs
            return (f"sync_col_kernel<double,{V},H={H}> (temporal-blocked strips: {V}-point "
                    f"lanes, chunks of tiles whose later tiles take their left neighbour from a "
                    f"carried boundary column instead of a halo; {k['exact']} exact of "
                    f"{k['exact'] + 2 * H + (k['exact'] - (32 * V - 2 * H)) // (32 * V - H) * H} "
                    f"points stepped per chunk; {H} steps per HBM pass)")
        return (f"sync_tb_kernel<double,{V},{k['buffers']},0,H={H}> "
                f"(temporal-blocked: {V}-point lanes, {H}-point halo, "
                f"{k['exact']} exact points per warp tile, {H} steps per HBM pass)")
    except Exception as e:  # the bench itself fails later if the library is missing
        return f"sync_tb_kernel (info unavailable: {e})"


def k5_geometry(per_pe):
    """The stream kernel's tile geometry for PEs of per_pe points (heat_k5_geometry)."""
    try:
        import ctypes
        from paper_1510_08982_b200 import _lib
        v, h = ctypes.c_int(), ctypes.c_int()
        _lib.lib().heat_k5_geometry(per_pe, ctypes.byref(v), ctypes.byref(h))
        return f"{v.value},{h.value}"
    except Exception:
        return "?"


def slab_halo():
    try:
        from paper_1510_08982_b200 import _lib
        return int(_lib.lib().heat_slab_halo())
    except Exception:
        return STEPS_PER_PASS


def steps_per_pass():
    try:
        return sync_kernel_info()["steps_per_pass"]
    except Exception:
        return STEPS_PER_PASS


N_STRONG_TOTAL = 1 << 33  # BASELINE configs[3] (cfg4): strong scaling at N = 2^33


def points_per_gpu(args, world):
    return N_STRONG_TOTAL // world if getattr(args, "strong", False) else N_PER_GPU


def config_dict(world, n=N_PER_GPU, strong=False, impl="b200", steps=10):
    if strong:
        work = (f"cfg4: N=2^33 FP64 in total ({n} points per GPU), r=0.4, Dirichlet(0,0), "
                f"sine IC, 1000-step bench steps; strong scaling over {world} GPU(s)")
    elif impl == "reference":
        work = (f"cfg3: N=2^30 FP64, r=0.4, Dirichlet(0,0), sine IC; each bench step is a "
                f"bounded sample of {REF_SAMPLE_STEPS} FTCS steps (the cfg3 run is 10^4)")
    else:
        work = (f"cfg3: N=2^30 FP64 per GPU, r=0.4, Dirichlet(0,0), sine IC; {steps} bench steps "
                f"of 1000 FTCS steps = {steps * 1000} steps timed (cfg3 is 10^4)" +
                ("" if world == 1 else f"; {world}-GPU slab decomposition, N=2^30*{world}"))
    d = {
        "workload": work,
        "N_per_gpu": n, "N_total": n * world, "r": R,
        "time_steps_per_bench_step": REF_SAMPLE_STEPS if impl == "reference"
        else STEPS_PER_BENCH_STEP,
        "l2": "inputs larger than L2 (8 GiB per array vs 126 MB L2)",
    }
    if impl == "reference":  # nothing of the GPU library is loaded on this arm
        d["kernel"] = "reference exec_run(Barriered), std::barrier per step, host threads"
        d["parallelism"] = "host threads"
        return d
    if world == 1:
        d["steps_per_pass"] = steps_per_pass()
        d["kernel"] = sync_kernel_name()
        d["parallelism"] = "single GPU"
    else:
        d["kernel"] = ("async_stream_kernel<48,64> with q=1 (the exact synchronous scheme), "
                       "one persistent launch per rank for the whole run")
        d["parallelism"] = (f"slab x{world}: halos by P2P stores into IPC-mapped neighbour "
                            "receive rings over NVLink (NCCL/gloo only ship the IPC handles, "
                            "seed barriers and the final gather)")
    return d


def run_b200(args, rank, world, local):
    import torch
    import torch.distributed as dist
    from paper_1510_08982_b200 import heat as H
    from paper_1510_08982_b200 import multigpu as MG

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    # a dedicated (non-legacy) stream: the kernels, the halo NCCL ops and the
    # timing events all live on it
    stream = torch.cuda.Stream(local)
    torch.cuda.set_stream(stream)
    n = points_per_gpu(args, world)
    bc = H.BoundaryCondition.dirichlet(0.0, 0.0)
    r = H.SolverParams.from_r(R).r()

    if world == 1:
        plan = H.Plan(n, local)
        plan.set_stream(stream.cuda_stream)
        plan.fill_sine()

        def advance(k):
            plan.sync_advance(r, bc, k)
    else:
        # N GPUs: K5 with q = 1 on each rank's slab -- the exact synchronous
        # scheme -- with the slab halos moving by P2P stores over NVLink into
        # the neighbours' receive rings; the timed region is ONE seeded run
        # of all its steps (one launch per rank, no collective inside)
        solver = MG.AsyncSlabSolver(n, n // ASYNC_PES, 1, bc, local, rank, world)
        solver.plan.fill_sine()  # each slab gets a sine profile (data-independent cost)
        plan = solver.plan

        def advance(k):
            solver.advance(r, k)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        advance(STEPS_PER_BENCH_STEP)
    plan.synchronize()
    barrier()
    # parity of the timed run: light-cone windows of the field as it enters
    # the timed region, checked against the oracle after it (outside the timing)
    chk = None
    if world == 1 and not args.skip_parity:
        from oracle.lightcone import WindowCheck
        chk = WindowCheck(n, STEPS_PER_BENCH_STEP * args.steps, sync_centres(n))
        chk.capture(plan.download_range)
        torch.cuda.synchronize()

    if world > 1:
        solver.prepare()  # seed the run (IPC rings) before the timed region
    launches0 = H.kernel_launches()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        e0.record(stream)
        if world == 1:
            for _ in range(args.steps):
                advance(STEPS_PER_BENCH_STEP)
        else:
            multi_stats = solver.run(r, STEPS_PER_BENCH_STEP * args.steps)
            if int(multi_stats.max_delay) != 0:  # q = 1 must read only current values
                raise RuntimeError(f"P2P sync run consumed a stale value "
                                   f"(max delay {multi_stats.max_delay})")
        e1.record(stream)
        barrier()
    plan.synchronize()
    launches = H.kernel_launches() - launches0
    ms = e0.elapsed_time(e1)
    parity = {}
    if chk is not None:
        from oracle import oracle as O
        port = O.port()
        kk = STEPS_PER_BENCH_STEP * args.steps
        parity["sync"] = chk.verify(plan.download_range,
                                    lambda w, lo: port.sync_window(w, lo, n, r, 0.0, 0.0, kk))
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    total_updates = float(n) * world * STEPS_PER_BENCH_STEP * args.steps
    glups = total_updates / (ms * 1e-3) / 1e9

    # Roofline of the dominant kernel (the K1 pass kernel, one launch per pass of
    # <= steps_per_pass() steps: 15 passes of 64 + one of 40 per 1000 steps).
    # The timed region is nothing but those back-to-back launches, so the
    # average launch duration is the timed region / launches.  With 64-step
    # temporal blocking a pass moves 0.25 B per lattice update through HBM;
    # the bound is the FP64 pipe (4 DP instructions per update: 2 DMUL +
    # 2 DADD with the shared r*u products), reported as the headline, and the
    # 16 B/update effective bandwidth beside it.
    if world == 1:
        spp = steps_per_pass()
        passes_per_step = -(-STEPS_PER_BENCH_STEP // spp)
        sync_launches = passes_per_step * args.steps
    else:
        sync_launches = 1  # one persistent K5 launch for the whole timed run
    per_launch_s = ms * 1e-3 / sync_launches
    updates = float(n) * STEPS_PER_BENCH_STEP * args.steps
    alg_bytes = BYTES_PER_UPDATE * updates / sync_launches  # per launch (average)
    alg_ops = FP64_OPS_PER_UPDATE * updates / sync_launches
    peak, peak_kind = measured_peaks()
    achieved = alg_bytes / per_launch_s / 1e9
    clk_mhz = clk.summary()["sm_mhz"] or 1965.0
    fp64_peak = 148 * 64 * 1.965e9 / 1e12  # SMs x FP64 lanes x max SM clock (T DP ops/s)
    fp64_achieved = alg_ops / per_launch_s / 1e12
    traffic = ncu_traffic_per_launch()
    roofline = {
        "kernel": "K1 pass kernel: " + sync_kernel_name() if world == 1 else "async_stream_kernel (K5, q=1)",
        "bound": "fp64", "achieved": round(fp64_achieved, 3), "peak": round(fp64_peak, 3),
        "unit": "TFLOP/s", "frac": round(fp64_achieved / fp64_peak, 4),
        # ncu DRAM bytes of one 64-step pass over 2^30 points (scales with the points)
        "traffic": None if traffic is None else traffic * n / N_PER_GPU,
        "peak_source": ("nominal 148 SMs x 64 FP64 lanes x 1965 MHz (MEASURED_PEAKS.json has no "
                        "FP64 figure; tools/fp64_micro.cu measured 18.55 T DMUL/DADD per s)"),
        "ops_per_update": FP64_OPS_PER_UPDATE,
        "algorithmic_ops_per_launch": alg_ops,
        "launch_ms": round(per_launch_s * 1e3, 3),
        "frac_at_measured_clock": round(fp64_achieved / (148 * 64 * clk_mhz * 1e6 / 1e12), 4),
        "hbm": {"achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4),
                "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
                "algorithmic_bytes_per_launch": alg_bytes,
                "dram_bytes_per_launch": None if traffic is None else traffic * n / N_PER_GPU,
                "note": "16 B per lattice update counted for every step (BASELINE.md §2): the "
                        "effective bandwidth temporal blocking buys; physical DRAM traffic is "
                        "one read + one write of the field per 64-step pass"},
    }

    # Asynchronous scheme on the same workload (single GPU): K5 streaming
    # kernel, PEs of 2^21 points, free-running with delays <= 7 and the
    # deterministic replay of a seeded q=2 stream.
    async_info = None
    if world == 1 and not args.skip_async:
        async_info = run_async(args, H, torch, plan, stream, n, r, bc, glups, parity)
    elif world > 1 and not args.skip_async:
        try:
            async_info = run_async_multi(args, H, MG, torch, stream, n, r, bc, glups, rank, world,
                                         local)
        except Exception as exc:  # report, do not lose the sync line
            async_info = {"error": f"{type(exc).__name__}: {exc}"[:300]}

    # End to end through the public API with host buffers (copies timed).
    e2e = None
    if not args.skip_e2e:
        e2e = run_e2e(args, H, torch, n, r, bc, rank, world, plan, advance, parity)

    cpu = None
    if rank == 0 and world == 1 and not args.skip_cpu:
        cpu = cpu_baseline_b200_arm(n)

    paper = None
    if rank == 0 and world == 1 and not args.skip_cpu:
        try:
            paper = run_paper_configs(H)
        except Exception as exc:  # report, do not lose the line
            paper = {"error": f"{type(exc).__name__}: {exc}"[:300]}

    line = {
        "metric": METRIC, "value": round(glups, 3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 3),
        "higher_is_better": True, "scaling": "strong" if args.strong else "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (sine IC generated on device)",
        "config": config_dict(world, n, args.strong, steps=args.steps),
        "parity": parity_summary(parity) if parity else None,
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
        "clocks": clk.summary(), "async": async_info, "paper_configs": paper,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def run_paper_configs(H):
    """BASELINE configs[0] / [1], the paper's own runs: N = 1024, r = 0.25,
    Dirichlet(0,0), sine IC, 1000 steps -- synchronous, and asynchronous with
    8 PEs, q = 2, seeded delays.  GPU: wall time of one call through the
    public API (upload, kernels, download), best of 20.  CPU: the reference's
    own sync_run / async_run (oracle/_ref, one host thread), best of 5; the
    GPU results must be bit-identical to it."""
    from oracle import oracle as O
    port = O.port()
    ref = O.ref() if O.Ref.available() else port
    n, k = 1024, 1000
    u0 = port.prepare_initial(port.sine_init(n), O.DIRICHLET, 0.0, 0.0)
    p = H.SolverParams.from_r(0.25)
    bc = H.BoundaryCondition.dirichlet(0.0, 0.0)
    part = H.PartitionSpec(n, n // 8)
    model = H.DelayModel.uniform(2, 1)

    def best(f, reps):
        out, ts = None, []
        for _ in range(reps):
            t0 = time.perf_counter()
            out = f()
            ts.append(time.perf_counter() - t0)
        return out, min(ts) * 1e6

    # the full API calls on both sides, each recording the trajectory every
    # 100 steps (default_stride for N > 1000) -- 11 snapshots
    f = H.TemperatureField(u0)
    g_sync, t_gs = best(lambda: H.sync_run(f, p, bc, k, 100).final().values(), 20)
    g_async, t_ga = best(lambda: H.async_run(f, p, bc, part, model, k, 100).final().values(), 20)
    c_sync, t_cs = best(lambda: ref.sync_run(u0, p.r(), O.DIRICHLET, 0.0, 0.0, k, stride=100), 5)
    c_async, t_ca = best(lambda: ref.async_run(u0, p.r(), O.DIRICHLET, 0.0, 0.0, n // 8,
                                               O.UNIFORM, 2, seed=1, k_end=k, stride=100), 5)
    kind = "reference" if ref is not port else "port"
    return {
        "workload": "N=1024, r=0.25, Dirichlet(0,0), sine IC, 1000 steps, trajectory every 100 "
                    "steps; wall per sync_run / async_run call",
        "cpu_kind": kind, "cpu_cores": 1,
        "cfg1_sync": {"gpu_us": round(t_gs, 1), "cpu_us": round(t_cs, 1),
                      "bit_exact": bool(np.array_equal(g_sync.view(np.uint64),
                                                        np.asarray(c_sync).view(np.uint64)))},
        "cfg2_async_q2": {"gpu_us": round(t_ga, 1), "cpu_us": round(t_ca, 1),
                          "bit_exact": bool(np.array_equal(g_async.view(np.uint64),
                                                            np.asarray(c_async).view(np.uint64)))},
    }


ASYNC_PES = 512  # 2^21 points per PE at N = 2^30


def sync_centres(n):
    """Points the parity leg checks: both ends, the points next to them, the
    middle, K1 tile boundaries (1408 exact points per tile, tiles start at 0),
    K5 PE boundaries (2^21 points) and a few seeded random points."""
    rng = np.random.default_rng(12345)
    c = [1, 2, n // 2 - 1, n // 2, 1408 * 1000, 1408 * 1000 - 1, 1408 * 381301,
         (n // ASYNC_PES) * 7, (n // ASYNC_PES) * 7 - 1, n - 3, n - 2]
    c += [int(x) for x in rng.integers(0, n, 6)]
    return c


def async_centres(n):
    pe = n // ASYNC_PES
    rng = np.random.default_rng(54321)
    c = [1, pe - 1, pe, 100 * pe - 1, 100 * pe, (ASYNC_PES // 2) * pe, n - pe - 1, n - pe,
         n - 2]
    c += [int(x) for x in rng.integers(0, n, 3)]
    return c


def parity_summary(parity):
    out = {k: bool(v["ok"]) for k, v in parity.items()}
    out["points"] = {k: int(v["points"]) for k, v in parity.items()}
    out["windows"] = {k: int(v["windows"]) for k, v in parity.items()}
    bad = {k: v["bad"] for k, v in parity.items() if v["bad"]}
    if bad:
        out["bad"] = bad
    out["oracle"] = ("oracle/heat_oracle.c orc_sync_window / orc_async_window: light-cone windows "
                     "of the field entering the timed region, every point > k from a held window "
                     "end compared bit for bit (SURVEY §8c)")
    return out


def run_async(args, H, torch, plan, stream, n, r, bc, sync_glups, parity):
    """Async vs sync on the cfg3 workload: same steps, device-timed."""
    per_pe = n // ASYNC_PES
    out = {"pes": ASYNC_PES, "points_per_pe": per_pe,
           "kernel": f"async_stream_kernel<{k5_geometry(per_pe)}> (persistent, PE-boundary "
                     f"acquire/release rings)"}
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    for name, call in (
            ("free", lambda: plan.async_advance(r, bc, per_pe, 8, STEPS_PER_BENCH_STEP)),
            ("deterministic", lambda: plan.async_replay(r, bc, per_pe, H.DelayModel.uniform(2, 1),
                                                        STEPS_PER_BENCH_STEP))):
        plan.fill_sine()
        for _ in range(max(1, args.warmup)):
            call()
        plan.synchronize()
        torch.cuda.synchronize()
        chk = None
        if name == "deterministic" and not args.skip_parity:
            from oracle.lightcone import WindowCheck
            chk = WindowCheck(n, STEPS_PER_BENCH_STEP * args.steps, async_centres(n))
            chk.capture(plan.download_range)
            torch.cuda.synchronize()
        e0.record(stream)
        stats = [call() for _ in range(args.steps)]
        e1.record(stream)
        plan.synchronize()
        ms = e0.elapsed_time(e1)
        v = float(n) * STEPS_PER_BENCH_STEP * args.steps / (ms * 1e-3) / 1e9
        st = stats[-1]
        if chk is not None:
            from oracle import oracle as O
            port = O.port()

            def replay(w, lo):  # each bench step is a fresh run: k from 0, stream restarted
                for _ in range(args.steps):
                    w = port.async_window(w, lo, n, r, 0.0, 0.0, per_pe, O.UNIFORM, 2, seed=1,
                                          k=STEPS_PER_BENCH_STEP)
                return w
            parity["async_det"] = chk.verify(plan.download_range, replay)
        out[name] = {
            "value": round(v, 3), "unit": UNIT, "ms_per_step": round(ms / args.steps, 3),
            "q": 8 if name == "free" else 2,
            "delay_law": "newest value with k-k* <= 7" if name == "free"
            else "DelayModel::uniform(q=2, seed=1) replayed bit-exactly",
            "reads_per_run": int(st.reads), "waits_per_run": int(st.waits),
            "max_delay": int(st.max_delay),
            "delay_histogram": [int(x) for x in st.delay_histogram[:8]],
            "vs_sync": round(v / sync_glups, 4),
        }
    if not args.skip_bound:
        try:
            out["free"]["bound"] = run_free_bound(H, plan, n, r, bc, per_pe, 8,
                                                  STEPS_PER_BENCH_STEP * args.steps)
        except Exception as exc:  # report, do not lose the line
            out["free"]["bound"] = {"error": f"{type(exc).__name__}: {exc}"[:300]}
    return out


def run_free_bound(H, plan, n, r, bc, per_pe, q, k):
    """SURVEY §8a row 12 at cfg3 (not timed): one free-running K5 run of all k
    steps from the sine IC with every PE edge value and read logged on the
    device, the a-posteriori bound sum_k ||u(k+1) - A u(k)||_inf formed from
    the logs, and the actual ||u_async(k) - u_sync(k)||_inf against the
    synchronous run of the same IC (heat_sync_run)."""
    import numpy as np
    t0 = time.perf_counter()
    plan.fill_sine()
    u0 = plan.download()
    part = H.PartitionSpec(n, per_pe)
    p = H.SolverParams.from_r(r)
    fin, st = H.async_free_run(u0, p, bc, part, q, k)
    sync = H.sync_final(u0, p, bc, k)
    err = 0.0
    for lo in range(0, n, 1 << 26):  # chunked: no 8 GiB temporaries
        err = max(err, float(np.max(np.abs(fin[lo:lo + (1 << 26)] - sync[lo:lo + (1 << 26)]))))
    return {"steps": k, "q": q, "error_inf": err, "bound": st.residual_sum,
            "within": bool(err <= st.residual_sum), "max_delay": int(st.max_delay),
            "reads": int(st.reads), "seconds": round(time.perf_counter() - t0, 1),
            "what": "one logged free-running K5 run of all steps (heat_async_free_run) vs "
                    "heat_sync_run of the same sine IC; bound = sum_k ||u(k+1) - A u(k)||_inf "
                    "+ k*8*eps*max|u| from the device logs"}


def run_async_multi(args, H, MG, torch, stream, n, r, bc, sync_glups, rank, world, local):
    """The other G-GPU legs: K5 free-running (q = 8) over the same P2P rings,
    timed as the headline (one seeded run of all steps), and -- for comparison
    only -- K1 slabs with the 64-point halos moved by NCCL every pass."""
    import torch.distributed as dist
    per_pe = n // ASYNC_PES
    out = {"pes_per_gpu": ASYNC_PES, "points_per_pe": per_pe,
           "transport": "P2P stores into IPC-mapped neighbour receive rings (NVLink)"}
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    total = STEPS_PER_BENCH_STEP * args.steps

    def timed(fn):
        torch.cuda.synchronize()
        dist.barrier()
        e0.record(stream)
        res = fn()
        e1.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
        t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        return res, float(n) * world * total / (ms * 1e-3) / 1e9

    solver = MG.AsyncSlabSolver(n, per_pe, 8, bc, local, rank, world)
    solver.plan.fill_sine()
    solver.advance(r, STEPS_PER_BENCH_STEP)  # warm-up run
    solver.prepare()
    st, v = timed(lambda: solver.run(r, total))
    out["free"] = {"value": round(v, 3), "unit": UNIT, "q": 8, "max_delay": int(st.max_delay),
                   "reads_per_run": int(st.reads), "vs_sync": round(v / sync_glups, 4)}
    solver.plan.close()

    slab = MG.SlabSolver(n, r, bc, local, rank, world)
    slab.plan.fill_sine()
    slab.advance(STEPS_PER_BENCH_STEP)

    def run_slab():
        for _ in range(args.steps):
            slab.advance(STEPS_PER_BENCH_STEP)
    _, v = timed(run_slab)
    out["sync_nccl_halo"] = {"value": round(v, 3), "unit": UNIT,
                             "what": "K1 slabs, 64-point halos by NCCL send/recv every pass "
                                     "(comparison only; the headline moves halos by P2P)",
                             "vs_p2p_sync": round(v / sync_glups, 4)}
    slab.plan.close()
    return out


def run_e2e(args, H, torch, n, r, bc, rank, world, plan, advance, parity):
    """Same metric through the public API with HOST buffers.  One e2e step is
    one call that runs the timed region's whole workload (cfg3: 10^4 FTCS
    steps, as a caller's sync_run(u0, params, bc, 10000) does): the host field
    goes H2D, the steps run, the result comes back D2H, all inside the timed
    call.  `per_call_1000` repeats it with 1000-step calls (the copies are
    then a larger share)."""
    kc = STEPS_PER_BENCH_STEP * args.steps  # FTCS steps per e2e call
    k = 2 if kc >= 5000 else 3
    host_in = torch.empty(n, dtype=torch.float64, pin_memory=True)
    host_out = torch.empty(n, dtype=torch.float64, pin_memory=True)
    plan.download(host_in.numpy())  # a valid (prepared) field to start from
    a_in, a_out = host_in.numpy(), host_out.numpy()

    def c_call(src, dst, steps):
        H._lib.check(H._lib.lib().heat_sync_run(
            H._lib.dptr(src), n, r, bc.kind, bc.c1, bc.c2, steps, steps, H._lib.dptr(dst), None,
            None, 0, None), "heat_sync_run")

    def timed_calls(src, dst, steps, reps):
        ts = []
        for i in range(reps + 1):
            if world == 1:
                t0 = time.perf_counter()
                c_call(src, dst, steps)
                t1 = time.perf_counter()
            else:
                import torch.distributed as dist
                dist.barrier()
                t0 = time.perf_counter()
                plan.upload(src)
                advance(steps)
                plan.download(dst)
                dist.barrier()
                t1 = time.perf_counter()
            if i > 0:
                ts.append(t1 - t0)
        return ts

    times = timed_calls(a_in, a_out, kc, k)
    if world == 1 and not args.skip_parity:  # the last call's output against its input
        from oracle import oracle as O
        from oracle.lightcone import WindowCheck
        port = O.port()
        chk = WindowCheck(n, kc, sync_centres(n))
        chk.capture(lambda lo, c: a_in[lo:lo + c])
        parity["e2e"] = chk.verify(
            lambda lo, c: a_out[lo:lo + c],
            lambda w, lo: port.sync_window(w, lo, n, r, 0.0, 0.0, kc))
    t = statistics.median(times)
    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([t], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
    v = float(n) * world * kc / t / 1e9
    out = {"value": round(v, 3), "unit": UNIT, "h2d_bytes_per_step": 8 * n,
           "d2h_bytes_per_step": 8 * n, "steps": k, "ftcs_steps_per_step": kc,
           "seconds_per_step": round(t, 4),
           "api": "heat_sync_run (C-ABI, pinned host buffers)" if world == 1 else
                  "heat.Plan upload/advance/download per rank"}
    if world == 1:
        # The drop-in caller's case: the reference's API takes std::vector
        # fields (integration/heat_core_b200.cpp passes their data pointers),
        # i.e. PAGEABLE host memory -- the same call with ordinary numpy arrays.
        import numpy as np
        p_in = np.empty(n)
        p_in[:] = a_in
        p_out = np.empty(n)
        pt = timed_calls(p_in, p_out, kc, 2)
        same = bool(np.array_equal(p_out.view(np.uint64), a_out.view(np.uint64)))
        out["pageable"] = {"value": round(float(n) * kc / statistics.median(pt) / 1e9, 3),
                           "unit": UNIT, "steps": len(pt), "same_result_as_pinned": same,
                           "api": "heat_sync_run (C-ABI) with pageable numpy host buffers, "
                                  "as heat::sync_run's std::vector fields arrive"}
        if kc != STEPS_PER_BENCH_STEP:
            t1k = statistics.median(timed_calls(a_in, a_out, STEPS_PER_BENCH_STEP, 3))
            p1k = statistics.median(timed_calls(p_in, p_out, STEPS_PER_BENCH_STEP, 2))
            out["per_call_1000"] = {
                "pinned": round(float(n) * STEPS_PER_BENCH_STEP / t1k / 1e9, 3),
                "pageable": round(float(n) * STEPS_PER_BENCH_STEP / p1k / 1e9, 3), "unit": UNIT,
                "what": "1000-step calls: 8 GiB in and out per 1000 steps (pageable: bound by the "
                        "host's memory bandwidth, DESIGN §5)"}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--skip-bound", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-async", action="store_true")
    ap.add_argument("--skip-parity", action="store_true",
                    help="do not check the timed runs against the oracle's light cones")
    ap.add_argument("--strong", action="store_true",
                    help="cfg4: N = 2^33 in total split over the GPUs (no host-buffer legs)")
    args = ap.parse_args()
    if args.strong:  # the field does not fit the host-buffer legs (e2e, CPU, paper configs)
        args.skip_e2e = args.skip_cpu = args.skip_bound = True
    rank, world, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_b200(args, rank, world, local)


if __name__ == "__main__":
    sys.exit(main())
