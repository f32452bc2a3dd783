#!/usr/bin/env python3
"""Benchmark of the FTCS hot path (BASELINE.json metric: FP64 lattice updates/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Workload (BASELINE.json configs[2], "cfg3"): N = 2^30 FP64 points per GPU,
r = from_r(0.4), Dirichlet(0,0), sine initial profile, 10^4 FTCS time steps.
One bench STEP = 1000 FTCS time steps over the whole field, so the default
--steps 10 is exactly the cfg3 run.  For N > 1 GPUs (torchrun, one rank per
GPU) each rank owns a 2^30-point slab of a G*2^30 domain (weak scaling; at
G = 8 the total is cfg4's 2^33) and exchanges heat_slab_halo()-point ghosts
(64) with its neighbours every pass of as many steps.

Arms
  b200       the sm_100a kernels (libheat_b200.so) -- value is device-timed
             with inputs resident in HBM; e2e is timed through the C-ABI
             (heat_sync_run with pinned host buffers, copies included).
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
CPU_SAMPLE_STEPS = 32  # ~5 s timed (+ ~8 s of the API's own 8 GiB copies) per sample at N = 2^30


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
        return d.get("sync_tb_kernel", {}).get("dram_bytes_per_launch")
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


def cpu_baseline_run(n: int, steps: int, warm: bool = True):
    """The reference's exec_run(Barriered) on all host threads (oracle/_ref),
    or the C port's threaded executor when the reference library is absent.
    Returns (GLUPS, cores, kind, sample description)."""
    from oracle import oracle as O
    port = O.port()
    u0 = _CPU_FIELDS.get(n)
    if u0 is None:  # 8 GiB at N = 2^30: built once per process, reused by every sample
        u0 = port.sine_init(n)
        u0[0] = 0.0
        u0[-1] = 0.0
        _CPU_FIELDS[n] = u0
    kind = "reference" if O.Ref.available() else "port"
    eng = O.ref() if kind == "reference" else port
    hw = os.cpu_count() or 1
    if kind == "reference":
        hw = eng.hardware_concurrency() or hw
    workers = 1
    while workers * 2 <= hw and n % (workers * 2) == 0:
        workers *= 2
    if kind == "reference":
        fin, dur, _ = eng.exec_run(u0, R, O.DIRICHLET, 0.0, 0.0, n // workers, workers, steps,
                                   O.BARRIERED)
    else:
        fin, dur = eng.exec_run(u0, R, O.DIRICHLET, 0.0, 0.0, n // workers, workers, steps,
                                O.BARRIERED)
    glups = n * steps / (dur * 1e-9) / 1e9
    sample = (f"N=2^{n.bit_length() - 1} FP64, {steps} FTCS steps, exec_run(Barriered) with P={workers} "
              f"threads; time = exec_run's own duration (thread spawn..join, async_exec.cpp:101-106)")
    return glups, workers, kind, sample


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    n = N_PER_GPU
    vals = []
    info = None
    for i in range(args.warmup + args.steps):
        g, cores, kind, sample = cpu_baseline_run(n, CPU_SAMPLE_STEPS)
        if i >= args.warmup:
            vals.append(g)
        info = (cores, kind, sample)
    v = statistics.median(vals)
    ms = n * CPU_SAMPLE_STEPS / (v * 1e9) * 1e3 * (STEPS_PER_BENCH_STEP / CPU_SAMPLE_STEPS)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(v, 4), "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (sine IC)",
        "config": config_dict(world),
        "cpu_baseline": {"value": round(v, 4), "unit": UNIT, "cores": info[0], "kind": info[1],
                         "sample": info[2] + f"; median of {args.steps} samples"},
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
        return (f"sync_tb_kernel<double,{k['V']},{k['buffers']},0,H={k['steps_per_pass']}> "
                f"(temporal-blocked: {k['V']}-point lanes, {k['steps_per_pass']}-point halo, "
                f"{k['exact']} exact points per warp tile, {k['steps_per_pass']} steps per HBM pass)")
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


def config_dict(world, n=N_PER_GPU, strong=False):
    if strong:
        work = (f"cfg4: N=2^33 FP64 in total ({n} points per GPU), r=0.4, Dirichlet(0,0), "
                f"sine IC, 1000-step bench steps; strong scaling over {world} GPU(s)")
    else:
        work = ("cfg3: N=2^30 FP64 per GPU, r=0.4, Dirichlet(0,0), sine IC, "
                "10^4 FTCS steps (= 10 bench steps of 1000)" +
                ("" if world == 1 else f"; {world}-GPU slab decomposition, N=2^30*{world}"))
    return {
        "workload": work,
        "N_per_gpu": n, "N_total": n * world, "r": R,
        "time_steps_per_bench_step": STEPS_PER_BENCH_STEP, "steps_per_pass": (steps_per_pass() if world == 1
                           else min(steps_per_pass(), slab_halo())),
        "kernel": sync_kernel_name(),
        "l2": "inputs larger than L2 (8 GiB per array vs 126 MB L2)",
        "parallelism": "single GPU" if world == 1 else f"slab x{world} (NCCL halo exchange)",
    }


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
        solver = MG.SlabSolver(n, r, bc, local, rank, world)
        solver.plan.fill_sine()  # each slab gets a sine profile (data-independent cost)
        plan = solver.plan

        def advance(k):
            solver.advance(k)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        advance(STEPS_PER_BENCH_STEP)
    plan.synchronize()
    barrier()

    launches0 = H.kernel_launches()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            advance(STEPS_PER_BENCH_STEP)
        e1.record(stream)
        barrier()
    plan.synchronize()
    launches = H.kernel_launches() - launches0
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    total_updates = float(n) * world * STEPS_PER_BENCH_STEP * args.steps
    glups = total_updates / (ms * 1e-3) / 1e9

    # Roofline of the dominant kernel (sync_tb_kernel, one launch per pass of
    # <= steps_per_pass() steps, e.g. 31 passes of 32 + one of 8 per 1000 steps).
    # achieved = algorithmic bytes of all its launches / their device time;
    # the timed region is nothing but those back-to-back launches.
    # multi-GPU slabs exchange heat_slab_halo() ghosts: passes of at most as many steps
    spp = steps_per_pass() if world == 1 else min(steps_per_pass(), slab_halo())
    passes_per_step = -(-STEPS_PER_BENCH_STEP // spp)
    sync_launches = passes_per_step * args.steps
    per_launch_s = ms * 1e-3 / sync_launches
    alg_bytes_total = BYTES_PER_UPDATE * float(n) * STEPS_PER_BENCH_STEP * args.steps
    alg_bytes = alg_bytes_total / sync_launches  # per launch (average)
    peak, peak_kind = measured_peaks()
    achieved = alg_bytes / per_launch_s / 1e9
    fp64_peak = 148 * 64 * 1.965e9 / 1e12  # DP lanes x SMs x boost clock, T ops/s (nominal)
    fp64_achieved = FP64_OPS_PER_UPDATE * float(n) * STEPS_PER_BENCH_STEP * args.steps / (
        ms * 1e-3) / 1e12
    roofline = {
        "bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
        "frac": round(achieved / peak, 4),
        # the capture is one pass over 2^30 points; DRAM bytes scale with the points
        "traffic": (None if ncu_traffic_per_launch() is None
                    else ncu_traffic_per_launch() * n / N_PER_GPU),
        "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
        "algorithmic_bytes_per_launch": alg_bytes,
        "note": "effective bandwidth with temporal blocking (16 B/update counted for every "
                "step); the pass itself is FP64-pipe bound, see fp64",
        "fp64": {"ops_per_update": FP64_OPS_PER_UPDATE, "achieved_tops": round(fp64_achieved, 3),
                 "peak_tops_nominal": round(fp64_peak, 3),
                 "frac": round(fp64_achieved / fp64_peak, 4)},
    }

    # Asynchronous scheme on the same workload (single GPU): K5 streaming
    # kernel, PEs of 2^21 points, free-running with delays <= 7 and the
    # deterministic replay of a seeded q=2 stream.
    async_info = None
    if world == 1 and not args.skip_async:
        async_info = run_async(args, H, torch, plan, stream, n, r, bc, glups)
    elif world > 1 and not args.skip_async:
        try:
            async_info = run_async_multi(args, H, MG, torch, stream, n, r, bc, glups, rank, world,
                                         local)
        except Exception as exc:  # report, do not lose the sync line
            async_info = {"error": f"{type(exc).__name__}: {exc}"[:300]}

    # End to end through the public API with host buffers (copies timed).
    e2e = None
    if not args.skip_e2e:
        e2e = run_e2e(args, H, torch, n, r, bc, rank, world, plan, advance)

    cpu = None
    if rank == 0 and world == 1 and not args.skip_cpu:
        g, cores, kind, sample = cpu_baseline_run(n, CPU_SAMPLE_STEPS)
        cpu = {"value": round(g, 4), "unit": UNIT, "cores": cores, "kind": kind,
               "sample": sample}

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
        "config": config_dict(world, n, args.strong),
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


def run_async(args, H, torch, plan, stream, n, r, bc, sync_glups):
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
        e0.record(stream)
        stats = [call() for _ in range(args.steps)]
        e1.record(stream)
        plan.synchronize()
        ms = e0.elapsed_time(e1)
        v = float(n) * STEPS_PER_BENCH_STEP * args.steps / (ms * 1e-3) / 1e9
        st = stats[-1]
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
    return out


def run_async_multi(args, H, MG, torch, stream, n, r, bc, sync_glups, rank, world, local):
    """G-GPU legs over NVLink P2P (heat_plan_xlink_*): each rank runs K5 on its
    2^30-point slab; PE boundaries between GPUs exchange edge values by P2P
    stores into the neighbour's receive rings.  q=1 free mode is the exact
    synchronous scheme with no collective in the loop; q=8 free-running."""
    import torch.distributed as dist
    per_pe = n // ASYNC_PES
    out = {"pes_per_gpu": ASYNC_PES, "points_per_pe": per_pe,
           "transport": "P2P stores into IPC-mapped neighbour receive rings (NVLink)"}
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    for name, q in (("sync_p2p", 1), ("free", 8)):
        solver = MG.AsyncSlabSolver(n, per_pe, q, bc, local, rank, world)
        solver.plan.fill_sine()
        for _ in range(max(1, args.warmup)):
            solver.advance(r, STEPS_PER_BENCH_STEP)
        torch.cuda.synchronize()
        dist.barrier()
        e0.record(stream)
        st = None
        for _ in range(args.steps):
            st = solver.advance(r, STEPS_PER_BENCH_STEP)
        e1.record(stream)
        solver.plan.synchronize()
        ms = e0.elapsed_time(e1)
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        v = float(n) * world * STEPS_PER_BENCH_STEP * args.steps / (ms * 1e-3) / 1e9
        out[name] = {"value": round(v, 3), "unit": UNIT, "q": q,
                     "max_delay": int(st.max_delay), "reads_per_run": int(st.reads),
                     "vs_sync_nccl_halo": round(v / sync_glups, 4)}
        solver.plan.close()
    return out


def run_e2e(args, H, torch, n, r, bc, rank, world, plan, advance):
    """Same metric through the public API with HOST buffers: per step the
    pinned host field goes H2D, 1000 FTCS steps run, the result comes back D2H."""
    k = max(1, min(args.steps, 3))
    host_in = torch.empty(n, dtype=torch.float64, pin_memory=True)
    host_out = torch.empty(n, dtype=torch.float64, pin_memory=True)
    plan.download(host_in.numpy())  # a valid (prepared) field to start from
    a_in, a_out = host_in.numpy(), host_out.numpy()
    times = []
    for i in range(k + 1):
        if world == 1:
            t0 = time.perf_counter()
            H._lib.check(H._lib.lib().heat_sync_run(
                H._lib.dptr(a_in), n, r, bc.kind, bc.c1, bc.c2, STEPS_PER_BENCH_STEP,
                STEPS_PER_BENCH_STEP, H._lib.dptr(a_out), None, None, 0, None), "heat_sync_run")
            t1 = time.perf_counter()
        else:
            import torch.distributed as dist
            dist.barrier()
            t0 = time.perf_counter()
            plan.upload(a_in)
            advance(STEPS_PER_BENCH_STEP)
            plan.download(a_out)
            dist.barrier()
            t1 = time.perf_counter()
        if i > 0:
            times.append(t1 - t0)
    t = statistics.median(times)
    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([t], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
    v = float(n) * world * STEPS_PER_BENCH_STEP / t / 1e9
    return {"value": round(v, 3), "unit": UNIT, "h2d_bytes_per_step": 8 * n,
            "d2h_bytes_per_step": 8 * n, "steps": k,
            "api": "heat_sync_run (C-ABI, pinned host buffers)" if world == 1 else
                   "heat.Plan upload/advance/download per rank"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-async", action="store_true")
    ap.add_argument("--strong", action="store_true",
                    help="cfg4: N = 2^33 in total split over the GPUs (no host-buffer legs)")
    args = ap.parse_args()
    if args.strong:  # the field does not fit the host-buffer legs (e2e, CPU, paper configs)
        args.skip_e2e = args.skip_cpu = True
    rank, world, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_b200(args, rank, world, local)


if __name__ == "__main__":
    sys.exit(main())
