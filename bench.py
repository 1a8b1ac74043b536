"""Benchmark: phase-space DOF-updates/s per Strang step (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--impl ours|reference]

Our arm: the full device-resident Strang step (half-x, rho, Poisson, full-v,
half-x, diagnostics) of BASELINE config 2 (Q2, 32^3 velocity cells, N_x=64,
p_x=2, synthetic Landau initial data) on N GPUs, timed with CUDA events on
the launching stream, max over ranks.  f is 1.36 GB (> 126 MB L2), so every
step streams from HBM; no L2 flush needed.

Reference arm (--impl reference): the reference algorithm on the host's CPU
cores (oracle/ port, all threads): whole Strang steps of the full state of the
same config, wall-clock timed (CpuSteps).  The reference is pure Python (nothing
to compile), so the oracle restatement is what runs.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Phase-space DOF-updates/s per Strang step; achieved HBM GB/s vs 8 TB/s"
UNIT = "DOF-updates/s"
CONFIGS = {
    "cfg1": dict(dim=3, n_base=16, levels=0, degree=1, n_x=16),
    "cfg2": dict(dim=3, n_base=32, levels=0, degree=2, n_x=64),
    "cfg3": dict(dim=3, n_base=4, levels=1, degree=2, n_x=64),
    "cfg4": dict(dim=3, n_base=4, levels=2, degree=3, n_x=128),
    "cfg5": dict(dim=3, n_base=48, levels=2, degree=2, n_x=512),
    # cfg4's 4^3 base is 35 MB, launch-bound at 8 GPUs; the scaling
    # claim also uses this larger-base variant (8.1e8 DOFs)
    "cfg4L": dict(dim=3, n_base=32, levels=2, degree=3, n_x=128),
}
NAMES = {
    "cfg1": "1X+3V Landau, 16^3 uniform, Q1, Nx=16",
    "cfg2": "1X+3V Landau damping, uniform 32^3 velocity mesh, Q2 DG, Nx=64, p_x=2",
    "cfg3": "1X+3V Landau, 4^3+AMR1, Q2, Nx=64",
    "cfg4": "1X+3V Landau, 4^3+AMR2, Q3, Nx=128",
    "cfg5": "1X+3V Landau, 48^3+AMR2, Q2, Nx=512",
    "cfg4L": "1X+3V Landau, 32^3+AMR2, Q3, Nx=128 (cfg4 with a 32^3 base)",
}
SWEEP_BYTES_PER_DOF = 16      # read + write each fp64 coefficient once
STEP_BYTES_PER_DOF = 64       # Strang step as structured by Simulation.step (incl. diagnostics)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def ncu_traffic(config, kernel="sweep"):
    """dram bytes per launch of `kernel` ("sweep" | "step_fused") from the committed ncu
    capture (profiles/ncu_summary.json, written by tools/ncu_summary.py), or None."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(path):
        return None
    with open(path) as fh:
        d = json.load(fh)
    ent = d.get(config, {}).get(kernel)
    return None if not ent else ent.get("dram_bytes_per_launch")


class ClockSampler:
    """NVML sampling of SM clock + throttle reasons in a background thread."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index, period=0.01):
        self.samples = []
        self.period = period
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                mhz = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((time.perf_counter(), mhz, rs))
            except Exception:
                pass
            time.sleep(self.period)

    def start(self):
        if self.ok:
            self.th = threading.Thread(target=self._run, daemon=True)
            self.th.start()
        return self

    def stop(self):
        if self.ok:
            self._stop.set()
            self.th.join()

    def summary(self, t0, t1):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        win = [s for s in self.samples if t0 <= s[0] <= t1]
        note = "timed region"
        if len(win) < 3:    # short timed region: widen to the warm-up + timed window
            win = self.samples
            note = "warm-up + timed region"
        mhz = [s[1] for s in win] or [0]
        mask = 0
        for s in win:
            mask |= s[2]
        reasons = [v for k, v in self.REASONS.items() if mask & k]
        return {"sm_mhz": float(np.median(mhz)), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(win), "window": note}


def parallelism_for(config, world):
    """(scaling, parallelism) of our arm at `world` ranks; the reference arm reports the same
    so the two lines carry identical config dicts.  Uniform velocity meshes shard by
    pencils (the fused step's items), AMR meshes by x-slabs; both split
    the same global problem over the ranks (strong scaling)."""
    if world == 1:
        return "weak", "x-slab x1"
    if CONFIGS[config]["levels"] == 0:
        return "strong", f"pencils x{world}"
    return "strong", f"x-slab x{world}"


def config_dict(config, n_v, n_x, parallelism, world=1):
    dofs = n_v * n_x
    per_rank = dofs // max(world, 1)
    return {"workload": NAMES[config], "config_id": config, "phase_dofs": dofs,
            "velocity_dofs": n_v, "x_dofs": n_x, "bc": "absorbing", "dt": 0.1,
            "parallelism": parallelism,
            "l2": ("inputs larger than L2 (state %.2f GB per rank)" % (per_rank * 8 / 1e9)
                   if per_rank * 8 > 126e6 else
                   "state %.1f MB per rank fits in the 126 MB L2, not flushed: a latency/"
                   "throughput figure, not an HBM-roofline one (SURVEY 8d)" % (per_rank * 8 / 1e6)),
            "initial_data": "Landau f=(2pi)^-1.5 exp(-|v|^2/2)(1+0.01cos(0.5x))"}


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2603_19959_b200 as sv
    from paper_2603_19959_b200 import _capi

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfgd = dict(CONFIGS[args.config])
    cfg = sv.SimConfig(**cfgd, n_steps=args.steps)
    scaling, parallelism = parallelism_for(args.config, world)
    if world > 1:
        from paper_2603_19959_b200.shard import PencilShardedSimulation, ShardedSimulation
        if parallelism.startswith("pencils"):
            sim = PencilShardedSimulation(cfg, rank, world)
        else:
            sim = ShardedSimulation(cfg, rank, world)
    else:
        sim = sv.Simulation(cfg)
    n_v = sim.f.shape[0]
    n_x_global = sim.xgrid.n_dofs
    dofs_total = n_v * n_x_global
    dofs_local = dofs_total // world   # pencils: a 1/world share of the items; slabs: ~1/world
    stream = torch.cuda.current_stream()
    rec = torch.empty(5, dtype=torch.float64, device=sim.f.device)
    lib = _capi.lib()

    sampler = ClockSampler(local).start()
    table = torch.empty((max(args.steps, args.warmup), 5), dtype=torch.float64,
                        device=sim.f.device)
    sim.advance(args.warmup, table[:args.warmup])
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    # timed region: K full Strang steps through the pipelined path run() uses, with
    # nothing else in the stream (an event between two kernels would break the
    # programmatic-dependent-launch overlap of the field chain and the fused step)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = lib.sldg_launch_count()
    t_wall0 = time.perf_counter()
    ev0.record(stream)
    sim.advance(args.steps, table[:args.steps])
    ev1.record(stream)
    torch.cuda.synchronize()
    t_wall1 = time.perf_counter()
    launches = lib.sldg_launch_count() - launches0
    if world > 1:
        dist.barrier()
    sampler.stop()
    ms = ev0.elapsed_time(ev1) / args.steps
    # the same K steps again with CUDA events around every v-sweep / fused-step launch
    # (on the launching stream): the dominant kernel's duration for the roofline
    ev_v = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            for _ in range(args.steps)]
    sim.advance(args.steps, table[:args.steps], v_events=ev_v)
    torch.cuda.synchronize()
    # the last step of advance() runs the fused kernel's last-step mode (no second
    # half-x, 16 B/DOF but less work): the roofline averages the steady-state launches
    fused_run = sim.fused_step_supported() and args.steps > 1
    ev_k = ev_v[:-1] if fused_run else ev_v
    sweep_ms = float(np.mean([a.elapsed_time(b) for a, b in ev_k]))
    if world > 1:
        t = torch.tensor([ms, sweep_ms], dtype=torch.float64, device=sim.f.device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, sweep_ms = float(t[0]), float(t[1])
    clocks = sampler.summary(t_wall0, t_wall1)

    # operator breakdown (separate short loop, same stream, CUDA events)
    def timed(fn, reps=3):
        fn()   # untimed first call: scratch allocation, function attributes
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps
    breakdown = {} if world > 1 else {   # single-device operators
        "xx_fused_moments_rho": timed(lambda: sim._xx(rec[2:5])),
        "x_half_plain": timed(sim._advect_x),
        "x_half_rho": timed(sim._lead_x_rho),
        "poisson": timed(lambda: sim.poisson.solve_into(sim._rho, sim._phi, sim._e)),
        "advect_v": timed(lambda: sim._advect_v(sim._e)),
        "rho_standalone": timed(lambda: sim._field(sim._e)),
        "moments_standalone": timed(lambda: sim._diag_into(sim._e, rec)),
    }

    # end to end through the public API with HOST buffers: every step copies the
    # state host->device (pinned), steps, copies it back and reads the record.
    e2e = None
    if world == 1 and not args.no_e2e:
        f_host = torch.empty(sim.f.shape, dtype=torch.float64, pin_memory=True)
        f_host.copy_(sim.f)
        rec_host = torch.empty(5, dtype=torch.float64, pin_memory=True)
        ke = max(2, min(args.steps, 5))
        for it in range(ke + 1):
            if it == 1:
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
            r = sim.step_host(f_host, rec_host)
        b.record(stream)
        torch.cuda.synchronize()
        e_ms = a.elapsed_time(b) / ke
        nbytes = sim.f.numel() * 8
        e2e = {"value": dofs_total / (e_ms * 1e-3), "unit": UNIT, "ms_per_step": e_ms,
               "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes + 40,
               "api": "Simulation.step_host(f_host_pinned): H2D state, Strang step, D2H state "
                      "+ diagnostics record", "record_finite": bool(np.isfinite(r.m0))}

    # the fast-path pencil sweep on its own (the north-star kernel), same state, same stream
    sweep_alone_ms = timed(lambda: sim._advect_v(sim._e), reps=5)
    peak, peak_kind = measured_peaks()
    fused = sim.fused_step_supported()
    algo = SWEEP_BYTES_PER_DOF * dofs_local           # read + write every coefficient once
    algo_sweep = SWEEP_BYTES_PER_DOF * sim.f.numel()  # the stand-alone sweep: whole buffer
    achieved = algo / (sweep_ms * 1e-3) / 1e9
    ach_sweep = algo_sweep / (sweep_alone_ms * 1e-3) / 1e9
    out = {
        "metric": METRIC, "value": dofs_total / (ms * 1e-3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args.config, n_v, n_x_global, parallelism, world),
        "pipeline": ("one HBM pass per step: k_step_fused (v-sweep + trailing half-x + "
                     "moments + next leading half-x + rho), 16 B/DOF" if fused else
                     "v-sweep pass + fused X.X pass (moments, rho), 32 B/DOF"),
        "step_hbm_gbs_at_reference_64B_per_dof":
            STEP_BYTES_PER_DOF * dofs_local / (ms * 1e-3) / 1e9,
        "breakdown_ms": breakdown,
        "roofline": {"bound": "hbm",
                     "timing": ("CUDA events around each launch on its stream, in a second "
                                "K-step advance() right after the timed one (same steps; "
                                "events kept out of the timed region)"),
                     "kernel": ("k_step_fused (dominant kernel of the timed steps)" if fused
                                else "k_level_mats + k_sweep_stream (v-sweep)"),
                     "achieved": achieved, "peak": peak, "peak_kind": peak_kind,
                     "unit": "GB/s", "frac": achieved / peak,
                     "frac_of_8TBs": achieved / 8000.0,
                     "traffic": ncu_traffic(args.config, "step_fused" if fused else "sweep"),
                     "algorithmic_bytes_per_launch": algo, "kernel_ms": sweep_ms},
        "roofline_sweep": {"bound": "hbm",
                           "kernel": "k_level_mats + k_sweep_stream (fast-path pencil sweep)",
                           "achieved": ach_sweep, "peak": peak, "peak_kind": peak_kind,
                           "unit": "GB/s", "frac": ach_sweep / peak,
                           "frac_of_8TBs": ach_sweep / 8000.0,
                           "traffic": ncu_traffic(args.config, "sweep"),
                           "algorithmic_bytes_per_launch": algo_sweep,
                           "kernel_ms": sweep_alone_ms},
        "clocks": clocks, "gpu_launches": int(launches), "e2e": e2e,
    }
    if not args.no_amr:
        # the AMR configurations of the scaling claim (BASELINE configs 4 and 5), each on
        # all N GPUs (x-slab sharding, the same global problem at every N: strong scaling)
        del sim
        torch.cuda.empty_cache()
        out["amr_scaling"] = {}
        for c in (c for c in args.amr_configs.split(",") if c):
            try:
                out["amr_scaling"][c] = time_amr(c, world, rank, args.amr_steps, sv,
                                                 args.amr_slab1)
            except Exception as exc:   # the headline line must still print
                out["amr_scaling"][c] = {"error": f"{type(exc).__name__}: {exc}"[:300]}
                torch.cuda.empty_cache()
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline_1core(args.config)
    if world > 1:
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(out))


def time_amr(config, world, rank, steps, sv, slab1=False):
    """ms per Strang step of `config` on `world` GPUs: Simulation at N = 1, x-slab
    ShardedSimulation (NCCL halo exchange overlapped with the X.X pass) at N > 1.
    CUDA events on the launching stream after 2 warm-up steps, max over ranks."""
    import torch
    import torch.distributed as dist
    cfg = sv.SimConfig(**CONFIGS[config], n_steps=steps)
    t0 = time.perf_counter()
    if world > 1 or slab1:
        from paper_2603_19959_b200.shard import ShardedSimulation
        sim = ShardedSimulation(cfg, rank, world)
        par = f"x-slab x{world}" + (" (sharded path)" if world == 1 else "")
    else:
        sim = sv.Simulation(cfg)
        par = "x-slab x1"
    setup_s = time.perf_counter() - t0
    sim.advance(2)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    table = sim.advance(steps)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t[0])
    n_v = len(sim.vweights)
    dofs = n_v * sim.xgrid.n_dofs
    fin = bool(torch.isfinite(table).all().item())
    del sim
    torch.cuda.empty_cache()
    return {"workload": NAMES[config], "n_gpus": world, "scaling": "strong",
            "parallelism": par, "phase_dofs": dofs, "steps": steps, "warmup": 2,
            "ms_per_step": ms, "value": dofs / (ms * 1e-3), "unit": UNIT,
            "setup_s": setup_s, "records_finite": fin,
            "timing": "CUDA events around advance(steps) on the launching stream, max over ranks"}


class CpuSteps:
    """The reference algorithm (oracle/sldg_oracle.py, a numpy restatement of the reference
    package, which is pure Python) stepping the FULL state of the config: each step is one
    whole Strang step (half-x, rho + Poisson + E, v-sweep over every column, half-x,
    diagnostics), timed by wall clock.  `workers` threads over columns / speed groups,
    exactly like the reference's ThreadPoolExecutor (vsweep.py:436-440, xfield.py:101-103),
    BLAS pinned to one thread (SURVEY.md §8(d) protocol)."""

    def __init__(self, config, workers):
        from oracle import sldg_oracle as so
        self.config = config
        self.workers = workers
        cfgd = CONFIGS[config]
        t0 = time.perf_counter()
        self.sim = so.Sim(dim=cfgd["dim"], n_base=cfgd["n_base"], levels=cfgd["levels"],
                          degree=cfgd["degree"], n_x=cfgd["n_x"], workers=workers)
        self.setup_s = time.perf_counter() - t0
        self.n_v, self.n_x = self.sim.f.shape

    def step(self):
        from threadpoolctl import threadpool_limits
        with threadpool_limits(limits=1):
            t0 = time.perf_counter()
            self.sim.step()
            return time.perf_counter() - t0

    def describe(self, n_steps):
        return (f"oracle/sldg_oracle.py (reference algorithm, numpy) Sim.step() on the full "
                f"{self.config} state ({self.n_v} x {self.n_x}): {n_steps} whole Strang "
                f"step(s), {self.workers} worker thread(s), BLAS 1 thread; setup "
                f"{self.setup_s:.1f}s excluded")


def cpu_baseline_1core(config):
    """One full Strang step at 1 core (the GPU arm's cpu_baseline)."""
    cs = CpuSteps(config, workers=1)
    t = cs.step()
    return {"value": cs.n_v * cs.n_x / t, "unit": UNIT, "cores": 1, "kind": "port",
            "ms_per_step": t * 1e3, "sample": cs.describe(1)}


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    workers = os.cpu_count() or 1
    t_start = time.perf_counter()
    cs = CpuSteps(args.config, workers)
    warm = args.warmup
    times = []
    for k in range(args.warmup + args.steps):
        t = cs.step()
        if k == 0 and (args.warmup + args.steps) * t > args.cpu_budget:
            # keep the whole run within a few minutes: the CPU needs no warm-up beyond
            # the first step (no JIT, no clocks to ramp)
            warm = 1
        if k < warm:
            continue
        times.append(t)
        if len(times) == args.steps:
            break
    t_wall = time.perf_counter() - t_start
    ms = float(np.mean(times)) * 1e3
    dofs = cs.n_v * cs.n_x
    value = dofs / (ms * 1e-3)
    scaling, parallelism = parallelism_for(args.config, world)
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": len(times),
           "warmup": warm, "ms_per_step": ms, "higher_is_better": True,
           "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "impl": "reference",
           "config": config_dict(args.config, cs.n_v, cs.n_x, parallelism),
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "kind": "port",
                            "sample": cs.describe(len(times))},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0},
           "wall_s": t_wall, "timing": "wall clock per whole step, mean over the timed steps"}
    print(json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-amr", action="store_true",
                    help="skip the AMR scaling lines (configs 4 and 5 on the same N GPUs)")
    ap.add_argument("--amr-configs", default="cfg4,cfg4L,cfg5")
    ap.add_argument("--amr-steps", type=int, default=10)
    ap.add_argument("--amr-slab1", action="store_true",
                    help="at N = 1 run the AMR lines through the sharded (x-slab) path")
    ap.add_argument("--cpu-budget", type=float, default=240.0,
                    help="reference arm: seconds for warm-up + timed steps before the "
                         "warm-up is cut to one step")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
