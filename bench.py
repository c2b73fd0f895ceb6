"""Throughput benchmark of the B200 VP-FV RK4 step (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--workload landau2d-128]

Metric (BASELINE.json): phase-space cell-updates per second per RK4 step
(sum over species of interior cells / wall time of one RK4 step; a step is 4
fused stages + moments + rho + Poisson + tables, the per-step non-finite check
included).  Default workload: 2D-2V Landau damping 128^2 x 128^2, fp64
(config 4), fixed dt = 0.9 * max_dt at t = 0.  Inputs
(2.58 GB per buffer) are far larger than L2, so no flush is needed.

Multi-GPU (torchrun, one rank per GPU): the same global problem is split
along x across ranks (strong scaling) by paper_2410_12155_b200.parallel.

``--impl reference`` times the reference algorithm on the host cores: the
threaded C restatement of the reference kernels in oracle/ (bitwise equal to
the reference numba kernels; the reference itself is pure Python and absent
on the GPU box), rank 0 only.
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

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (config description, builder args)
    "landau2d-128": "2D2V Landau damping 128^2 x 128^2, single electron species (BASELINE config 4)",
    "landau1d-128": "1D1V Landau damping 128 x 128, alpha = 0.01 (BASELINE config 1)",
    "landau2d-64": "2D2V Landau damping 64^2 x 64^2 (reduced, for quick runs)",
    "landau2d-32": "2D2V Landau damping 32^2 x 32^2 (single-core numpy CPU-leg sample only)",
    "twostream-1024": "1D1V two-stream 1024 x 1024 (BASELINE config 2)",
    "weibel-256": "1D2V bi-Maxwellian 256^3 (BASELINE config 3)",
    "ep2d2v-64": "2D2V electron-proton m_r=1836, 64^4 per species (BASELINE config 5, per GPU)",
}

KERNEL_OF = {  # the dominant (stage) kernel of each workload
    "landau2d-128": "stage2d2v_rb_kernel (fused 2D-2V RHS + RK4 update, TMA-tiled)",
    "landau2d-64": "stage2d2v_rb_kernel (fused 2D-2V RHS + RK4 update, TMA-tiled)",
    "landau2d-32": "stage2d2v_rb_kernel (fused 2D-2V RHS + RK4 update, TMA-tiled)",
    "ep2d2v-64": "stage2d2v_rb_kernel (fused 2D-2V RHS + RK4 update, TMA-tiled)",
    "weibel-256": "stage1d2v_rb_kernel (fused 1D-2V RHS + RK4 update, TMA-tiled)",
    "twostream-1024": "stage_1d1v_march_kernel (fused 1D-1V RHS + RK4 update, x-marching, bulk-copied rows)",
    "landau1d-128": "stage_1d1v_kernel (fused 1D-1V RHS + RK4 update)",
}

STAGE_BYTES = (16, 24, 24, 32)  # algorithmic bytes/cell of RK stages 1..4


WEAK = {"ep2d2v-64"}  # per-GPU box fixed: the global x extent grows with the rank count (BASELINE config 5)


def make_setup(name, world=1, device=None):
    """The workload's set-up; ``device``: padded arrays built on the GPU
    (problems.separable_on_device, bitwise the host builder)."""
    from paper_2410_12155_b200 import problems as P

    kw = {"device": device}
    if name == "landau2d-128":
        return P.make_problem(P.landau_spec(), 128, 128, **kw)
    if name == "landau1d-128":
        return P.make_landau_1d(P.landau_spec(alpha=0.01), 128, 128, **kw)
    if name == "landau2d-64":
        return P.make_problem(P.landau_spec(), 64, 64, **kw)
    if name == "landau2d-32":
        return P.make_problem(P.landau_spec(), 32, 32, **kw)
    if name == "twostream-1024":
        return P.make_problem(P.ProblemSpec("two-stream"), 1024, 1024, **kw)
    if name == "weibel-256":
        return P.make_bimaxwellian_1d2v(256, 256, 256, **kw)
    if name == "ep2d2v-64":  # 64^4 per species per GPU; N ranks hold N x-slabs of 64 planes
        return P.make_electron_proton_2d2v((64 * world, 64), (64, 64), **kw)
    raise ValueError(name)


PROFILE_SUMMARY = os.path.join(ROOT, "profiles", "r2_rb_summary.json")


def load_traffic():
    """Per-launch DRAM bytes of the stage kernel from the committed ncu --set full
    captures (mean over the four RK stages), with the capture it came from."""
    try:
        with open(PROFILE_SUMMARY) as f:
            caps = json.load(f)["captures"]
        vals = [c["traffic_bytes"] for c in caps if c.get("traffic_bytes")]
        return (sum(vals) / len(vals) if vals else None), os.path.relpath(PROFILE_SUMMARY, ROOT)
    except (OSError, KeyError, ValueError):
        return None, None


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)

REASON_BITS = {
    0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
    0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
    0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
}


class ClockSampler:
    """SM clock and clock-event reasons sampled through NVML every few ms while
    the timed region runs (nvidia-smi as a fallback when pynvml is missing)."""

    def __init__(self, gpu_index, period_s=0.005):
        self.gpu = gpu_index
        self.period = period_s
        self.samples = []
        self._stop = threading.Event()
        self._thread = None
        self._proc = None
        self.power_limit_w = None
        self._viol0 = None
        self.violations_ms = None

    def _violations(self, pynvml, h):
        """Cumulative time (ns) the driver held clocks down for power / thermal
        reasons: NVML violation counters, which a sparse reason sample can miss."""
        out = {}
        for name, pol in (("power", pynvml.NVML_PERF_POLICY_POWER), ("thermal", pynvml.NVML_PERF_POLICY_THERMAL),
                          ("reliability", pynvml.NVML_PERF_POLICY_RELIABILITY)):
            try:
                out[name] = int(pynvml.nvmlDeviceGetViolationStatus(h, pol).violationTime)
            except pynvml.NVMLError:
                pass
        return out

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            smax = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            try:
                self.power_limit_w = pynvml.nvmlDeviceGetEnforcedPowerLimit(h) / 1e3
            except pynvml.NVMLError:
                self.power_limit_w = None
            self._nvml, self._h = pynvml, h
            self._viol0 = self._violations(pynvml, h)

            def poll():
                while not self._stop.is_set():
                    try:
                        try:
                            pw = pynvml.nvmlDeviceGetPowerUsage(h) / 1e3
                        except pynvml.NVMLError:
                            pw = None
                        self.samples.append((float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)),
                                             float(smax),
                                             int(pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)), pw))
                    except pynvml.NVMLError:
                        pass
                    self._stop.wait(self.period)

            self._thread = threading.Thread(target=poll, daemon=True)
            self._thread.start()
        except Exception:  # noqa: BLE001 -- no NVML: fall back to nvidia-smi
            try:
                self._proc = subprocess.Popen(
                    ["nvidia-smi", "-i", str(self.gpu),
                     "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                     "--format=csv,noheader,nounits", "-lms", "100"],
                    stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
                self._thread = threading.Thread(target=self._read, daemon=True)
                self._thread.start()
            except (OSError, ValueError):
                self._proc = None
        return self

    def _read(self):
        for line in self._proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 3:
                try:
                    self.samples.append((float(parts[0]), float(parts[1]), int(parts[2], 16), None))
                except ValueError:
                    pass

    def __exit__(self, *exc):
        self._stop.set()
        if self._viol0 is not None:
            v1 = self._violations(self._nvml, self._h)
            self.violations_ms = {k: (v1[k] - self._viol0[k]) / 1e6 for k in v1 if k in self._viol0}
        if self._proc is not None:
            self._proc.terminate()
            try:
                self._proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self._proc.kill()
        if self._thread is not None:
            self._thread.join(timeout=5)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [s[0] for s in self.samples]
        reasons = set()
        for _, _, bits, _ in self.samples:
            for b, n in REASON_BITS.items():
                if bits & b and n != "gpu_idle":
                    reasons.add(n)
            unknown = bits & ~sum(REASON_BITS)
            if unknown:
                reasons.add(f"unmapped_bits_{unknown:#x}")
        out = {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(s[1] for s in self.samples),
               "reasons": sorted(reasons), "samples": len(sm), "sm_mhz_min": min(sm)}
        if self.violations_ms is not None:
            # time the driver spent holding clocks down while the region ran
            out["violation_ms"] = {k: round(v, 3) for k, v in self.violations_ms.items()}
            if self.violations_ms.get("power", 0.0) > 0.0:
                reasons.add("sw_power_cap")
            out["reasons"] = sorted(reasons)
        pw = [s[3] for s in self.samples if s[3] is not None]
        if pw:  # board power while the step runs: a kernel held at the power limit clocks below max
            out["power_w_median"] = statistics.median(pw)
            out["power_w_max"] = max(pw)
            out["power_limit_w"] = self.power_limit_w
        return out


# ---------------------------------------------------------------------------
# CPU baseline: the threaded C restatement of the reference (oracle/)


def cpu_reference_steps(setup, dt, steps, budget_s=60.0):
    """Time RK4 steps of the oracle's C restatement; returns (cells/s, info)."""
    from oracle import cbackend as C

    grids = [f.grid for f in setup.dists]
    sim = C.CSimulation(grids, setup.species, [np.array(f.data) for f in setup.dists], dt=dt)
    cells = sum(int(np.prod(g.N)) for g in grids)
    t0 = time.perf_counter()
    sim.advance(dt)  # first step also warms the C library / page-faults the buffers
    first = time.perf_counter() - t0
    n = max(1, min(steps, int(budget_s / max(first, 1e-9))))
    t0 = time.perf_counter()
    for _ in range(n):
        sim.advance(dt)
    el = time.perf_counter() - t0
    return cells * n / el, dict(steps=n, seconds=el, cores=C.num_threads())


# ---------------------------------------------------------------------------
# B200 arm


def run_b200(args, rank, world, device):
    import torch

    from paper_2410_12155_b200 import runner as R
    from paper_2410_12155_b200.kernels import stream_handle  # noqa: F401

    import torch as _t

    t0 = time.perf_counter()
    setup = make_setup(args.workload, world, device=device if world == 1 else None)
    _t.cuda.synchronize(device)
    setup_s = time.perf_counter() - t0
    if world > 1:
        from paper_2410_12155_b200.parallel import DistributedSimulation

        halo = args.halo
        if halo == "auto":  # the fused NVLink push where it applies, else NCCL send/recv
            ok = (args.velocity_parts == 1 and all(f.grid.v == 2 for f in setup.dists)
                  and setup.dists[0].grid.N[0] % world == 0)
            halo = "peer" if ok else "nccl"
        try:
            sim = DistributedSimulation(setup, dt=None, device=device, velocity_parts=args.velocity_parts, halo=halo)
        except Exception as e:  # noqa: BLE001 -- e.g. no peer access between these GPUs
            if halo != "peer" or args.halo == "peer":
                raise
            print(f"[bench] halo='peer' unavailable ({e}); using NCCL send/recv", file=sys.stderr)
            halo = "nccl"
            sim = DistributedSimulation(setup, dt=None, device=device, velocity_parts=args.velocity_parts, halo=halo)
        args.halo_used = halo
        dt = 0.9 * sim.max_dt()
        sim.fixed_dt = dt
    else:
        sim = R.Simulation(setup, device=device)
        dt = 0.9 * sim.max_dt()
        sim.fixed_dt = dt
    cells_global = sum(int(np.prod(f.grid.N)) for f in setup.dists)
    cells_local = sim.local_cells() if hasattr(sim, "local_cells") else cells_global
    stream = torch.cuda.current_stream(device)

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize(device)

    # The timed region replays the plain step graph.  The stage kernels'
    # launch durations come from CUDA events captured around every stage
    # launch into the graph, in a second pass of the same K steps: those event
    # nodes cost ~8 us each on a 1D step (+60% at 128^2) and break up the
    # concurrent species branches of a two-species step (+13% on ep2d2v-64).
    sim.enable_stage_timing(False)
    for _ in range(args.warmup):
        sim.advance(dt)
    barrier()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    marks = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with ClockSampler(device.index) as clocks:
        start.record(stream)
        marks[0].record(stream)
        for k in range(args.steps):
            sim.advance(dt)
            marks[k + 1].record(stream)
        stop.record(stream)
        barrier()
        ms_local = start.elapsed_time(stop)
    per_step = sorted(marks[k].elapsed_time(marks[k + 1]) for k in range(args.steps))
    sim.enable_stage_timing(True)
    sim.advance(dt)  # captures the evented graph variant
    sim.enable_stage_timing(True)  # reset the accumulators
    barrier()
    time.sleep(1.0)  # let the power limiter recover (sw_power_cap) so both passes start alike
    barrier()
    with ClockSampler(device.index) as clocks_rp:
        start.record(stream)
        for _ in range(args.steps):
            sim.advance(dt)
        stop.record(stream)
        barrier()
        ms_roofline_pass = start.elapsed_time(stop)
    stage_ms = sim.stage_kernel_ms()  # per RK stage slot, summed over the pass's steps and species
    sim.enable_stage_timing(False)
    launches_per_step = sim.launches_per_step()
    p2p = measured_p2p_gbs(device, world) if world > 1 and rank == 0 else None
    nvlink = nvlink_line(sim, world, ms_local / args.steps, p2p)
    ms = ms_local
    if world > 1:
        t = torch.tensor([ms_local], dtype=torch.float64, device=device)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    value = cells_global * args.steps / (ms / 1e3)
    q = lambda f: per_step[min(len(per_step) - 1, int(f * len(per_step)))]  # noqa: E731
    step_stats = {"median_ms": statistics.median(per_step), "p10_ms": q(0.1), "p90_ms": q(0.9),
                  "min_ms": per_step[0], "max_ms": per_step[-1], "rank": rank,
                  "how": "CUDA events between consecutive steps of the timed region (rank 0's stream)"}

    # roofline of the dominant kernel (the fused stage), from in-graph events
    stage_bytes = sum(b * cells_local for b in STAGE_BYTES) * args.steps
    stage_s = sum(stage_ms) / 1e3
    peak, peak_kind = load_peaks()
    traffic, traffic_src = load_traffic()
    if args.workload != "landau2d-128" or world != 1:  # the capture is of that configuration
        traffic, traffic_src = None, None
    achieved = stage_bytes / stage_s / 1e9 if stage_s > 0 else None
    share = stage_s / (ms_local / 1e3)
    per_stage = [{"stage": k + 1, "ms": m / args.steps, "algorithmic_bytes_per_cell": STAGE_BYTES[k],
                  "hbm_frac": (STAGE_BYTES[k] * cells_local * args.steps / (m / 1e3) / 1e9 / peak) if m > 0 else None}
                 for k, m in enumerate(stage_ms)]
    fp64 = fp64_roofline(args.workload, stage_ms, cells_local, args.steps)

    # end to end through the public API with host buffers:
    # H2D of the step's input state from pinned memory, step, D2H of the result
    e2e = None
    if rank == 0 and world == 1 and args.e2e_steps > 0:
        # at least ~50 ms of wall clock, so host jitter does not dominate a short step
        e2e = e2e_measure(sim, dt, max(args.e2e_steps, min(2000, int(50.0 / max(ms_per_step, 1e-3)))), device,
                          cells_global)

    e2e_dropin = None
    if rank == 0 and world == 1 and args.e2e_steps > 0 and len(setup.dists) == 1:
        E_host = sim._E_host(sim.ctx.f0)
        h0 = sim._host_state()[0]
        del sim
        torch.cuda.empty_cache()
        e2e_dropin = e2e_dropin_measure(setup, h0, E_host, dt, device, cells_global)

    cpu, parity, host_setup_s = None, None, None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sim = None
        parity = parity_check(args.workload, dt, device)
        t0 = time.perf_counter()
        host_setup = make_setup(args.workload)
        host_setup_s = time.perf_counter() - t0
        v, info = cpu_reference_steps(host_setup, dt, 2, budget_s=args.cpu_budget)
        del host_setup
        legs = cpu_legs(args.workload)
        cpu = {"value": v, "unit": "cell-updates/s", "cores": info["cores"], "kind": "port",
               "sample": f"{info['steps']} full RK4 step(s) of the same {args.workload} problem "
                         f"({info['seconds']:.1f} s), threaded C restatement of the reference kernels "
                         f"(oracle/stage_ref.c, bitwise = reference numba) + numpy FFT; built -O3 without "
                         f"-march (portable baseline)", "single_core_legs": legs}
    launches = launches_per_step * args.steps
    line = {
        "metric": "phase-space cell-updates/sec per RK4 step",
        "value": value, "unit": "cell-updates/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak" if args.workload in WEAK else "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": args.workload, "description": WORKLOADS[args.workload],
                   "cells": cells_global, "dt": dt, "l2": l2_note(setup),
                   "halo": getattr(args, "halo_used", None),
                   "parallelism": (f"x-slab x{world // args.velocity_parts}, vx x{args.velocity_parts}"
                                   if world > 1 else "single GPU")},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                     "traffic_source": traffic_src,
                     "algorithmic_bytes_per_launch": sum(b * cells_local for b in STAGE_BYTES) / 4,
                     "kernel": KERNEL_OF[args.workload],
                     "algorithmic_bytes_per_cell_per_step": sum(STAGE_BYTES),
                     "stage_ms_per_step": [m / args.steps for m in stage_ms],
                     "share_of_step": share, "peak_kind": peak_kind,
                     "per_stage": per_stage, "fp64": fp64,
                     "fp64_frac": fp64["frac"] if fp64 else None,
                     "timing": (f"stage-kernel launch durations from CUDA events captured around every "
                                f"stage launch in a second pass of the same {args.steps} steps, right after "
                                f"the timed region, under the same clock sampling "
                                f"({ms_roofline_pass / args.steps:.3f} ms/step with the event nodes; the "
                                f"timed region replays the plain graph)"),
                     "clocks_roofline_pass": clocks_rp.summary()},
        "step_roofline": {"achieved_GBs": 96 * cells_local * args.steps / (ms_local / 1e3) / 1e9,
                          "frac": 96 * cells_local * args.steps / (ms_local / 1e3) / 1e9 / peak},
        "step_stats": step_stats,
        "e2e": e2e, "e2e_dropin": e2e_dropin, "cpu_baseline": cpu,
        "setup": {"built_on": "device" if world == 1 else "host", "seconds": setup_s, "host_build_seconds": host_setup_s,
                  "how": "make_problem factor arrays on the host, the padded product on the GPU "
                         "(vpfv_init_separable, bitwise the host builder); host_build_seconds: the numpy "
                         "builder of the same set-up (built for the cpu_baseline leg)"}, "parity": parity, "gpu_launches": launches,
        "nvlink": nvlink,
        "clocks": clocks.summary(),
    }
    return line


FP64_PEAK_FILE = os.path.join(ROOT, "profiles", "r2_fp64_peak.json")
STAGE_PROFILE = os.path.join(ROOT, "profiles", "r2_stage_profile.json")


def fp64_roofline(workload, stage_ms, cells, steps):
    """FP64 issue roofline of the stage kernel: fp64 instructions per cell per
    RK stage (DFMA + DMUL + DADD lane ops, counted in the committed ncu SASS
    capture of the same kernel, profiles/r2_stage_profile.json) x cells / the
    stage's event-timed duration, against the measured DFMA throughput of
    this B200 (profiles/r2_fp64_peak.json, scripts/probes/fp64_peak.cu)."""
    try:
        with open(FP64_PEAK_FILE) as f:
            peak = float(json.load(f)["fp64_dfma_per_s"])
        with open(STAGE_PROFILE) as f:
            prof = json.load(f)
    except (OSError, KeyError, ValueError):
        return None
    ops = prof.get("dp_ops_per_cell", {}).get(workload)
    if not ops or len(ops) != 4:
        return None
    per = [o * cells * steps / (m / 1e3) if m > 0 else None for o, m in zip(ops, stage_ms)]
    tot_ops = sum(o * cells * steps for o in ops)
    tot_s = sum(stage_ms) / 1e3
    achieved = tot_ops / tot_s if tot_s > 0 else None
    return {"bound": "fp64", "dp_ops_per_cell_per_stage": ops, "achieved": achieved, "peak": peak,
            "unit": "fp64 ops/s (DFMA, DMUL, DADD lane instructions)",
            "frac": achieved / peak if achieved else None,
            "per_stage_frac": [p / peak if p else None for p in per],
            "source": os.path.relpath(STAGE_PROFILE, ROOT) + " + " + os.path.relpath(FP64_PEAK_FILE, ROOT)}


def parity_check(workload, dt, device):
    """One RK4 step of the benchmarked problem on the GPU against the threaded
    C restatement of the reference (oracle/, the cpu_baseline leg), from the
    same initial state with the same dt: relative L2 per species (north-star
    bar 1e-12) and a checksum of each side."""
    from oracle import cbackend as C
    from paper_2410_12155_b200 import runner as R

    setup = make_setup(workload)
    sim = R.Simulation(setup, device=device)
    sim.fixed_dt = dt
    sim.advance(dt)
    got = sim.interiors()
    del sim
    ref = C.CSimulation([f.grid for f in setup.dists], setup.species,
                        [np.array(f.data) for f in make_setup(workload).dists], dt=dt)
    ref.advance(dt)
    want = ref.interiors()
    rels = [float(np.linalg.norm(a - b) / np.linalg.norm(b)) for a, b in zip(got, want)]
    return {"steps": 1, "rel_l2": rels, "bar": 1e-12, "ok": all(r <= 1e-12 for r in rels),
            "checksum_gpu": [float(np.sum(a)) for a in got], "checksum_oracle": [float(np.sum(b)) for b in want],
            "oracle": "oracle/stage_ref.c (threaded C restatement, bitwise = reference numba) + numpy FFT"}


def l2_note(setup):
    """Whether the step's buffers exceed the 126 MB L2 (no flush needed) or not."""
    per = sum(int(np.prod(f.grid.padded_shape)) * 8 for f in setup.dists)
    if per > 126e6:
        return f"inputs larger than L2 ({per / 1e9:.2f} GB per state buffer)"
    return (f"inputs smaller than L2 ({per / 1e6:.1f} MB per state buffer): L2-resident, "
            f"not flushed -- a parity configuration, not the bench line of record")


def measured_p2p_gbs(device, world):
    """NVLink peer copy bandwidth from this rank's GPU to the next one
    (scripts/probes/nvlink_p2p.py's measurement, 256 MiB, best of 5), or None
    when the ranks share a GPU or have no peer access."""
    try:
        import torch

        sys.path.insert(0, os.path.join(ROOT, "scripts", "probes"))
        from nvlink_p2p import p2p_gbs

        src = device.index if device.index is not None else torch.cuda.current_device()
        if torch.cuda.device_count() < 2:
            return None
        return p2p_gbs(src, (src + 1) % torch.cuda.device_count(), mib=256)
    except Exception:  # noqa: BLE001 -- a probe; the line falls back to the nominal peak
        return None


def nvlink_line(sim, world, ms_per_step, p2p=None):
    """Halo traffic of the multi-GPU step against the NVLink 5 roofline: the
    bytes each rank sends per step and the rate they would need if the
    exchange were not overlapped with compute (a lower bound on the link
    share of the step), against the measured peer copy bandwidth of this box
    when there is one (else the nominal 900 GB/s per direction,
    B200_PROFILING.md)."""
    if world == 1 or not hasattr(sim, "traffic_report"):
        return None
    t = sim.traffic_report()
    per_step = 4 * t["total_bytes"]
    gbs = per_step / (ms_per_step / 1e3) / 1e9
    peak = p2p if p2p else 900.0
    return {"bytes_per_rank_per_step": per_step, "x_halo_bytes_per_stage": t["x_halo_bytes"],
            "v_face_bytes_per_stage": t["v_face_bytes"], "density_bytes_per_stage": t["density_bytes"],
            "rate_at_step_time_GBs": gbs, "peak_GBs": peak, "peak_kind": "measured p2p copy" if p2p else "nominal",
            "frac": gbs / peak}


def e2e_measure(sim, dt, steps, device, cells):
    """Host-buffer throughput through the library's host entry
    (runner.HostPipeline): every step uploads its input state from pinned host
    memory and downloads its result; uploads, steps and downloads of
    consecutive steps overlap on separate streams (two warm-up steps first,
    which capture the step graphs)."""
    from paper_2410_12155_b200.runner import HostPipeline

    pipe = HostPipeline(sim)
    host_in = pipe.host_state()
    host_out = [[torch_empty_pinned_like(h) for h in host_in] for _ in range(2)]
    pipe.run(lambda k: host_in, lambda k: host_out[k & 1], dt, 2)
    t0 = time.perf_counter()
    pipe.run(lambda k: host_in, lambda k: host_out[k & 1], dt, steps)
    el = time.perf_counter() - t0
    nbytes = pipe.bytes_per_step()
    return {"value": cells * steps / el, "unit": "cell-updates/s", "h2d_bytes_per_step": nbytes,
            "d2h_bytes_per_step": nbytes, "steps": steps,
            "how": "per step: H2D of the input state (interior; ghosts are frozen or periodic images) from "
                   "pinned host memory, the graph-replayed RK4 step, D2H of the new state; "
                   "runner.HostPipeline overlaps the upload of step k+1 and the download of step k-1 with "
                   "step k (copy streams on contiguous device staging buffers, interior unpack/pack by "
                   "vpfv_box_copy on the compute stream; wall clock, host-synchronised at the end)"}


def e2e_dropin_measure(setup, f0, E, dt, device, cells, steps=1):
    """Throughput of the drop-in operator: one RK4
    step = the reference's four ``fused_stage`` calls (timestepping.py's
    3-buffer protocol, RK4_STAGES) on host numpy arrays -- every call uploads
    the arrays it reads and downloads dest's interior (kernels._DropIn /
    _HostStager, allocation-free after the first call).  E is held fixed at
    the initial field (the caller's host field solve is not part of the
    operator).  Fast path (exact=False); wall clock."""
    from paper_2410_12155_b200 import kernels as K
    from paper_2410_12155_b200.timestepping import RK4_STAGES

    g, sp = setup.dists[0].grid, setup.species[0]
    bufs = {"f0": f0, "f1": np.zeros(g.padded_shape), "fout": np.zeros(g.padded_shape)}
    h2d = d2h = 0
    n_int = int(np.prod(g.N)) * 8
    plane = int(np.prod(g.padded_shape[1:])) * 8

    def step(count):
        nonlocal h2d, d2h
        for dn, an, bn, sn, ca, cb, cd, div in RK4_STAGES:
            K.fused_stage(bufs[dn], bufs[an], bufs[bn], bufs[sn], ca, cb, cd, dt / div, g, sp, E, exact=False)
            if count:
                seen = {id(bufs[sn])}
                h2d += plane * g.padded_shape[0]
                for x, c in ((bufs[an], ca), (bufs[bn], cb), (bufs[dn], cd)):
                    if c != 0.0 and id(x) not in seen:
                        seen.add(id(x))
                        h2d += plane * g.N[0]
                d2h += n_int
        bufs["f0"], bufs["fout"] = bufs["fout"], bufs["f0"]

    step(False)  # builds the cached context (device buffers, pinned chunks, tables)
    t0 = time.perf_counter()
    for _ in range(steps):
        step(True)
    el = time.perf_counter() - t0
    K._DROPIN.clear()
    return {"value": cells * steps / el, "unit": "cell-updates/s", "h2d_bytes_per_step": h2d // steps,
            "d2h_bytes_per_step": d2h // steps, "steps": steps, "seconds": el,
            "how": "4 drop-in fused_stage calls per RK4 step on host numpy arrays (reference calling "
                   "convention): src uploaded whole, the read RK operands over the interior x-planes, dest's "
                   "interior downloaded, through two 64 MB pinned chunks; E fixed; wall clock"}


def torch_empty_pinned_like(h):
    import torch

    return torch.empty_like(h).pin_memory()


# ---------------------------------------------------------------------------
# reference arm


def run_reference(args):
    setup = make_setup(args.workload, int(os.environ.get("WORLD_SIZE", "1")))
    from paper_2410_12155_b200.fvm import max_speed_per_dim
    from oracle import vpfv_oracle as O
    from oracle import cbackend as C

    grids = [f.grid for f in setup.dists]
    sim0 = C.CSimulation(grids, setup.species, [np.array(f.data) for f in setup.dists])
    dt = 0.9 * sim0.max_dt()
    del sim0
    cells = sum(int(np.prod(g.N)) for g in grids)
    sim = C.CSimulation(grids, setup.species, [np.array(f.data) for f in setup.dists], dt=dt)
    for _ in range(min(args.warmup, 1)):
        sim.advance(dt)
    budget = args.cpu_budget * 2
    t0 = time.perf_counter()
    n = 0
    while n < args.steps:
        sim.advance(dt)
        n += 1
        if time.perf_counter() - t0 > budget:
            break
    el = time.perf_counter() - t0
    value = cells * n / el
    _ = (max_speed_per_dim, O)
    sample = (f"{n} of {args.steps} requested RK4 steps of the full {args.workload} problem "
              f"(time-capped at {budget:.0f} s), warmup {min(args.warmup, 1)}")
    return {
        "impl": "reference", "metric": "phase-space cell-updates/sec per RK4 step", "value": value,
        "unit": "cell-updates/s", "n_gpus": 0, "steps": n, "warmup": min(args.warmup, 1),
        "ms_per_step": el / n * 1e3, "higher_is_better": True,
        "scaling": "weak" if args.workload in WEAK else "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": args.workload, "description": WORKLOADS[args.workload], "cells": cells,
                   "dt": dt},
        "cpu_baseline": {"value": value, "unit": "cell-updates/s", "cores": C.num_threads(),
                         "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "cell-updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


LEG_WORKLOAD = {"landau2d-128": "landau2d-64", "ep2d2v-64": "ep2d2v-64", "weibel-256": "weibel-256",
                "twostream-1024": "twostream-1024", "landau1d-128": "landau1d-128", "landau2d-64": "landau2d-64"}


def cpu_leg_child(kind, workload):
    """One single-core CPU leg (run in a subprocess with OMP_NUM_THREADS=1):
    ``numpy`` = the oracle's restatement of the reference's production driver
    (OracleSimulation, rhs="numpy": runner.py:183-191's vlasov_rhs path);
    ``c1`` = the C restatement of the numba kernels on one thread
    (_kernels.py:320-373 driven per stage, = the numba-driven step on one
    core).  Prints one JSON object."""
    from oracle import cbackend as C
    from oracle import vpfv_oracle as O

    setup = make_setup(workload)
    grids = [f.grid for f in setup.dists]
    datas = [np.array(f.data) for f in setup.dists]
    c0 = C.CSimulation(grids, setup.species, datas)
    dt = 0.9 * c0.max_dt()
    del c0
    cells = sum(int(np.prod(g.N)) for g in grids)
    if kind == "numpy":
        sim = O.OracleSimulation(grids, setup.species, datas, dt=dt, rhs="numpy")
    else:
        sim = C.CSimulation(grids, setup.species, datas, dt=dt)
    t0 = time.perf_counter()
    n = 0
    while n < 1 or time.perf_counter() - t0 < 5.0:
        sim.advance(dt)
        n += 1
    el = time.perf_counter() - t0
    print(json.dumps({"value": cells * n / el, "steps": n, "seconds": el, "cells": cells,
                      "threads": C.num_threads() if kind == "c1" else 1}))


def cpu_legs(workload):
    """BASELINE.md section 3's single-core legs, each on a bounded sample
    (per-cell costs; the numpy driver at 64^4 would take ~30 s a step)."""
    out = []
    for kind, what in (("numpy", "reference production driver restated in numpy (vlasov_rhs + fold-tree "
                                 "moment + FFT Poisson), OracleSimulation rhs='numpy', 1 core"),
                       ("c1", "numba-equivalent fused kernels (oracle/stage_ref.c, bitwise = numba) driven "
                              "stage by stage, OMP_NUM_THREADS=1")):
        wl = LEG_WORKLOAD.get(workload, workload)
        if kind == "numpy" and wl in ("landau2d-64", "ep2d2v-64", "weibel-256", "twostream-1024"):
            wl = {"landau2d-64": "landau2d-32", "ep2d2v-64": "landau2d-32", "weibel-256": "landau2d-32",
                  "twostream-1024": "landau1d-128"}[wl]
        env = dict(os.environ, OMP_NUM_THREADS="1", OPENBLAS_NUM_THREADS="1", MKL_NUM_THREADS="1")
        try:
            r = subprocess.run([sys.executable, os.path.abspath(__file__), "--cpu-leg", kind, "--workload", wl],
                               env=env, capture_output=True, text=True, timeout=300)
            d = json.loads(r.stdout.strip().splitlines()[-1])
        except Exception as e:  # noqa: BLE001 -- a leg that fails is reported, not fatal
            out.append({"kind": kind, "error": str(e)[:200]})
            continue
        out.append({"kind": "port", "leg": kind, "value": d["value"], "unit": "cell-updates/s", "cores": 1,
                    "what": what, "sample": f"{d['steps']} RK4 step(s) of {wl} ({d['cells']} cells, "
                                            f"{d['seconds']:.1f} s)"})
    return out


def spawn_ranks(n):
    """``python bench.py --gpus N`` without a launcher: re-exec through
    torch.distributed.run with one rank per GPU on 127.0.0.1 (the driver's own
    launch line), after checking that N GPUs are visible (VPFV_SAME_DEVICE=1
    puts every rank on GPU 0 -- validation only).  Returns the exit code."""
    import socket

    import torch

    have = torch.cuda.device_count()
    if have < n and not os.environ.get("VPFV_SAME_DEVICE"):
        print(f"[bench] --gpus {n} requested but only {have} GPU(s) are visible", file=sys.stderr)
        return 2
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd, check=False).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="landau2d-128", choices=sorted(WORKLOADS))
    ap.add_argument("--e2e-steps", type=int, default=32)
    ap.add_argument("--cpu-budget", type=float, default=30.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--halo", default="auto", choices=["auto", "nccl", "peer"],
                    help="multi-GPU x-halo: fused NVLink push from the stage kernel (peer) or NCCL send/recv")
    ap.add_argument("--cpu-leg", choices=["numpy", "c1"], help=argparse.SUPPRESS)
    ap.add_argument("--velocity-parts", type=int, default=1,
                    help="multi-GPU: partitions of the first velocity dim (ranks = x-slabs x this)")
    args = ap.parse_args()
    if args.cpu_leg:
        cpu_leg_child(args.cpu_leg, args.workload)
        return
    if args.warmup < 3 and args.impl == "b200":
        args.warmup = 3
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "b200":
        sys.exit(spawn_ranks(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "b200" and world != args.gpus:
        print(f"[bench] --gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU", file=sys.stderr)
        sys.exit(2)
    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args)), flush=True)
        return
    import torch

    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("VPFV_SAME_DEVICE"):  # validation only: all ranks on GPU 0 (gloo transport)
        local = 0
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        backend = os.environ.get("VPFV_DIST_BACKEND", "nccl")
        if backend == "nccl":
            torch.distributed.init_process_group("nccl", device_id=device)
        else:
            torch.distributed.init_process_group(backend)
    line = run_b200(args, rank, world, device)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
