#!/usr/bin/env python
"""Benchmark: grid-point updates per second of the constant-density acoustic
propagator (BASELINE.json metric), B200 (sm_100a) vs the reference CPU path.

One bench "step" = one complete forward propagation of the workload from the
quiescent state (Solver<T>::forward, kernel.hpp:237-263): source injection,
receiver sampling every time step and health checks included.
  N = 1 : C4, 3D Overthrust-shaped 217x811x811 extended grid, SO=8, 2650 steps.
  N > 1 : weak scaling -- one C4-sized slab (217 extended Z planes) per GPU,
          Z-slab decomposition with an R-plane NCCL halo exchange every step.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
Launched with torchrun for N > 1 (one rank per GPU, RANK/LOCAL_RANK/WORLD_SIZE).
Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Gpts/s (grid-point updates/s) and % HBM roofline"
UNIT = "Gpts/s"
BYTES_PER_POINT = 20  # fp32: read u_cur, u_prev, c2dt2, eta; write u_next
BASELINE_GPTS = {"C4": 5.58}  # V100 OpenMP offload 3D SO8


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--workload", default="auto", help="auto | C1 | C2 | C3 | C4")
    p.add_argument("--math", default="exact", choices=["exact", "fma"])
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=12.0)
    return p.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def workload_cfg(name, world):
    from paper_2201_05278_b200 import configs
    if name == "auto":
        name = "C4"
    if name == "C4" and world > 1:
        return "C4w", configs.overthrust3d(8, z_planes_ext=217 * world)
    return name, configs.CONFIGS[name]()


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.dev = device_index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in self.rows if len(r) > 2 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 2 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for k, nm in enumerate(names):
                if len(r) > 5 + k and r[5 + k].lower().startswith("active"):
                    reasons.add(nm)
        loaded = [v for v in sm if v > 0.5 * max(sm)] if sm else []
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons), "samples": len(self.rows)}


def traffic_for(workload):
    """dram bytes (read+write) per sweep launch from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(workload)
    except Exception:
        return None


# --------------------------------------------------------------------------
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2201_05278_b200 import DampingField, Solver, make_material_model
    from paper_2201_05278_b200._lib import FDW_MATH_EXACT, FDW_MATH_FMA, lib
    from paper_2201_05278_b200.configs import build_workload

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            raise SystemExit("--gpus N > 1 must be launched with torchrun (one rank per GPU)")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    wname, cfg = workload_cfg(args.workload, world)
    math_mode = FDW_MATH_EXACT if args.math == "exact" else FDW_MATH_FMA

    t0 = time.time()
    w = build_workload(cfg, np.float32, rank=rank, world=world)
    setup_s = time.time() - t0
    slab = None
    # halo transport for N > 1: "peer" (default; the sweep stores the halo
    # planes straight into the neighbours' levels over NVLink) or "nccl"
    halo = os.environ.get("FDW_HALO", "peer")
    if world > 1 and halo == "nccl":
        import ctypes as C
        idbuf = (C.c_ubyte * 128)()
        if rank == 0:
            lib().fdw_nccl_unique_id(C.byref(idbuf))
        obj = [bytes(idbuf)]
        dist.broadcast_object_list(obj, src=0)
        slab = (*w.slab, obj[0])
    elif world > 1:
        slab = (*w.slab, None)
    stream = torch.cuda.Stream()

    def make_solver(vel, eta, mats=None):
        t0 = time.perf_counter()
        s = Solver(w.grid, mats or make_material_model(vel), DampingField(eta=eta), w.spec, w.axis, w.coeffs,
                   device=local, math=math_mode, slab=slab)
        t1 = time.perf_counter()
        s.set_stream(stream.cuda_stream)
        if world > 1 and halo != "nccl":
            from paper_2201_05278_b200 import dist as fdist
            fdist.link_peers(s)
        t2 = time.perf_counter()
        s.set_sources(w.sources, w.wavelet)
        s.set_receivers(w.receivers)
        if os.environ.get("FDW_BENCH_DEBUG"):
            print(f"  make_solver: Solver() {t1 - t0:.3f}, set_stream {t2 - t1:.3f}, maps "
                  f"{time.perf_counter() - t2:.3f}", file=sys.stderr, flush=True)
        return s

    solver = make_solver(w.velocity, w.eta)
    n_steps = w.axis.n_steps
    local_pts = int(np.prod([solver._shape[0] - 2 * w.grid.halo] + list(w.grid.extended_shape[1:w.grid.ndim])))
    total_pts = w.grid.extended_points()

    def one_forward():
        solver.reset_state()
        solver.refresh_boundary()
        lib().fdw_record(solver.ctx)
        solver.advance_raw(n_steps, record=True)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
            torch.cuda.synchronize()

    for _ in range(args.warmup):
        one_forward()
    barrier()
    l0 = solver.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            one_forward()
        ev1.record(stream)
        barrier()
    launches = solver.launch_count() - l0
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    value = total_pts * n_steps / (ms_per_step * 1e-3) / 1e9

    # per-kernel device times (CUDA events around every launch, same stream),
    # continuing from the state the timed forwards left: a developed wavefield
    # at step n_steps.  (A field that is still mostly zero draws less power
    # and runs the sweep at a higher clock: about 10% faster on B200 under the
    # power cap, so timing kernels from rest would flatter the roofline.)
    prof = solver.profile_steps(min(200, n_steps))
    sweep_ms = prof[0]
    hbm, hbm_src = peaks()
    achieved = local_pts * BYTES_PER_POINT / (sweep_ms * 1e-3) / 1e9
    step_ms_dev = ms_per_step / n_steps
    # whole-step figure: the same algorithmic bytes over the timed step time
    # (sweep + inject + receivers + health + launch gaps, in the CUDA graph)
    step_achieved = local_pts * BYTES_PER_POINT / (step_ms_dev * 1e-3) / 1e9
    tr = traffic_for(wname)

    # e2e: the public API with host buffers (pinned), H2D + D2H inside the region
    e2e = None
    if not args.no_e2e:
        solver.close()
        del solver
        torch.cuda.empty_cache()
        vel_h = torch.from_numpy(w.velocity).pin_memory().numpy()
        eta_h = torch.from_numpy(w.eta).pin_memory().numpy()
        seis_bytes = (n_steps + 1) * w.receivers.n_points * 4
        ext_bytes = local_pts * 4
        # host-side input validation (make_material_model: velocity > 0, c_max)
        # is input preparation, done once outside the timed region
        mats = make_material_model(vel_h)
        pinned = {}

        def pinned_alloc(shape, dtype):  # reused pinned result buffers
            key = (tuple(shape), np.dtype(dtype).str)
            if key not in pinned:
                pinned[key] = torch.empty(shape, dtype=torch.from_numpy(np.zeros(0, dtype)).dtype).pin_memory().numpy()
            return pinned[key]

        e2e_times = []
        for it in range(max(1, args.steps) + 1):
            barrier()
            e0 = time.perf_counter()
            s = make_solver(vel_h, eta_h, mats)
            e1 = time.perf_counter()
            s.set_host_allocator(pinned_alloc)
            r = s.forward()
            _ = r.seismogram.data, r.snapshots[-1]
            e2 = time.perf_counter()
            s.close()
            barrier()
            el = time.perf_counter() - e0
            if os.environ.get("FDW_BENCH_DEBUG"):
                print(f"e2e iter {it}: {el:.3f} s (ctor {e1 - e0:.3f}, forward {e2 - e1:.3f}, kernel "
                      f"{r.kernel_seconds:.3f}, close {el - (e2 - e0):.3f})", file=sys.stderr, flush=True)
            if it > 0:  # first call pays graph capture
                e2e_times.append(el)
        el = statistics.mean(e2e_times)
        if world > 1:
            t = torch.tensor([el], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        e2e = {"value": round(total_pts * n_steps / el / 1e9, 3), "unit": UNIT,
               "h2d_bytes_per_step": int(vel_h.nbytes + eta_h.nbytes + w.sources.weight.nbytes * 2
                                         + w.receivers.weight.nbytes * 2 + w.wavelet.nbytes),
               "d2h_bytes_per_step": int(seis_bytes + ext_bytes),
               "api": "paper_2201_05278_b200.Solver(...) + set_sources/receivers + forward() over "
                      "libfdwave_cuda.so; pinned host buffers; velocity/eta H2D, seismogram + final "
                      "snapshot D2H inside the timed region",
               "seconds_per_step": round(el, 4)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(cfg, args.cpu_seconds)

    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank != 0:
        return None
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_per_step, 3), "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": round(value / BASELINE_GPTS["C4"], 2) if wname in BASELINE_GPTS else None,
        "dtype": "f32", "data": "synthetic",
        "config": {
            "workload": wname, "name": cfg.name, "extended_shape": list(w.grid.extended_shape[:w.grid.ndim]),
            "space_order": cfg.space_order, "time_steps": n_steps, "points_per_gpu": local_pts,
            "total_points": total_pts, "receivers": w.receivers.n_points, "sources": w.sources.n_points,
            "math": args.math,
            "parallelism": f"z-slab x{world} ({halo} halo)" if world > 1 else "single GPU",
            "step": "one full forward propagation from rest (inject + record every time step, health every 100)",
            "l2": "inputs exceed L2 (4 fields x ~0.7 GB >> 126 MB); no flush needed",
            "setup_seconds": round(setup_s, 2),
            "vs_baseline_ref": "BASELINE.md 3D SO8 V100 OpenMP offload 63.12 s -> 5.58 Gpts/s (PAPER.md:93)",
        },
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                     "frac": round(achieved / hbm, 4), "traffic": tr, "peak_source": hbm_src,
                     "kernel": "sweep (stencil3d/2d)", "bytes_per_point": BYTES_PER_POINT,
                     "state": "developed wavefield (kernels timed after the timed forwards, from step n_steps)",
                     "step_achieved": round(step_achieved, 1), "step_frac": round(step_achieved / hbm, 4),
                     "sweep_ms": round(sweep_ms, 5), "step_ms": round(step_ms_dev, 5),
                     "sweep_share": round(sweep_ms / step_ms_dev, 4),
                     "kernel_ms": {k: round(v, 5) for k, v in zip(
                         ["sweep", "inject", "boundary", "receivers", "health", "halo"], prof)}},
        "e2e": e2e,
        "cpu_baseline": cpu,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    return line


def cpu_baseline(cfg, seconds):
    """The reference's own Solver<float> (oracle/_ref, compiled in place from the
    reference headers) on this host's cores: bounded sample of the same workload."""
    try:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle as O
        if O.rlib() is None:
            raise RuntimeError("no reference library")
        kind = "reference"
        t0 = time.time()
        run = O.RefRun(cfg, np.float32, threads=0)
        setup = time.time() - t0
        pts = int(np.prod(run.extended))
        probe = run.time_steps(1)
        k = max(1, min(60, int(seconds / max(probe, 1e-6)) - 1))
        el = probe + run.time_steps(k)
        n = k + 1
        cores = int(O.rlib().ref_max_threads())
        return {"value": round(pts * n / el / 1e9, 4), "unit": UNIT, "cores": cores, "kind": kind,
                "sample": f"first {n} time steps of {cfg.name} ({pts} ext pts) from rest, reference "
                          f"Solver<float> Backend::Parallel, {el:.1f} s loop (setup {setup:.1f} s excluded)",
                "cpu_model": _cpu_model()}
    except Exception as e:  # keep the GPU line valid
        return {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                "sample": f"unavailable: {e}"}


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def run_reference(args):
    """--impl reference: the reference's own CPU implementation of the path
    (oracle/_ref) on the same workload, each step a bounded sample."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return None
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    wname, cfg = workload_cfg(args.workload, 1)
    if O.rlib() is None:
        return {"impl": "reference", "unavailable": "oracle/_ref/libfdwave_ref.so not built"}
    t0 = time.time()
    run = O.RefRun(cfg, np.float32, threads=0)
    setup = time.time() - t0
    pts = int(np.prod(run.extended))
    # size one step to ~2 s of CPU work
    probe = run.time_steps(1)
    per = max(1, min(50, int(2.0 / max(probe, 1e-6))))
    for _ in range(args.warmup):
        run.time_steps(per)
    times = [run.time_steps(per) for _ in range(args.steps)]
    el = sum(times)
    value = pts * per * args.steps / el / 1e9
    cores = int(O.rlib().ref_max_threads())
    return {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(el / args.steps * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": wname, "name": cfg.name, "extended_shape": list(run.extended),
                   "step": f"{per} reference time steps (bounded sample of the forward run)",
                   "setup_seconds": round(setup, 2)},
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": f"{args.steps} x {per} time steps of {cfg.name} from rest, reference "
                                   "Solver<float> (oracle/_ref, -O3, no fast-math) Backend::Parallel",
                         "cpu_model": _cpu_model()},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    args = parse()
    line = run_reference(args) if args.impl == "reference" else run_ours(args)
    if line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
