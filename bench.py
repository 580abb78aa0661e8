#!/usr/bin/env python
"""Benchmark: grid-point updates per second of the constant-density acoustic
propagator (BASELINE.json metric), B200 (sm_100a) vs the reference CPU path.

One bench "step" = one complete forward propagation of the workload from the
quiescent state (Solver<T>::forward, kernel.hpp:237-263): source injection,
receiver sampling every time step and health checks included.
  N = 1 : C4, 3D Overthrust-shaped 217x811x811 extended grid, SO=8, 2650 steps.
  N > 1 : C5 weak scaling (BASELINE config 5) -- 200 extended Z planes x 811 x
          811 per GPU, SO=8, 500 steps; --workload C4 is the strong-scaling
          split of C4 (BASELINE config 4: slabs 109/108, 55/54, 28/27).
          Z slabs; each step's sweep stores its R boundary planes straight
          into the neighbours' ghost planes over NVLink peer memory.  Before
          timing, a reduced grid over the same ranks is checked bit for bit
          against one domain ("parity" in the line).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload auto|C1..C5|C4w] [--devices 0,1,...]
N > 1 runs under torchrun (one process per GPU, RANK/LOCAL_RANK/WORLD_SIZE) or,
launched directly, as one process with a host thread per GPU.
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
    p.add_argument("--workload", default="auto", help="auto | C1 | C2 | C3 | C4 | C5 | C4w")
    p.add_argument("--devices", default="", help="N > 1 without torchrun: CUDA ordinals, one per rank "
                                                  "(default 0..N-1; repeated ordinals = host-ordered emulation)")
    p.add_argument("--no-parity", action="store_true")
    p.add_argument("--math", default="exact", choices=["exact", "fma"])
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=24.0)
    return p.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def replicated(cfg, world):
    """2D does not shard: N GPUs run N independent replicas."""
    return world > 1 and cfg.ndim == 2


def l2_flush_needed(points, l2_bytes):
    """Timing rule: inputs larger than L2, or L2 flushed between timed steps.
    The working set is 4 fp32 fields (two levels, c2dt2, damping) of `points`."""
    return 4 * points * 4 < 2 * l2_bytes


def workload_cfg(name, world):
    """auto: C4 on one GPU, C5 (weak scaling, 200 planes per GPU) on N > 1.
    C3 / C4 on N > 1 are strong scaling (the one grid split into N slabs);
    C4w is weak scaling with one C4-sized slab (217 planes) per GPU."""
    from paper_2201_05278_b200 import configs
    if name == "auto":
        name = "C4" if world == 1 else "C5"
    if name == "C5":
        return name, configs.weak3d(world)
    if name == "C4w":
        return name, configs.overthrust3d(8, z_planes_ext=217 * world)
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
        if self.dev is None:  # ranks other than 0 do not sample
            return self
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


SWEEP_END_MARKER = "// 2D: one persistent cooperative kernel runs a whole chunk"


def sweep_source_sha():
    """SHA-256 of fdw_kernels.cuh up to the end of the 3D TMA sweep: the sweep
    and everything it can use is defined before the 2D section, so edits
    further down (2D kernels, small helpers) do not invalidate a capture."""
    import hashlib
    with open(os.path.join(ROOT, "paper_2201_05278_b200", "csrc", "fdw_kernels.cuh"), "rb") as f:
        src = f.read()
    end = src.find(SWEEP_END_MARKER.encode())
    return hashlib.sha256(src if end < 0 else src[:end]).hexdigest()


def traffic_for(workload):
    """DRAM bytes (read + write) per sweep launch from the committed ncu capture
    (profiles/ncu_traffic.json).  Valid only for the kernel source it was
    captured from: the capture records the SHA-256 of the sweep's source
    (sweep_source_sha), and a changed sweep reports null instead of a stale
    number."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f)
        if d.get("sweep_source_sha256") != sweep_source_sha():
            return None, "stale: the sweep's source changed since the ncu capture"
        return d.get(workload), d.get("source")
    except Exception as e:
        return None, f"unavailable: {e}"


class TorchEnv:
    """One process per GPU under torchrun (RANK / LOCAL_RANK / WORLD_SIZE):
    torch.distributed carries only control traffic; the ranks' levels and
    sync blocks are IPC-mapped (dist.link_peers)."""

    def __init__(self, world, rank, local):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.world, self.rank, self.device = world, rank, local
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        self.transport = "peer: NVLink P2P stores from the sweep into IPC-mapped neighbour levels, halo epochs"

    def barrier(self):
        self.torch.cuda.synchronize()
        self.dist.barrier()
        self.torch.cuda.synchronize()

    def gather(self, obj):
        out = [None] * self.world
        self.dist.all_gather_object(out, obj)
        return out

    def allmax(self, x):
        return max(self.gather(float(x)))

    def link(self, solver):
        from paper_2201_05278_b200 import dist as fdist
        fdist.link_peers(solver)

    def close(self):
        self.dist.barrier()
        self.dist.destroy_process_group()


class ThreadShared:
    def __init__(self, devices):
        self.devices = list(devices)
        self.world = len(self.devices)
        self.bar = threading.Barrier(self.world, timeout=1800)
        self.slots = [None] * self.world


class ThreadEnv:
    """One process driving N GPUs, one host thread per rank (no torchrun):
    the slab Solvers are linked in-process (fdw_peer_link).  Ranks that share
    a GPU (--devices 0,0: emulation) run host-ordered."""

    def __init__(self, shared, rank):
        import torch
        self.torch, self.sh = torch, shared
        self.world, self.rank, self.device = shared.world, rank, shared.devices[rank]
        torch.cuda.set_device(self.device)
        shared_gpu = len(set(shared.devices)) < shared.world
        self.transport = ("host-ordered peer stores (ranks share a GPU: emulation, not a scaling number)"
                          if shared_gpu else
                          "peer: NVLink P2P stores from the sweep into the neighbours' levels, halo epochs "
                          "(one process, a thread per GPU)")

    def barrier(self):
        self.torch.cuda.synchronize()
        self.sh.bar.wait()

    def gather(self, obj):
        self.sh.slots[self.rank] = obj
        self.sh.bar.wait()
        out = list(self.sh.slots)
        self.sh.bar.wait()
        return out

    def allmax(self, x):
        return max(self.gather(float(x)))

    def link(self, solver):
        solver.peer_link(self.gather(solver))

    def close(self):
        self.sh.bar.wait()


class SoloEnv:
    world, rank, transport = 1, 0, None

    def __init__(self, device=0):
        import torch
        self.torch, self.device = torch, device
        torch.cuda.set_device(device)

    def barrier(self):
        self.torch.cuda.synchronize()

    def gather(self, obj):
        return [obj]

    def allmax(self, x):
        return float(x)

    def link(self, solver):
        pass

    def close(self):
        pass


def parity_check(env, math_mode):
    """N > 1 self-check before timing: a reduced grid decomposed over the same
    ranks as the timed run (same kernels, same peer transport, a point source
    whose taps straddle a slab face), started from a random state so that
    every halo exchange matters from the first step, compared with the same
    grid as one domain on rank 0's GPU.  Field and seismogram bit for bit
    (the straddling receivers are merged from the ranks' per-tap products)."""
    from paper_2201_05278_b200 import DampingField, Solver, make_material_model
    from paper_2201_05278_b200.configs import SyntheticConfig, build_workload
    world, rank = env.world, env.rank
    per, h = 24, 20.0
    nz_int = per * world - 10
    z_face = h * (per - 5) + h / 2  # extended plane 24.5: taps on both sides of the first slab face
    cfg = SyntheticConfig(
        name=f"parity-p{world}", ndim=3, bbox=[0.0, h * (nz_int - 1), 0.0, h * 120, 0.0, h * 120],
        spacing=[h, h, h], space_order=8, damping=[100.0] * 6, vmin=2000.0, vmax=6000.0, tf=0.0,
        sources=[(z_face, h * 60.5, h * 60.5), (h * (per * world - 14) + h / 2, h * 30.5, h * 80.5)],
        receivers=[(h * (per - 6) + h / 2, h * (3 + k), h * 60.5) for k in range(100)], fixed_steps=24)
    w = build_workload(cfg, np.float32, rank=rank, world=world)
    R = w.grid.halo
    P = w.grid.padded_shape()
    rng = np.random.default_rng(2201)
    prev = (rng.standard_normal(P) * 1e-3).astype(np.float32)
    curr = (rng.standard_normal(P) * 1e-3).astype(np.float32)
    zb, ze = w.slab[2], w.slab[3]
    s = Solver(w.grid, make_material_model(w.velocity), DampingField(eta=w.eta), w.spec, w.axis, w.coeffs,
               device=env.device, math=math_mode, slab=w.slab)
    env.link(s)
    s.set_sources(w.sources, w.wavelet)
    s.set_receivers(w.receivers)
    s.previous_level()[...] = prev[zb:ze + 2 * R]
    s.current_level()[...] = curr[zb:ze + 2 * R]
    s.refresh_boundary()
    from paper_2201_05278_b200._lib import lib
    lib().fdw_record(s.ctx)
    s.advance_raw(w.axis.n_steps, record=True)
    from paper_2201_05278_b200.dist import merge_seismogram, split_products
    rows = w.axis.n_steps + 1
    parts = env.gather((s.extended_level(), s.seismogram_f64(rows), split_products(s, rows)))
    s.close()
    if rank != 0:
        env.barrier()
        return None
    wf = build_workload(cfg, np.float32)
    r = Solver(wf.grid, make_material_model(wf.velocity), DampingField(eta=wf.eta), wf.spec, wf.axis, wf.coeffs,
               device=env.device, math=math_mode)
    r.set_sources(wf.sources, wf.wavelet)
    r.set_receivers(wf.receivers)
    r.previous_level()[...] = prev
    r.current_level()[...] = curr
    r.refresh_boundary()
    lib().fdw_record(r.ctx)
    r.advance_raw(wf.axis.n_steps, record=True)
    ref_field, ref_seis = r.extended_level(), r.seismogram_f64()
    r.close()
    env.barrier()
    field = np.concatenate([p[0] for p in parts], axis=0)
    seis = merge_seismogram([p[1] for p in parts], [p[2] for p in parts], wf.receivers.n_points)
    exact = bool(np.array_equal(field, ref_field))
    seis_exact = bool(np.array_equal(seis, ref_seis))
    return {"ok": bool(exact and seis_exact and np.abs(ref_field).max() > 0), "field_bit_exact": exact,
            "seismogram_bit_exact": seis_exact,
            "case": f"{cfg.name}: {world} slabs of {per} planes x 131 x 131, SO8, random start, 24 steps, receivers "
                    f"straddling a slab face, vs one domain on rank 0's GPU"}


def run_ours(args):
    """Dispatch: N = 1 (one GPU), torchrun (one process per GPU), or one
    process with a thread per GPU when --gpus N > 1 is launched directly."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        if world != args.gpus:
            raise SystemExit(f"WORLD_SIZE {world} != --gpus {args.gpus}")
        env = TorchEnv(world, int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")))
        return bench_rank(args, env)
    if args.gpus <= 1:
        return bench_rank(args, SoloEnv(int(args.devices.split(",")[0]) if args.devices else 0))
    devices = [int(x) for x in args.devices.split(",")] if args.devices else list(range(args.gpus))
    if len(devices) != args.gpus:
        raise SystemExit("--devices must list --gpus ordinals")
    sh = ThreadShared(devices)
    out, errs = [None] * args.gpus, []

    def go(r):
        try:
            out[r] = bench_rank(args, ThreadEnv(sh, r))
        except BaseException as e:  # surfaced below; unblock the other ranks
            import traceback
            errs.append(f"rank {r}: {traceback.format_exc()}")
            sh.bar.abort()

    th = [threading.Thread(target=go, args=(r,), daemon=True) for r in range(args.gpus)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise SystemExit("\n".join(errs))
    return out[0]


def bench_rank(args, env):
    import torch

    from paper_2201_05278_b200 import DampingField, Solver, make_material_model
    from paper_2201_05278_b200._lib import FDW_MATH_EXACT, FDW_MATH_FMA, lib
    from paper_2201_05278_b200.configs import build_workload

    world, rank, dev = env.world, env.rank, env.device
    wname, cfg = workload_cfg(args.workload, world)
    math_mode = FDW_MATH_EXACT if args.math == "exact" else FDW_MATH_FMA
    # 2D does not shard (775k points take ~5 us per step, a
    # split would be latency-dominated): N GPUs run N independent replicas
    replicas = replicated(cfg, world)
    parity = parity_check(env, math_mode) if world > 1 and not replicas and not args.no_parity else None

    t0 = time.time()
    w = build_workload(cfg, np.float32, rank=0 if replicas else rank, world=1 if replicas else world)
    setup_s = time.time() - t0
    slab = w.slab if world > 1 and not replicas else None
    stream = torch.cuda.Stream(device=dev)

    def make_solver(vel, eta, mats=None):
        s = Solver(w.grid, mats or make_material_model(vel), DampingField(eta=eta), w.spec, w.axis, w.coeffs,
                   device=dev, math=math_mode, slab=slab)
        s.set_stream(stream.cuda_stream)
        if not replicas:
            env.link(s)
        s.set_sources(w.sources, w.wavelet)
        s.set_receivers(w.receivers)
        return s

    solver = make_solver(w.velocity, w.eta)
    n_steps = w.axis.n_steps
    local_pts = int(np.prod([solver._shape[0] - 2 * w.grid.halo] + list(w.grid.extended_shape[1:w.grid.ndim])))
    total_pts = w.grid.extended_points() * (world if replicas else 1)

    def one_forward():
        solver.reset_state()
        solver.refresh_boundary()
        lib().fdw_record(solver.ctx)
        solver.advance_raw(n_steps, record=True)

    for _ in range(args.warmup):
        one_forward()
    env.barrier()
    # Timing rule: inputs larger than L2, or L2 flushed between timed steps.
    # 3D fields (0.6-0.8 GB each) exceed the 126 MB L2; a 2D working set
    # (C1/C2: 4 fields x ~4 MB) fits, so every 2D forward is preceded by a
    # write of twice the L2 size and timed by its own event pair (the flush
    # stays outside the timed region).
    l2_bytes = torch.cuda.get_device_properties(dev).L2_cache_size
    work_bytes = 4 * local_pts * 4
    flush = l2_flush_needed(local_pts, l2_bytes)
    scrub = torch.empty(2 * l2_bytes // 4 + 1024, dtype=torch.float32, device=dev) if flush else None
    l0 = solver.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev if rank == 0 else None) as clk:
        env.barrier()
        if flush:
            evs = []
            for _ in range(args.steps):
                with torch.cuda.stream(stream):
                    scrub.fill_(1.0)
                a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a0.record(stream)
                one_forward()
                a1.record(stream)
                evs.append((a0, a1))
            env.barrier()
            torch.cuda.synchronize()
            t_ms = sum(a.elapsed_time(b) for a, b in evs)
        else:
            ev0.record(stream)
            for _ in range(args.steps):
                one_forward()
            ev1.record(stream)
            env.barrier()
            torch.cuda.synchronize()
            t_ms = ev0.elapsed_time(ev1)
    launches = solver.launch_count() - l0
    ms = env.allmax(t_ms)  # device time, max over ranks
    ms_per_step = ms / args.steps
    value = total_pts * n_steps / (ms_per_step * 1e-3) / 1e9

    # per-kernel device times (CUDA events around every launch, same stream),
    # continuing from the state the timed forwards left: a developed wavefield
    # at step n_steps.  (A field that is still mostly zero draws less power
    # and runs the sweep at a higher clock: about 10% faster on B200 under the
    # power cap, so timing kernels from rest would flatter the roofline.)
    # the states at n_steps / 2 and n_steps seed the CPU baseline's samples
    # (the reference's CPU rate changes over a run: subnormal arithmetic in the
    # numerical precursor ahead of the wavefront slows the middle of the run)
    cpu_states = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu_states = {"end": (solver.previous_level().copy(), solver.current_level().copy())}
        solver._host_view = False
    # Power state: the host-side pause after the timed region (and the level
    # downloads above) lets the power limiter lift the SM clock for the next
    # ~100 ms, which made a profile taken right away ~5% faster than the same
    # kernel inside the chain (464 vs 490 us at C4).  A back-to-back settle
    # of graph-captured steps first puts the sweep back in the chain's
    # (sw_power_cap) state, so `achieved` describes the kernel as it runs.
    solver.advance_raw(min(300, n_steps), record=True)
    prof = solver.profile_steps(min(200, n_steps))
    sweep_ms = prof[0]
    if os.environ.get("FDW_BENCH_DEBUG"):
        for m in (20, 200, 20):
            print(f"profile_steps({m}) sweep {solver.profile_steps(m)[0]:.4f} ms", file=sys.stderr, flush=True)
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record(stream)
        solver.advance_raw(100, record=True)
        c1.record(stream)
        c1.synchronize()
        print(f"graph chunk: {c0.elapsed_time(c1) / 100:.4f} ms/step", file=sys.stderr, flush=True)
    if cpu_states is not None:
        one_half = n_steps // 2
        solver.reset_state()
        solver.refresh_boundary()
        solver.advance_raw(one_half)
        cpu_states["mid"] = (solver.previous_level().copy(), solver.current_level().copy())
        solver._host_view = False
    hbm, hbm_src = peaks()
    achieved = local_pts * BYTES_PER_POINT / (sweep_ms * 1e-3) / 1e9
    step_ms_dev = ms_per_step / n_steps
    # whole-step figure: the same algorithmic bytes over the timed step time
    # (sweep + inject + receivers + health + launch gaps, in the CUDA graph)
    step_achieved = local_pts * BYTES_PER_POINT / (step_ms_dev * 1e-3) / 1e9
    tr, tr_src = traffic_for(wname)

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
            env.barrier()
            e0 = time.perf_counter()
            s = make_solver(vel_h, eta_h, mats)
            e1 = time.perf_counter()
            s.set_host_allocator(pinned_alloc)
            r = s.forward()
            _ = r.seismogram.data, r.snapshots[-1]
            e2 = time.perf_counter()
            s.close()
            env.barrier()
            el = time.perf_counter() - e0
            if os.environ.get("FDW_BENCH_DEBUG"):
                print(f"e2e iter {it}: {el:.3f} s (ctor {e1 - e0:.3f}, forward {e2 - e1:.3f}, kernel "
                      f"{r.kernel_seconds:.3f}, close {el - (e2 - e0):.3f})", file=sys.stderr, flush=True)
            if it > 0:  # first call pays graph capture
                e2e_times.append(el)
        el = env.allmax(statistics.mean(e2e_times))
        e2e = {"value": round(total_pts * n_steps / el / 1e9, 3), "unit": UNIT,
               "h2d_bytes_per_step": int(vel_h.nbytes + eta_h.nbytes + w.sources.weight.nbytes * 2
                                         + w.receivers.weight.nbytes * 2 + w.wavelet.nbytes),
               "d2h_bytes_per_step": int(seis_bytes + ext_bytes),
               "api": "paper_2201_05278_b200.Solver(...) + set_sources/receivers + forward() over "
                      "libfdwave_cuda.so; pinned host buffers; velocity/eta H2D, seismogram + final "
                      "snapshot D2H inside the timed region" + (" (per rank: its slab)" if world > 1 else ""),
               "seconds_per_step": round(el, 4)}
    else:
        solver.close()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(cfg, args.cpu_seconds, cpu_states, wname, n_steps)

    env.close()
    if rank != 0:
        return None
    strong = world > 1 and wname in ("C3", "C4")
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_per_step, 3), "higher_is_better": True,
        "scaling": "strong" if strong else "weak",
        "vs_baseline": round(value / BASELINE_GPTS["C4"], 2) if wname in BASELINE_GPTS else None,
        "dtype": "f32", "data": "synthetic",
        "config": {
            "workload": wname, "name": cfg.name, "extended_shape": list(w.grid.extended_shape[:w.grid.ndim]),
            "space_order": cfg.space_order, "time_steps": n_steps, "points_per_gpu": local_pts,
            "total_points": total_pts, "receivers": w.receivers.n_points, "sources": w.sources.n_points,
            "math": args.math,
            "parallelism": (f"independent replicas x{world} (2D does not shard)" if replicas else
                            f"z-slab x{world}" if world > 1 else "single GPU"),
            "step": "one full forward propagation from rest (inject + record every time step, health every 100)",
            "l2": (f"working set {work_bytes / 2**20:.0f} MiB fits the {l2_bytes / 2**20:.0f} MiB L2: L2 flushed "
                   f"({2 * l2_bytes / 2**20:.0f} MiB write) before every timed forward, outside its events"
                   if flush else f"inputs exceed L2 (4 fields x {local_pts * 4 / 2**30:.2f} GiB >> "
                   f"{l2_bytes / 2**20:.0f} MiB); no flush needed"),
            "setup_seconds": round(setup_s, 2),
            "vs_baseline_ref": "BASELINE.md 3D SO8 V100 OpenMP offload 63.12 s -> 5.58 Gpts/s (PAPER.md:93)",
        },
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                     "frac": round(achieved / hbm, 4), "traffic": tr, "traffic_source": tr_src,
                     "peak_source": hbm_src,
                     "kernel": "sweep (stencil3d/2d)", "bytes_per_point": BYTES_PER_POINT,
                     "state": "developed wavefield, power-capped like the timed chain (kernels timed after the timed forwards and a 300-step settle, from step n_steps + 300)",
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
    if world > 1:
        line["transport"] = "none: independent replicas" if replicas else env.transport
        line["parity"] = parity
    return line


def cpu_baseline(cfg, seconds, states=None, wname=None, n_steps=None):
    """The reference's own Solver<float> (oracle/_ref, compiled in place from the
    reference headers) on this host's cores: bounded samples of the same
    workload.  The CPU's rate is not constant over a run (a field of exact
    zeros is fast; subnormals in the numerical precursor ahead of the
    wavefront are slow), so the value samples three points of the run --
    from rest, and from the GPU's states at n/2 and n loaded into the reference
    Solver's levels -- and reports points x steps / seconds over all three.
    The full-length run of the fixture generator is reported beside it."""
    try:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle as O
        if O.rlib() is None:
            raise RuntimeError("no reference library")
        t0 = time.time()
        run = O.RefRun(cfg, np.float32, threads=0)
        setup = time.time() - t0
        pts = int(np.prod(run.extended))
        cores = int(O.rlib().ref_max_threads())
        parts = ["rest"] + ([k for k in ("mid", "end") if k in states] if states else [])
        per = seconds / len(parts)
        run.time_steps(1)  # OpenMP pool and first-touch warm-up, untimed
        samples = {}
        for name in parts:
            if name != "rest":
                run.set_levels(*states[name])
            probe = run.time_steps(1)
            k = max(1, min(60, int(per / max(probe, 1e-6)) - 1))
            el = probe + run.time_steps(k)
            samples[name] = (k + 1, el)
        n_all = sum(v[0] for v in samples.values())
        t_all = sum(v[1] for v in samples.values())
        at = {"rest": "step 0", "mid": f"step {n_steps // 2}" if n_steps else "mid-run",
              "end": f"step {n_steps}" if n_steps else "end"}
        out = {"value": round(pts * n_all / t_all / 1e9, 4), "unit": UNIT, "cores": cores, "kind": "reference",
               "sample": f"{n_all} time steps of {cfg.name} ({pts} ext pts) in {len(samples)} runs of ~{per:.0f} s from "
                         + ", ".join(f"{at[k]} ({v[0]} steps, {v[1]:.1f} s)" for k, v in samples.items())
                         + " (states after step 0 are the GPU's, loaded into the reference Solver's levels); "
                           f"reference Solver<float> Backend::Parallel; setup {setup:.1f} s excluded",
               "per_state_gpts": {k: round(pts * v[0] / v[1] / 1e9, 4) for k, v in samples.items()},
               "cpu_model": _cpu_model()}
        # the whole forward, measured once on a GPU box of this pool next to a
        # bench line (tools/cpu_full_run.py; bit-identical to the fixtures)
        full = os.path.join(ROOT, "profiles", "r02", f"cpu_full_{(wname or '').lower()}.json")
        if os.path.exists(full):
            with open(full) as f:
                m = json.load(f)
            out["full_run"] = {"gpts": m["gpts"], "seconds": m["kernel_seconds"], "steps": m["n_steps"],
                               "threads": m["threads"], "bit_identical_to_fixture": m["matches_fixture"],
                               "where": f"GPU box of this pool, earlier run ({os.path.relpath(full, ROOT)})"}
        return out
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
    # the same workload as our arm at this N (C5 at N > 1 is 200 planes per GPU)
    wname, cfg = workload_cfg(args.workload, max(world, args.gpus))
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
        "higher_is_better": True, "scaling": "strong" if max(world, args.gpus) > 1 and wname in ("C3", "C4") else "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
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
