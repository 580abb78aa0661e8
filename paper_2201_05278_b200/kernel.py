"""Propagator -- Python mirror of fdwave/kernel.hpp over libfdwave_cuda.so.

`Solver` keeps the reference's public API (kernel.hpp:170-273): constructor,
set_sources, set_receivers, add_volume_source, set_backend, set_verbose,
set_snapshot_cap, grid, time_axis, current_level, previous_level, step_index,
refresh_boundary, step, forward, max_abs.  The wavefield lives on the GPU; the
host levels returned by current_level()/previous_level() are mirrors kept in
sync on access (writes to them are uploaded before the next device step),
so the reference's "mutable reference to a member" semantics hold.
"""
from __future__ import annotations

import ctypes as C
import enum
import sys
import time
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _lib
from ._lib import FDW_ADVANCE_ASYNC, FDW_ADVANCE_RECORD, FDW_EINSTABLE, FDW_EINVAL, FDW_OK, ptr


class BoundaryCondition(enum.IntEnum):  # kernel.hpp:27
    NullDirichlet = 0
    NullNeumann = 1
    None_ = 2


def boundary_condition_from_string(s: str) -> BoundaryCondition:
    """kernel.hpp:29-34."""
    table = {"null_dirichlet": BoundaryCondition.NullDirichlet,
             "null_neumann": BoundaryCondition.NullNeumann, "none": BoundaryCondition.None_}
    if s not in table:
        raise ValueError("unknown boundary condition: " + s)
    return table[s]


@dataclass
class BoundarySpec:  # kernel.hpp:37-45, face[axis][low/high]
    face: list = field(default_factory=lambda: [[BoundaryCondition.NullDirichlet] * 2 for _ in range(3)])

    @staticmethod
    def uniform(bc: BoundaryCondition) -> "BoundarySpec":
        return BoundarySpec([[bc, bc] for _ in range(3)])


class InstabilityError(RuntimeError):  # kernel.hpp:48-62 instability_error
    def __init__(self, step: int, max_abs: float):
        super().__init__(f"non-finite wavefield at step {step} (max |p| = {max_abs}); "
                         "timestep is likely unstable")
        self._step = step
        self._max_abs = max_abs

    def step(self) -> int:
        return self._step

    def max_abs(self) -> float:
        return self._max_abs


class FdwError(RuntimeError):
    """CUDA-side (or peer-transport) failure reported through the C-ABI."""


def apply_boundary(f: np.ndarray, grid, spec: BoundarySpec) -> None:
    """kernel.hpp:67-102 on a host padded field (in place), axis by axis over
    the full padded extent of the other axes."""
    h = grid.halo
    for axis in range(grid.ndim):
        n_ext = grid.extended_shape[axis]
        v = np.moveaxis(f, axis, 0)
        for side in range(2):
            bc = spec.face[axis][side]
            face = h if side == 0 else h + n_ext - 1
            out = -1 if side == 0 else 1
            if bc == BoundaryCondition.NullDirichlet:
                v[face] = 0
                for k in range(1, h + 1):
                    v[face + out * k] = -v[face - out * k]
            elif bc == BoundaryCondition.NullNeumann:
                for k in range(1, h + 1):
                    v[face + out * k] = v[face - out * k]
            else:
                for k in range(1, h + 1):
                    v[face + out * k] = 0


@dataclass
class ModulatedField:  # kernel.hpp:140-144
    field: np.ndarray
    amplitude: list


@dataclass
class Seismogram:  # kernel.hpp:146-153
    n_receivers: int = 0
    data: np.ndarray = field(default_factory=lambda: np.zeros(0))
    coordinates: list = field(default_factory=list)

    def at(self, row: int, rec: int):
        return self.data[row * self.n_receivers + rec]


@dataclass
class ForwardResult:  # kernel.hpp:155-161
    snapshots: List[np.ndarray] = field(default_factory=list)
    snapshot_steps: List[int] = field(default_factory=list)
    seismogram: Seismogram = field(default_factory=Seismogram)
    kernel_seconds: float = 0.0


class Backend(enum.IntEnum):  # kernel.hpp:163
    Serial = 0
    Parallel = 1


def _check(ctx, rc: int, what: str):
    if rc == FDW_OK:
        return
    msg = _lib.lib().fdw_last_error(ctx).decode(errors="replace")
    if rc == FDW_EINVAL:
        raise ValueError(f"{what}: {msg}")
    raise FdwError(f"{what}: {msg} (status {rc})")


class Solver:
    """fdwave::Solver<T> on the GPU.  T follows materials.velocity.dtype
    (float32 / float64).  Extra keyword-only knobs: device, variant
    (FDW_KERNEL_*), math (FDW_MATH_*), z_segments, and slab=(rank, world,
    z_begin, z_end) for a Z-slab rank of a multi-GPU run (then the field
    arrays are the rank's local padded slab; link the ranks with peer_link /
    dist.link_peers before stepping)."""

    def __new__(cls, grid=None, *args, devices=None, slab=None, **kw):
        """Like the C++ drop-in: several devices (devices=[...], or FDW_DEVICES
        in the environment) make a 3D Solver a SlabSolver, one Z slab per GPU."""
        if cls is Solver and slab is None and grid is not None and grid.ndim == 3:
            from .multi import SlabSolver, devices_from_env
            devs = list(devices) if devices is not None else devices_from_env()
            if len(devs) > 1 and grid.extended_shape[0] >= 2 * grid.halo * len(devs):
                kw.pop("device", None)
                return SlabSolver(grid, *args, devices=devs, **kw)
        return super().__new__(cls)

    def __init__(self, grid, materials, damping, boundary: BoundarySpec, time_axis, coeffs, *,
                 device: int = 0, variant: int = 0, math: int = 0, z_segments: int = 0,
                 slab=None, devices=None):
        if coeffs.order != grid.space_order:
            raise ValueError("stencil order does not match grid order")
        L = _lib.lib()
        self._grid = grid
        self._time = time_axis
        self._coeffs = coeffs
        self._boundary = boundary
        vel = np.ascontiguousarray(materials.velocity)
        self._dtype = vel.dtype
        if self._dtype not in (np.float32, np.float64):
            raise ValueError("velocity must be float32 or float64")
        eta = np.ascontiguousarray(damping.eta, dtype=self._dtype)
        d = _lib.fdw_desc()
        L.fdw_desc_init(C.byref(d))
        d.ndim = grid.ndim
        d.space_order = grid.space_order
        d.dtype_bytes = self._dtype.itemsize
        for a in range(3):
            d.extended[a] = int(grid.extended_shape[a]) if a < grid.ndim else 1
            d.spacing[a] = float(grid.spacing[a]) if a < grid.ndim else 1.0
            for s in range(2):
                d.bc[a][s] = int(boundary.face[a][s])
        for j, v in enumerate(coeffs.second):
            d.coeffs[j] = float(v)
        for j, v in enumerate(coeffs.first):
            d.coeffs1[j] = float(v)
        d.dt = float(time_axis.dt)
        d.n_steps = int(time_axis.n_steps)
        d.device = int(device)
        d.variant = int(variant)
        d.math = int(math)
        d.z_segments = int(z_segments)
        P = list(grid.padded_shape())
        if slab is not None:
            rank, world, zb, ze = slab[:4]
            d.rank, d.world, d.z_begin, d.z_end = int(rank), int(world), int(zb), int(ze)
            P[0] = int(ze - zb) + 2 * grid.halo
        self._shape = tuple(P[:grid.ndim]) if grid.ndim == 3 else (P[0], P[1])
        if vel.size != int(np.prod(self._shape)) or eta.size != vel.size:
            raise ValueError("velocity/eta shape does not match the padded grid")
        self._ctx = C.c_void_p()
        rc = L.fdw_create(C.byref(d), C.byref(self._ctx))
        if rc != FDW_OK:
            msg = L.fdw_last_error(None).decode(errors="replace")
            if rc == FDW_EINVAL:
                raise ValueError(msg)
            raise FdwError(f"fdw_create: {msg} (status {rc})")
        self._desc = d
        _check(self._ctx, L.fdw_set_medium(self._ctx, ptr(vel), ptr(eta), 0), "fdw_set_medium")
        if materials.density is not None:  # kernel.hpp:295-296
            rho = np.ascontiguousarray(materials.density, dtype=self._dtype)
            if rho.size != vel.size:
                raise ValueError("density shape does not match the padded grid")
            _check(self._ctx, L.fdw_set_density(self._ctx, ptr(rho), 0), "fdw_set_density")
        self._sources = None
        self._wavelet = None
        self._receivers = None
        self._receiver_coordinates = []
        self._n_rec = 0
        self._verbose = False
        self._verbose_quiet = False  # a slab rank other than 0 (SlabSolver): checks, no line
        self._loop_start = time.perf_counter()  # kernel.hpp:494 (reset by forward)
        self._snapshot_cap = 4 << 30
        self._prev = None
        self._curr = None
        self._host_view = False
        self._alloc = np.empty

    def set_host_allocator(self, fn):
        """fn(shape, dtype) -> ndarray used for forward() results (snapshots,
        seismogram); pass a pinned-memory allocator for full-speed D2H."""
        self._alloc = fn or np.empty

    # -- lifetime --
    def close(self):
        if getattr(self, "_ctx", None):
            _lib.lib().fdw_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- reference API --
    def set_sources(self, sources, wavelet):
        """kernel.hpp:188-193."""
        wavelet = np.ascontiguousarray(wavelet, dtype=np.float64)
        if sources.n_points > 0 and len(wavelet) < self._time.sample_count():
            raise ValueError("wavelet shorter than the time axis")
        self._sources, self._wavelet = sources, wavelet
        _check(self._ctx, _lib.lib().fdw_set_sources(
            self._ctx, sources.n_points, ptr(np.ascontiguousarray(sources.offsets, np.uint64)),
            ptr(np.ascontiguousarray(sources.index, np.uint64)),
            ptr(np.ascontiguousarray(sources.weight, np.float64)), ptr(wavelet), len(wavelet)),
            "fdw_set_sources")

    def set_receivers(self, receivers, coordinates=None):
        """kernel.hpp:194-198."""
        self._receivers = receivers
        self._receiver_coordinates = list(coordinates or [])
        self._n_rec = receivers.n_points
        _check(self._ctx, _lib.lib().fdw_set_receivers(
            self._ctx, receivers.n_points, ptr(np.ascontiguousarray(receivers.offsets, np.uint64)),
            ptr(np.ascontiguousarray(receivers.index, np.uint64)),
            ptr(np.ascontiguousarray(receivers.weight, np.float64))), "fdw_set_receivers")

    def add_volume_source(self, source):
        """kernel.hpp:199-203: dense forcing field (padded shape) times a
        per-step amplitude, added after the point sources (:439-452)."""
        if len(source.amplitude) < self._time.n_steps:
            raise ValueError("volume source amplitude shorter than run")
        f = np.ascontiguousarray(source.field, dtype=self._dtype)
        if f.size != int(np.prod(self._shape)):
            raise ValueError("volume source field shape does not match the padded grid")
        amp = np.ascontiguousarray(source.amplitude, np.float64)
        _check(self._ctx, _lib.lib().fdw_add_volume_source(self._ctx, ptr(f), ptr(amp), len(amp), 0),
               "fdw_add_volume_source")

    def set_backend(self, backend, workers: int = 0):
        """kernel.hpp:204-211 -- accepted and ignored (one GPU code path)."""

    def set_verbose(self, verbose: bool):
        self._verbose = bool(verbose)

    def set_snapshot_cap(self, nbytes: int):
        self._snapshot_cap = int(nbytes)

    def grid(self):
        return self._grid

    def time_axis(self):
        return self._time

    def step_index(self) -> int:
        v = C.c_uint64()
        _lib.lib().fdw_step_index(self._ctx, C.byref(v))
        return int(v.value)

    def _ensure_host(self):
        if self._curr is None:
            self._prev = np.zeros(self._shape, self._dtype)
            self._curr = np.zeros(self._shape, self._dtype)

    def _download(self):
        self._ensure_host()
        _check(self._ctx, _lib.lib().fdw_get_levels(self._ctx, ptr(self._prev), ptr(self._curr)),
               "fdw_get_levels")

    def _upload_if_viewed(self):
        if self._host_view:
            _check(self._ctx, _lib.lib().fdw_set_levels(self._ctx, ptr(self._prev), ptr(self._curr)),
                   "fdw_set_levels")

    def current_level(self) -> np.ndarray:
        """kernel.hpp:217 -- host mirror (same array object across calls)."""
        if not self._host_view:
            self._download()
            self._host_view = True
        return self._curr

    def previous_level(self) -> np.ndarray:
        """kernel.hpp:218."""
        if not self._host_view:
            self._download()
            self._host_view = True
        return self._prev

    def refresh_boundary(self):
        """kernel.hpp:223."""
        self._upload_if_viewed()
        _check(self._ctx, _lib.lib().fdw_refresh_boundary(self._ctx), "fdw_refresh_boundary")
        if self._host_view:
            self._download()

    def _advance(self, n: int, flags: int):
        if self._verbose:  # check_health's progress line (kernel.hpp:456-466)
            self._verbose_advance(n, flags & ~FDW_ADVANCE_ASYNC)
            return
        self._advance_raw(n, flags)

    def _verbose_advance(self, n: int, flags: int):
        """Steps in pieces that end at the health checks (step % 100 == 0 or
        the last step); after each, the reference's line
        "step s/N  t s  max|p| = m" on stderr, t since forward() began its loop."""
        ci, total = 100, self._time.n_steps
        s = self.step_index()
        end = s + n
        while s < end:
            nxt = (s // ci + 1) * ci
            if total > s:
                nxt = min(nxt, total)
            nxt = min(nxt, end)
            self._advance_raw(nxt - s, flags)
            s = nxt
            if s % ci == 0 or s == total:
                v = C.c_double()
                _check(self._ctx, _lib.lib().fdw_max_abs(self._ctx, C.byref(v)), "fdw_max_abs")
                if not self._verbose_quiet:
                    sys.stderr.write("step %d/%d  %.3fs  max|p| = %.6e\n"
                                     % (s, total, time.perf_counter() - self._loop_start, v.value))

    def _advance_raw(self, n: int, flags: int):
        bad_step = C.c_uint64()
        bad_max = C.c_double()
        rc = _lib.lib().fdw_advance(self._ctx, n, flags, C.byref(bad_step), C.byref(bad_max))
        if rc == FDW_EINSTABLE:
            if self._host_view:
                self._download()
            raise InstabilityError(int(bad_step.value), float(bad_max.value))
        _check(self._ctx, rc, "fdw_advance")

    def _wait(self):
        bad_step = C.c_uint64()
        bad_max = C.c_double()
        rc = _lib.lib().fdw_wait(self._ctx, C.byref(bad_step), C.byref(bad_max))
        if rc == FDW_EINSTABLE:
            if self._host_view:
                self._download()
            raise InstabilityError(int(bad_step.value), float(bad_max.value))
        _check(self._ctx, rc, "fdw_wait")

    def step(self):
        """kernel.hpp:226-233."""
        self._upload_if_viewed()
        self._advance(1, 0)
        if self._host_view:
            self._download()

    def forward(self) -> ForwardResult:
        """kernel.hpp:237-263."""
        res = ForwardResult()
        res.seismogram.n_receivers = self._n_rec
        res.seismogram.coordinates = list(self._receiver_coordinates)
        ext_pts = int(np.prod(self._grid.extended_shape))
        snap_bytes = self._time.snapshot_count() * ext_pts * self._dtype.itemsize
        if snap_bytes > self._snapshot_cap:
            raise ValueError(f"snapshot storage ({snap_bytes} bytes) exceeds the configured cap; "
                             "raise the cap or the stride")
        self.refresh_boundary()
        L = _lib.lib()
        _check(self._ctx, L.fdw_record(self._ctx), "fdw_record")
        start = self.step_index()
        n_total = self._time.n_steps
        stride = self._time.saving_stride

        def store(step):  # kernel.hpp:305-306
            return step == n_total if stride == 0 else step % stride == 0

        if store(start):
            self._snapshot(res, start)
        # steps at which a snapshot is due inside (start, start + n_total]
        end = start + n_total
        if stride == 0:
            events = [n_total] if start < n_total <= end else []
        else:
            events = list(range((start // stride + 1) * stride, end + 1, stride))
        events.append(end)
        t0 = time.perf_counter()
        self._loop_start = t0
        cur = start
        # steps and snapshot copies are queued without host syncs: each
        # snapshot streams out on the copy stream while later steps run
        for ev in sorted(set(events)):
            if ev > cur:
                self._advance(ev - cur, FDW_ADVANCE_RECORD | FDW_ADVANCE_ASYNC)
                cur = ev
            if store(cur) and cur != start:
                self._snapshot(res, cur, stream=True)
        self._wait()
        res.kernel_seconds = time.perf_counter() - t0
        if self._n_rec:
            data = self._alloc(((n_total + 1) * self._n_rec,), self._dtype)
            _check(self._ctx, L.fdw_download_seismogram(self._ctx, ptr(data), n_total + 1),
                   "fdw_download_seismogram")
            res.seismogram.data = data
        if self._host_view:
            self._download()
        return res

    def _snapshot(self, res, step, stream=False):
        out = self._alloc(tuple(self._extended_local()), self._dtype)
        if stream:  # valid after _wait()
            _check(self._ctx, _lib.lib().fdw_snapshot_async(self._ctx, ptr(out)), "fdw_snapshot_async")
        else:
            _check(self._ctx, _lib.lib().fdw_get_extended(self._ctx, ptr(out)), "fdw_get_extended")
        res.snapshots.append(out)
        res.snapshot_steps.append(step)

    def max_abs(self) -> float:
        """kernel.hpp:265-273."""
        self._upload_if_viewed()
        v = C.c_double()
        _check(self._ctx, _lib.lib().fdw_max_abs(self._ctx, C.byref(v)), "fdw_max_abs")
        return float(v.value)

    # -- device-side extras (not in the reference API) --
    def seismogram_f64(self, rows: Optional[int] = None) -> np.ndarray:
        rows = self._time.n_steps + 1 if rows is None else rows
        out = np.empty(rows * self._n_rec, np.float64)
        _check(self._ctx, _lib.lib().fdw_download_seismogram_f64(self._ctx, ptr(out), rows),
               "fdw_download_seismogram_f64")
        return out

    def _extended_local(self):
        ext = list(self._grid.extended_shape[:self._grid.ndim])
        if self._desc.world > 1:
            ext[0] = int(self._desc.z_end - self._desc.z_begin)
        return ext

    def extended_level(self) -> np.ndarray:
        out = np.empty(tuple(self._extended_local()), self._dtype)
        _check(self._ctx, _lib.lib().fdw_get_extended(self._ctx, ptr(out)), "fdw_get_extended")
        return out

    def layout(self) -> dict:
        ld, plane, base, planes = (C.c_uint64() for _ in range(4))
        var = C.c_int32()
        _lib.lib().fdw_layout(self._ctx, C.byref(ld), C.byref(plane), C.byref(base), C.byref(planes),
                              C.byref(var))
        return {"ld": ld.value, "plane": plane.value, "base": base.value, "planes": planes.value,
                "variant": var.value & 0xFF, "z_segments": (var.value >> 8) & 0xFF,
                "ctas_per_sm": (var.value >> 16) & 0xFF, "tma_pd": var.value >> 24}

    # -- peer transport (Z slabs over NVLink peer memory) --
    def peer_export(self) -> bytes:
        """IPC handles of this rank's levels and sync block (fdw_peer_export)."""
        buf = (C.c_ubyte * _lib.FDW_PEER_BLOB_BYTES)()
        _check(self._ctx, _lib.lib().fdw_peer_export(self._ctx, C.byref(buf)), "fdw_peer_export")
        return bytes(buf)

    def peer_import(self, blobs) -> None:
        """Every rank's peer_export() blob in rank order (one process per GPU)."""
        data = b"".join(bytes(b) for b in blobs)
        buf = (C.c_ubyte * len(data)).from_buffer_copy(data)
        _check(self._ctx, _lib.lib().fdw_peer_import(self._ctx, C.byref(buf), len(blobs)), "fdw_peer_import")

    def peer_link(self, solvers) -> None:
        """All ranks' Solvers driven from this process (one thread per rank)."""
        arr = (C.c_void_p * len(solvers))(*[s._ctx.value for s in solvers])
        _check(self._ctx, _lib.lib().fdw_peer_link(self._ctx, arr, len(solvers)), "fdw_peer_link")

    def debug_check_guards(self) -> int:
        """Guard / slack violations (context created with FDW_GUARD_CHECK=1)."""
        v = C.c_uint64()
        _check(self._ctx, _lib.lib().fdw_debug_check_guards(self._ctx, C.byref(v)), "fdw_debug_check_guards")
        return int(v.value)

    def peer_loopback(self) -> None:
        """Profiling: emulated neighbours on this GPU (fdw_peer_loopback)."""
        _check(self._ctx, _lib.lib().fdw_peer_loopback(self._ctx), "fdw_peer_loopback")

    def set_stream(self, stream_ptr: int):
        _check(self._ctx, _lib.lib().fdw_set_stream(self._ctx, C.c_void_p(stream_ptr)), "fdw_set_stream")

    def advance_raw(self, n: int, record: bool = False):
        """n device steps without host-mirror traffic (for timing loops)."""
        self._advance(n, FDW_ADVANCE_RECORD if record else 0)

    def reset_state(self):
        """Quiescent restart on the same medium: zero levels, step 0."""
        _check(self._ctx, _lib.lib().fdw_zero_levels(self._ctx), "fdw_zero_levels")
        self.set_step_index(0)

    def set_step_index(self, step: int):
        _check(self._ctx, _lib.lib().fdw_set_step_index(self._ctx, step), "fdw_set_step_index")

    def profile_steps(self, n: int) -> list:
        ms = (C.c_double * 6)()
        _check(self._ctx, _lib.lib().fdw_profile_steps(self._ctx, n, ms), "fdw_profile_steps")
        return list(ms)

    def launch_count(self) -> int:
        v = C.c_uint64()
        _lib.lib().fdw_launch_count(self._ctx, C.byref(v))
        return int(v.value)

    @property
    def ctx(self):
        return self._ctx
