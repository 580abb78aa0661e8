"""SlabSolver -- fdwave::Solver<T> over several GPUs from one process.

The Python counterpart of the C++ drop-in's FDW_DEVICES mode
(include/fdwave/kernel.hpp): a 3D grid is split into Z slabs with
fdw_slab_range, one slab Solver per device, linked in-process
(fdw_peer_link).  The halo planes travel inside each step over NVLink peer
memory; this class only scatters and gathers the host
views and drives every collective call from one host thread per rank.  It
replaces the reference's only parallelism, the OpenMP loop over Z planes
(kernel.hpp:392-393), with one GPU per slab, behind the same public API as
Solver (kernel.hpp:170-273).

Repeated device ordinals (devices=[0, 0]) emulate slabs on one GPU; the
library then orders the ranks on the host (host-ordered group).
"""
from __future__ import annotations

import os
import time
from concurrent.futures import ThreadPoolExecutor
from typing import List, Optional, Sequence

import numpy as np

from .kernel import ForwardResult, InstabilityError, Solver
from .model import DampingField, MaterialModel


def devices_from_env() -> List[int]:
    """FDW_DEVICES="0-7" or "0,1,2" (as the C++ drop-in reads it)."""
    spec = os.environ.get("FDW_DEVICES", "").strip()
    out: List[int] = []
    for tok in filter(None, (t.strip() for t in spec.split(","))):
        if "-" in tok:
            lo, hi = tok.split("-", 1)
            out.extend(range(int(lo), int(hi) + 1))
        else:
            out.append(int(tok))
    return out


class SlabSolver:
    """Solver over len(devices) Z slabs.  Same methods and semantics as Solver;
    the host arrays it takes and returns are the full padded grid."""

    def __init__(self, grid, materials, damping, boundary, time_axis, coeffs, *, devices: Sequence[int],
                 variant: int = 0, math: int = 0, z_segments: int = 0):
        from .dist import slab_range
        if grid.ndim != 3:
            raise ValueError("slab decomposition is 3D only")
        self._grid, self._time = grid, time_axis
        self._devices = list(devices)
        world = len(self._devices)
        R = grid.halo
        if grid.extended_shape[0] < 2 * R * world:
            raise ValueError(f"{grid.extended_shape[0]} extended planes cannot give {world} slabs of >= {2 * R}")
        self._slabs = [slab_range(grid.extended_shape[0], world, r) for r in range(world)]
        vel = np.ascontiguousarray(materials.velocity)
        eta = np.ascontiguousarray(damping.eta, dtype=vel.dtype)
        rho = None if materials.density is None else np.ascontiguousarray(materials.density, dtype=vel.dtype)
        self._dtype = vel.dtype
        self._shape = tuple(grid.padded_shape()[:3])
        self._ranks: List[Solver] = []
        for r, (zb, ze) in enumerate(self._slabs):
            sl = slice(zb, ze + 2 * R)  # the rank's padded slab: contiguous Z planes
            mats = MaterialModel(velocity=vel[sl], density=None if rho is None else rho[sl], c_max=materials.c_max)
            self._ranks.append(Solver(grid, mats, DampingField(eta=eta[sl]), boundary, time_axis, coeffs,
                                      device=self._devices[r], variant=variant, math=math, z_segments=z_segments,
                                      slab=(r, world, zb, ze)))
        for s in self._ranks:
            s.peer_link(self._ranks)
        for s in self._ranks[1:]:
            s._verbose_quiet = True  # rank 0 prints the progress line
        self._pool = ThreadPoolExecutor(max_workers=world)
        self._prev: Optional[np.ndarray] = None
        self._curr: Optional[np.ndarray] = None
        self._host_view = False
        self._n_rec = 0
        self._receiver_coordinates: list = []

    # -- lifetime --
    def close(self):
        for s in getattr(self, "_ranks", []):
            s.close()
        self._ranks = []
        if getattr(self, "_pool", None):
            self._pool.shutdown(wait=True)
            self._pool = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def devices(self) -> List[int]:
        return list(self._devices)

    # every rank at once (collective calls wait for each other)
    def _all(self, fn):
        futs = [self._pool.submit(fn, r, s) for r, s in enumerate(self._ranks)]
        out, err = [], []
        for f in futs:
            try:
                out.append(f.result())
            except BaseException as e:  # noqa: BLE001 -- re-raised below
                out.append(None)
                err.append(e)
        if err:
            inst = [e for e in err if isinstance(e, InstabilityError)]
            raise inst[0] if inst else err[0]
        return out

    # -- reference API --
    def set_sources(self, sources, wavelet):
        for s in self._ranks:  # each slab keeps the taps it owns
            s.set_sources(sources, wavelet)

    def set_receivers(self, receivers, coordinates=None):
        for s in self._ranks:
            s.set_receivers(receivers, coordinates)
        self._n_rec = receivers.n_points
        self._receiver_coordinates = list(coordinates or [])

    def add_volume_source(self, source):
        from .kernel import ModulatedField
        R = self._grid.halo
        f = np.ascontiguousarray(source.field, dtype=self._dtype)
        for s, (zb, ze) in zip(self._ranks, self._slabs):
            s.add_volume_source(ModulatedField(field=f[zb:ze + 2 * R], amplitude=source.amplitude))

    def set_backend(self, backend, workers: int = 0):
        """kernel.hpp:204-211 -- accepted and ignored."""

    def set_verbose(self, verbose: bool):
        for s in self._ranks:
            s.set_verbose(verbose)

    def set_snapshot_cap(self, nbytes: int):
        for s in self._ranks:
            s.set_snapshot_cap(nbytes)

    def grid(self):
        return self._grid

    def time_axis(self):
        return self._time

    def step_index(self) -> int:
        return self._ranks[0].step_index()

    # host views of the full padded grid: gathered from the slabs (owned
    # planes, plus the global Z ghost planes of the first / last rank) and
    # scattered back before the next device call
    def _gather(self):
        if self._curr is None:
            self._prev = np.zeros(self._shape, self._dtype)
            self._curr = np.zeros(self._shape, self._dtype)
        R, world = self._grid.halo, len(self._ranks)
        for r, (s, (zb, ze)) in enumerate(zip(self._ranks, self._slabs)):
            s._download()
            nl = ze - zb + 2 * R
            lo, hi = (0 if r == 0 else R), (nl if r == world - 1 else nl - R)
            self._prev[zb + lo:zb + hi] = s._prev[lo:hi]
            self._curr[zb + lo:zb + hi] = s._curr[lo:hi]

    def _scatter(self):
        if not self._host_view:
            return
        R = self._grid.halo
        for s, (zb, ze) in zip(self._ranks, self._slabs):
            s._ensure_host()
            s._prev[...] = self._prev[zb:ze + 2 * R]
            s._curr[...] = self._curr[zb:ze + 2 * R]
            s._host_view = True
            s._upload_if_viewed()
            s._host_view = False

    def current_level(self) -> np.ndarray:
        if not self._host_view:
            self._gather()
            self._host_view = True
        return self._curr

    def previous_level(self) -> np.ndarray:
        if not self._host_view:
            self._gather()
            self._host_view = True
        return self._prev

    def refresh_boundary(self):
        self._scatter()
        self._all(lambda r, s: s.refresh_boundary())
        if self._host_view:
            self._gather()

    def step(self):
        self._scatter()
        self._all(lambda r, s: s._advance(1, 0))
        if self._host_view:
            self._gather()

    def forward(self) -> ForwardResult:
        self._scatter()
        t0 = time.perf_counter()
        outs = self._all(lambda r, s: s.forward())
        res = ForwardResult()
        res.kernel_seconds = time.perf_counter() - t0
        res.snapshot_steps = list(outs[0].snapshot_steps)
        res.snapshots = [np.concatenate([o.snapshots[i] for o in outs], axis=0)
                         for i in range(len(outs[0].snapshots))]
        res.seismogram.n_receivers = self._n_rec
        res.seismogram.coordinates = list(self._receiver_coordinates)
        if self._n_rec:
            res.seismogram.data = self.seismogram_f64().astype(self._dtype)
        if self._host_view:
            self._gather()
        return res

    def max_abs(self) -> float:
        self._scatter()
        return self._all(lambda r, s: s.max_abs())[0]  # reduced over every slab

    # -- device-side extras --
    def seismogram_f64(self, rows: Optional[int] = None) -> np.ndarray:
        """The reference's accumulation (acquisition.hpp:155-158) over all
        slabs, bit for bit: per-slab partials plus the straddling receivers'
        per-tap products merged in entry order (dist.merge_seismogram)."""
        from .dist import merge_seismogram, split_products
        rows = self._time.n_steps + 1 if rows is None else rows
        parts = [s.seismogram_f64(rows) for s in self._ranks]
        return merge_seismogram(parts, [split_products(s, rows) for s in self._ranks], self._n_rec)
