"""ctypes wrappers of the CPU checkers -- TEST INFRASTRUCTURE ONLY.

  Oracle     -> oracle/liboracle.so          (C restatement, fdw_oracle.c)
  Reference  -> oracle/_ref/libfdwave_ref.so (the reference headers compiled in
                                              place by oracle/Makefile)

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libfdwave_ref.so")

_P = C.c_void_p
_U64 = C.c_uint64
_U64P = C.POINTER(C.c_uint64)
_DP = C.POINTER(C.c_double)


class fdwo_grid(C.Structure):
    _fields_ = [("ndim", C.c_int32), ("halo", C.c_int32), ("space_order", C.c_int32), ("_pad", C.c_int32),
                ("bbox", (C.c_double * 2) * 3), ("spacing", C.c_double * 3), ("interior", C.c_uint64 * 3),
                ("damping_cells", (C.c_uint64 * 2) * 3), ("damping_length", (C.c_double * 2) * 3),
                ("extended", C.c_uint64 * 3), ("padded", C.c_uint64 * 3)]


class ref_config(C.Structure):
    _fields_ = [("ndim", C.c_int32), ("space_order", C.c_int32), ("dtype", C.c_int32),
                ("window_radius", C.c_int32), ("bc", (C.c_int32 * 2) * 3), ("bbox", C.c_double * 6),
                ("spacing", C.c_double * 3), ("damping", C.c_double * 6), ("tf", C.c_double),
                ("dt", C.c_double), ("alpha", C.c_double), ("power", C.c_double), ("f0", C.c_double),
                ("saving_stride", C.c_uint64)]


def build(force: bool = False) -> None:
    """make -C oracle (liboracle.so always; _ref/ when /root/reference exists)."""
    if force or not os.path.exists(ORACLE_SO) or (os.path.isdir("/root/reference") and not os.path.exists(REF_SO)):
        subprocess.run(["make", "-s", "-C", HERE], check=True)


def _ptr(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


def _bc(bc):
    arr = ((C.c_int32 * 2) * 3)()
    for a in range(3):
        for s in range(2):
            arr[a][s] = int(bc[a][s])
    return arr


_olib = None
_rlib = None


def olib():
    global _olib
    if _olib is None:
        build()
        L = C.CDLL(ORACLE_SO)
        L.fdwo_stable_dt.restype = C.c_double
        L.fdwo_stable_dt.argtypes = [C.c_double, _DP, C.c_int, C.c_int, C.c_int]
        L.fdwo_n_steps.restype = _U64
        L.fdwo_n_steps.argtypes = [C.c_double, C.c_double]
        L.fdwo_build_grid.argtypes = [C.c_int, _DP, _DP, C.c_int, _DP, C.POINTER(fdwo_grid)]
        L.fdwo_second_derivative_coefficients.argtypes = [C.c_int, _DP]
        L.fdwo_first_derivative_coefficients.argtypes = [C.c_int, _DP]
        L.fdwo_resample_model.argtypes = [C.POINTER(fdwo_grid), _P, _P, C.c_int, _P]
        L.fdwo_damping_field.argtypes = [C.POINTER(fdwo_grid), C.c_double, C.c_double, C.c_int, _P]
        for f in ("fdwo_bessel_i0", "fdwo_sinc"):
            getattr(L, f).restype = C.c_double
            getattr(L, f).argtypes = [C.c_double]
        L.fdwo_kaiser_window.restype = C.c_double
        L.fdwo_kaiser_window.argtypes = [C.c_double, C.c_int, C.c_double]
        L.fdwo_default_kaiser_b.restype = C.c_double
        L.fdwo_default_kaiser_b.argtypes = [C.c_int]
        L.fdwo_build_injection_map.restype = C.c_int64
        L.fdwo_build_injection_map.argtypes = [C.POINTER(fdwo_grid), _P, _U64, C.c_int, C.c_double, _P, _P, _P, _U64]
        L.fdwo_ricker_samples.argtypes = [_U64, C.c_double, C.c_double, _P]
        L.fdwo_apply_boundary.argtypes = [C.POINTER(fdwo_grid), _P, C.c_int, _P]
        L.fdwo_solver_create.argtypes = [C.POINTER(fdwo_grid), C.c_int, _DP, C.c_double, _U64, _P, _P, _P,
                                         C.POINTER(_P)]
        L.fdwo_solver_destroy.argtypes = [_P]
        L.fdwo_solver_set_density.argtypes = [_P, _P]
        L.fdwo_density_log_gradient.argtypes = [C.POINTER(fdwo_grid), C.c_int, _P, _P]
        L.fdwo_solver_set_threads.argtypes = [_P, C.c_int]
        L.fdwo_solver_add_volume_source.argtypes = [_P, _P, _P, _U64]
        L.fdwo_solver_set_sources.argtypes = [_P, _U64, _P, _P, _P, _P, _U64]
        L.fdwo_solver_set_receivers.argtypes = [_P, _U64, _P, _P, _P]
        L.fdwo_solver_current.restype = _P
        L.fdwo_solver_current.argtypes = [_P]
        L.fdwo_solver_previous.restype = _P
        L.fdwo_solver_previous.argtypes = [_P]
        L.fdwo_solver_step_index.restype = _U64
        L.fdwo_solver_step_index.argtypes = [_P]
        L.fdwo_solver_refresh_boundary.argtypes = [_P]
        L.fdwo_solver_step.argtypes = [_P, _U64P, _DP]
        L.fdwo_solver_max_abs.restype = C.c_double
        L.fdwo_solver_max_abs.argtypes = [_P]
        L.fdwo_solver_sample.argtypes = [_P, _P]
        L.fdwo_solver_forward.argtypes = [_P, _P, _P, _DP, _U64P, _DP]
        _olib = L
    return _olib


def rlib():
    """The reference compiled in place; None when it was never built."""
    global _rlib
    if _rlib is None:
        build()
        if not os.path.exists(REF_SO):
            return None
        L = C.CDLL(REF_SO)
        L.ref_last_error.restype = C.c_char_p
        L.ref_run_create.restype = _P
        L.ref_run_create.argtypes = [C.POINTER(ref_config), _P, _P, _P, _U64, _P, _U64]
        L.ref_solver_create.restype = _P
        L.ref_solver_create.argtypes = [C.c_int, C.c_int, C.c_int, _P, _P, C.c_double, _U64, _P, _P, _P]
        L.ref_destroy.argtypes = [_P]
        L.ref_solver_create_vd.restype = _P
        L.ref_solver_create_vd.argtypes = [C.c_int, C.c_int, C.c_int, _P, _P, C.c_double, _U64, _P, _P, _P, _P]
        L.ref_density_log_gradient.argtypes = [C.c_int, C.c_int, C.c_int, _P, _P, _P, _P]
        L.ref_info.restype = _U64
        L.ref_info.argtypes = [_P, _P, _DP, _U64P, _U64P]
        L.ref_get_fields.argtypes = [_P, _P, _P]
        L.ref_get_map.argtypes = [_P, C.c_int, _P, _P, _P]
        L.ref_get_wavelet.argtypes = [_P, _P]
        L.ref_set_threads.argtypes = [_P, C.c_int]
        L.ref_solver_add_volume_source.argtypes = [_P, _P, _P, _U64]
        L.ref_step.argtypes = [_P, _U64P, _DP]
        L.ref_level.restype = _P
        L.ref_level.argtypes = [_P, C.c_int]
        L.ref_refresh.argtypes = [_P]
        L.ref_max_abs.restype = C.c_double
        L.ref_max_abs.argtypes = [_P]
        L.ref_sample.argtypes = [_P, _P]
        L.ref_forward.argtypes = [_P, _P, _P, _DP, _U64P, _DP]
        L.ref_time_steps.argtypes = [_P, _U64, _DP]
        L.ref_solver_set_sources.argtypes = [_P, _U64, _P, _P, _P, _P, _U64]
        L.ref_solver_set_receivers.argtypes = [_P, _U64, _P, _P, _P]
        L.ref_second_derivative.argtypes = [C.c_int, _P]
        L.ref_stable_dt.restype = C.c_double
        L.ref_stable_dt.argtypes = [C.c_double, _P, C.c_int, C.c_int, C.c_int]
        for f in ("ref_bessel_i0", "ref_sinc"):
            getattr(L, f).restype = C.c_double
            getattr(L, f).argtypes = [C.c_double]
        L.ref_ricker.argtypes = [_U64, C.c_double, C.c_double, _P]
        L.ref_max_threads.restype = C.c_int
        _rlib = L
    return _rlib


def oracle_grid(ndim, bbox, spacing, order, damping):
    g = fdwo_grid()
    b = np.asarray(bbox, np.float64)
    s = np.asarray(spacing, np.float64)
    d = np.asarray(damping, np.float64)
    rc = olib().fdwo_build_grid(ndim, b.ctypes.data_as(_DP), s.ctypes.data_as(_DP), order,
                                d.ctypes.data_as(_DP), C.byref(g))
    if rc:
        raise ValueError("fdwo_build_grid failed")
    return g


class OracleSolver:
    """fdwo_solver handle: the C restatement of Solver<T> on caller arrays."""

    def __init__(self, ndim, order, dtype, extended, spacing, dt, n_steps, bc, velocity, eta, threads=0,
                 density=None):
        L = olib()
        g = fdwo_grid()
        g.ndim, g.halo, g.space_order = ndim, order // 2, order
        for a in range(3):
            g.spacing[a] = float(spacing[a]) if a < ndim else 1.0
            g.extended[a] = int(extended[a]) if a < ndim else 1
            g.interior[a] = g.extended[a]
            g.padded[a] = g.extended[a] + (order if a < ndim else 0)
        self.grid = g
        self.dtype = np.dtype(dtype)
        self.shape = tuple(int(g.padded[a]) for a in range(ndim))
        coeffs = np.zeros(11)
        L.fdwo_second_derivative_coefficients(order, coeffs.ctypes.data_as(_DP))
        self.vel = np.ascontiguousarray(velocity, self.dtype).reshape(self.shape)
        self.eta = np.ascontiguousarray(eta, self.dtype).reshape(self.shape)
        self.h = _P()
        rc = L.fdwo_solver_create(C.byref(g), self.dtype.itemsize, coeffs.ctypes.data_as(_DP), dt, n_steps,
                                  _bc(bc), _ptr(self.vel), _ptr(self.eta), C.byref(self.h))
        if rc:
            raise ValueError("fdwo_solver_create failed")
        L.fdwo_solver_set_threads(self.h, threads)
        self.n_steps = n_steps
        self.n_rec = 0
        if density is not None:
            self.rho = np.ascontiguousarray(density, self.dtype).reshape(self.shape)
            if L.fdwo_solver_set_density(self.h, _ptr(self.rho)):
                raise ValueError("fdwo_solver_set_density failed")

    def __del__(self):
        if getattr(self, "h", None):
            olib().fdwo_solver_destroy(self.h)
            self.h = None

    def _view(self, p):
        n = int(np.prod(self.shape))
        buf = (C.c_char * (n * self.dtype.itemsize)).from_address(p)
        return np.frombuffer(buf, self.dtype).reshape(self.shape)

    def current(self):
        return self._view(olib().fdwo_solver_current(self.h))

    def previous(self):
        return self._view(olib().fdwo_solver_previous(self.h))

    def set_sources(self, imap, wavelet):
        wav = np.ascontiguousarray(wavelet, np.float64)
        self._src = (np.ascontiguousarray(imap.offsets, np.uint64), np.ascontiguousarray(imap.index, np.uint64),
                     np.ascontiguousarray(imap.weight, np.float64), wav)
        rc = olib().fdwo_solver_set_sources(self.h, imap.n_points, *(_ptr(a) for a in self._src), len(wav))
        if rc:
            raise ValueError("wavelet shorter than the time axis")

    def set_receivers(self, imap):
        self._rec = (np.ascontiguousarray(imap.offsets, np.uint64), np.ascontiguousarray(imap.index, np.uint64),
                     np.ascontiguousarray(imap.weight, np.float64))
        olib().fdwo_solver_set_receivers(self.h, imap.n_points, *(_ptr(a) for a in self._rec))
        self.n_rec = imap.n_points

    def add_volume_source(self, field, amplitude):
        """kernel.hpp:199-203 (ModulatedField, :140-144)."""
        f = np.ascontiguousarray(field, self.dtype).reshape(self.shape)
        a = np.ascontiguousarray(amplitude, np.float64)
        if olib().fdwo_solver_add_volume_source(self.h, _ptr(f), _ptr(a), len(a)):
            raise ValueError("volume source amplitude shorter than run")
        self._vol = getattr(self, "_vol", []) + [(f, a)]

    def refresh_boundary(self):
        olib().fdwo_solver_refresh_boundary(self.h)

    def step(self):
        bs, bm = C.c_uint64(), C.c_double()
        rc = olib().fdwo_solver_step(self.h, C.byref(bs), C.byref(bm))
        if rc == 4:
            return int(bs.value), float(bm.value)
        return None

    def step_index(self):
        return int(olib().fdwo_solver_step_index(self.h))

    def max_abs(self):
        return float(olib().fdwo_solver_max_abs(self.h))

    def forward(self):
        seis = np.zeros((self.n_steps + 1) * max(self.n_rec, 1), self.dtype)
        ext = tuple(int(self.grid.extended[a]) for a in range(self.grid.ndim))
        final = np.zeros(ext, self.dtype)
        secs, bs, bm = C.c_double(), C.c_uint64(), C.c_double()
        rc = olib().fdwo_solver_forward(self.h, _ptr(seis), _ptr(final), C.byref(secs), C.byref(bs), C.byref(bm))
        if rc == 4:
            return {"unstable": (int(bs.value), float(bm.value))}
        return {"seismogram": seis[: (self.n_steps + 1) * self.n_rec], "final": final, "seconds": secs.value}


class RefRun:
    """A whole synthetic run built by the reference's own setup chain."""

    def __init__(self, cfg, dtype=np.float32, raw=None, threads=0):
        from paper_2201_05278_b200.configs import synthetic_raw  # raw generator only
        L = rlib()
        if L is None:
            raise RuntimeError("oracle/_ref/libfdwave_ref.so is not built (reference tree absent)")
        rc_ = ref_config()
        rc_.ndim, rc_.space_order, rc_.dtype = cfg.ndim, cfg.space_order, np.dtype(dtype).itemsize
        rc_.window_radius = cfg.window_radius
        for a in range(3):
            for s in range(2):
                rc_.bc[a][s] = int(cfg.bc[a][s])
        for i, v in enumerate(cfg.bbox):
            rc_.bbox[i] = v
        for i, v in enumerate(cfg.spacing):
            rc_.spacing[i] = v
        for i, v in enumerate(cfg.damping):
            rc_.damping[i] = v
        rc_.tf = cfg.tf
        rc_.dt = cfg.dt or 0.0
        if cfg.fixed_steps is not None:
            from paper_2201_05278_b200.stencil import stable_dt
            dt = stable_dt(float(np.dtype(dtype).type(cfg.vmax)), cfg.spacing[:cfg.ndim], cfg.space_order, cfg.ndim)
            rc_.dt, rc_.tf = dt, dt * cfg.fixed_steps
        rc_.alpha, rc_.power, rc_.f0 = cfg.alpha, cfg.power, cfg.f0
        g = oracle_grid(cfg.ndim, cfg.bbox, cfg.spacing[:cfg.ndim], cfg.space_order, cfg.damping)
        raw_shape = np.array([g.interior[a] for a in range(cfg.ndim)], np.uint64)
        if raw is None:
            raw = synthetic_raw(tuple(int(v) for v in raw_shape), cfg.vmin, cfg.vmax)
        self.raw = np.ascontiguousarray(raw, np.float64)
        self.raw_shape = raw_shape
        src = np.ascontiguousarray(np.asarray(cfg.sources, np.float64).reshape(-1, 3))
        rec = np.ascontiguousarray(np.asarray(cfg.receivers, np.float64).reshape(-1, 3))
        self.h = L.ref_run_create(C.byref(rc_), _ptr(self.raw), _ptr(raw_shape), _ptr(src), len(src),
                                  _ptr(rec), len(rec))
        if not self.h:
            raise ValueError(L.ref_last_error().decode())
        self.dtype = np.dtype(dtype)
        shapes = np.zeros(6, np.uint64)
        dt_, ns, nr = C.c_double(), C.c_uint64(), C.c_uint64()
        self.n_steps = int(L.ref_info(self.h, _ptr(shapes), C.byref(dt_), C.byref(ns), C.byref(nr)))
        self.dt = dt_.value
        self.ndim = cfg.ndim
        self.extended = tuple(int(v) for v in shapes[:cfg.ndim])
        self.padded = tuple(int(v) for v in shapes[3:3 + cfg.ndim])
        self.n_src_entries, self.n_rec_entries = int(ns.value), int(nr.value)
        self.n_src, self.n_rec = len(src), len(rec)
        L.ref_set_threads(self.h, threads)

    def __del__(self):
        if getattr(self, "h", None):
            rlib().ref_destroy(self.h)
            self.h = None

    def fields(self):
        v = np.zeros(self.padded, self.dtype)
        e = np.zeros(self.padded, self.dtype)
        rlib().ref_get_fields(self.h, _ptr(v), _ptr(e))
        return v, e

    def maps(self):
        out = []
        for which, n, m in ((0, self.n_src, self.n_src_entries), (1, self.n_rec, self.n_rec_entries)):
            off = np.zeros(n + 1, np.uint64)
            idx = np.zeros(max(m, 1), np.uint64)
            w = np.zeros(max(m, 1), np.float64)
            rlib().ref_get_map(self.h, which, _ptr(off), _ptr(idx), _ptr(w))
            out.append((off, idx[:m], w[:m]))
        return out

    def wavelet(self):
        w = np.zeros(self.n_steps + 1, np.float64)
        if self.n_src:
            rlib().ref_get_wavelet(self.h, _ptr(w))
        return w

    def forward(self):
        seis = np.zeros((self.n_steps + 1) * max(self.n_rec, 1), self.dtype)
        final = np.zeros(self.extended, self.dtype)
        secs, bs, bm = C.c_double(), C.c_uint64(), C.c_double()
        rc = rlib().ref_forward(self.h, _ptr(seis), _ptr(final), C.byref(secs), C.byref(bs), C.byref(bm))
        if rc == 4:
            return {"unstable": (int(bs.value), float(bm.value))}
        return {"seismogram": seis[: (self.n_steps + 1) * self.n_rec], "final": final, "seconds": secs.value}

    def set_levels(self, prev, curr):
        """Overwrites the reference Solver's levels (current_level() /
        previous_level() are mutable references, kernel.hpp:217-218), e.g. with
        a developed wavefield for a representative CPU timing sample."""
        L = rlib()
        for which, a in ((0, prev), (1, curr)):
            a = np.ascontiguousarray(a, self.dtype)
            n = int(np.prod(self.padded))
            if a.size != n:
                raise ValueError("level shape does not match the padded grid")
            C.memmove(L.ref_level(self.h, which), a.ctypes.data, a.nbytes)

    def time_steps(self, n):
        secs = C.c_double()
        rc = rlib().ref_time_steps(self.h, n, C.byref(secs))
        if rc:
            raise RuntimeError("reference went unstable while timing")
        return secs.value


class RefSolver:
    """Reference Solver<T> built on caller arrays (test_kernel.cpp make_solver style)."""

    def __init__(self, ndim, order, dtype, extended, spacing, dt, n_steps, bc, velocity, eta, density=None):
        L = rlib()
        if L is None:
            raise RuntimeError("reference library not built")
        self.dtype = np.dtype(dtype)
        self.shape = tuple(int(e) + order for e in extended[:ndim])
        ext = np.array(list(extended) + [1] * (3 - len(extended)), np.uint64)
        sp = np.array(list(spacing) + [1.0] * (3 - len(spacing)), np.float64)
        self.vel = np.ascontiguousarray(velocity, self.dtype)
        self.eta = np.ascontiguousarray(eta, self.dtype)
        bcs = np.array([[int(bc[a][s]) for s in range(2)] for a in range(3)], np.int32)
        self.rho = None if density is None else np.ascontiguousarray(density, self.dtype)
        self.h = L.ref_solver_create_vd(ndim, order, self.dtype.itemsize, _ptr(ext), _ptr(sp), dt, n_steps,
                                        _ptr(bcs), _ptr(self.vel), _ptr(self.eta), _ptr(self.rho))
        if not self.h:
            raise ValueError(L.ref_last_error().decode())
        self.n_steps = n_steps

    def __del__(self):
        if getattr(self, "h", None):
            rlib().ref_destroy(self.h)
            self.h = None

    def _view(self, which):
        p = rlib().ref_level(self.h, which)
        n = int(np.prod(self.shape))
        buf = (C.c_char * (n * self.dtype.itemsize)).from_address(p)
        return np.frombuffer(buf, self.dtype).reshape(self.shape)

    def current(self):
        return self._view(1)

    def previous(self):
        return self._view(0)

    def set_sources(self, imap, wavelet):
        self._src = (np.ascontiguousarray(imap.offsets, np.uint64), np.ascontiguousarray(imap.index, np.uint64),
                     np.ascontiguousarray(imap.weight, np.float64), np.ascontiguousarray(wavelet, np.float64))
        rlib().ref_solver_set_sources(self.h, imap.n_points, *(_ptr(a) for a in self._src), len(self._src[3]))

    def set_receivers(self, imap):
        self._rec = (np.ascontiguousarray(imap.offsets, np.uint64), np.ascontiguousarray(imap.index, np.uint64),
                     np.ascontiguousarray(imap.weight, np.float64))
        rlib().ref_solver_set_receivers(self.h, imap.n_points, *(_ptr(a) for a in self._rec))

    def add_volume_source(self, field, amplitude):
        f = np.ascontiguousarray(field, self.dtype)
        a = np.ascontiguousarray(amplitude, np.float64)
        if rlib().ref_solver_add_volume_source(self.h, _ptr(f), _ptr(a), len(a)):
            raise ValueError(rlib().ref_last_error().decode())

    def refresh_boundary(self):
        rlib().ref_refresh(self.h)

    def step(self):
        bs, bm = C.c_uint64(), C.c_double()
        rc = rlib().ref_step(self.h, C.byref(bs), C.byref(bm))
        if rc == 4:
            return int(bs.value), float(bm.value)
        return None

    def max_abs(self):
        return float(rlib().ref_max_abs(self.h))

    def sample(self, n_rec):
        row = np.zeros(n_rec, self.dtype)
        rlib().ref_sample(self.h, _ptr(row))
        return row
