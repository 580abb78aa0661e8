"""paper_2201_05278_b200 -- B200-native (sm_100a) constant-density acoustic
propagator of simwave (arXiv 2201.05278), behind the reference's
fdwave::Solver<T> API.

The compute path is libfdwave_cuda.so (include/fdwave_cuda.h); this package is
the Python mirror of the reference's host API (grid / stencil / time axis /
model / acquisition setup producers and Solver) over that C-ABI.
"""
from .acquisition import (InterpolationMap, PointSet, bessel_i0, build_injection_map,
                          default_kaiser_b, hicks_weights_1d, kaiser_window, make_point_set,
                          resample_wavelet, ricker_samples, ricker_wavelet, sample_receivers, sinc)
from .grid import Grid, Precision, build_grid, extend_with_damping
from .kernel import (Backend, BoundaryCondition, BoundarySpec, FdwError, ForwardResult,
                     InstabilityError, ModulatedField, Seismogram, Solver, apply_boundary,
                     boundary_condition_from_string)
from .model import DampingField, MaterialModel, damping_field, make_material_model, resample_model
from .multi import SlabSolver
from .stencil import (StencilCoeffs, first_derivative_coefficients, make_stencil,
                      second_derivative_coefficients, stable_dt)
from .time_axis import TimeAxis, build_time_axis

__all__ = [n for n in dir() if not n.startswith("_")]
