// ref_wrapper.cpp -- extern "C" shim over the UNMODIFIED reference headers
// (/root/reference/proj/include/fdwave/*.hpp, compiled in place; nothing is
// copied).  TEST INFRASTRUCTURE ONLY: built into oracle/_ref/libfdwave_ref.so
// by oracle/Makefile and used (a) to pin the C restatement in fdw_oracle.c,
// (b) to generate tests/golden fixtures, (c) as bench.py's reference CPU arm.
//
// Two entry families:
//   ref_run_*    -- a whole synthetic run built with the reference's own setup
//                  producers (build_grid, extend_with_damping, resample_model,
//                  make_material_model, damping_field, build_time_axis,
//                  build_injection_map, ricker_wavelet) -- runner.hpp:42-110.
//   ref_solver_* -- a Solver<T> built from caller arrays, stepped one step at a
//                  time (mirrors test_kernel.cpp:37-66 make_solver).
#include <array>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "fdwave/acquisition.hpp"
#include "fdwave/grid.hpp"
#include "fdwave/kernel.hpp"
#include "fdwave/model.hpp"
#include "fdwave/stencil.hpp"
#include "fdwave/time_axis.hpp"

using namespace fdwave;

extern "C" {

struct ref_config {
    int32_t ndim, space_order, dtype, window_radius;
    int32_t bc[3][2];
    double bbox[6];
    double spacing[3];
    double damping[6];
    double tf, dt;  // dt <= 0: stable bound
    double alpha, power, f0;
    uint64_t saving_stride;
};

}  // extern "C"

namespace {

BoundarySpec to_spec(const int32_t bc[3][2]) {
    BoundarySpec s;
    for (int a = 0; a < 3; ++a)
        for (int side = 0; side < 2; ++side)
            s.face[a][side] = static_cast<BoundaryCondition>(bc[a][side]);
    return s;
}

thread_local std::string g_err;

struct RunBase {
    virtual ~RunBase() = default;
    Grid grid;
    TimeAxis axis;
    InterpolationMap src, rec;
    std::vector<double> wavelet;
    virtual void get_fields(void* vel, void* eta) = 0;
    virtual int step(uint64_t* bad_step, double* bad_max) = 0;
    virtual void* level(int which) = 0;
    virtual void refresh() = 0;
    virtual double max_abs() = 0;
    virtual void sample(void* row) = 0;
    virtual int forward(void* seis, void* final_ext, double* secs, uint64_t* bad_step,
                        double* bad_max) = 0;
    virtual void set_threads(int threads) = 0;
    virtual void set_maps() = 0;
    virtual int add_volume(const void* field, const double* amp, uint64_t n_amp) = 0;
};

template <typename T>
struct Run : RunBase {
    std::unique_ptr<Solver<T>> solver;
    Field<T> velocity_copy, eta_copy;

    void get_fields(void* vel, void* eta) override {
        if (vel) std::memcpy(vel, velocity_copy.data(), velocity_copy.size() * sizeof(T));
        if (eta) std::memcpy(eta, eta_copy.data(), eta_copy.size() * sizeof(T));
    }
    int step(uint64_t* bad_step, double* bad_max) override {
        try {
            solver->step();
        } catch (const instability_error& e) {
            if (bad_step) *bad_step = e.step();
            if (bad_max) *bad_max = e.max_abs();
            return 4;
        }
        return 0;
    }
    void* level(int which) override {
        return which == 0 ? solver->previous_level().data() : solver->current_level().data();
    }
    void refresh() override { solver->refresh_boundary(); }
    int add_volume(const void* field, const double* amp, uint64_t n_amp) override {
        fdwave::ModulatedField<T> m;
        m.field = Field<T>(grid.ndim, grid.padded_shape());
        std::memcpy(m.field.data(), field, m.field.size() * sizeof(T));
        m.amplitude.assign(amp, amp + n_amp);
        try {
            solver->add_volume_source(std::move(m));
        } catch (const std::exception& e) {
            g_err = e.what();
            return 1;
        }
        return 0;
    }
    double max_abs() override { return solver->max_abs(); }
    void sample(void* row) override {
        const auto r = sample_receivers(solver->current_level(), rec);
        std::memcpy(row, r.data(), r.size() * sizeof(T));
    }
    int forward(void* seis, void* final_ext, double* secs, uint64_t* bad_step,
                double* bad_max) override {
        try {
            const ForwardResult<T> res = solver->forward();
            if (seis)
                std::memcpy(seis, res.seismogram.data.data(),
                            res.seismogram.data.size() * sizeof(T));
            if (final_ext && !res.snapshots.empty())
                std::memcpy(final_ext, res.snapshots.back().data(),
                            res.snapshots.back().size() * sizeof(T));
            if (secs) *secs = res.kernel_seconds;
        } catch (const instability_error& e) {
            if (bad_step) *bad_step = e.step();
            if (bad_max) *bad_max = e.max_abs();
            return 4;
        }
        return 0;
    }
    void set_threads(int threads) override {
        solver->set_backend(threads == 1 ? Backend::Serial : Backend::Parallel, threads);
    }
    void set_maps() override {
        if (!src.points.empty()) solver->set_sources(src, wavelet);
        if (!rec.points.empty()) solver->set_receivers(rec);
    }
};

std::vector<std::array<double, 3>> to_coords(const double* c, uint64_t n) {
    std::vector<std::array<double, 3>> out(n);
    for (uint64_t i = 0; i < n; ++i) out[i] = {c[3 * i], c[3 * i + 1], c[3 * i + 2]};
    return out;
}

template <typename T>
RunBase* make_run(const ref_config* cfg, const double* raw, const uint64_t* raw_shape,
                  const double* src_xyz, uint64_t n_src, const double* rec_xyz,
                  uint64_t n_rec) {
    auto run = std::make_unique<Run<T>>();
    const int nd = cfg->ndim;
    Grid grid = build_grid(std::span<const double>(cfg->bbox, 2 * nd),
                           std::span<const double>(cfg->spacing, nd), cfg->space_order,
                           sizeof(T) == 4 ? Precision::Single : Precision::Double);
    grid = extend_with_damping(grid, std::span<const double>(cfg->damping, 2 * nd));
    std::vector<std::size_t> shape(raw_shape, raw_shape + nd);
    std::size_t count = 1;
    for (auto n : shape) count *= n;
    Field<T> velocity = resample_model<T>(std::span<const double>(raw, count), shape, grid);
    run->velocity_copy = velocity;
    MaterialModel<T> materials = make_material_model<T>(std::move(velocity));
    const double c_max = static_cast<double>(materials.c_max);
    DampingField<T> damping = damping_field<T>(grid, cfg->alpha, cfg->power);
    run->eta_copy = damping.eta;
    std::optional<double> dt;
    if (cfg->dt > 0.0) dt = cfg->dt;
    TimeAxis axis = build_time_axis(cfg->tf, dt, cfg->saving_stride, c_max, grid);
    const StencilCoeffs coeffs = make_stencil(cfg->space_order);
    run->solver = std::make_unique<Solver<T>>(grid, std::move(materials), std::move(damping),
                                              to_spec(cfg->bc), axis, coeffs);
    const int radius = cfg->window_radius > 0 ? cfg->window_radius : 4;
    if (n_src) {
        run->src = build_injection_map(make_point_set(to_coords(src_xyz, n_src), radius), grid);
        run->wavelet = ricker_wavelet(axis, cfg->f0);
    }
    if (n_rec)
        run->rec = build_injection_map(make_point_set(to_coords(rec_xyz, n_rec), radius), grid);
    run->grid = grid;
    run->axis = axis;
    run->set_maps();
    return run.release();
}

template <typename T>
RunBase* make_solver_from_arrays(int ndim, int order, const uint64_t* extended,
                                 const double* spacing, double dt, uint64_t n_steps,
                                 const int32_t bc[3][2], const void* vel, const void* eta,
                                 const void* rho = nullptr) {
    auto run = std::make_unique<Run<T>>();
    Grid grid;
    grid.ndim = ndim;
    grid.space_order = order;
    grid.halo = order / 2;
    for (int a = 0; a < ndim; ++a) {
        grid.extended_shape[a] = extended[a];
        grid.interior_shape[a] = extended[a];
        grid.spacing[a] = spacing[a];
        grid.bbox[a] = {0.0, static_cast<double>(extended[a] - 1) * spacing[a]};
    }
    const auto padded = grid.padded_shape();
    Field<T> v(ndim, padded), e(ndim, padded);
    std::memcpy(v.data(), vel, v.size() * sizeof(T));
    std::memcpy(e.data(), eta, e.size() * sizeof(T));
    run->velocity_copy = v;
    run->eta_copy = e;
    MaterialModel<T> materials;  // bypass the >0 check so tests may pass any field
    materials.velocity = std::move(v);
    if (rho) {  // VariableDensity = true branch of the sweep (kernel.hpp:365-373, :407-417)
        Field<T> r(ndim, padded);
        std::memcpy(r.data(), rho, r.size() * sizeof(T));
        materials.density = std::move(r);
    }
    DampingField<T> damping;
    damping.eta = std::move(e);
    TimeAxis axis;
    axis.dt = dt;
    axis.n_steps = n_steps;
    axis.tf = dt * static_cast<double>(n_steps);
    run->solver = std::make_unique<Solver<T>>(grid, std::move(materials), std::move(damping),
                                              to_spec(bc), axis, make_stencil(order));
    run->grid = grid;
    run->axis = axis;
    return run.release();
}


}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void* ref_run_create(const ref_config* cfg, const double* raw, const uint64_t* raw_shape,
                     const double* src_xyz, uint64_t n_src, const double* rec_xyz,
                     uint64_t n_rec) {
    try {
        if (cfg->dtype == 4)
            return make_run<float>(cfg, raw, raw_shape, src_xyz, n_src, rec_xyz, n_rec);
        return make_run<double>(cfg, raw, raw_shape, src_xyz, n_src, rec_xyz, n_rec);
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void* ref_solver_create(int ndim, int order, int dtype, const uint64_t* extended,
                        const double* spacing, double dt, uint64_t n_steps,
                        const int32_t* bc /* 3x2 */, const void* vel, const void* eta) {
    try {
        const auto* b = reinterpret_cast<const int32_t(*)[2]>(bc);
        if (dtype == 4)
            return make_solver_from_arrays<float>(ndim, order, extended, spacing, dt, n_steps,
                                                  b, vel, eta);
        return make_solver_from_arrays<double>(ndim, order, extended, spacing, dt, n_steps, b,
                                               vel, eta);
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void* ref_solver_create_vd(int ndim, int order, int dtype, const uint64_t* extended,
                           const double* spacing, double dt, uint64_t n_steps, const int32_t* bc,
                           const void* vel, const void* eta, const void* rho) {
    try {
        const auto* b = reinterpret_cast<const int32_t(*)[2]>(bc);
        if (dtype == 4)
            return make_solver_from_arrays<float>(ndim, order, extended, spacing, dt, n_steps, b,
                                                  vel, eta, rho);
        return make_solver_from_arrays<double>(ndim, order, extended, spacing, dt, n_steps, b, vel,
                                               eta, rho);
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

// density_log_gradient (kernel.hpp:104-136) of a padded rho: 3 padded fields out
void ref_density_log_gradient(int ndim, int order, int dtype, const uint64_t* extended,
                              const double* spacing, const void* rho, void* out) {
    Grid grid;
    grid.ndim = ndim;
    grid.space_order = order;
    grid.halo = order / 2;
    for (int a = 0; a < ndim; ++a) {
        grid.extended_shape[a] = extended[a];
        grid.spacing[a] = spacing[a];
    }
    const auto padded = grid.padded_shape();
    auto run = [&](auto tag) {
        using T = decltype(tag);
        Field<T> r(ndim, padded);
        std::memcpy(r.data(), rho, r.size() * sizeof(T));
        const auto g = density_log_gradient(r, grid, make_stencil(order));
        for (int a = 0; a < 3; ++a)
            if (g[a].size())
                std::memcpy(static_cast<char*>(out) + a * r.size() * sizeof(T), g[a].data(),
                            r.size() * sizeof(T));
    };
    if (dtype == 4)
        run(float{});
    else
        run(double{});
}

void ref_destroy(void* h) { delete static_cast<RunBase*>(h); }

// shapes[0..2] extended, [3..5] padded; returns n_steps
uint64_t ref_info(void* h, uint64_t* shapes, double* dt, uint64_t* n_src_entries,
                  uint64_t* n_rec_entries) {
    auto* r = static_cast<RunBase*>(h);
    const auto p = r->grid.padded_shape();
    for (int a = 0; a < 3; ++a) {
        shapes[a] = r->grid.extended_shape[a];
        shapes[3 + a] = p[a];
    }
    if (dt) *dt = r->axis.dt;
    auto count = [](const InterpolationMap& m) {
        uint64_t n = 0;
        for (const auto& e : m.points) n += e.size();
        return n;
    };
    if (n_src_entries) *n_src_entries = count(r->src);
    if (n_rec_entries) *n_rec_entries = count(r->rec);
    return r->axis.n_steps;
}

void ref_get_fields(void* h, void* vel, void* eta) { static_cast<RunBase*>(h)->get_fields(vel, eta); }

// which: 0 sources, 1 receivers; CSR copy-out
void ref_get_map(void* h, int which, uint64_t* offsets, uint64_t* idx, double* w) {
    auto* r = static_cast<RunBase*>(h);
    const InterpolationMap& m = which == 0 ? r->src : r->rec;
    uint64_t k = 0;
    offsets[0] = 0;
    for (std::size_t p = 0; p < m.points.size(); ++p) {
        for (const auto& e : m.points[p]) {
            idx[k] = e.index;
            w[k] = e.weight;
            ++k;
        }
        offsets[p + 1] = k;
    }
}

void ref_get_wavelet(void* h, double* out) {
    auto* r = static_cast<RunBase*>(h);
    std::memcpy(out, r->wavelet.data(), r->wavelet.size() * sizeof(double));
}

void ref_set_threads(void* h, int threads) { static_cast<RunBase*>(h)->set_threads(threads); }

int ref_step(void* h, uint64_t* bad_step, double* bad_max) {
    return static_cast<RunBase*>(h)->step(bad_step, bad_max);
}

void* ref_level(void* h, int which) { return static_cast<RunBase*>(h)->level(which); }
void ref_refresh(void* h) { static_cast<RunBase*>(h)->refresh(); }
double ref_max_abs(void* h) { return static_cast<RunBase*>(h)->max_abs(); }
void ref_sample(void* h, void* row) { static_cast<RunBase*>(h)->sample(row); }

int ref_forward(void* h, void* seis, void* final_ext, double* secs, uint64_t* bad_step,
                double* bad_max) {
    return static_cast<RunBase*>(h)->forward(seis, final_ext, secs, bad_step, bad_max);
}

// Bounded timing sample for the CPU arm: n reference steps (+ receiver record
// per step, as forward() does), wall seconds of the loop only.
int ref_time_steps(void* h, uint64_t n, double* secs) {
    auto* r = static_cast<RunBase*>(h);
    std::vector<double> row(r->rec.points.size() + 1);
    const auto t0 = std::chrono::steady_clock::now();
    for (uint64_t i = 0; i < n; ++i) {
        uint64_t bs;
        double bm;
        if (r->step(&bs, &bm)) return 4;
        if (!r->rec.points.empty()) r->sample(row.data());
    }
    *secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return 0;
}

// ref_solver_*: sources/receivers from caller CSR (indices into the padded field)
int ref_solver_set_sources(void* h, uint64_t n, const uint64_t* off, const uint64_t* idx,
                           const double* w, const double* wavelet, uint64_t n_samples) {
    auto* r = static_cast<RunBase*>(h);
    r->src.points.assign(n, {});
    for (uint64_t p = 0; p < n; ++p)
        for (uint64_t e = off[p]; e < off[p + 1]; ++e) r->src.points[p].push_back({idx[e], w[e]});
    r->wavelet.assign(wavelet, wavelet + n_samples);
    try {
        r->set_maps();
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
    return 0;
}

// Solver::add_volume_source (kernel.hpp:199-203)
int ref_solver_add_volume_source(void* h, const void* field, const double* amp, uint64_t n_amp) {
    return static_cast<RunBase*>(h)->add_volume(field, amp, n_amp);
}

int ref_solver_set_receivers(void* h, uint64_t n, const uint64_t* off, const uint64_t* idx,
                             const double* w) {
    auto* r = static_cast<RunBase*>(h);
    r->rec.points.assign(n, {});
    for (uint64_t p = 0; p < n; ++p)
        for (uint64_t e = off[p]; e < off[p + 1]; ++e) r->rec.points[p].push_back({idx[e], w[e]});
    r->set_maps();
    return 0;
}

// reference setup producers exposed individually
void ref_second_derivative(int order, double* out) {
    const auto v = second_derivative_coefficients(order);
    std::memcpy(out, v.data(), v.size() * sizeof(double));
}
double ref_stable_dt(double c_max, const double* spacing, int n, int order, int ndim) {
    return stable_dt(c_max, std::span<const double>(spacing, n), order, ndim);
}
double ref_bessel_i0(double x) { return bessel_i0(x); }
double ref_sinc(double x) { return sinc(x); }
void ref_ricker(uint64_t count, double dt, double f, double* out) {
    const auto s = ricker_samples(count, dt, f);
    std::memcpy(out, s.data(), s.size() * sizeof(double));
}
int ref_max_threads() {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

}  // extern "C"
