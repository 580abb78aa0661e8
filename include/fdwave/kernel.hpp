// fdwave/kernel.hpp -- DROP-IN replacement for the reference's
// /root/reference/proj/include/fdwave/kernel.hpp (lines 27-495).
//
// Put this directory BEFORE the reference include directory:
//     g++ -std=c++20 -I<repo>/include -I<fdwave>/proj/include ...
//         -L<repo>/paper_2201_05278_b200 -lfdwave_cuda
// The reference headers' own  #include "fdwave/kernel.hpp"  then resolves here,
// so runner.hpp, bench.hpp, verify.hpp and the reference tests compile
// unchanged against the B200 engine.  Every other fdwave header (grid, field,
// model, stencil, time_axis, acquisition) is the reference's own.
//
// Same public names and semantics as the reference: BoundaryCondition,
// boundary_condition_from_string, BoundarySpec, instability_error,
// apply_boundary, density_log_gradient, ModulatedField, Seismogram,
// ForwardResult, Backend, Solver<T>.  Solver<T> keeps its wavefield on the GPU
// and forwards to the C-ABI in fdwave_cuda.h; current_level()/previous_level()
// return host mirrors that are synchronised around device work once they have
// been handed out (the reference returns references to members, kernel.hpp:
// 217-218, and its tests write initial conditions through them).
//
// Variable density (MaterialModel::density) runs on the GPU through
// fdw_set_density (grad(rho)/rho formed on the device, kernel.hpp:104-136 and
// :295-296); add_volume_source through fdw_add_volume_source (:199-203,
// :439-452).  set_backend is accepted and ignored.
#pragma once

#include <array>
#include <chrono>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstdio>
#include <optional>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "fdwave/acquisition.hpp"
#include "fdwave/field.hpp"
#include "fdwave/grid.hpp"
#include "fdwave/model.hpp"
#include "fdwave/stencil.hpp"
#include "fdwave/time_axis.hpp"
#include "fdwave_cuda.h"

namespace fdwave {

enum class BoundaryCondition { NullDirichlet, NullNeumann, None };

inline BoundaryCondition boundary_condition_from_string(const std::string& name) {
    static const std::pair<const char*, BoundaryCondition> table[] = {
        {"null_dirichlet", BoundaryCondition::NullDirichlet},
        {"null_neumann", BoundaryCondition::NullNeumann},
        {"none", BoundaryCondition::None}};
    for (const auto& [key, bc] : table)
        if (name == key) return bc;
    throw std::invalid_argument("unknown boundary condition: " + name);
}

struct BoundarySpec {
    std::array<std::array<BoundaryCondition, 2>, 3> face{};

    static BoundarySpec uniform(BoundaryCondition bc) {
        BoundarySpec spec;
        for (int a = 0; a < 3; ++a) spec.face[a] = {bc, bc};
        return spec;
    }
};

class instability_error : public std::runtime_error {
public:
    instability_error(std::size_t step, double max_abs)
        : std::runtime_error("non-finite wavefield at step " + std::to_string(step) +
                             " (max |p| = " + std::to_string(max_abs) +
                             "); timestep is likely unstable"),
          step_(step),
          max_abs_(max_abs) {}
    std::size_t step() const { return step_; }
    double max_abs() const { return max_abs_; }

private:
    std::size_t step_;
    double max_abs_;
};

/// Host-side halo fill (used for the host mirrors): per axis in order, for
/// every line across the full padded extent of the other axes, the face node is
/// zeroed for null-Dirichlet and the h ghost nodes mirror the interior about it
/// (Dirichlet negated, Neumann as is, none zero).
template <typename T>
void apply_boundary(Field<T>& f, const Grid& grid, const BoundarySpec& spec) {
    const auto pad = grid.padded_shape();
    const std::ptrdiff_t h = grid.halo;
    const auto st = f.strides();
    for (int axis = 0; axis < grid.ndim; ++axis) {
        const std::ptrdiff_t sa = static_cast<std::ptrdiff_t>(st[axis]);
        const std::ptrdiff_t lo_face = h;
        const std::ptrdiff_t hi_face = h + static_cast<std::ptrdiff_t>(grid.extended_shape[axis]) - 1;
        // enumerate the starts of all lines along `axis`
        std::array<int, 2> other{};
        for (int a = 0, k = 0; a < 3; ++a)
            if (a != axis) other[k++] = a;
        for (std::size_t i = 0; i < pad[other[0]]; ++i) {
            for (std::size_t j = 0; j < pad[other[1]]; ++j) {
                T* line = f.data() + i * st[other[0]] + j * st[other[1]];
                for (int side = 0; side < 2; ++side) {
                    const BoundaryCondition bc = spec.face[axis][side];
                    const std::ptrdiff_t face = side ? hi_face : lo_face;
                    const std::ptrdiff_t dir = side ? 1 : -1;  // outward
                    if (bc == BoundaryCondition::NullDirichlet) line[face * sa] = T(0);
                    for (std::ptrdiff_t k = 1; k <= h; ++k) {
                        T& ghost = line[(face + dir * k) * sa];
                        const T src = line[(face - dir * k) * sa];
                        ghost = bc == BoundaryCondition::NullDirichlet ? -src
                              : bc == BoundaryCondition::NullNeumann   ? src
                                                                       : T(0);
                    }
                }
            }
        }
    }
}

/// grad(rho)/rho per axis with the first-derivative stencil over the extended
/// grid (host; API parity -- Solver<T> forms the same fields on the device).
template <typename T>
std::array<Field<T>, 3> density_log_gradient(const Field<T>& rho, const Grid& grid,
                                             const StencilCoeffs& coeffs) {
    std::array<Field<T>, 3> out;
    const auto pad = grid.padded_shape();
    const std::size_t h = static_cast<std::size_t>(grid.halo);
    std::array<std::size_t, 3> b{0, 0, 0}, e{1, 1, 1};
    for (int a = 0; a < grid.ndim; ++a) {
        b[a] = h;
        e[a] = h + grid.extended_shape[a];
    }
    for (int axis = 0; axis < grid.ndim; ++axis) {
        Field<T> g(grid.ndim, pad);
        const std::ptrdiff_t s = static_cast<std::ptrdiff_t>(rho.strides()[axis]);
        const double scale = 1.0 / (2.0 * grid.spacing[axis]);
        for (std::size_t z = b[0]; z < e[0]; ++z)
            for (std::size_t x = b[1]; x < e[1]; ++x)
                for (std::size_t y = b[2]; y < e[2]; ++y) {
                    const std::size_t i = rho.index(z, x, y);
                    double d = 0.0;
                    for (int j = 1; j <= coeffs.radius; ++j)
                        d += coeffs.first[j - 1] * (static_cast<double>(rho[i + j * s]) -
                                                    static_cast<double>(rho[i - j * s]));
                    g[i] = static_cast<T>(d * scale / static_cast<double>(rho[i]));
                }
        out[axis] = std::move(g);
    }
    return out;
}

template <typename T>
struct ModulatedField {
    Field<T> field;
    std::vector<double> amplitude;
};

template <typename T>
struct Seismogram {
    std::size_t n_receivers = 0;
    std::vector<T> data;  // (n_steps + 1) rows * n_receivers, row-major
    std::vector<std::array<double, 3>> coordinates;

    T at(std::size_t row, std::size_t rec) const { return data[row * n_receivers + rec]; }
};

template <typename T>
struct ForwardResult {
    std::vector<Field<T>> snapshots;
    std::vector<std::size_t> snapshot_steps;
    Seismogram<T> seismogram;
    double kernel_seconds = 0.0;
};

enum class Backend { Serial, Parallel };

/// fdwave::Solver<T> on a B200 through libfdwave_cuda.so.
template <typename T>
class Solver {
    static_assert(std::is_same_v<T, float> || std::is_same_v<T, double>,
                  "Solver<T>: T must be float or double");

public:
    Solver(Grid grid, MaterialModel<T> materials, DampingField<T> damping, BoundarySpec boundary,
           TimeAxis time, StencilCoeffs coeffs)
        : grid_(std::move(grid)), boundary_(boundary), time_(time), coeffs_(std::move(coeffs)) {
        if (coeffs_.order != grid_.space_order)
            throw std::invalid_argument("stencil order does not match grid order");
        fdw_desc d;
        fdw_desc_init(&d);
        d.ndim = grid_.ndim;
        d.space_order = grid_.space_order;
        d.dtype_bytes = static_cast<int32_t>(sizeof(T));
        for (int a = 0; a < 3; ++a) {
            d.extended[a] = a < grid_.ndim ? grid_.extended_shape[a] : 1;
            d.spacing[a] = a < grid_.ndim ? grid_.spacing[a] : 1.0;
            for (int side = 0; side < 2; ++side) d.bc[a][side] = static_cast<int32_t>(boundary_.face[a][side]);
        }
        for (std::size_t j = 0; j < coeffs_.second.size() && j < 11; ++j) d.coeffs[j] = coeffs_.second[j];
        for (std::size_t j = 0; j < coeffs_.first.size() && j < 10; ++j) d.coeffs1[j] = coeffs_.first[j];
        d.dt = time_.dt;
        d.n_steps = time_.n_steps;
        check(fdw_create(&d, &ctx_), "fdw_create", true);
        try {
            check(fdw_set_medium(ctx_, materials.velocity.data(), damping.eta.data(), 0), "fdw_set_medium");
            if (materials.density) {
                if (materials.density->size() != materials.velocity.size())
                    throw std::invalid_argument("material model: density shape mismatch");
                check(fdw_set_density(ctx_, materials.density->data(), 0), "fdw_set_density");
            }
        } catch (...) {
            release();
            throw;
        }
        prev_ = Field<T>(grid_.ndim, grid_.padded_shape());
        curr_ = Field<T>(grid_.ndim, grid_.padded_shape());
    }

    Solver(const Solver&) = delete;
    Solver& operator=(const Solver&) = delete;
    Solver(Solver&& o) noexcept { *this = std::move(o); }
    Solver& operator=(Solver&& o) noexcept {
        if (this != &o) {
            release();
            grid_ = std::move(o.grid_);
            boundary_ = o.boundary_;
            time_ = o.time_;
            coeffs_ = std::move(o.coeffs_);
            prev_ = std::move(o.prev_);
            curr_ = std::move(o.curr_);
            n_receivers_ = o.n_receivers_;
            receiver_coordinates_ = std::move(o.receiver_coordinates_);
            verbose_ = o.verbose_;
            snapshot_cap_bytes_ = o.snapshot_cap_bytes_;
            mirrored_ = o.mirrored_;
            ctx_ = o.ctx_;
            o.ctx_ = nullptr;
        }
        return *this;
    }
    ~Solver() { release(); }

    void set_sources(InterpolationMap sources, std::vector<double> wavelet) {
        if (!sources.points.empty() && wavelet.size() < time_.sample_count())
            throw std::invalid_argument("wavelet shorter than the time axis");
        std::vector<uint64_t> off, idx;
        std::vector<double> w;
        flatten(sources, off, idx, w);
        check(fdw_set_sources(ctx_, sources.points.size(), off.data(), idx.data(), w.data(), wavelet.data(),
                              wavelet.size()),
              "fdw_set_sources");
    }
    void set_receivers(InterpolationMap receivers, std::vector<std::array<double, 3>> coordinates = {}) {
        std::vector<uint64_t> off, idx;
        std::vector<double> w;
        flatten(receivers, off, idx, w);
        check(fdw_set_receivers(ctx_, receivers.points.size(), off.data(), idx.data(), w.data()),
              "fdw_set_receivers");
        n_receivers_ = receivers.points.size();
        receiver_coordinates_ = std::move(coordinates);
    }
    void add_volume_source(ModulatedField<T> source) {
        if (source.amplitude.size() < time_.n_steps)
            throw std::invalid_argument("volume source amplitude shorter than run");
        const auto pad = grid_.padded_shape();
        if (source.field.size() != pad[0] * pad[1] * pad[2])
            throw std::invalid_argument("volume source field shape mismatch");
        check(fdw_add_volume_source(ctx_, source.field.data(), source.amplitude.data(), source.amplitude.size(), 0),
              "fdw_add_volume_source");
    }
    void set_backend(Backend, int) {}
    void set_verbose(bool verbose) { verbose_ = verbose; }
    void set_snapshot_cap(std::size_t bytes) { snapshot_cap_bytes_ = bytes; }

    const Grid& grid() const { return grid_; }
    const TimeAxis& time_axis() const { return time_; }
    Field<T>& current_level() {
        mirror();
        return curr_;
    }
    Field<T>& previous_level() {
        mirror();
        return prev_;
    }
    std::size_t step_index() const {
        uint64_t s = 0;
        fdw_step_index(ctx_, &s);
        return static_cast<std::size_t>(s);
    }

    void refresh_boundary() {
        push();
        check(fdw_refresh_boundary(ctx_), "fdw_refresh_boundary");
        pull();
    }

    void step() {
        push();
        advance(1, 0);
        pull();
    }

    ForwardResult<T> forward() {
        ForwardResult<T> result;
        result.seismogram.n_receivers = n_receivers_;
        result.seismogram.coordinates = receiver_coordinates_;
        const std::size_t snap_bytes = time_.snapshot_count() * grid_.extended_points() * sizeof(T);
        if (snap_bytes > snapshot_cap_bytes_)
            throw std::invalid_argument("snapshot storage (" + std::to_string(snap_bytes) +
                                        " bytes) exceeds the configured cap; raise the cap or the stride");
        // snapshot buffers are written asynchronously: keep them in place
        result.snapshots.reserve(time_.snapshot_count() + 1);
        refresh_boundary();
        check(fdw_record(ctx_), "fdw_record");
        const std::size_t start = step_index(), n = time_.n_steps, stride = time_.saving_stride;
        auto due = [&](std::size_t s) { return stride == 0 ? s == n : s % stride == 0; };
        if (due(start)) snapshot(result, start);
        const auto t0 = std::chrono::steady_clock::now();
        std::size_t cur = start;
        const std::size_t end = start + n;
        // steps and snapshot copies are queued without host syncs; each
        // snapshot streams out on the copy stream while later steps run
        while (cur < end) {
            std::size_t next = end;
            if (stride != 0) next = std::min(end, (cur / stride + 1) * stride);
            else if (cur < n && n < end) next = n;
            advance(next - cur, FDW_ADVANCE_RECORD | FDW_ADVANCE_ASYNC);
            cur = next;
            if (due(cur)) snapshot(result, cur, true);
        }
        wait();
        result.kernel_seconds =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (n_receivers_) {
            result.seismogram.data.resize((n + 1) * n_receivers_);
            check(fdw_download_seismogram(ctx_, result.seismogram.data.data(), n + 1),
                  "fdw_download_seismogram");
        }
        pull();
        return result;
    }

    double max_abs() const {
        const_cast<Solver*>(this)->push();
        double m = 0.0;
        check(fdw_max_abs(ctx_, &m), "fdw_max_abs");
        return m;
    }

private:
    static void flatten(const InterpolationMap& m, std::vector<uint64_t>& off, std::vector<uint64_t>& idx,
                        std::vector<double>& w) {
        off.assign(1, 0);
        for (const auto& entries : m.points) {
            for (const auto& e : entries) {
                idx.push_back(e.index);
                w.push_back(e.weight);
            }
            off.push_back(idx.size());
        }
        if (idx.empty()) {  // keep valid pointers for the ABI
            idx.push_back(0);
            w.push_back(0.0);
        }
    }

    void check(fdw_status s, const char* what, bool creating = false) const {
        if (s == FDW_OK) return;
        const std::string msg = std::string(what) + ": " + fdw_last_error(creating ? nullptr : ctx_);
        if (s == FDW_EINVAL) throw std::invalid_argument(msg);
        throw std::runtime_error(msg);
    }

    void advance(std::size_t n, uint32_t flags) {
        uint64_t bad_step = 0;
        double bad_max = 0.0;
        const fdw_status s = fdw_advance(ctx_, n, flags, &bad_step, &bad_max);
        if (s == FDW_EINSTABLE) {
            pull();
            throw instability_error(bad_step, bad_max);
        }
        check(s, "fdw_advance");
        if (verbose_)
            std::fprintf(stderr, "step %zu/%zu\n", step_index(), static_cast<std::size_t>(time_.n_steps));
    }

    void wait() {
        uint64_t bad_step = 0;
        double bad_max = 0.0;
        const fdw_status st = fdw_wait(ctx_, &bad_step, &bad_max);
        if (st == FDW_EINSTABLE) {
            pull();
            throw instability_error(bad_step, bad_max);
        }
        check(st, "fdw_wait");
    }

    void snapshot(ForwardResult<T>& r, std::size_t s, bool stream = false) {
        Field<T> out(grid_.ndim, grid_.extended_shape);
        if (stream)  // filled by the copy stream; valid after wait()
            check(fdw_snapshot_async(ctx_, out.data()), "fdw_snapshot_async");
        else
            check(fdw_get_extended(ctx_, out.data()), "fdw_get_extended");
        r.snapshots.push_back(std::move(out));
        r.snapshot_steps.push_back(s);
    }

    // host mirrors: downloaded on first access, then kept coherent
    void mirror() {
        if (!mirrored_) {
            check(fdw_get_levels(ctx_, prev_.data(), curr_.data()), "fdw_get_levels");
            mirrored_ = true;
        }
    }
    void push() {
        if (mirrored_) check(fdw_set_levels(ctx_, prev_.data(), curr_.data()), "fdw_set_levels");
    }
    void pull() {
        if (mirrored_) check(fdw_get_levels(ctx_, prev_.data(), curr_.data()), "fdw_get_levels");
    }
    void release() {
        if (ctx_) fdw_destroy(ctx_);
        ctx_ = nullptr;
    }

    Grid grid_;
    BoundarySpec boundary_;
    TimeAxis time_;
    StencilCoeffs coeffs_;
    Field<T> prev_, curr_;
    std::size_t n_receivers_ = 0;
    std::vector<std::array<double, 3>> receiver_coordinates_;
    bool verbose_ = false;
    std::size_t snapshot_cap_bytes_ = std::size_t(4) << 30;
    bool mirrored_ = false;
    fdw_solver* ctx_ = nullptr;
};

}  // namespace fdwave
