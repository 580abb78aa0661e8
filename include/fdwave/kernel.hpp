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

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <optional>
#include <stdexcept>
#include <string>
#include <thread>
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

namespace detail {

/// FDW_DEVICES: the GPUs one Solver spreads a 3D grid over as Z slabs, e.g.
/// "0-7" or "0,1,2,3" (repeated ordinals emulate slabs on one GPU; the
/// library then orders the ranks on the host).  Unset: device 0 only.
inline std::vector<int> devices_from_env() {
    std::vector<int> out;
    const char* env = std::getenv("FDW_DEVICES");
    if (!env || !*env) return out;
    std::string spec(env);
    std::size_t pos = 0;
    while (pos <= spec.size()) {
        const std::size_t comma = spec.find(',', pos);
        const std::string tok = spec.substr(pos, comma == std::string::npos ? std::string::npos : comma - pos);
        const std::size_t dash = tok.find('-');
        if (!tok.empty()) {
            if (dash != std::string::npos) {
                const int lo = std::stoi(tok.substr(0, dash)), hi = std::stoi(tok.substr(dash + 1));
                for (int d = lo; d <= hi; ++d) out.push_back(d);
            } else {
                out.push_back(std::stoi(tok));
            }
        }
        if (comma == std::string::npos) break;
        pos = comma + 1;
    }
    return out;
}

/// Runs f(r) for every rank concurrently (one host thread each: the ranks of
/// a slab decomposition wait on each other inside collective calls) and
/// rethrows the first failure.
template <class F>
void on_ranks(std::size_t n, F&& f) {
    if (n == 1) {
        f(std::size_t(0));
        return;
    }
    std::vector<std::exception_ptr> err(n);
    std::vector<std::thread> th;
    th.reserve(n);
    for (std::size_t r = 0; r < n; ++r)
        th.emplace_back([&, r] {
            try {
                f(r);
            } catch (...) {
                err[r] = std::current_exception();
            }
        });
    for (auto& t : th) t.join();
    for (auto& e : err)
        if (e) std::rethrow_exception(e);
}

}  // namespace detail

/// fdwave::Solver<T> on a B200 through libfdwave_cuda.so.  With FDW_DEVICES
/// naming several GPUs, a 3D Solver is one Z slab per GPU (the reference's
/// OpenMP loop over Z planes, kernel.hpp:392-393, becomes a loop over GPUs):
/// the slabs exchange their halo planes over NVLink peer memory inside each
/// step, and this class scatters / gathers the host-side views.
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
        std::vector<int> devs = detail::devices_from_env();
        if (devs.empty()) devs.push_back(0);
        if (grid_.ndim != 3 || devs.size() > grid_.extended_shape[0] / (2 * std::size_t(grid_.halo)))
            devs.resize(1);  // 2D, or slabs thinner than 2R planes: one GPU
        const std::size_t world = devs.size();
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
        const auto pad = grid_.padded_shape();
        plane_ = pad[1] * pad[2];
        ctxs_.assign(world, nullptr);
        slabs_.assign(world, {0, grid_.extended_shape[0]});
        try {
            for (std::size_t r = 0; r < world; ++r) {
                fdw_desc dr = d;
                dr.device = devs[r];
                if (world > 1) {
                    uint64_t zb = 0, ze = 0;
                    check_ctx(fdw_slab_range(grid_.extended_shape[0], static_cast<int32_t>(world),
                                             static_cast<int32_t>(r), &zb, &ze),
                              nullptr, "fdw_slab_range");
                    dr.rank = static_cast<int32_t>(r);
                    dr.world = static_cast<int32_t>(world);
                    dr.z_begin = zb;
                    dr.z_end = ze;
                    slabs_[r] = {zb, ze};
                }
                check_ctx(fdw_create(&dr, &ctxs_[r]), nullptr, "fdw_create");
                const std::size_t off = slabs_[r].first * plane_;  // local padded slab = contiguous planes
                check_ctx(fdw_set_medium(ctxs_[r], materials.velocity.data() + off, damping.eta.data() + off, 0),
                          ctxs_[r], "fdw_set_medium");
                if (materials.density) {
                    if (materials.density->size() != materials.velocity.size())
                        throw std::invalid_argument("material model: density shape mismatch");
                    check_ctx(fdw_set_density(ctxs_[r], materials.density->data() + off, 0), ctxs_[r],
                              "fdw_set_density");
                }
            }
            if (world > 1)
                for (std::size_t r = 0; r < world; ++r)
                    check_ctx(fdw_peer_link(ctxs_[r], ctxs_.data(), static_cast<int32_t>(world)), ctxs_[r],
                              "fdw_peer_link");
        } catch (...) {
            release();
            throw;
        }
        ctx_ = ctxs_[0];
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
            loop_start_ = o.loop_start_;
            plane_ = o.plane_;
            ctxs_ = std::move(o.ctxs_);
            slabs_ = std::move(o.slabs_);
            ctx_ = o.ctx_;
            o.ctx_ = nullptr;
            o.ctxs_.clear();
        }
        return *this;
    }
    ~Solver() { release(); }

    /// Number of GPUs (Z slabs) this Solver runs on.
    std::size_t devices() const { return ctxs_.size(); }

    void set_sources(InterpolationMap sources, std::vector<double> wavelet) {
        if (!sources.points.empty() && wavelet.size() < time_.sample_count())
            throw std::invalid_argument("wavelet shorter than the time axis");
        std::vector<uint64_t> off, idx;
        std::vector<double> w;
        flatten(sources, off, idx, w);
        for (auto* c : ctxs_)  // each slab keeps the taps it owns
            check_ctx(fdw_set_sources(c, sources.points.size(), off.data(), idx.data(), w.data(), wavelet.data(),
                                      wavelet.size()),
                      c, "fdw_set_sources");
    }
    void set_receivers(InterpolationMap receivers, std::vector<std::array<double, 3>> coordinates = {}) {
        std::vector<uint64_t> off, idx;
        std::vector<double> w;
        flatten(receivers, off, idx, w);
        for (auto* c : ctxs_)
            check_ctx(fdw_set_receivers(c, receivers.points.size(), off.data(), idx.data(), w.data()), c,
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
        for (std::size_t r = 0; r < ctxs_.size(); ++r)
            check_ctx(fdw_add_volume_source(ctxs_[r], source.field.data() + slabs_[r].first * plane_,
                                            source.amplitude.data(), source.amplitude.size(), 0),
                      ctxs_[r], "fdw_add_volume_source");
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
        detail::on_ranks(ctxs_.size(),
                         [&](std::size_t r) { check_ctx(fdw_refresh_boundary(ctxs_[r]), ctxs_[r], "fdw_refresh_boundary"); });
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
        for (auto* c : ctxs_) check_ctx(fdw_record(c), c, "fdw_record");
        const std::size_t start = step_index(), n = time_.n_steps, stride = time_.saving_stride;
        auto due = [&](std::size_t s) { return stride == 0 ? s == n : s % stride == 0; };
        if (due(start)) snapshot(result, start);
        const auto t0 = std::chrono::steady_clock::now();
        loop_start_ = t0;
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
            if (ctxs_.size() == 1) {
                check(fdw_download_seismogram(ctx_, result.seismogram.data.data(), n + 1),
                      "fdw_download_seismogram");
            } else {
                const std::vector<double> acc = merged_seismogram(n + 1);
                for (std::size_t i = 0; i < acc.size(); ++i) result.seismogram.data[i] = static_cast<T>(acc[i]);
            }
        }
        pull();
        return result;
    }

    double max_abs() const {
        const_cast<Solver*>(this)->push();
        std::vector<double> m(ctxs_.size(), 0.0);
        detail::on_ranks(ctxs_.size(),
                         [&](std::size_t r) { check_ctx(fdw_max_abs(ctxs_[r], &m[r]), ctxs_[r], "fdw_max_abs"); });
        return m[0];  // reduced over every slab
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

    // The seismogram of a slab decomposition, bit-identical to the
    // reference's accumulation (acquisition.hpp:155-158): receivers inside
    // one slab come from that rank's partial sum (the others hold 0); a
    // receiver whose taps straddle a face is re-summed from every rank's
    // per-tap products in entry order, sequentially from +0.0.
    std::vector<double> merged_seismogram(std::size_t rows) {
        std::vector<double> acc(rows * n_receivers_, 0.0), part(acc.size());
        struct Tap {
            uint64_t entry;
            std::size_t rank, slot;
        };
        std::vector<std::vector<Tap>> split(n_receivers_);
        std::vector<std::vector<double>> prod(ctxs_.size());
        std::vector<uint64_t> nslot(ctxs_.size(), 0);
        for (std::size_t r = 0; r < ctxs_.size(); ++r) {
            check_ctx(fdw_download_seismogram_f64(ctxs_[r], part.data(), rows), ctxs_[r], "fdw_download_seismogram");
            for (std::size_t i = 0; i < acc.size(); ++i) acc[i] += part[i];
            check_ctx(fdw_receiver_split_info(ctxs_[r], &nslot[r], nullptr, nullptr), ctxs_[r], "fdw_receiver_split_info");
            if (!nslot[r]) continue;
            std::vector<uint64_t> rec(nslot[r]), ent(nslot[r]);
            check_ctx(fdw_receiver_split_info(ctxs_[r], &nslot[r], rec.data(), ent.data()), ctxs_[r],
                      "fdw_receiver_split_info");
            prod[r].resize(rows * nslot[r]);
            check_ctx(fdw_download_receiver_products(ctxs_[r], prod[r].data(), rows), ctxs_[r],
                      "fdw_download_receiver_products");
            for (std::size_t j = 0; j < nslot[r]; ++j) split[rec[j]].push_back({ent[j], r, j});
        }
        for (std::size_t p = 0; p < n_receivers_; ++p) {
            auto& taps = split[p];
            if (taps.empty()) continue;
            std::sort(taps.begin(), taps.end(), [](const Tap& a, const Tap& b) { return a.entry < b.entry; });
            for (std::size_t row = 0; row < rows; ++row) {
                double s = 0.0;
                for (const Tap& t : taps) s += prod[t.rank][row * nslot[t.rank] + t.slot];
                acc[row * n_receivers_ + p] = s;
            }
        }
        return acc;
    }

    static void check_ctx(fdw_status s, const fdw_solver* c, const char* what) {
        if (s == FDW_OK) return;
        const std::string msg = std::string(what) + ": " + fdw_last_error(c);
        if (s == FDW_EINVAL) throw std::invalid_argument(msg);
        throw std::runtime_error(msg);
    }
    void check(fdw_status s, const char* what) const { check_ctx(s, ctx_, what); }

    // fdw_advance on every slab; an instability (the same step on every rank:
    // the health check is reduced across slabs) becomes instability_error
    void advance_ranks(std::size_t n, uint32_t flags) {
        std::vector<uint64_t> bad_step(ctxs_.size(), 0);
        std::vector<double> bad_max(ctxs_.size(), 0.0);
        std::vector<fdw_status> st(ctxs_.size(), FDW_OK);
        detail::on_ranks(ctxs_.size(), [&](std::size_t r) {
            st[r] = fdw_advance(ctxs_[r], n, flags, &bad_step[r], &bad_max[r]);
        });
        for (std::size_t r = 0; r < ctxs_.size(); ++r)
            if (st[r] == FDW_EINSTABLE) {
                pull();
                throw instability_error(bad_step[r], bad_max[r]);
            }
        for (std::size_t r = 0; r < ctxs_.size(); ++r) check_ctx(st[r], ctxs_[r], "fdw_advance");
    }

    void advance(std::size_t n, uint32_t flags) {
        if (verbose_) {  // the reference's progress line at every health check
            verbose_advance(n, flags & ~uint32_t(FDW_ADVANCE_ASYNC));
            return;
        }
        advance_ranks(n, flags);
    }

    // check_health's verbose branch (kernel.hpp:456-466): the steps run in
    // pieces that end at the health checks (step % 100 == 0 or the last
    // step); after each, the line "step s/N  t s  max|p| = m" with the time
    // since forward() started its loop (or since construction, as there).
    void verbose_advance(std::size_t n, uint32_t flags) {
        const std::size_t ci = 100, total = time_.n_steps;
        std::size_t s = step_index();
        const std::size_t end = s + n;
        while (s < end) {
            std::size_t next = (s / ci + 1) * ci;
            if (total > s) next = std::min(next, total);
            next = std::min(next, end);
            advance_ranks(next - s, flags);
            s = next;
            if (s % ci == 0 || s == total) {
                std::vector<double> m(ctxs_.size(), 0.0);
                detail::on_ranks(ctxs_.size(), [&](std::size_t r) {
                    check_ctx(fdw_max_abs(ctxs_[r], &m[r]), ctxs_[r], "fdw_max_abs");
                });
                const double el =
                    std::chrono::duration<double>(std::chrono::steady_clock::now() - loop_start_).count();
                std::fprintf(stderr, "step %zu/%zu  %.3fs  max|p| = %.6e\n", s, total, el, m[0]);
            }
        }
    }

    void wait() {
        std::vector<uint64_t> bad_step(ctxs_.size(), 0);
        std::vector<double> bad_max(ctxs_.size(), 0.0);
        std::vector<fdw_status> st(ctxs_.size(), FDW_OK);
        for (std::size_t r = 0; r < ctxs_.size(); ++r) st[r] = fdw_wait(ctxs_[r], &bad_step[r], &bad_max[r]);
        for (std::size_t r = 0; r < ctxs_.size(); ++r)
            if (st[r] == FDW_EINSTABLE) {
                pull();
                throw instability_error(bad_step[r], bad_max[r]);
            }
        for (std::size_t r = 0; r < ctxs_.size(); ++r) check_ctx(st[r], ctxs_[r], "fdw_wait");
    }

    void snapshot(ForwardResult<T>& res, std::size_t s, bool stream = false) {
        Field<T> out(grid_.ndim, grid_.extended_shape);
        const std::size_t eplane = grid_.ndim == 3 ? grid_.extended_shape[1] * grid_.extended_shape[2] : 0;
        for (std::size_t r = 0; r < ctxs_.size(); ++r) {  // each slab fills its own planes
            T* dst = out.data() + slabs_[r].first * eplane;
            if (stream)  // filled by the copy stream; valid after wait()
                check_ctx(fdw_snapshot_async(ctxs_[r], dst), ctxs_[r], "fdw_snapshot_async");
            else
                check_ctx(fdw_get_extended(ctxs_[r], dst), ctxs_[r], "fdw_get_extended");
        }
        res.snapshots.push_back(std::move(out));
        res.snapshot_steps.push_back(s);
    }

    // host mirrors: downloaded on first access, then kept coherent.  Slabs:
    // each rank's owned planes (plus the global Z ghost planes on the first
    // and last rank) are gathered; uploads hand every rank its padded slab.
    void gather_levels() {
        if (ctxs_.size() == 1) {
            check(fdw_get_levels(ctx_, prev_.data(), curr_.data()), "fdw_get_levels");
            return;
        }
        const std::size_t h = static_cast<std::size_t>(grid_.halo), world = ctxs_.size();
        detail::on_ranks(world, [&](std::size_t r) {
            const std::size_t zb = slabs_[r].first, ze = slabs_[r].second, nl = ze - zb + 2 * h;
            std::vector<T> p(nl * plane_), c(nl * plane_);
            check_ctx(fdw_get_levels(ctxs_[r], p.data(), c.data()), ctxs_[r], "fdw_get_levels");
            const std::size_t lo = r == 0 ? 0 : h, hi = r + 1 == world ? nl : nl - h;
            std::copy(p.begin() + lo * plane_, p.begin() + hi * plane_, prev_.data() + (zb + lo) * plane_);
            std::copy(c.begin() + lo * plane_, c.begin() + hi * plane_, curr_.data() + (zb + lo) * plane_);
        });
    }
    void mirror() {
        if (!mirrored_) {
            gather_levels();
            mirrored_ = true;
        }
    }
    void push() {
        if (!mirrored_) return;
        for (std::size_t r = 0; r < ctxs_.size(); ++r) {
            const std::size_t off = slabs_[r].first * plane_;
            check_ctx(fdw_set_levels(ctxs_[r], prev_.data() + off, curr_.data() + off), ctxs_[r], "fdw_set_levels");
        }
    }
    void pull() {
        if (mirrored_) gather_levels();
    }
    void release() {
        for (auto*& c : ctxs_) {
            if (c) fdw_destroy(c);
            c = nullptr;
        }
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
    std::size_t plane_ = 0;                                    // padded elements per Z plane
    std::vector<fdw_solver*> ctxs_;                            // one context per GPU (Z slab)
    std::vector<std::pair<std::size_t, std::size_t>> slabs_;   // owned extended Z planes per rank
    fdw_solver* ctx_ = nullptr;                                // rank 0
    std::chrono::steady_clock::time_point loop_start_ = std::chrono::steady_clock::now();
};

}  // namespace fdwave
