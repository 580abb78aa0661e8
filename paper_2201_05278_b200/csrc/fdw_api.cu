// fdw_api.cu -- C-ABI (include/fdwave_cuda.h) over the sm_100a kernels.
//
// Host-side restatement of fdwave::Solver<T> (kernel.hpp:170-495) for the
// device: layout and upload/download of the padded fields, source/receiver
// index remapping, the step sequence (sweep -> inject -> swap -> boundary ->
// health) captured as CUDA-graph chunks, and the Z-slab halo exchange over
// NVLink peer memory for multi-GPU runs (no NCCL on the data path).  No CPU
// fallback: every compute path is a kernel.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <unordered_map>
#include <vector>

#include <nvtx3/nvToolsExt.h>
#include <unistd.h>

#include "../../include/fdwave_cuda.h"
#include "fdw_inst.h"
#include "fdw_kernels.cuh"

using fdw::Ctrl;
using fdw::SweepArgs;
using fdwi::TMA_BX;
using fdwi::TMA_PD;
using fdwi::tma_kernel;
using fdwi::tma_vd_kernel;
using fdwi::fused2d_kernel;
using fdwi::res2d_kernel;
using fdwi::res2d2_kernel;

namespace {

thread_local std::string g_create_error;

struct ProfileSink {
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> marks;
};

}  // namespace

// NVTX ranges (header-only NVTX3, no link dependency) around the host calls
// that enqueue device work, so an nsys / ncu timeline groups the kernels by
// chunk, health check, upload and snapshot.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

// FDW_DEBUG_TIMING=1: host-side phase timings of the setup/teardown calls
struct PhaseTimer {
    const char* fn;
    bool on;
    std::chrono::steady_clock::time_point t;
    explicit PhaseTimer(const char* f) : fn(f), on(getenv("FDW_DEBUG_TIMING") != nullptr), t(std::chrono::steady_clock::now()) {}
    void lap(const char* what) {
        if (!on) return;
        const auto n = std::chrono::steady_clock::now();
        fprintf(stderr, "%s %-14s %8.3f ms\n", fn, what, std::chrono::duration<double, std::milli>(n - t).count());
        t = n;
    }
};

// Pinned host mirrors of Ctrl, recycled across solvers (cudaMallocHost /
// cudaFreeHost are device-synchronising and slow under memory pressure).
static std::mutex g_ctrl_mu;
static std::vector<Ctrl*> g_ctrl_free;

static Ctrl* pinned_ctrl_get() {
    {
        std::lock_guard<std::mutex> lk(g_ctrl_mu);
        if (!g_ctrl_free.empty()) {
            Ctrl* p = g_ctrl_free.back();
            g_ctrl_free.pop_back();
            return p;
        }
    }
    void* p = nullptr;
    if (cudaMallocHost(&p, sizeof(Ctrl)) != cudaSuccess) return nullptr;
    return static_cast<Ctrl*>(p);
}

static void pinned_ctrl_put(Ctrl* p) {
    std::lock_guard<std::mutex> lk(g_ctrl_mu);
    g_ctrl_free.push_back(p);
}

struct fdw_solver {
    fdw_desc d{};
    std::string err;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int sm_count = 148;

    int ndim = 3, R = 1, tsize = 4;
    long long P[3] = {1, 1, 1};  // global padded shape
    long long nzl = 0;           // 3D: owned extended planes; 2D: extended rows (Z)
    long long nxl = 0, nyl = 0;  // 3D: ext X, ext Y; 2D: ext X (fast), unused
    long long Lz = 0;            // 3D: stored planes = nzl + 2R; 2D: 1
    long long rows_alloc = 0;    // rows per stored plane (3D) / total rows (2D)
    long long ld = 0, plane = 0, base = 0, origin = 0, origin_pad = 0;
    size_t level_elems = 0;

    void* lvl[2] = {nullptr, nullptr};
    int cur = 1;  // lvl[cur] is the current level (Solver::curr_)
    // ghost-cell state per level: 0 stored & consistent with the boundary
    // conditions, 1 virtual (stored ghosts stale; the TMA kernel mirrors on
    // the fly), 2 raw (uploaded by the caller; stored ghosts authoritative)
    int gstate[2] = {0, 0};
    void* c2dt2 = nullptr;
    void* eta = nullptr;
    void* grad[3] = {nullptr, nullptr, nullptr};  // variable density: grad(rho)/rho per axis
    bool vd = false;
    int2* d_ezr = nullptr;  // TMA: eta-zero Z range per tile column
    // volume sources (ModulatedField): device fields, pointer table, amplitudes
    std::vector<void*> vs_fields;
    void* d_vs_ptrs = nullptr;
    void* d_vs_amp = nullptr;
    unsigned long long* d_vs_len = nullptr;
    unsigned long long vs_namp = 0;
    std::vector<std::vector<double>> vs_amps;  // host copy of the amplitudes
    Ctrl* ctrl = nullptr;
    Ctrl* h_ctrl = nullptr;  // pinned mirror
    bool medium_set = false;

    int n_tgt = 0;
    long long* d_tgt = nullptr;
    unsigned int* d_ent_off = nullptr;
    double* d_ent_w = nullptr;
    double* d_wavelet = nullptr;
    unsigned long long n_wavelet = 0;

    int n_rec = 0;
    long long* d_rec_idx = nullptr;
    unsigned int* d_rec_off = nullptr;
    double* d_rec_w = nullptr;
    double* d_seis = nullptr;
    // slabs: taps of receivers that straddle a slab face -> per-tap products
    int n_split = 0;                       // product slots on this rank
    long long* d_sp_idx = nullptr;
    double* d_sp_w = nullptr;
    double* d_sp_prod = nullptr;           // [seis_rows][n_split]
    std::vector<uint64_t> sp_rec, sp_entry; // per slot: receiver, entry position within it
    unsigned long long seis_rows = 0;

    unsigned long long host_step = 0;
    int variant = FDW_KERNEL_SIMPLE;
    int zseg = 1;
    int bx = 16;
    int occupancy = 0;
    int tma_minb = 3;
    int tma_pd = 0;  // > 0: split-ring TMA sweep with that many planes in flight
    // damping table (split-ring fp32 sweep): 1-byte eta index per point, (om, iop) per index
    unsigned char* d_eidx = nullptr;
    void* d_etab = nullptr;  // float2 / double2 pairs
    int n_etab = 0;          // entries incl. index 0; 0: no table (the sweep streams fp32 eta)
    CUtensorMap tm_eb{};     // TMA map over d_eidx

    std::map<std::tuple<unsigned long long, int, int, int>, cudaGraphExec_t> graphs;
    std::map<std::tuple<unsigned long long, int, int, int>, unsigned long long> graph_kernels;
    bool capturing = false;
    bool pdl_sweep = false;  // next TMA sweep launch: programmatic dependent launch (enqueue_step)
    unsigned long long capture_kernels = 0;
    unsigned long long launches = 0;  // kernels launched (graph nodes included)
    ProfileSink* prof = nullptr;
    // TMA descriptors (variant FDW_KERNEL_TMA): u-tile box for each level, and
    // the prev/c2dt2/eta tile box for each level, c2dt2 and eta
    CUtensorMap tm_u[2], tm_p[2], tm_c, tm_e;
    CUtensorMap tm_g[3] = {};    // variable density: grad(rho)/rho tiles
    int* d_tmap = nullptr;       // FUSED2D: dense injection-target map over the extended grid
    // asynchronous advances (FDW_ADVANCE_ASYNC) not yet checked for an abort
    // receivers of step k run on a side stream beside the sweep of step k+1
    // (they only read level k, which step k+2's sweep overwrites)
    cudaStream_t side = nullptr;
    cudaEvent_t fork_ev[2] = {nullptr, nullptr};
    cudaEvent_t rec_ev[2] = {nullptr, nullptr};
    std::vector<long long> h_tgt;             // host copy of the merged targets
    std::vector<std::vector<double>> h_tw;    // and their entry weights
    bool mirror_tgt = false;                  // a point-source target lies in a neighbour's ghost planes
    bool pending = false;
    unsigned long long pend_start = 0;
    int pend_cur = 0;
    // snapshot streaming (fdw_snapshot_async): device pack slots, pinned
    // bounce slots, a copy stream and per-slot events
    struct SnapJob {
        void* dst = nullptr;
        const void* src = nullptr;
        size_t bytes = 0;
    };
    static constexpr int SNAP_SLOTS = 2;
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t snap_packed[SNAP_SLOTS] = {nullptr, nullptr};
    cudaEvent_t snap_free[SNAP_SLOTS] = {nullptr, nullptr};
    void* snap_dev[SNAP_SLOTS] = {nullptr, nullptr};
    void* snap_host[SNAP_SLOTS] = {nullptr, nullptr};
    size_t snap_bytes = 0;
    int snap_next = 0;
    int fused_grid = 0;          // FUSED2D: co-resident blocks of the cooperative kernel
    // FUSED2D, shared-memory resident kernel (constant density): block rows,
    // blocks per grid row, blocks, dynamic smem; per-block source / tap lists
    bool res2d = false;
    bool res_pair = false;  // two steps per grid barrier (step2d_resident2)
    size_t res_smem2 = 0, res_smem2_base = 0;
    int res_BZ = 0, res_xb = 0, res_nb = 0;
    size_t res_smem = 0;
    int* d_blk_toff = nullptr;
    int* d_blk_tgt = nullptr;
    int* d_blk_tpos = nullptr;
    int* d_blk_roff = nullptr;
    int* d_blk_rpack = nullptr;
    int* d_tap_ix = nullptr;
    int res_tapcap = 0;
    size_t res_smem_base = 0;
    void* d_tapbuf = nullptr;
    int n_ent = 0;
    void* d_res_hbuf = nullptr;  // two-step resident 2D kernel: strip buffers (2 levels)
    // peer transport (Z slabs, world > 1): halo planes stored straight into
    // the neighbours' levels over NVLink, halo epochs and the health reduction
    // through per-rank sync blocks
    bool peer_mode = false;
    bool peers_ready = false;
    bool ipc_same_device = false;  // an IPC-imported neighbour shares this GPU (cannot step)
    struct HostGroup* group = nullptr;  // host-ordered ranks (fdw_peer_link with a shared GPU)
    bool no_pdl = false;           // FDW_NO_PDL at create time
    int prio_hi = 0, prio_lo = 0;  // launch priorities: step chain / side-stream receivers (FDW_NO_PRIO: equal)
    bool tail_pdl_aware = false;   // last kernel of the previous step on `stream` is PDL-aware
    fdw::PeerSync* psync = nullptr;                        // own sync block (cudaMalloc, IPC-exportable)
    fdw::PeerSync* peer_sync[fdw::PEER_MAX_WORLD] = {};    // every rank's block, mapped
    void* peer_lvl[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};  // [lower, upper][level], mapped
    long long peer_delta[2] = {0, 0};                      // neighbour element = local element + delta
    std::vector<void*> ipc_mapped;                         // cudaIpcCloseMemHandle on destroy
    // FDW_GUARD_CHECK=1: a patterned zone after each field allocation
    static constexpr size_t GUARD = 1 << 16;
    size_t guard_bytes = 0;
    // fdw_peer_loopback (profiling): emulated neighbours on this GPU
    bool loopback = false;
    // timing experiments (tools/peer_overhead.py), read at create: FDW_DBG_NO_SEGROT,
    // FDW_DBG_NO_HALO_STORE (loopback only), FDW_DBG_FENCE_ALL
    bool dbg_no_rot = false, dbg_no_store = false, dbg_fence_all = false, dbg_fence_sc = false;
    void* loop_lvl[2] = {nullptr, nullptr};
    fdw::PeerSync* loop_sync = nullptr;
};

namespace {

fdw_status fail(fdw_solver* c, fdw_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    if (c)
        c->err = buf;
    else
        g_create_error = buf;
    return s;
}

#define CU(call)                                                                        \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess)                                                          \
            return fail(c, FDW_ECUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                        __FILE__, __LINE__);                                            \
    } while (0)

#define CHECK_LAUNCH()                      \
    do {                                    \
        CU(cudaGetLastError());             \
        if (c->capturing)                   \
            ++c->capture_kernels;           \
        else                                \
            ++c->launches;                  \
    } while (0)

unsigned long long align_up(unsigned long long v, unsigned long long a) { return (v + a - 1) / a * a; }

// cudaFuncAttributeMaxDynamicSharedMemorySize is per function and shared by
// every context of the process on a device: contexts on different host
// threads share it.  It is only ever raised (a larger limit does not change
// occupancy), under one lock, so no thread can lower it between another
// thread's set and launch.  Tracked per (device, function): the attribute is
// applied to the function as loaded on the current device, and one process
// may drive several GPUs (fdw_peer_link, FDW_DEVICES).
cudaError_t raise_smem_limit(const void* f, size_t bytes) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, size_t> cur;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> lk(mu);
    size_t& have = cur[{dev, f}];
    if (bytes <= have) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) have = bytes;
    return e;
}

}  // namespace

// Ranks linked in one process whose GPUs are shared (one GPU emulating a
// slab decomposition, e.g. the test suite) must never have a kernel spin on a
// flag another launch on the same GPU sets: nothing guarantees the two run
// concurrently.  Such a group is HOST-ORDERED: at every cross-rank point each
// rank records an event, the rank threads meet at a host barrier, and each
// stream waits on its peers' events before the kernel that checks the flags,
// which then finds them already set.  Steps run as direct launches (no graph:
// a captured graph cannot wait on another stream's per-step event).
struct HostGroup {
    int world = 0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    unsigned long long gen = 0;
    bool broken = false;
    fdw_solver* member[fdw::PEER_MAX_WORLD] = {};
    cudaEvent_t ev[fdw::PEER_MAX_WORLD][2] = {};
    unsigned long long round[fdw::PEER_MAX_WORLD] = {};
    int alive = 0;
    // false after 60 s without every rank arriving (a rank thread died or a
    // caller skipped a collective call): the group is then broken for good
    bool barrier() {
        std::unique_lock<std::mutex> lk(mu);
        if (broken) return false;
        const unsigned long long g = gen;
        if (++arrived == world) {
            arrived = 0;
            ++gen;
            cv.notify_all();
            return true;
        }
        if (!cv.wait_for(lk, std::chrono::seconds(60), [&] { return gen != g || broken; })) broken = true;
        if (broken) cv.notify_all();
        return !broken;
    }
};

namespace {
std::mutex g_group_mu;
std::map<const fdw_solver*, HostGroup*> g_groups;  // keyed by the rank-0 context
}  // namespace

namespace {

// ---------------------------------------------------------------------------
// kernel dispatch

// Region table for fdw::boundary_kernel: ghost shells (global Z faces only
// for slabs) and the nodes of active null-Dirichlet faces.
fdw::BoundaryArgs boundary_args(const fdw_solver* c) {
    fdw::BoundaryArgs b{};
    const int h = c->R;
    b.nd = c->ndim;
    b.h = h;
    b.origin_pad = c->origin_pad;
    const bool lo_z = c->d.rank == 0, hi_z = c->d.rank == c->d.world - 1;
    int ext[3], P[3];
    if (c->ndim == 3) {
        ext[0] = (int)c->nzl; ext[1] = (int)c->nxl; ext[2] = (int)c->nyl;
        P[0] = (int)c->Lz; P[1] = (int)c->P[1]; P[2] = (int)c->P[2];
        b.s[0] = c->plane; b.s[1] = c->ld; b.s[2] = 1;
    } else {
        ext[0] = (int)c->nzl; ext[1] = (int)c->nxl; ext[2] = 1;
        P[0] = (int)c->P[0]; P[1] = (int)c->P[1]; P[2] = 1;
        b.s[0] = c->ld; b.s[1] = 1; b.s[2] = 0;
    }
    for (int a = 0; a < 3; ++a) {
        b.ext[a] = ext[a];
        for (int sd = 0; sd < 2; ++sd) {
            const int bc = c->d.bc[a][sd];
            b.f[a][sd] = bc == FDW_BC_NULL_DIRICHLET ? -1 : bc == FDW_BC_NULL_NEUMANN ? 1 : 0;
            b.act[a][sd] = a < c->ndim ? 1 : 0;
        }
    }
    if (c->ndim == 3) {
        b.act[0][0] = lo_z;
        b.act[0][1] = hi_z;
    }
    int n = 0;
    auto add = [&](int z0, int x0, int y0, int nz, int nx, int ny, int zero) {
        if (nz <= 0 || nx <= 0 || ny <= 0) return;
        b.reg[n] = {{z0, x0, y0}, {nz, nx, ny}, zero};
        ++n;
    };
    const int yP = c->ndim == 3 ? P[2] : 1;
    const int yh = c->ndim == 3 ? h : 0;
    const int ny = c->ndim == 3 ? ext[2] : 1;
    // ghost cells
    if (b.act[0][0]) add(0, 0, 0, h, P[1], yP, 0);
    if (b.act[0][1]) add(P[0] - h, 0, 0, h, P[1], yP, 0);
    add(h, 0, 0, ext[0], h, yP, 0);
    add(h, P[1] - h, 0, ext[0], h, yP, 0);
    if (c->ndim == 3) {
        add(h, h, 0, ext[0], ext[1], h, 0);
        add(h, h, P[2] - h, ext[0], ext[1], h, 0);
    }
    // Dirichlet face nodes
    if (b.act[0][0] && b.f[0][0] < 0) add(h, h, yh, 1, ext[1], ny, 1);
    if (b.act[0][1] && b.f[0][1] < 0) add(h + ext[0] - 1, h, yh, 1, ext[1], ny, 1);
    if (b.f[1][0] < 0) add(h, h, yh, ext[0], 1, ny, 1);
    if (b.f[1][1] < 0) add(h, h + ext[1] - 1, yh, ext[0], 1, ny, 1);
    if (c->ndim == 3) {
        if (b.f[2][0] < 0) add(h, h, h, ext[0], ext[1], 1, 1);
        if (b.f[2][1] < 0) add(h, h, h + ext[2] - 1, ext[0], ext[1], 1, 1);
    }
    b.n_regions = n;
    b.start[0] = 0;
    for (int r = 0; r < n; ++r)
        b.start[r + 1] = b.start[r] + (long long)b.reg[r].n[0] * b.reg[r].n[1] * b.reg[r].n[2];
    return b;
}

template <typename T>
fdw_status launch_faces_t(fdw_solver* c, int lv) {
    const fdw::BoundaryArgs b = boundary_args(c);
    if (b.n_regions == 0) return FDW_OK;
    long long mx = 0;
    for (int r = 0; r < b.n_regions; ++r) mx = std::max(mx, b.start[r + 1] - b.start[r]);
    dim3 grid((unsigned)((mx + 255) / 256), (unsigned)b.n_regions);
    fdw::boundary_kernel<T><<<grid, 256, 0, c->stream>>>(static_cast<T*>(c->lvl[lv]), b, c->ctrl);
    CHECK_LAUNCH();
    return FDW_OK;
}

fdw_status launch_faces(fdw_solver* c, int lv) {
    return c->tsize == 4 ? launch_faces_t<float>(c, lv) : launch_faces_t<double>(c, lv);
}

template <typename T>
SweepArgs<T> sweep_args(fdw_solver* c, int src, int dst) {
    SweepArgs<T> a{};
    a.u = static_cast<const T*>(c->lvl[src]);
    a.out = static_cast<T*>(c->lvl[dst]);
    a.c2dt2 = static_cast<const T*>(c->c2dt2);
    a.eta = static_cast<const T*>(c->eta);
    for (int j = 0; j <= c->R; ++j) a.v[j] = static_cast<T>(c->d.coeffs[j]);
    for (int k = 0; k < 3; ++k) a.ih[k] = T(1);
    for (int k = 0; k < c->ndim; ++k)
        a.ih[k] = static_cast<T>(1.0 / (c->d.spacing[k] * c->d.spacing[k]));
    a.dt = c->d.dt;
    a.ld = c->ld;
    a.plane = c->plane;
    a.origin = c->origin;
    a.nz = (int)c->nzl;
    a.nx = (int)c->nxl;
    a.ny = (int)c->nyl;
    for (int ax = 0; ax < 3; ++ax)
        for (int sd = 0; sd < 2; ++sd) {
            const int bc = c->d.bc[ax][sd];
            a.gf[ax][sd] = bc == FDW_BC_NULL_DIRICHLET ? -1 : bc == FDW_BC_NULL_NEUMANN ? 1 : 0;
            a.gact[ax][sd] = ax < c->ndim ? 1 : 0;
        }
    if (c->ndim == 3) {
        a.gact[0][0] = c->d.rank == 0;
        a.gact[0][1] = c->d.rank == c->d.world - 1;
    }
    a.ctrl = c->ctrl;
    a.ezr = c->d_ezr;
    a.seg_rot = 0;
    a.etab = static_cast<const typename fdw::EtabPair<T>::type*>(c->d_etab);
    a.n_etab = c->n_etab;
    a.negz = static_cast<T>(-0.0);
    if (c->vd) {
        a.vd = 1;
        for (int k = 0; k < 3; ++k) {
            a.grad[k] = static_cast<const T*>(c->grad[k < c->ndim ? k : 0]);
            a.i2h[k] = k < c->ndim ? static_cast<T>(1.0 / (2.0 * c->d.spacing[k])) : T(0);
        }
        for (int j = 0; j < c->R; ++j) a.w1[j] = static_cast<T>(c->d.coeffs1[j]);
    }
    return a;
}

#define R_SWITCH(R, MACRO) \
    switch (R) {           \
        MACRO(1)           \
        MACRO(2)           \
        MACRO(3)           \
        MACRO(4)           \
        MACRO(5)           \
        MACRO(6)           \
        MACRO(7)           \
        MACRO(8)           \
        MACRO(9)           \
        MACRO(10)          \
        default: break;    \
    }

template <typename T, bool EX>
void launch_simple(fdw_solver* c, const SweepArgs<T>& a) {
    if (c->ndim == 3) {
        dim3 block(32, 8), grid((unsigned)((a.ny + 31) / 32), (unsigned)((a.nx + 7) / 8), (unsigned)a.nz);
#define L3(RR) \
    case RR: fdw::sweep3d_simple<T, RR, EX><<<grid, block, 0, c->stream>>>(a); break;
        R_SWITCH(c->R, L3)
#undef L3
    } else {
        dim3 block(128, 2), grid((unsigned)((a.nx + 127) / 128), (unsigned)((a.nz + 1) / 2));
#define L2(RR) \
    case RR: fdw::sweep2d_simple<T, RR, EX><<<grid, block, 0, c->stream>>>(a); break;
        R_SWITCH(c->R, L2)
#undef L2
    }
}

template <typename T, int BX>
dim3 zmarch_grid(const fdw_solver* c) {
    using S = fdw::ZMarchShape<T, BX>;
    return dim3((unsigned)((c->nyl + S::TYW - 1) / S::TYW), (unsigned)((c->nxl + BX - 1) / BX),
                (unsigned)c->zseg);
}

template <typename T, bool EX>
bool launch_zmarch(fdw_solver* c, const SweepArgs<T>& a) {
    constexpr int BX = 16;
    using S = fdw::ZMarchShape<T, BX>;
    dim3 block(S::NTY, BX), grid = zmarch_grid<T, BX>(c);
    switch (c->R) {
        case 1: fdw::sweep3d_zmarch<T, 1, BX, EX><<<grid, block, 0, c->stream>>>(a); return true;
        case 2: fdw::sweep3d_zmarch<T, 2, BX, EX><<<grid, block, 0, c->stream>>>(a); return true;
        case 4: fdw::sweep3d_zmarch<T, 4, BX, EX><<<grid, block, 0, c->stream>>>(a); return true;
        default: return false;
    }
}

bool zmarch_supported(int R) { return R == 1 || R == 2 || R == 4; }


template <typename T>
int tma_smem(int R, bool vd = false, int pd = 0) {
    if (pd > 0 && vd) {
        switch (R) {
            case 1: return fdw::TmaShape<T, 1, TMA_BX, 6, TMA_PD>::SMEM;
            case 2: return fdw::TmaShape<T, 2, TMA_BX, 6, TMA_PD>::SMEM;
            default: return fdw::TmaShape<T, 4, TMA_BX, 6, TMA_PD>::SMEM;
        }
    }
    if (pd > 0 && !vd) {
        switch (R) {
            case 1: return fdw::TmaShape<T, 1, TMA_BX, 3, TMA_PD>::SMEM;
            case 2: return fdw::TmaShape<T, 2, TMA_BX, 3, TMA_PD>::SMEM;
            default: return fdw::TmaShape<T, 4, TMA_BX, 3, TMA_PD>::SMEM;
        }
    }
    if (vd) {
        switch (R) {
            case 1: return fdw::TmaShape<T, 1, TMA_BX, 6>::SMEM;
            case 2: return fdw::TmaShape<T, 2, TMA_BX, 6>::SMEM;
            default: return fdw::TmaShape<T, 4, TMA_BX, 6>::SMEM;
        }
    }
    switch (R) {
        case 1: return fdw::TmaShape<T, 1, TMA_BX>::SMEM;
        case 2: return fdw::TmaShape<T, 2, TMA_BX>::SMEM;
        default: return fdw::TmaShape<T, 4, TMA_BX>::SMEM;
    }
}

fdw::PeerArgs peer_args(fdw_solver* c);
bool fused_halo(const fdw_solver* c, bool virt);

template <typename T, bool EX>
bool launch_tma(fdw_solver* c, const SweepArgs<T>& a0, int src, int dst) {
    using S4 = fdw::TmaShape<T, 4, TMA_BX>;
    const cudaStream_t st = c->stream;
    SweepArgs<T> a = a0;
    dim3 block(S4::NTY, TMA_BX);
    dim3 grid((unsigned)((c->nyl + S4::TYW - 1) / S4::TYW), (unsigned)((c->nxl + TMA_BX - 1) / TMA_BX),
              (unsigned)c->zseg);
    if (fused_halo(c, true) && c->peers_ready) {
        // the sweep runs the step's halo epoch (enqueue_step): boundary CTAs
        // wait for the neighbours, store the halo planes into their ghost
        // planes, and the last of them publishes; the boundary segments
        // (S-1, 0) are rotated into the first wave
        a.peer_lo = static_cast<T*>(c->peer_lvl[0][dst]);
        a.peer_hi = static_cast<T*>(c->peer_lvl[1][dst]);
        a.peer_lo_delta = c->peer_delta[0];
        a.peer_hi_delta = c->peer_delta[1];
        a.peer = peer_args(c);
        a.publish = c->mirror_tgt ? 0 : 1;
        const int S = c->zseg, R = c->R;
        const long long nz = c->nzl;
        unsigned nseg = 0;
        for (int sg = 0; sg < S; ++sg) {
            const long long zs = nz * sg / S, ze = nz * (sg + 1) / S;
            if ((a.peer_lo && zs < R) || (a.peer_hi && ze > nz - R)) ++nseg;
        }
        a.n_bnd = nseg * grid.x * grid.y;
        a.seg_rot = c->dbg_no_rot ? 0 : S - 1;
        a.halo_store = c->loopback && c->dbg_no_store ? 0 : 1;
        a.fence_all = c->dbg_fence_all ? 1 : c->dbg_fence_sc ? 2 : 0;
    }
    const int col_base = (int)(c->base + c->R);
    const bool etab = c->tma_pd > 0 && c->n_etab > 0;
    // density: split rings only together with the damping table (vd_fast)
    const int pd = c->vd ? (etab ? c->tma_pd : 0) : c->tma_pd;
    const int smem = tma_smem<T>(c->R, c->vd, pd);
    const CUtensorMap& g0 = c->tm_g[0];
    const CUtensorMap& g1 = c->tm_g[1];
    const CUtensorMap& g2 = c->tm_g[2];
    // programmatic dependent launch: the sweep's prologue (mbarrier setup,
    // eta-range load) overlaps the predecessor's tail; it waits in-kernel
    // the time-step chain runs at high priority: a receiver kernel on the
    // side stream only takes the SM slots the sweep's last wave leaves free
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (c->prio_hi != c->prio_lo) {
        attr[na].id = cudaLaunchAttributePriority;
        attr[na++].val.priority = c->prio_hi;
    }
    if (c->pdl_sweep) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na++].val.programmaticStreamSerializationAllowed = 1;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = (size_t)smem;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = na;
    if (c->R != 1 && c->R != 2 && c->R != 4) return false;
    const void* kern = nullptr;
    if (c->vd) {
        kern = tma_vd_kernel<T>(c->R, EX, etab);
    } else if (pd > 0) {
        kern = tma_kernel<T>(c->R, EX, 3, pd, etab);
    } else {
        kern = tma_kernel<T>(c->R, EX, c->tma_minb == 3 ? 3 : 2);
    }
    if (!kern) return false;
    // an error is left for the caller's CHECK_LAUNCH (cudaGetLastError)
    // tm_p[src]: the split rings' head tile (interior box on the current level);
    // with the damping table the eta stream is the 1-byte index map
    CUtensorMap maps[8] = {c->tm_u[src], c->tm_p[dst], c->tm_c, etab ? c->tm_eb : c->tm_e, g0, g1, g2, c->tm_p[src]};
    int cb = col_base;
    void* args[10] = {&a, &maps[0], &maps[1], &maps[2], &maps[3], &maps[4], &maps[5], &maps[6], &maps[7], &cb};
    (void)cudaLaunchKernelExC(&cfg, kern, args);
    return true;
}

size_t res2d2_smem(const fdw_solver* c, int BZ, int tapcap) {
    const int V = 16 / c->tsize, TX = 16 * V, R = c->R;
    const int H1 = ((R + V - 1) / V) * V, H2 = ((2 * R + V - 1) / V) * V;
    return (size_t)(2 * (BZ + 4 * R) * (TX + 2 * H2) + 3 * (BZ + 2 * R) * (TX + 2 * H1)) * c->tsize +
           8 * fdw::F2D_CHUNK * sizeof(double) + (size_t)tapcap * sizeof(int);
}

template <typename T>
fdw_status launch_res2d_t(fdw_solver* c, int L, int cur0, bool record) {
    fdw::Res2DArgs<T> a{};
    a.lvl[0] = static_cast<T*>(c->lvl[0]);
    a.lvl[1] = static_cast<T*>(c->lvl[1]);
    a.c2dt2 = static_cast<const T*>(c->c2dt2);
    a.eta = static_cast<const T*>(c->eta);
    for (int j = 0; j <= c->R; ++j) a.v[j] = static_cast<T>(c->d.coeffs[j]);
    for (int k = 0; k < 2; ++k) a.ih[k] = static_cast<T>(1.0 / (c->d.spacing[k] * c->d.spacing[k]));
    a.dt = c->d.dt;
    a.ld = c->ld;
    a.origin = c->origin;
    a.nz = (int)c->nzl;
    a.nx = (int)c->nxl;
    for (int ax = 0; ax < 2; ++ax)
        for (int sd = 0; sd < 2; ++sd) {
            const int bc = c->d.bc[ax][sd];
            a.gf[ax][sd] = bc == FDW_BC_NULL_DIRICHLET ? -1 : bc == FDW_BC_NULL_NEUMANN ? 1 : 0;
        }
    a.BZ = c->res_BZ;
    a.xb = c->res_xb;
    a.blk_toff = c->d_blk_toff;
    a.blk_tgt = c->d_blk_tgt;
    a.blk_tpos = c->d_blk_tpos;
    a.ent_off = c->d_ent_off;
    a.ent_w = c->d_ent_w;
    a.wavelet = c->d_wavelet;
    a.n_wavelet = c->n_wavelet;
    a.blk_roff = c->d_blk_roff;
    a.blk_rpack = c->d_blk_rpack;
    a.tap_ix = c->d_tap_ix;
    a.tapcap = c->res_tapcap;
    a.tapbuf = static_cast<T*>(c->d_tapbuf);
    a.n_ent = c->n_ent;
    a.roff = c->d_rec_off;
    a.rw = c->d_rec_w;
    a.seis = c->d_seis;
    a.n_rec = c->d_seis ? c->n_rec : 0;
    a.n_rows = c->seis_rows;
    a.ctrl = c->ctrl;
    int rec = record && c->d_seis && c->d_tapbuf ? 1 : 0;
    const bool ex = c->d.math == FDW_MATH_EXACT;
    int Lp = c->res_pair ? (L & ~1) : 0, k0 = 0;
    a.hbuf[0] = static_cast<T*>(c->d_res_hbuf);
    a.hbuf[1] = a.hbuf[0] + c->level_elems;
    if (Lp >= 2) {  // pairs of steps, one grid barrier each
        void* args2[] = {&a, &Lp, &cur0, &rec};
        const void* f2 = res2d2_kernel<T>(c->R, ex);
        if (!f2) return fail(c, FDW_EINVAL, "resident 2D kernel not built for this configuration");
        // the smem attribute is per function, shared by every context of the process
        CU(raise_smem_limit(f2, c->res_smem2));
        CU(cudaLaunchCooperativeKernel(f2, dim3((unsigned)c->res_nb), dim3(256), args2, c->res_smem2, c->stream));
        if (c->capturing)
            ++c->capture_kernels;
        else
            ++c->launches;
        k0 = Lp;
    }
    int Ls = L - k0, cur = cur0 ^ (k0 & 1);
    if (Ls > 0) {
        void* args[] = {&a, &Ls, &cur, &rec, &k0};
        const void* f = res2d_kernel<T>(c->R, ex);
        if (!f) return fail(c, FDW_EINVAL, "resident 2D kernel not built for this configuration");
        CU(raise_smem_limit(f, c->res_smem));
        CU(cudaLaunchCooperativeKernel(f, dim3((unsigned)c->res_nb), dim3(256), args, c->res_smem, c->stream));
        if (c->capturing)
            ++c->capture_kernels;
        else
            ++c->launches;
    }
    return FDW_OK;
}

// Block decomposition of the resident 2D kernel: the largest co-resident
// occupancy whose blocks fit shared memory and leave every block at least
// 2R rows and 2*HY columns (mirror sources and strips stay inside a block).
template <typename T>
bool res2d_configure(fdw_solver* c) {
    if (std::getenv("FDW_NO_RESIDENT2D")) return false;
    const int V = 16 / (int)sizeof(T), TX = 16 * V, R = c->R, HY = ((R + V - 1) / V) * V, UW = TX + 2 * HY;
    const long long nz = c->nzl, nx = c->nxl;
    const int xb = (int)((nx + TX - 1) / TX);
    if (nx - (long long)(xb - 1) * TX < 2 * HY) return false;
    const void* f = res2d_kernel<T>(R, c->d.math == FDW_MATH_EXACT);
    if (!f) return false;
    // two steps per barrier: 2R strips and halos; blocks >= 2R rows, >= 2*H2 columns
    const int H2 = ((2 * R + V - 1) / V) * V;
    const void* f2 = res2d2_kernel<T>(R, c->d.math == FDW_MATH_EXACT);
    if (!std::getenv("FDW_NO_RES2D_PAIR") && f2 && nx - (long long)(xb - 1) * TX >= 2 * H2) {
        // 2 CTAs/SM first: measured faster than 3 smaller blocks (more ring per block) on C1
        for (int occ : {2, 3, 1}) {
            const long long cap = (long long)occ * c->sm_count;
            const long long zbn0 = std::min<long long>(nz, cap / xb);
            if (zbn0 < 1) continue;
            const int BZ = (int)((nz + zbn0 - 1) / zbn0);
            const int zbn = (int)((nz + BZ - 1) / BZ);
            if (BZ < 2 * R || nz - (long long)(zbn - 1) * BZ < 2 * R) continue;
            const size_t smem2 = res2d2_smem(c, BZ, 0);
            const size_t smem1 =
                (size_t)(2 * (BZ + 2 * R) * UW + 3 * BZ * TX) * sizeof(T) + 8 * fdw::F2D_CHUNK * sizeof(double);
            if (smem2 > 227 * 1024) continue;
            if (raise_smem_limit(f2, smem2) != cudaSuccess ||
                raise_smem_limit(f, smem1) != cudaSuccess) {
                cudaGetLastError();
                continue;
            }
            int got = 0;
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&got, f2, 256, smem2) != cudaSuccess) {
                cudaGetLastError();
                continue;
            }
            if ((long long)zbn * xb > (long long)got * c->sm_count) continue;
            const size_t hb = 2 * c->level_elems * sizeof(T);
            if (cudaMallocAsync(&c->d_res_hbuf, hb, c->stream) != cudaSuccess ||
                cudaMemsetAsync(c->d_res_hbuf, 0, hb, c->stream) != cudaSuccess) {
                cudaGetLastError();
                if (c->d_res_hbuf) cudaFreeAsync(c->d_res_hbuf, c->stream);
                c->d_res_hbuf = nullptr;
                break;  // the one-step kernel below
            }
            c->res2d = true;
            c->res_pair = true;
            c->res_BZ = BZ;
            c->res_xb = xb;
            c->res_nb = zbn * xb;
            c->res_smem = c->res_smem_base = smem1;
            c->res_smem2 = c->res_smem2_base = smem2;
            c->occupancy = got;
            return true;
        }
    }
    for (int occ = 3; occ >= 1; --occ) {
        const long long cap = (long long)occ * c->sm_count;
        const long long zbn0 = std::min<long long>(nz, cap / xb);
        if (zbn0 < 1) continue;
        const int BZ = (int)((nz + zbn0 - 1) / zbn0);
        const int zbn = (int)((nz + BZ - 1) / BZ);
        if (BZ < 2 * R || nz - (long long)(zbn - 1) * BZ < 2 * R) continue;
        const size_t smem =
            (size_t)(2 * (BZ + 2 * R) * UW + 3 * BZ * TX) * sizeof(T) + 8 * fdw::F2D_CHUNK * sizeof(double);
        if (smem > 227 * 1024) continue;
        if (raise_smem_limit(f, smem) != cudaSuccess) {
            cudaGetLastError();
            continue;
        }
        int got = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&got, f, 256, smem) != cudaSuccess) {
            cudaGetLastError();
            continue;
        }
        if ((long long)zbn * xb > (long long)got * c->sm_count) continue;
        c->res2d = true;
        c->res_BZ = BZ;
        c->res_xb = xb;
        c->res_nb = zbn * xb;
        c->res_smem = smem;
        c->res_smem_base = smem;
        c->occupancy = got;
        return true;
    }
    return false;
}

// block of extended (z, x) in the resident 2D decomposition, and its packed
// block-local coordinates (fdw::res2d_pack)
long long res2d_block_of(const fdw_solver* c, long long z, long long x, int* pos) {
    const int TX = 16 * (16 / c->tsize);
    const long long bz = z / c->res_BZ, bx = x / TX;
    *pos = fdw::res2d_pack((int)(z - bz * c->res_BZ), (int)(x - bx * TX));
    return bz * c->res_xb + bx;
}

// Per-block point-source list of the resident 2D kernel (merged targets).
fdw_status res2d_sources(fdw_solver* c);
// Per-block receiver-tap list of the resident 2D kernel (ghost taps mirrored).
fdw_status res2d_receivers(fdw_solver* c, const std::vector<long long>& ri);

template <typename T>
fdw_status launch_fused2d_t(fdw_solver* c, int L, int cur0, bool record, int k0) {
    if (c->res2d && !c->vd && k0 == 0) return launch_res2d_t<T>(c, L, cur0, record);
    fdw::Fused2DArgs<T> a{};
    a.lvl[0] = static_cast<T*>(c->lvl[0]);
    a.lvl[1] = static_cast<T*>(c->lvl[1]);
    a.c2dt2 = static_cast<const T*>(c->c2dt2);
    a.eta = static_cast<const T*>(c->eta);
    for (int j = 0; j <= c->R; ++j) a.v[j] = static_cast<T>(c->d.coeffs[j]);
    for (int k = 0; k < 2; ++k) a.ih[k] = static_cast<T>(1.0 / (c->d.spacing[k] * c->d.spacing[k]));
    a.ih[2] = T(1);
    a.dt = c->d.dt;
    a.ld = c->ld;
    a.origin = c->origin;
    a.nz = (int)c->nzl;
    a.nx = (int)c->nxl;
    for (int ax = 0; ax < 2; ++ax)
        for (int sd = 0; sd < 2; ++sd) {
            const int bc = c->d.bc[ax][sd];
            a.gf[ax][sd] = bc == FDW_BC_NULL_DIRICHLET ? -1 : bc == FDW_BC_NULL_NEUMANN ? 1 : 0;
        }
    a.tmap = c->d_tmap;
    a.ent_off = c->d_ent_off;
    a.ent_w = c->d_ent_w;
    a.wavelet = c->d_wavelet;
    a.n_wavelet = c->n_wavelet;
    a.ridx = c->d_rec_idx;
    a.roff = c->d_rec_off;
    a.rw = c->d_rec_w;
    a.seis = c->d_seis;
    a.n_rec = c->d_seis ? c->n_rec : 0;
    a.n_rows = c->seis_rows;
    a.ctrl = c->ctrl;
    if (c->vd) {
        for (int k = 0; k < 2; ++k) {
            a.grad[k] = static_cast<const T*>(c->grad[k]);
            a.i2h[k] = static_cast<T>(1.0 / (2.0 * c->d.spacing[k]));
        }
        for (int j = 0; j < c->R; ++j) a.w1[j] = static_cast<T>(c->d.coeffs1[j]);
    }
    {
        const char* dbg = std::getenv("FDW_DEBUG_FUSED");
        a.dbg = dbg ? std::atoi(dbg) : 0;
    }
    int rec = record && c->d_seis ? 1 : 0;
    void* args[] = {&a, &L, &cur0, &rec, &k0};
    const void* f = fused2d_kernel<T>(c->R, c->d.math == FDW_MATH_EXACT, c->vd);
    if (!f) return fail(c, FDW_EINVAL, "fused 2D kernel not built for this configuration");
    CU(cudaLaunchCooperativeKernel(f, dim3((unsigned)c->fused_grid), dim3(256), args, 0, c->stream));
    if (c->capturing)
        ++c->capture_kernels;
    else
        ++c->launches;
    return FDW_OK;
}

fdw_status launch_fused2d(fdw_solver* c, int L, int cur0, bool record, int k0) {
    return c->tsize == 4 ? launch_fused2d_t<float>(c, L, cur0, record, k0)
                         : launch_fused2d_t<double>(c, L, cur0, record, k0);
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// L2 promotion of the TMA loads: FDW_TMA_PROMO_U (u tiles, default 64 B) /
// FDW_TMA_PROMO_P (prev, c2dt2, eta tiles, default 256 B) = 0, 64, 128 or 256.
// The u tile rows start 16 B before a 128-B line (the Y halo); promoting those
// slivers to 256 B fetched neighbour data that missed L2 later: C4 sweep DRAM
// reads 2.155 -> 2.100 GB with 64 B (profiles/r01/power_cap.txt).
CUtensorMapL2promotion promo_env(const char* name, int dflt) {
    const char* e = std::getenv(name);
    const int v = e ? std::atoi(e) : dflt;
    return v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
         : v == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
         : v == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                    : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
}

// 3D map over one pitched level: dims (ld, rows_alloc, planes), box (bw, bh, 1)
bool make_map(const fdw_solver* c, CUtensorMap* m, void* base, int bw, int bh,
              CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B, int esize = 0) {
    auto fn = encode_fn();
    if (!fn) return false;
    if (!esize) esize = c->tsize;
    // The tensor ends at the padded box: row / column slack beyond it is
    // out of bounds, which TMA zero-fills without touching DRAM (the last
    // tile of a row or column would otherwise stream up to 63 slack columns /
    // 15 slack rows of every field).  No kernel reads a value from there.
    // FDW_TMA_FULL_PITCH=1: the whole allocated pitch (A/B).
    static const bool full = std::getenv("FDW_TMA_FULL_PITCH") != nullptr;
    const cuuint64_t dims[3] = {(cuuint64_t)(full ? c->ld : c->base + c->P[2]),
                                (cuuint64_t)(full ? c->rows_alloc : c->P[1]), (cuuint64_t)(c->Lz + 1)};
    const cuuint64_t strides[2] = {(cuuint64_t)c->ld * esize, (cuuint64_t)c->plane * esize};
    const cuuint32_t box[3] = {(cuuint32_t)bw, (cuuint32_t)bh, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUtensorMapDataType dt = esize == 1   ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                   : esize == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                                : CU_TENSOR_MAP_DATA_TYPE_FLOAT64;
    const CUresult r = fn(m, dt, 3,
                          base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_NONE, promo,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

template <typename T>
bool make_maps_t(fdw_solver* c) {
    int uw, uh, pw, ph;
    switch (c->R) {
#define SH(RR)                                                                   \
    case RR:                                                                     \
        uw = fdw::TmaShape<T, RR, TMA_BX>::UW;                                    \
        uh = fdw::TmaShape<T, RR, TMA_BX>::UH;                                    \
        pw = fdw::TmaShape<T, RR, TMA_BX>::TYW;                                   \
        ph = TMA_BX;                                                             \
        break;
        SH(1)
        SH(2)
        SH(4)
#undef SH
        default: return false;
    }
    bool ok = true;
    const CUtensorMapL2promotion pu = promo_env("FDW_TMA_PROMO_U", 64), pp = promo_env("FDW_TMA_PROMO_P", 256);
    for (int l = 0; l < 2; ++l) {
        ok &= make_map(c, &c->tm_u[l], c->lvl[l], uw, uh, pu);
        ok &= make_map(c, &c->tm_p[l], c->lvl[l], pw, ph, pp);
    }
    ok &= make_map(c, &c->tm_c, c->c2dt2, pw, ph, pp);
    ok &= make_map(c, &c->tm_e, c->eta, pw, ph, pp);
    return ok;
}

template <typename T>
int zmarch_occupancy(int R, bool exact) {
    constexpr int BX = 16;
    using S = fdw::ZMarchShape<T, BX>;
    int occ = 0;
    const void* f = nullptr;
    if (exact) {
        f = R == 1 ? (const void*)fdw::sweep3d_zmarch<T, 1, BX, true>
          : R == 2 ? (const void*)fdw::sweep3d_zmarch<T, 2, BX, true>
                   : (const void*)fdw::sweep3d_zmarch<T, 4, BX, true>;
    } else {
        f = R == 1 ? (const void*)fdw::sweep3d_zmarch<T, 1, BX, false>
          : R == 2 ? (const void*)fdw::sweep3d_zmarch<T, 2, BX, false>
                   : (const void*)fdw::sweep3d_zmarch<T, 4, BX, false>;
    }
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, f, S::THREADS, 0) != cudaSuccess) occ = 1;
    return occ < 1 ? 1 : occ;
}

template <typename T>
fdw_status launch_sweep_t(fdw_solver* c, int src, int dst, bool virt) {
    const SweepArgs<T> a = sweep_args<T>(c, src, dst);
    const bool ex = c->d.math == FDW_MATH_EXACT;
    if (c->vd && !(c->variant == FDW_KERNEL_TMA && virt)) {
        // density terms: the TMA kernel (virtual ghosts) or the element-wise sweep
        if (ex)
            launch_simple<T, true>(c, a);
        else
            launch_simple<T, false>(c, a);
    } else if (c->variant == FDW_KERNEL_TMA && !virt) {
        // stored-ghost step (caller-uploaded level): the LDG-fed Z-march
        const bool ok = ex ? launch_zmarch<T, true>(c, a) : launch_zmarch<T, false>(c, a);
        if (!ok) return fail(c, FDW_EINVAL, "zmarch kernel not built for radius %d", c->R);
    } else if (c->variant == FDW_KERNEL_TMA) {
        const bool ok = ex ? launch_tma<T, true>(c, a, src, dst) : launch_tma<T, false>(c, a, src, dst);
        if (!ok) return fail(c, FDW_EINVAL, "TMA kernel not built for radius %d", c->R);
    } else if (c->variant == FDW_KERNEL_ZMARCH) {
        const bool ok = ex ? launch_zmarch<T, true>(c, a) : launch_zmarch<T, false>(c, a);
        if (!ok) return fail(c, FDW_EINVAL, "zmarch kernel not built for radius %d", c->R);
    } else {
        if (ex)
            launch_simple<T, true>(c, a);
        else
            launch_simple<T, false>(c, a);
    }
    CHECK_LAUNCH();
    return FDW_OK;
}

fdw_status launch_sweep(fdw_solver* c, int src, int dst, bool virt) {
    return c->tsize == 4 ? launch_sweep_t<float>(c, src, dst, virt) : launch_sweep_t<double>(c, src, dst, virt);
}

template <typename T>
fdw_status launch_inject_t(fdw_solver* c, int dst, int k, int t0 = 0, int cnt = -1, cudaStream_t st = nullptr,
                           bool pdl = false) {
    if (cnt < 0) cnt = c->n_tgt - t0;
    if (cnt <= 0) return FDW_OK;
    if (!st) st = c->stream;
    const int tb = 128;
    fdw::PeerMirror<T> pm;
    if (c->peer_mode && c->peers_ready) {  // targets in the halo planes reach the neighbour too
        pm.lo = static_cast<T*>(c->peer_lvl[0][dst]);
        pm.hi = static_cast<T*>(c->peer_lvl[1][dst]);
        pm.lo_delta = c->peer_delta[0];
        pm.hi_delta = c->peer_delta[1];
        pm.lo_end = c->origin + (long long)c->R * c->plane;
        pm.hi_begin = c->origin + (c->nzl - c->R) * c->plane;
    }
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (c->prio_hi != c->prio_lo) {
        attr[na].id = cudaLaunchAttributePriority;
        attr[na++].val.priority = c->prio_hi;
    }
    if (pdl) {  // PDL: setup-time loads overlap the sweep's tail (inject_kernel)
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na++].val.programmaticStreamSerializationAllowed = 1;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)((cnt + tb - 1) / tb));
    cfg.blockDim = dim3(tb);
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = na;
    (void)cudaLaunchKernelEx(&cfg, fdw::inject_kernel<T, true>, static_cast<T*>(c->lvl[dst]),
                             static_cast<const T*>(c->c2dt2), static_cast<const T*>(c->eta), c->d.dt,
                             static_cast<const long long*>(c->d_tgt + t0),
                             static_cast<const unsigned int*>(c->d_ent_off + t0),
                             static_cast<const double*>(c->d_ent_w), static_cast<const double*>(c->d_wavelet),
                             c->n_wavelet, cnt, k, static_cast<const fdw::Ctrl*>(c->ctrl), pm);
    CHECK_LAUNCH();
    return FDW_OK;
}

template <typename T>
fdw_status launch_volume_t(fdw_solver* c, int dst, int k) {
    if (c->vs_fields.empty()) return FDW_OK;
    const long long ny = c->ndim == 3 ? c->nyl : 1;
    const long long n = c->nzl * c->nxl * ny;
    const int tb = 256;
    int dface = 0;
    for (int a = 0; a < c->ndim; ++a)
        for (int sd = 0; sd < 2; ++sd) {
            if (c->d.bc[a][sd] != FDW_BC_NULL_DIRICHLET) continue;
            if (a == 0 && c->ndim == 3 && ((sd == 0 && c->d.rank != 0) || (sd == 1 && c->d.rank != c->d.world - 1)))
                continue;  // internal slab face
            dface |= 1 << (2 * a + sd);
        }
    fdw::volume_source_kernel<T><<<(unsigned)((n + tb - 1) / tb), tb, 0, c->stream>>>(
        static_cast<T*>(c->lvl[dst]), static_cast<const T*>(c->c2dt2), static_cast<const T*>(c->eta), c->d.dt,
        static_cast<const T* const*>(c->d_vs_ptrs), static_cast<const T*>(c->d_vs_amp), c->d_vs_len, (int)c->vs_fields.size(),
        c->vs_namp, c->origin, c->ndim == 3 ? c->plane : c->ld, c->ndim == 3 ? c->ld : 1, (int)c->nzl,
        (int)c->nxl, (int)ny, dface, k, c->ctrl);
    CHECK_LAUNCH();
    return FDW_OK;
}

fdw_status launch_inject(fdw_solver* c, int dst, int k, bool pdl = false) {
    fdw_status s = c->tsize == 4 ? launch_inject_t<float>(c, dst, k, 0, -1, nullptr, pdl)
                                 : launch_inject_t<double>(c, dst, k, 0, -1, nullptr, pdl);
    if (s) return s;
    return c->tsize == 4 ? launch_volume_t<float>(c, dst, k) : launch_volume_t<double>(c, dst, k);
}

// apply_boundary (kernel.hpp:67-102) on level `lv`: axis 0, 1, 2 in order.
// For Z-slabs the Z phase runs only on global faces and the X/Y phases skip
// the internal ghost planes (those arrive complete from the neighbour).
template <typename T>
fdw_status launch_boundary_t(fdw_solver* c, int lv, int mode) {
    const Ctrl* ctrl = c->ctrl;
    T* f = static_cast<T*>(c->lvl[lv]);
    const int h = c->R;
    const int tb = 256;
    auto go = [&](long long origin_pad, long long sa, int n_ext, long long s1, int n1, long long s2,
                  int n2, int bc_lo, int bc_hi, int do_lo, int do_hi) -> fdw_status {
        const long long n = (long long)n1 * n2;
        if (n <= 0 || (!do_lo && !do_hi)) return FDW_OK;
        fdw::ghost_lines<T><<<(unsigned)((n + tb - 1) / tb), tb, 0, c->stream>>>(
            f, origin_pad, sa, n_ext, h, s1, n1, s2, n2, bc_lo, bc_hi, do_lo, do_hi, ctrl, mode);
        CHECK_LAUNCH();
        return FDW_OK;
    };
    fdw_status s;
    const auto& bc = c->d.bc;
    if (c->ndim == 3) {
        const int rank = c->d.rank, world = c->d.world;
        // axis 0 (Z): lines over all padded (X, Y)
        s = go(c->origin_pad, c->plane, (int)c->nzl, c->ld, (int)c->P[1], 1, (int)c->P[2], bc[0][0],
               bc[0][1], rank == 0, rank == world - 1);
        if (s) return s;
        const long long p_lo = rank > 0 ? h : 0;
        const long long p_hi = rank < world - 1 ? c->Lz - h : c->Lz;
        const long long o = c->origin_pad + p_lo * c->plane;
        // axis 1 (X): lines over (planes, padded Y)
        s = go(o, c->ld, (int)c->nxl, c->plane, (int)(p_hi - p_lo), 1, (int)c->P[2], bc[1][0],
               bc[1][1], 1, 1);
        if (s) return s;
        // axis 2 (Y): lines over (planes, padded X)
        s = go(o, 1, (int)c->nyl, c->plane, (int)(p_hi - p_lo), c->ld, (int)c->P[1], bc[2][0],
               bc[2][1], 1, 1);
        if (s) return s;
    } else {
        // axis 0 (Z = rows): lines over padded X columns
        s = go(c->origin_pad, c->ld, (int)c->nzl, 0, 1, 1, (int)c->P[1], bc[0][0], bc[0][1], 1, 1);
        if (s) return s;
        // axis 1 (X = fast): lines over padded Z rows
        s = go(c->origin_pad, 1, (int)c->nxl, c->ld, (int)c->P[0], 0, 1, bc[1][0], bc[1][1], 1, 1);
        if (s) return s;
    }
    return FDW_OK;
}

fdw_status launch_boundary(fdw_solver* c, int lv, int mode) {
    return c->tsize == 4 ? launch_boundary_t<float>(c, lv, mode) : launch_boundary_t<double>(c, lv, mode);
}

fdw::PeerArgs peer_args(fdw_solver* c) {
    fdw::PeerArgs p{};
    p.self = c->psync;
    for (int r = 0; r < fdw::PEER_MAX_WORLD; ++r) p.peer[r] = c->peer_sync[r];
    p.rank = c->d.rank;
    p.world = c->d.world;
    p.ctrl = c->ctrl;
    return p;
}

bool slab_peers(const fdw_solver* c) { return c->d.world > 1 && c->peer_mode; }

// Host-ordered group: this rank's stream waits for its neighbours' (or every
// rank's) work enqueued before this point.  See HostGroup.
fdw_status group_point(fdw_solver* c, bool all_ranks) {
    HostGroup* g = c->group;
    if (!g) return FDW_OK;
    const int r = c->d.rank;
    const int slot = (int)(g->round[r]++ & 1);
    CU(cudaEventRecord(g->ev[r][slot], c->stream));
    if (!g->barrier())
        return fail(c, FDW_EPEER, "host-ordered slab group: a rank did not reach the same collective call within 60 s");
    for (int s = 0; s < c->d.world; ++s) {
        if (s == r || (!all_ranks && s != r - 1 && s != r + 1)) continue;
        CU(cudaStreamWaitEvent(c->stream, g->ev[s][slot], 0));
    }
    return FDW_OK;
}

fdw_status peers_usable(fdw_solver* c) {
    if (!c->peers_ready) return fail(c, FDW_ESTATE, "peer transport: fdw_peer_import / fdw_peer_link first");
    if (c->ipc_same_device)
        return fail(c, FDW_ESTATE,
                    "peer transport: a neighbour in another process shares this GPU; its kernels and ours would "
                    "wait on each other -- drive ranks that share a GPU from one process (fdw_peer_link)");
    return FDW_OK;
}

// Start of a halo epoch (before an operation that reads ghost planes or
// stores into a neighbour's): wait until both neighbours published it.
// `in_kernel`: the TMA sweep waits itself (only the host-ordered point here).
fdw_status launch_peer_wait(fdw_solver* c, bool in_kernel, int honor_abort = 1) {
    fdw_status s = peers_usable(c);
    if (s) return s;
    if ((s = group_point(c, false))) return s;
    if (in_kernel) return FDW_OK;
    fdw::peer_wait_kernel<<<1, 32, 0, c->stream>>>(peer_args(c), honor_abort);
    CHECK_LAUNCH();
    return FDW_OK;
}

fdw_status launch_peer_publish(fdw_solver* c, int honor_abort = 1) {
    fdw_status s = peers_usable(c);
    if (s) return s;
    fdw::peer_publish_kernel<<<1, 32, 0, c->stream>>>(peer_args(c), honor_abort);
    CHECK_LAUNCH();
    return FDW_OK;
}

// Copies the first / last R owned planes of level lv into the neighbours'
// ghost planes (full padded planes); the caller brackets it with
// launch_peer_wait / launch_peer_publish.
fdw_status launch_peer_push(fdw_solver* c, int lv) {
    fdw_status s = peers_usable(c);
    if (s) return s;
    const long long n = (long long)c->R * c->plane;
    const long long lo_src = (long long)c->R * c->plane, hi_src = c->nzl * c->plane;
    const unsigned grid = (unsigned)std::min<long long>((n / (16 / c->tsize) + 255) / 256, (long long)c->sm_count * 4);
    if (c->tsize == 4)
        fdw::peer_push<float><<<grid, 256, 0, c->stream>>>(static_cast<const float*>(c->lvl[lv]),
                                                            static_cast<float*>(c->peer_lvl[0][lv]),
                                                            static_cast<float*>(c->peer_lvl[1][lv]), lo_src,
                                                            c->peer_delta[0], hi_src, c->peer_delta[1], n);
    else
        fdw::peer_push<double><<<grid, 256, 0, c->stream>>>(static_cast<const double*>(c->lvl[lv]),
                                                             static_cast<double*>(c->peer_lvl[0][lv]),
                                                             static_cast<double*>(c->peer_lvl[1][lv]), lo_src,
                                                             c->peer_delta[0], hi_src, c->peer_delta[1], n);
    CHECK_LAUNCH();
    return FDW_OK;
}

// A whole halo epoch that only pushes level lv (refresh_boundary).
fdw_status peer_exchange(fdw_solver* c, int lv) {
    if (!slab_peers(c) || c->ndim != 3) return FDW_OK;
    fdw_status s;
    if ((s = launch_peer_wait(c, false, 0))) return s;
    if ((s = launch_peer_push(c, lv))) return s;
    return launch_peer_publish(c, 0);
}

// Teardown of a linked slab context, before its levels and sync block are
// freed.  Host-ordered group: wait for the other members' queued work (their
// stores into this rank's memory) and break the group, so a member that keeps
// calling collectives fails at once instead of waiting for this rank.  Peer
// ranks on other GPUs: a bounded device-side wait until every rank finished
// the halo / health epochs this rank went through.
void peer_leave(fdw_solver* c) {
    if (!c->peer_mode || !c->peers_ready) return;
    if (HostGroup* g = c->group) {
        std::lock_guard<std::mutex> lk(g_group_mu);
        {
            std::lock_guard<std::mutex> gl(g->mu);
            g->broken = true;
            g->cv.notify_all();
        }
        for (int r = 0; r < g->world; ++r)
            if (g->member[r] && g->member[r] != c) cudaStreamSynchronize(g->member[r]->stream);
        g->member[c->d.rank] = nullptr;
        c->group = nullptr;
        // a broken group is never joined again: drop its key now (a new rank-0
        // context may reuse this address while other members still live)
        for (auto it = g_groups.begin(); it != g_groups.end();)
            it = it->second == g ? g_groups.erase(it) : std::next(it);
        if (--g->alive == 0) {
            for (auto& e2 : g->ev)
                for (cudaEvent_t e : e2)
                    if (e) cudaEventDestroy(e);
            delete g;
        }
        return;
    }
    if (c->ipc_same_device || c->loopback) return;  // never stepped (peers_usable) / no real peers
    fdw::peer_quiesce<<<1, 32, 0, c->stream>>>(peer_args(c), 5000000000ull);
    cudaStreamSynchronize(c->stream);
    cudaGetLastError();
}

// Cross-rank health reduction: post, (host-ordered point), reduce.
fdw_status launch_peer_health(fdw_solver* c, int honor_abort) {
    fdw_status s = peers_usable(c);
    if (s) return s;
    fdw::peer_health_post<<<1, 32, 0, c->stream>>>(peer_args(c), honor_abort);
    CHECK_LAUNCH();
    if ((s = group_point(c, true))) return s;
    fdw::peer_health_reduce<<<1, 32, 0, c->stream>>>(peer_args(c), honor_abort);
    CHECK_LAUNCH();
    return FDW_OK;
}

template <typename T>
fdw_status launch_receivers_t(fdw_solver* c, int lv, int row_add, cudaStream_t st) {
    if (c->n_rec == 0 || !c->d_seis) return FDW_OK;
    if (c->n_split > 0) {
        fdw::receiver_products_kernel<T><<<(c->n_split + 255) / 256, 256, 0, st>>>(
            static_cast<const T*>(c->lvl[lv]), c->d_sp_idx, c->d_sp_w, c->d_sp_prod, c->n_split, c->seis_rows,
            row_add, c->ctrl);
        CHECK_LAUNCH();
    }
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributePriority;
    attr[0].val.priority = c->prio_lo;  // below the step chain (launch_tma)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)((c->n_rec + fdw::REC_WARPS - 1) / fdw::REC_WARPS));
    cfg.blockDim = dim3(32 * fdw::REC_WARPS);
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = c->prio_hi != c->prio_lo ? 1 : 0;
    (void)cudaLaunchKernelEx(&cfg, fdw::receivers_kernel<T>, static_cast<const T*>(c->lvl[lv]),
                             static_cast<const long long*>(c->d_rec_idx), static_cast<const unsigned int*>(c->d_rec_off),
                             static_cast<const double*>(c->d_rec_w), c->d_seis, c->n_rec, c->seis_rows, row_add,
                             static_cast<const fdw::Ctrl*>(c->ctrl));
    CHECK_LAUNCH();
    return FDW_OK;
}

fdw_status launch_receivers(fdw_solver* c, int lv, int row_add, cudaStream_t st = nullptr) {
    if (!st) st = c->stream;
    return c->tsize == 4 ? launch_receivers_t<float>(c, lv, row_add, st)
                         : launch_receivers_t<double>(c, lv, row_add, st);
}

bool overlap_receivers(const fdw_solver* c) { return c->side && !c->prof && c->n_rec > 0 && c->d_seis; }

// Health reduction over this rank's owned padded planes (global faces keep
// their ghost planes; internal ghost planes belong to the neighbour).
// check_health / max_abs (kernel.hpp:265-273, :456-458): a scan of the
// extended points gives max |u| (ghost cells only repeat those magnitudes or
// hold 0); only if a non-finite value exists are the ghost cells materialised
// (exact apply_boundary) and the padded slab rescanned for the first
// non-finite flat index, as the reference's padded scan returns it.
template <typename T>
fdw_status launch_health_t(fdw_solver* c, int lv, int honor_abort) {
    // a caller-uploaded level keeps its own ghost values: scan it as stored
    const bool raw = c->gstate[lv] == 2;
    fdw::health_reset<<<1, 1, 0, c->stream>>>(c->ctrl, honor_abort);
    CHECK_LAUNCH();
    const T* u = static_cast<const T*>(c->lvl[lv]);
    const int h = c->R;
    long long p_lo = 0, p_hi = 1, n_rows, n_cols;
    unsigned long long gp_lo = 0, gp_hi = 0;
    int ext_planes = 1, ext_rows, ext_cols, e_p0 = 0;
    if (c->ndim == 3) {
        p_lo = c->d.rank > 0 ? h : 0;
        p_hi = c->d.rank < c->d.world - 1 ? c->Lz - h : c->Lz;
        gp_lo = c->d.z_begin;  // global padded plane of local plane 0
        gp_hi = c->d.z_begin + c->Lz;
        n_rows = c->P[1];
        n_cols = c->P[2];
        ext_planes = (int)c->nzl;
        e_p0 = h;
        ext_rows = (int)c->nxl;
        ext_cols = (int)c->nyl;
    } else {
        n_rows = c->P[0];
        n_cols = c->P[1];
        ext_rows = (int)c->nzl;
        ext_cols = (int)c->nxl;
    }
    const unsigned long long P1 = (unsigned long long)c->P[1], P2 = (unsigned long long)c->P[2];
    const int is3d = c->ndim == 3;
    if (!raw) {
        (void)e_p0;
        fdw::health_scan_ext<T><<<c->sm_count * 8, 256, 0, c->stream>>>(
            u, c->origin, c->ld, c->plane, ext_planes, ext_rows, ext_cols, h, gp_lo, P1, P2, is3d, c->ctrl,
            honor_abort);
        CHECK_LAUNCH();
    }
    if (slab_peers(c)) {
        fdw_status s = launch_peer_health(c, honor_abort);
        if (s) return s;
    }
    {
        if (!raw) {
            fdw_status s = launch_boundary(c, lv, 2);
            if (s) return s;
        }
        const long long rows = (p_hi - p_lo) * n_rows;
        const int blocks = (int)std::min<long long>(rows, (long long)c->sm_count * 8);
        fdw::health_kernel<T><<<blocks, 256, 0, c->stream>>>(u, c->origin_pad, c->ld, c->plane, (int)p_lo,
                                                             (int)(p_hi - p_lo), 0, (int)n_rows, 0, (int)n_cols,
                                                             gp_lo, P1, P2, is3d, c->ctrl, honor_abort, raw ? 0 : 1);
        CHECK_LAUNCH();
    }
    if (slab_peers(c)) {
        fdw_status s = launch_peer_health(c, honor_abort);
        if (s) return s;
    }
    fdw::health_classify<T><<<1, 1, 0, c->stream>>>(u, c->ctrl, c->origin_pad, c->ld, c->plane, gp_lo, gp_hi, P1, P2,
                                                    is3d, honor_abort);
    CHECK_LAUNCH();
    if (slab_peers(c)) {
        fdw_status s = launch_peer_health(c, honor_abort);
        if (s) return s;
    }
    return FDW_OK;
}

fdw_status launch_health(fdw_solver* c, int lv, int honor_abort) {
    NvtxRange nv("fdw health check");
    return c->tsize == 4 ? launch_health_t<float>(c, lv, honor_abort) : launch_health_t<double>(c, lv, honor_abort);
}

// -- profiling marks (direct-launch mode only) --
struct Mark {
    fdw_solver* c;
    int cls;
    cudaEvent_t a = nullptr, b = nullptr;
    Mark(fdw_solver* c_, int cls_) : c(c_), cls(cls_) {
        if (c->prof) {
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaEventRecord(a, c->stream);
        }
    }
    ~Mark() {
        if (c->prof) {
            cudaEventRecord(b, c->stream);
            c->prof->marks.push_back({cls, {a, b}});
        }
    }
};

// One Solver::step (kernel.hpp:226-233) with relative index k inside a chunk;
// `src` is the current level before the step.
// Virtual-ghost path for a step reading level `src`: only the TMA kernel, and
// only when src's stored ghosts are not caller-provided raw values.
bool virtual_step(const fdw_solver* c, int gstate_src) {
    // FUSED2D reads stored ghosts (any state) and leaves corner ghosts stale
    if (c->variant == FDW_KERNEL_FUSED2D) return true;
    return c->variant == FDW_KERNEL_TMA && gstate_src != 2;
}

template <typename P>
fdw_status dev_upload(fdw_solver* c, P** dst, const std::vector<P>& v) {
    // stream-ordered pool memory: a synchronous cudaFree costs a device-wide
    // sync and, measured on B200, up to seconds while the driver trims
    if (*dst) cudaFreeAsync(*dst, c->stream);
    *dst = nullptr;
    const size_t n = std::max<size_t>(v.size(), 1);
    CU(cudaMallocAsync(reinterpret_cast<void**>(dst), n * sizeof(P), c->stream));
    if (!v.empty()) CU(cudaMemcpyAsync(*dst, v.data(), v.size() * sizeof(P), cudaMemcpyHostToDevice, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    return FDW_OK;
}

fdw_status res2d_sources(fdw_solver* c) {
    const int nb = c->res_nb;
    std::vector<std::vector<std::pair<int, int>>> per((size_t)nb);
    const int TX = 16 * (16 / c->tsize), ring = c->res_pair ? c->R : 0;
    const int zbn = c->res_nb / c->res_xb;
    for (size_t t = 0; t < c->h_tgt.size(); ++t) {
        const long long rem = c->h_tgt[t] - c->origin;
        const long long z = rem / c->ld, x = rem % c->ld;
        if (rem < 0 || z >= c->nzl || x >= c->nxl) return fail(c, FDW_EINVAL, "source target outside the grid");
        // the owning block, and (two-step kernel) every block whose R-wide ring holds it
        for (int bzi = 0; bzi < zbn; ++bzi)
            for (int bxi = 0; bxi < c->res_xb; ++bxi) {
                const long long z0 = (long long)bzi * c->res_BZ, x0 = (long long)bxi * TX;
                const long long z1 = std::min<long long>(z0 + c->res_BZ, c->nzl), x1 = std::min<long long>(x0 + TX, c->nxl);
                if (z < z0 - ring || z >= z1 + ring || x < x0 - ring || x >= x1 + ring) continue;
                const bool in = z >= z0 && z < z1 && x >= x0 && x < x1;
                per[(size_t)(bzi * c->res_xb + bxi)].push_back(
                    {(int)t, fdw::res2d_pack((int)(z - z0), (int)(x - x0)) | (in ? fdw::RES2D_IN_BLOCK : 0)});
            }
    }
    std::vector<int> off(1, 0), tg, ps;
    for (auto& v : per) {
        for (auto& e : v) {
            tg.push_back(e.first);
            ps.push_back(e.second);
        }
        off.push_back((int)tg.size());
    }
    fdw_status s;
    if ((s = dev_upload(c, &c->d_blk_toff, off))) return s;
    if ((s = dev_upload(c, &c->d_blk_tgt, tg))) return s;
    return dev_upload(c, &c->d_blk_tpos, ps);
}

// Receiver taps as apply_boundary leaves the level (kernel.hpp:67-102): a tap
// in a ghost cell reads the mirrored extended point times the faces' factors
// (-1 Dirichlet, +1 Neumann; "none" gives 0), corners both axes.
fdw_status res2d_receivers(fdw_solver* c, const std::vector<long long>& ri) {
    const int nb = c->res_nb;
    const int n = (int)ri.size();
    std::vector<std::vector<std::tuple<int, int, int>>> per((size_t)nb);  // (entry, smem offset, factor)
    auto fac = [&](int ax, int side) {
        const int bc = c->d.bc[ax][side];
        return bc == FDW_BC_NULL_DIRICHLET ? -1 : bc == FDW_BC_NULL_NEUMANN ? 1 : 0;
    };
    for (int e = 0; e < n; ++e) {
        // offset = origin + z*ld + x with x in [-R, nx+R) and ld > nx + 2R
        const long long q = ri[(size_t)e] - c->origin + c->R;
        long long z = q >= 0 ? q / c->ld : -((-q + c->ld - 1) / c->ld);
        long long x = q - z * c->ld - c->R;
        int f = 1;
        if (z < 0) { z = -z; f *= fac(0, 0); }
        if (z >= c->nzl) { z = 2 * (c->nzl - 1) - z; f *= fac(0, 1); }
        if (x < 0) { x = -x; f *= fac(1, 0); }
        if (x >= c->nxl) { x = 2 * (c->nxl - 1) - x; f *= fac(1, 1); }
        if (z < 0 || z >= c->nzl || x < 0 || x >= c->nxl) return fail(c, FDW_EINVAL, "receiver tap outside the grid");
        if (f == 0) {  // "none" face: the tap reads +0 (any in-block position, factor 0)
            per[0].push_back({e, fdw::res2d_pack(0, 0), 0});
            continue;
        }
        int pos = 0;
        const long long b = res2d_block_of(c, z, x, &pos);
        per[(size_t)b].push_back({e, pos, f});
    }
    // One tap-buffer slot per distinct (block, position, mirror factor): the
    // windows of neighbouring receivers overlap (C2: 108,800 entries on 14,7k
    // points), so the blocks that hold them store each value once per row.
    std::vector<int> off(1, 0), pack, ix((size_t)std::max(n, 1), 0);
    int most = 0;
    for (auto& v : per) {
        std::unordered_map<int, int> uniq;
        for (auto& t : v) {
            const int key = (std::get<1>(t) << 2) | (std::get<2>(t) + 1);
            auto it = uniq.find(key);
            if (it == uniq.end()) {
                it = uniq.emplace(key, (int)pack.size()).first;
                pack.push_back(key);
            }
            ix[(size_t)std::get<0>(t)] = it->second;
        }
        most = std::max(most, (int)uniq.size());
        off.push_back((int)pack.size());
    }
    const int n_slots = (int)pack.size();
    fdw_status s;
    if ((s = dev_upload(c, &c->d_blk_roff, off))) return s;
    if ((s = dev_upload(c, &c->d_blk_rpack, pack))) return s;
    if ((s = dev_upload(c, &c->d_tap_ix, ix))) return s;
    // cache each block's tap list in shared memory when the grid still fits
    c->res_tapcap = 0;
    c->res_smem = c->res_smem_base;
    c->res_smem2 = c->res_smem2_base;
    if (most > 0 && most <= 16384) {
        const bool ex = c->d.math == FDW_MATH_EXACT;
        auto fits = [&](const void* f, size_t smem) {
            int got = 0;
            return smem <= 227 * 1024 &&
                   raise_smem_limit(f, smem) == cudaSuccess &&
                   cudaOccupancyMaxActiveBlocksPerMultiprocessor(&got, f, 256, smem) == cudaSuccess &&
                   (long long)c->res_nb <= (long long)got * c->sm_count;
        };
        const size_t s1 = c->res_smem_base + (size_t)most * sizeof(int);
        const size_t s2 = c->res_smem2_base + (size_t)most * sizeof(int);
        const void* f1 = c->tsize == 4 ? res2d_kernel<float>(c->R, ex) : res2d_kernel<double>(c->R, ex);
        const void* f2 = c->tsize == 4 ? res2d2_kernel<float>(c->R, ex) : res2d2_kernel<double>(c->R, ex);
        if (fits(f1, s1) && (!c->res_pair || fits(f2, s2))) {
            c->res_tapcap = most;
            c->res_smem = s1;
            c->res_smem2 = s2;
        }
        cudaGetLastError();
    }
    if (c->d_tapbuf) cudaFreeAsync(c->d_tapbuf, c->stream);
    c->d_tapbuf = nullptr;
    c->n_ent = n_slots;
    CU(cudaMallocAsync(&c->d_tapbuf, (size_t)std::max(1, 8 * n_slots) * c->tsize, c->stream));  // 8 rows in flight
    CU(cudaMemsetAsync(c->d_tapbuf, 0, (size_t)std::max(1, 8 * n_slots) * c->tsize, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    return FDW_OK;
}

bool use_pdl(const fdw_solver* c) {
    // host-ordered groups put an event wait between steps: plain launches there
    return !c->no_pdl && c->variant == FDW_KERNEL_TMA && !c->prof && c->vs_fields.empty() && !c->group;
}

// Whether the TMA sweep reading level `src` runs the slab's halo epoch itself
// (waits in its boundary CTAs, stores the halo planes, publishes).
bool fused_halo(const fdw_solver* c, bool virt) {
    return slab_peers(c) && c->variant == FDW_KERNEL_TMA && virt && c->vs_fields.empty();
}

// One Solver::step (kernel.hpp:226-233) with relative index k inside a chunk;
// `src` is the current level before the step.  For Z slabs the step is one
// halo epoch: the neighbours' previous step must be complete before this
// step's boundary CTAs read the ghost planes or store into theirs.
fdw_status enqueue_step(fdw_solver* c, int k, int src, bool record, bool virt) {
    const int dst = 1 - src;
    fdw_status s;
    const bool ovl = record && overlap_receivers(c);
    // this sweep overwrites level `dst`, which step k-2's receivers read
    if (ovl && k >= 2) CU(cudaStreamWaitEvent(c->stream, c->rec_ev[k & 1], 0));
    const bool peers = slab_peers(c) && c->ndim == 3;
    const bool fused = fused_halo(c, virt);
    if (peers && (s = launch_peer_wait(c, fused))) return s;
    // programmatic dependent launch inside a chunk (TMA sweep on virtual
    // ghosts, no volume sources): the sweep follows the previous step's
    // point-source kernel (or sweep), which follows this sweep
    const bool pdl = use_pdl(c) && virt;
    c->pdl_sweep = pdl && k > 0 && c->tail_pdl_aware && !(peers && !fused);
    { Mark m(c, 0); s = launch_sweep(c, src, dst, virt); c->pdl_sweep = false; if (s) return s; }
    c->tail_pdl_aware = pdl;
    if (c->n_tgt > 0 || !c->vs_fields.empty()) {
        Mark m(c, 1);
        if ((s = launch_inject(c, dst, k, pdl && c->tail_pdl_aware))) return s;
        c->tail_pdl_aware = pdl && c->vs_fields.empty();
    }
    // swap: dst is now the current level
    if (!virt) { Mark m(c, 2); if ((s = launch_faces(c, dst))) return s; c->tail_pdl_aware = false; }
    if (peers) {
        Mark m(c, 5);
        if (!fused) {  // the sweep did not store the halo planes itself
            if ((s = launch_peer_push(c, dst))) return s;
        }
        // the sweep publishes unless a point source wrote into the halo
        // planes after it (its mirrored store must be visible first)
        if (!fused || c->mirror_tgt) {
            if ((s = launch_peer_publish(c))) return s;
            c->tail_pdl_aware = false;
        }
    }
    if (record && ovl) {
        CU(cudaEventRecord(c->fork_ev[k & 1], c->stream));
        CU(cudaStreamWaitEvent(c->side, c->fork_ev[k & 1], 0));
        if ((s = launch_receivers(c, dst, k + 1, c->side))) return s;
        CU(cudaEventRecord(c->rec_ev[k & 1], c->side));
    } else if (record) {
        Mark m(c, 3);
        if ((s = launch_receivers(c, dst, k + 1))) return s;
        c->tail_pdl_aware = false;
    }
    return FDW_OK;
}

fdw_status enqueue_chunk(fdw_solver* c, unsigned long long L, int cur0, bool check, bool record, bool first_virt,
                         bool rest_virt) {
    fdw_status s;
    c->tail_pdl_aware = false;  // the chunk's first sweep follows an ordinary launch
    if (c->variant == FDW_KERNEL_FUSED2D) {
        // one cooperative launch for the chunk (one per step when profiling);
        // a raw first level takes one stored-ghost step first
        unsigned long long k0 = 0;
        (void)first_virt;  // stored ghosts: a raw (caller-uploaded) level is read as stored
        if (c->prof) {
            for (unsigned long long k = k0; k < L; ++k) {
                Mark m(c, 0);
                if ((s = launch_fused2d(c, 1, cur0 ^ (int)(k & 1), record, (int)k))) return s;
            }
        } else if (L > k0) {
            if ((s = launch_fused2d(c, (int)(L - k0), cur0 ^ (int)(k0 & 1), record, (int)k0))) return s;
        }
    } else {
        for (unsigned long long k = 0; k < L; ++k)
            if ((s = enqueue_step(c, (int)k, cur0 ^ (int)(k & 1), record, k == 0 ? first_virt : rest_virt))) return s;
        if (record && overlap_receivers(c)) {  // join the side stream before the chunk ends
            CU(cudaStreamWaitEvent(c->stream, c->rec_ev[(L - 1) & 1], 0));
            if (L >= 2) CU(cudaStreamWaitEvent(c->stream, c->rec_ev[(L - 2) & 1], 0));
        }
    }
    fdw::step_advance<<<1, 1, 0, c->stream>>>(c->ctrl, L);
    CHECK_LAUNCH();
    if (check) {
        const int lv = cur0 ^ (int)(L & 1);
        Mark m(c, 4);
        if ((s = launch_health(c, lv, 1))) return s;
        fdw::health_latch<<<1, 1, 0, c->stream>>>(c->ctrl);
        CHECK_LAUNCH();
    }
    return FDW_OK;
}

fdw_status run_chunk(fdw_solver* c, unsigned long long L, bool check, bool record) {
    NvtxRange nv(check ? "fdw chunk + health" : "fdw chunk");
    const int cur0 = c->cur;
    const bool first_virt = virtual_step(c, c->gstate[cur0]);
    const bool rest_virt = virtual_step(c, 0);
    if (L < 8 || c->prof || c->variant == FDW_KERNEL_FUSED2D || c->group) {
        fdw_status s = enqueue_chunk(c, L, cur0, check, record, first_virt, rest_virt);
        if (s) return s;
    } else {
        const auto key = std::make_tuple(L, cur0 | (first_virt ? 2 : 0), (int)check, (int)record);
        auto it = c->graphs.find(key);
        if (it == c->graphs.end()) {
            cudaGraph_t g;
            CU(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
            c->capturing = true;
            c->capture_kernels = 0;
            fdw_status s = enqueue_chunk(c, L, cur0, check, record, first_virt, rest_virt);
            c->capturing = false;
            cudaError_t e = cudaStreamEndCapture(c->stream, &g);
            if (s) return s;
            if (e != cudaSuccess) return fail(c, FDW_ECUDA, "graph capture failed: %s", cudaGetErrorString(e));
            cudaGraphExec_t ge;
            CU(cudaGraphInstantiate(&ge, g, 0));
            cudaGraphDestroy(g);
            it = c->graphs.emplace(key, ge).first;
            c->graph_kernels[key] = c->capture_kernels;
        }
        CU(cudaGraphLaunch(it->second, c->stream));
        c->launches += c->graph_kernels[key];
    }
    // ghost state of the levels written by this chunk
    for (unsigned long long k = 0; k < L && k < 2; ++k) {
        const unsigned long long kk = L - 1 - k;  // last two steps
        const int dst = 1 - (cur0 ^ (int)(kk & 1));
        c->gstate[dst] = (kk == 0 ? first_virt : rest_virt) ? 1 : 0;
    }
    c->cur = cur0 ^ (int)(L & 1);
    c->host_step += L;
    return FDW_OK;
}

template <typename T>
fdw_status density_grad_t(fdw_solver* c, const T* rho) {
    // extended points of the local slab; per-axis strides of the device layout
    const long long nz = c->nzl, nx = c->nxl, ny = c->ndim == 3 ? c->nyl : 1;
    const long long stride[3] = {c->ndim == 3 ? c->plane : c->ld, c->ndim == 3 ? c->ld : 1, 1};
    const long long n = nz * nx * ny;
    double w[10] = {0};
    for (int j = 0; j < c->R; ++j) w[j] = c->d.coeffs1[j];
    const int tb = 256;
    for (int ax = 0; ax < c->ndim; ++ax) {
        fdw::density_grad_kernel<T><<<(unsigned)((n + tb - 1) / tb), tb, 0, c->stream>>>(
            rho, static_cast<T*>(c->grad[ax]), c->origin, stride[1], stride[0], (int)nz, (int)nx, (int)ny,
            stride[ax], c->R, w[0], w[1], w[2], w[3], w[4], w[5], w[6], w[7], w[8], w[9],
            1.0 / (2.0 * c->d.spacing[ax]));
        CHECK_LAUNCH();
    }
    return FDW_OK;
}

// Materialises the stored ghost cells of a level whose ghosts are virtual.
fdw_status settle_ghosts(fdw_solver* c, int lv) {
    if (c->gstate[lv] != 1) return FDW_OK;
    fdw_status s = launch_boundary(c, lv, 0);
    if (s) return s;
    c->gstate[lv] = 0;
    return FDW_OK;
}

fdw_status read_ctrl(fdw_solver* c) {
    CU(cudaMemcpyAsync(c->h_ctrl, c->ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    return FDW_OK;
}

// Picks the Z-segment count for the Z-march kernel: fill whole waves of
// resident CTAs while keeping the 2R-plane queue warm-up small.
int pick_zseg(fdw_solver* c, int occ) {
    // Thin slabs (strong scaling): 3 segments measured best at 27, 54 and 109
    // planes of C4 (middle ranks with emulated neighbours, split-ring sweep:
    // 93 / 149 / 261 us against 103 / 159 / 267 us for this model's pick,
    // tools/strong_probe.py, profiles/r02/strong_probe.json).
    if (c->nzl <= 128) return (int)std::max<long long>(1, std::min<long long>(3, c->nzl / c->R));
    // Cost model in units of plane-steps of one CTA, fitted on B200 (C4 and C3
    // sweeps over 4..14 segments): a segment of n planes costs n + 0.2*2R
    // (queue warm-up); the grid drains at `resident` CTAs; half a CTA of tail
    // plus half of the idle share of the last partial wave.
    const long long ty = (c->nyl + (64 / (c->tsize / 4)) - 1) / (64 / (c->tsize / 4));
    const long long tx = (c->nxl + 15) / 16;
    const double tiles = (double)(ty * tx);
    const double resident = (double)c->sm_count * occ;
    const double warm = 0.2 * 2.0 * c->R;
    double best = 0.0;
    int best_s = 1;
    for (int s = 1; s <= 16; ++s) {
        if (c->nzl / s < 4 * c->R) break;
        const double dur = (double)c->nzl / s + warm;
        const double waves = tiles * s / resident;
        const double t = tiles * s * dur / resident + 0.5 * dur + 0.5 * dur * (std::ceil(waves) - waves);
        if (s == 1 || t < best - 1e-9) {
            best = t;
            best_s = s;
        }
    }
    return best_s;
}

// Dense box (nz x nx x ny) <-> pitched device layout, on the device.
fdw_status launch_box_copy(fdw_solver* c, void* dst, long long d_plane, long long d_row, const void* src,
                           long long s_plane, long long s_row, long long nz, long long nx, long long ny) {
    const long long n = nz * nx * ny;
    if (n <= 0) return FDW_OK;
    const int tb = 256;
    const unsigned grid = (unsigned)std::min<long long>((n + tb - 1) / tb, (long long)c->sm_count * 16);
    if (c->tsize == 4)
        fdw::box_copy<float><<<grid, tb, 0, c->stream>>>(static_cast<float*>(dst), d_plane, d_row,
                                                         static_cast<const float*>(src), s_plane, s_row, (int)nz,
                                                         (int)nx, (int)ny);
    else
        fdw::box_copy<double><<<grid, tb, 0, c->stream>>>(static_cast<double*>(dst), d_plane, d_row,
                                                          static_cast<const double*>(src), s_plane, s_row, (int)nz,
                                                          (int)nx, (int)ny);
    CHECK_LAUNCH();
    return FDW_OK;
}

// Padded box of the local slab in the caller's dense layout: planes, rows, cols
void padded_box(const fdw_solver* c, long long& nz, long long& nx, long long& ny) {
    if (c->ndim == 3) {
        nz = c->Lz, nx = c->P[1], ny = c->P[2];
    } else {
        nz = 1, nx = c->P[0], ny = c->P[1];
    }
}

// Host (or device) dense padded array -> pitched level.  A host source goes
// through ONE contiguous H2D copy into pool memory and is scattered on the
// device (row-pitched cudaMemcpy2D from host runs at ~half the PCIe rate).
fdw_status copy_host_to_level(fdw_solver* c, void* dst, const void* src, int on_device) {
    long long nz, nx, ny;
    padded_box(c, nz, nx, ny);
    const size_t bytes = (size_t)(nz * nx * ny) * c->tsize;
    const void* from = src;
    void* tmp = nullptr;
    if (!on_device) {
        CU(cudaMallocAsync(&tmp, bytes, c->stream));
        CU(cudaMemcpyAsync(tmp, src, bytes, cudaMemcpyHostToDevice, c->stream));
        from = tmp;
    }
    fdw_status s = launch_box_copy(c, static_cast<char*>(dst) + (size_t)c->base * c->tsize, c->plane, c->ld, from,
                                   nx * ny, ny, nz, nx, ny);
    if (tmp) cudaFreeAsync(tmp, c->stream);
    return s;
}

// Pitched level -> host dense padded array (one contiguous D2H copy).
fdw_status copy_level_to_host(fdw_solver* c, void* dst, const void* src) {
    long long nz, nx, ny;
    padded_box(c, nz, nx, ny);
    const size_t bytes = (size_t)(nz * nx * ny) * c->tsize;
    void* tmp = nullptr;
    CU(cudaMallocAsync(&tmp, bytes, c->stream));
    fdw_status s = launch_box_copy(c, tmp, nx * ny, ny, static_cast<const char*>(src) + (size_t)c->base * c->tsize,
                                   c->plane, c->ld, nz, nx, ny);
    if (!s) CU(cudaMemcpyAsync(dst, tmp, bytes, cudaMemcpyDeviceToHost, c->stream));
    cudaFreeAsync(tmp, c->stream);
    return s;
}

// Global padded flat index -> device element offset (-1: not on this rank).
long long remap(const fdw_solver* c, unsigned long long flat) {
    if (c->ndim == 3) {
        const unsigned long long P12 = (unsigned long long)c->P[1] * c->P[2];
        const unsigned long long gp = flat / P12, rem = flat % P12;
        if (gp >= (unsigned long long)c->P[0]) return -1;
        const long long z = (long long)gp - c->R;  // extended Z (may be a ghost)
        const long long zb = (long long)c->d.z_begin, ze = (long long)c->d.z_end;
        const bool first = c->d.rank == 0, last = c->d.rank == c->d.world - 1;
        const bool owned = (z >= zb && z < ze) || (first && z < 0) || (last && z >= ze);
        if (!owned) return -1;
        const long long lp = (long long)gp - zb;
        return c->base + lp * c->plane + (long long)(rem / c->P[2]) * c->ld + (long long)(rem % c->P[2]);
    }
    const unsigned long long P1 = (unsigned long long)c->P[1];
    if (flat >= (unsigned long long)c->P[0] * P1) return -1;
    return c->base + (long long)(flat / P1) * c->ld + (long long)(flat % P1);
}

// Taps that apply_boundary (kernel.hpp:67-102) overwrites in the same step
// have no effect on the reference's result and are dropped: ghost cells, and
// points of a null-Dirichlet face (kernel.hpp:87-88).
bool dropped_target(const fdw_solver* c, unsigned long long flat) {
    long long p[3] = {0, 0, 0};
    if (c->ndim == 3) {
        const unsigned long long P12 = (unsigned long long)c->P[1] * c->P[2];
        p[0] = (long long)(flat / P12);
        p[1] = (long long)((flat % P12) / c->P[2]);
        p[2] = (long long)(flat % c->P[2]);
    } else {
        p[0] = (long long)(flat / c->P[1]);
        p[1] = (long long)(flat % c->P[1]);
    }
    for (int a = 0; a < c->ndim; ++a) {
        const long long e = p[a] - c->R;  // global extended coordinate
        const long long n = (long long)c->d.extended[a];
        if (e < 0 || e >= n) return true;
        if (c->d.bc[a][0] == FDW_BC_NULL_DIRICHLET && e == 0) return true;
        if (c->d.bc[a][1] == FDW_BC_NULL_DIRICHLET && e == n - 1) return true;
    }
    return false;
}


fdw_status prologue(fdw_solver* c) {
    if (!c) return FDW_EINVAL;
    CU(cudaSetDevice(c->d.device));
    return FDW_OK;
}

// Checks the device abort latch after advances (synchronising the stream).
// On an abort, restores the host bookkeeping to the frozen failing step and
// returns FDW_EINSTABLE with instability_error's (step, max_abs).
fdw_status resolve_pending(fdw_solver* c, uint64_t* bad_step, double* bad_max) {
    if (!c->pending) return FDW_OK;
    c->pending = false;
    fdw_status s;
    if ((s = read_ctrl(c))) return s;
    if (!c->h_ctrl->abort) return FDW_OK;
    if (c->h_ctrl->peer_err)
        return fail(c, FDW_EPEER,
                    "peer transport: a rank of the slab decomposition failed or did not signal within 20 s "
                    "(seen by rank %d of %d)",
                    c->d.rank, c->d.world);
    const unsigned long long done = c->h_ctrl->step - c->pend_start;
    c->host_step = c->h_ctrl->step;
    c->cur = c->pend_cur ^ (int)(done & 1);
    // levels written by executed steps: treat their ghosts as virtual
    // (settled from the extended values on download)
    if (c->variant == FDW_KERNEL_TMA) {
        c->gstate[c->cur] = 1;
        if (done >= 2) c->gstate[1 - c->cur] = 1;
    }
    if (bad_step) *bad_step = c->h_ctrl->bad_step;
    if (bad_max)
        *bad_max = c->h_ctrl->kind == 2 ? std::numeric_limits<double>::quiet_NaN()
                                        : std::numeric_limits<double>::infinity();
    const unsigned int zero = 0;
    CU(cudaMemcpyAsync(&c->ctrl->abort, &zero, sizeof(zero), cudaMemcpyHostToDevice, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    if (c->copy_stream) CU(cudaStreamSynchronize(c->copy_stream));
    return fail(c, FDW_EINSTABLE, "non-finite wavefield at step %llu; timestep is likely unstable",
                (unsigned long long)c->h_ctrl->bad_step);
}

// Entry of every call that reads or replaces device state: pending
// asynchronous advances are checked first (an instability surfaces here).
fdw_status enter(fdw_solver* c) {
    fdw_status s = prologue(c);
    if (s) return s;
    if (c->copy_stream) CU(cudaStreamSynchronize(c->copy_stream));
    return resolve_pending(c, nullptr, nullptr);
}

}  // namespace

extern "C" {

void fdw_desc_init(fdw_desc* d) {
    std::memset(d, 0, sizeof(*d));
    d->abi_version = FDW_ABI_VERSION;
    d->ndim = 3;
    d->space_order = 8;
    d->dtype_bytes = 4;
    for (int a = 0; a < 3; ++a) {
        d->extended[a] = 1;
        d->spacing[a] = 1.0;
        d->bc[a][0] = d->bc[a][1] = FDW_BC_NONE;
    }
    d->check_interval = 100;
    d->world = 1;
    d->variant = FDW_KERNEL_AUTO;
    d->math = FDW_MATH_EXACT;
}

const char* fdw_status_string(fdw_status s) {
    switch (s) {
        case FDW_OK: return "ok";
        case FDW_EINVAL: return "invalid argument";
        case FDW_ECUDA: return "CUDA error";
        case FDW_EPEER: return "peer transport error";
        case FDW_EINSTABLE: return "non-finite wavefield";
        case FDW_ENOMEM: return "out of memory";
        case FDW_ESTATE: return "invalid call order";
    }
    return "unknown";
}

const char* fdw_last_error(const fdw_solver* c) { return c ? c->err.c_str() : g_create_error.c_str(); }

fdw_status fdw_slab_range(uint64_t n_ext, int32_t world, int32_t rank, uint64_t* zb, uint64_t* ze) {
    if (world < 1 || rank < 0 || rank >= world || n_ext < (uint64_t)world) return FDW_EINVAL;
    // balanced split, floor(n*r/w) boundaries (217 over 8 -> 27 x7, then 28)
    *zb = n_ext * (uint64_t)rank / (uint64_t)world;
    *ze = n_ext * (uint64_t)(rank + 1) / (uint64_t)world;
    return FDW_OK;
}

int32_t fdw_owner_of(uint64_t flat, const uint64_t ext[3], int32_t halo, int32_t world) {
    const uint64_t P1 = ext[1] + 2 * (uint64_t)halo, P2 = ext[2] + 2 * (uint64_t)halo;
    const long long z = (long long)(flat / (P1 * P2)) - halo;
    if (z < 0 || z >= (long long)ext[0]) return -1;
    for (int32_t r = 0; r < world; ++r) {
        uint64_t b, e;
        if (fdw_slab_range(ext[0], world, r, &b, &e) == FDW_OK && (uint64_t)z >= b && (uint64_t)z < e) return r;
    }
    return -1;
}

namespace {
struct PeerBlob {
    uint32_t magic;
    int32_t rank, world, tsize, R, device;
    int64_t ld, plane, nzl, origin, pid;
    cudaIpcMemHandle_t lvl[2];
    cudaIpcMemHandle_t sync;
    char bus[32];  // PCI bus id of the rank's GPU (ordinals differ between processes)
};
static_assert(sizeof(PeerBlob) <= FDW_PEER_BLOB_BYTES, "peer blob size");
constexpr uint32_t PEER_MAGIC = 0x50574446u;  // "FDWP"

// Mapping of the neighbours' levels: neighbour element = local element + delta.
// Lower neighbour: local plane z in [0, R) is its plane nzl_lo + z.  Upper
// neighbour: local plane z in [nzl - R, nzl) is its plane z - nzl.
fdw_status peer_geometry(fdw_solver* c, int s, long long ld, long long plane, long long nzl, long long origin,
                         int tsize, int R) {
    if (ld != c->ld || plane != c->plane || tsize != c->tsize || R != c->R)
        return fail(c, FDW_EINVAL, "peer rank %d: slab layout differs (ld %lld/%lld, plane %lld/%lld)", s, ld,
                    c->ld, plane, c->plane);
    if (nzl < c->R) return fail(c, FDW_EINVAL, "peer rank %d owns fewer than R planes", s);
    if (s == c->d.rank - 1) c->peer_delta[0] = origin + nzl * plane - c->origin;
    if (s == c->d.rank + 1) c->peer_delta[1] = origin - c->nzl * plane - c->origin;
    return FDW_OK;
}
}  // namespace

fdw_status fdw_peer_export(fdw_solver* c, unsigned char out[FDW_PEER_BLOB_BYTES]) {
    fdw_status s = prologue(c);
    if (s) return s;
    if (!out) return fail(c, FDW_EINVAL, "null output");
    if (!c->peer_mode) return fail(c, FDW_EINVAL, "not a peer-transport slab context");
    PeerBlob b{};
    b.magic = PEER_MAGIC;
    b.rank = c->d.rank;
    b.world = c->d.world;
    b.tsize = c->tsize;
    b.R = c->R;
    b.device = c->d.device;
    b.ld = c->ld;
    b.plane = c->plane;
    b.nzl = c->nzl;
    b.origin = c->origin;
    b.pid = (int64_t)getpid();
    CU(cudaDeviceGetPCIBusId(b.bus, (int)sizeof(b.bus), c->d.device));
    for (int l = 0; l < 2; ++l) CU(cudaIpcGetMemHandle(&b.lvl[l], c->lvl[l]));
    CU(cudaIpcGetMemHandle(&b.sync, c->psync));
    std::memset(out, 0, FDW_PEER_BLOB_BYTES);
    std::memcpy(out, &b, sizeof(b));
    return FDW_OK;
}

fdw_status fdw_peer_import(fdw_solver* c, const unsigned char* blobs, int32_t world) {
    fdw_status s = prologue(c);
    if (s) return s;
    if (!c->peer_mode) return fail(c, FDW_EINVAL, "not a peer-transport slab context");
    if (!blobs || world != c->d.world) return fail(c, FDW_EINVAL, "need one blob per rank (%d)", c->d.world);
    if (c->peers_ready) return fail(c, FDW_ESTATE, "peers already imported");
    char bus[32] = {};
    CU(cudaDeviceGetPCIBusId(bus, (int)sizeof(bus), c->d.device));
    for (int r = 0; r < world; ++r) {
        if (r == c->d.rank) continue;
        PeerBlob b;
        std::memcpy(&b, blobs + (size_t)r * FDW_PEER_BLOB_BYTES, sizeof(b));
        if (b.magic != PEER_MAGIC || b.rank != r || b.world != world)
            return fail(c, FDW_EINVAL, "peer blob %d is not rank %d's export", r, r);
        if (b.pid == (int64_t)getpid())
            return fail(c, FDW_EINVAL, "peer rank %d lives in this process: use fdw_peer_link", r);
        if ((s = peer_geometry(c, r, b.ld, b.plane, b.nzl, b.origin, b.tsize, b.R))) return s;
        if (std::strncmp(b.bus, bus, sizeof(bus)) == 0) c->ipc_same_device = true;
        void* p = nullptr;
        CU(cudaIpcOpenMemHandle(&p, b.sync, cudaIpcMemLazyEnablePeerAccess));
        c->ipc_mapped.push_back(p);
        c->peer_sync[r] = static_cast<fdw::PeerSync*>(p);
        const int side = r == c->d.rank - 1 ? 0 : r == c->d.rank + 1 ? 1 : -1;
        if (side >= 0)
            for (int l = 0; l < 2; ++l) {
                CU(cudaIpcOpenMemHandle(&p, b.lvl[l], cudaIpcMemLazyEnablePeerAccess));
                c->ipc_mapped.push_back(p);
                c->peer_lvl[side][l] = p;
            }
    }
    c->peers_ready = true;
    return FDW_OK;
}

fdw_status fdw_peer_link(fdw_solver* c, fdw_solver* const* all, int32_t world) {
    fdw_status s = prologue(c);
    if (s) return s;
    if (!c->peer_mode) return fail(c, FDW_EINVAL, "not a peer-transport slab context");
    if (!all || world != c->d.world) return fail(c, FDW_EINVAL, "need one context per rank (%d)", c->d.world);
    if (c->peers_ready) return fail(c, FDW_ESTATE, "peers already linked");
    for (int r = 0; r < world; ++r) {
        const fdw_solver* o = all[r];
        if (r == c->d.rank) {
            if (o != c) return fail(c, FDW_EINVAL, "all[%d] must be this context", r);
            continue;
        }
        if (!o || !o->peer_mode || o->d.rank != r || o->d.world != world)
            return fail(c, FDW_EINVAL, "all[%d] is not rank %d of this decomposition", r, r);
        if ((s = peer_geometry(c, r, o->ld, o->plane, o->nzl, o->origin, o->tsize, o->R))) return s;
        if (o->d.device != c->d.device) {
            const cudaError_t e = cudaDeviceEnablePeerAccess(o->d.device, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
                return fail(c, FDW_ECUDA, "cudaDeviceEnablePeerAccess(%d): %s", o->d.device, cudaGetErrorString(e));
            cudaGetLastError();
        }
        c->peer_sync[r] = o->psync;
        const int side = r == c->d.rank - 1 ? 0 : r == c->d.rank + 1 ? 1 : -1;
        if (side >= 0)
            for (int l = 0; l < 2; ++l) c->peer_lvl[side][l] = o->lvl[l];
    }
    // ranks sharing a GPU (or FDW_PEER_HOST_ORDER=1): host-ordered group
    bool shared = std::getenv("FDW_PEER_HOST_ORDER") != nullptr;
    for (int r = 0; r < world; ++r)
        for (int q = r + 1; q < world; ++q) shared = shared || all[r]->d.device == all[q]->d.device;
    if (shared) {
        std::lock_guard<std::mutex> lk(g_group_mu);
        HostGroup*& g = g_groups[all[0]];
        if (!g) {
            g = new HostGroup();
            g->world = world;
        }
        const int r = c->d.rank;
        for (int k = 0; k < 2; ++k)
            if (!g->ev[r][k]) CU(cudaEventCreateWithFlags(&g->ev[r][k], cudaEventDisableTiming));
        g->member[r] = c;
        ++g->alive;
        c->group = g;
    }
    c->peers_ready = true;
    return FDW_OK;
}

fdw_status fdw_debug_check_guards(fdw_solver* c, uint64_t* n_bad) {
    fdw_status s = enter(c);
    if (s) return s;
    if (!n_bad) return fail(c, FDW_EINVAL, "null output");
    if (!c->guard_bytes) return fail(c, FDW_ESTATE, "guards are off: create the context with FDW_GUARD_CHECK=1");
    CU(cudaStreamSynchronize(c->side));
    unsigned long long* d_bad = nullptr;
    CU(cudaMallocAsync(reinterpret_cast<void**>(&d_bad), sizeof(*d_bad), c->stream));
    CU(cudaMemsetAsync(d_bad, 0, sizeof(*d_bad), c->stream));
    const size_t body = c->level_elems * c->tsize;
    const long long nrows = c->ndim == 3 ? c->P[1] : c->P[0];
    const long long ncols = c->ndim == 3 ? c->P[2] : c->P[1];
    const long long nplanes = c->ndim == 3 ? c->Lz : 1;
    int k = 0;
    for (void* p : {c->lvl[0], c->lvl[1], c->c2dt2, c->eta}) {
        const int slack = k++ < 2;  // levels: nothing may land outside the padded box
        fdw::guard_scan<<<c->sm_count * 4, 256, 0, c->stream>>>(
            static_cast<const unsigned int*>(p), (body + c->guard_bytes) / 4, body / 4, slack, c->ld, c->plane,
            c->base, nrows, ncols, nplanes, c->tsize, d_bad);
        CHECK_LAUNCH();
    }
    unsigned long long h = 0;
    CU(cudaMemcpyAsync(&h, d_bad, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    CU(cudaFreeAsync(d_bad, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    *n_bad = h;
    return FDW_OK;
}

fdw_status fdw_peer_loopback(fdw_solver* c) {
    fdw_status s = prologue(c);
    if (s) return s;
    if (!c->peer_mode) return fail(c, FDW_EINVAL, "not a peer-transport slab context");
    if (c->peers_ready) return fail(c, FDW_ESTATE, "peers already linked");
    const size_t bytes = c->level_elems * c->tsize;
    for (int l = 0; l < 2; ++l) CU(cudaMalloc(&c->loop_lvl[l], bytes));
    CU(cudaMalloc(reinterpret_cast<void**>(&c->loop_sync), sizeof(fdw::PeerSync)));
    CU(cudaMemset(c->loop_sync, 0, sizeof(fdw::PeerSync)));
    // the neighbours' epochs and health posts are already far ahead, their
    // inbox values neutral (no non-finite index, max 0, kind 0)
    fdw::PeerSync h{};
    CU(cudaMemcpy(&h, c->psync, sizeof(h), cudaMemcpyDeviceToHost));
    const int r = c->d.rank;
    for (int q = 0; q < c->d.world; ++q) {
        if (q == r) continue;
        h.halo_flag[q] = h.health_flag[q] = 1ull << 62;
        for (int k = 0; k < 2; ++k) {
            h.in_idx[k][q] = ~0ull;
            h.in_max[k][q] = 0ull;
            h.in_kind[k][q] = 0u;
        }
        c->peer_sync[q] = c->loop_sync;  // this rank's posts and publishes land in scratch
    }
    CU(cudaMemcpy(c->psync, &h, sizeof(h), cudaMemcpyHostToDevice));
    for (int side = 0; side < 2; ++side) {
        const bool has = side == 0 ? r > 0 : r < c->d.world - 1;
        for (int l = 0; l < 2; ++l) c->peer_lvl[side][l] = has ? c->loop_lvl[l] : nullptr;
        c->peer_delta[side] = 0;  // halo planes land at the same offsets of the scratch level
    }
    c->loopback = true;
    c->peers_ready = true;
    return FDW_OK;
}

fdw_status fdw_create(const fdw_desc* dp, fdw_solver** out) {
    NvtxRange nv("fdw_create");
    fdw_solver* c = nullptr;
    if (!dp || !out) return fail(nullptr, FDW_EINVAL, "null descriptor");
    const fdw_desc& d = *dp;
    if (d.abi_version != FDW_ABI_VERSION) return fail(nullptr, FDW_EINVAL, "ABI version mismatch");
    if (d.ndim != 2 && d.ndim != 3) return fail(nullptr, FDW_EINVAL, "Field: ndim must be 2 or 3");
    if (d.space_order < 2 || d.space_order > 20 || d.space_order % 2)
        return fail(nullptr, FDW_EINVAL, "spatial order must be even and in [2, 20]");
    if (d.dtype_bytes != 4 && d.dtype_bytes != 8) return fail(nullptr, FDW_EINVAL, "dtype must be 4 or 8 bytes");
    const int R = d.space_order / 2;
    for (int a = 0; a < d.ndim; ++a) {
        if (d.extended[a] < (uint64_t)(2 * R + 2))
            return fail(nullptr, FDW_EINVAL,
                        "extended extent %llu on axis %d is below 2*halo+2 = %d (mirror sources would "
                        "reach the opposite face)",
                        (unsigned long long)d.extended[a], a, 2 * R + 2);
        if (!(d.spacing[a] > 0.0)) return fail(nullptr, FDW_EINVAL, "spacing must be positive");
        for (int s = 0; s < 2; ++s)
            if (d.bc[a][s] < 0 || d.bc[a][s] > 2) return fail(nullptr, FDW_EINVAL, "bad boundary condition");
    }
    if (d.world < 1 || d.rank < 0 || d.rank >= d.world) return fail(nullptr, FDW_EINVAL, "bad rank/world");
    if (d.world > 1 && d.ndim != 3) return fail(nullptr, FDW_EINVAL, "slab decomposition is 3D only");
    if (d.world > 1) {
        if (!(d.z_end > d.z_begin) || d.z_end > d.extended[0] || d.z_end - d.z_begin < (uint64_t)(2 * R))
            return fail(nullptr, FDW_EINVAL, "slab [%llu, %llu) must own >= %d of %llu planes",
                        (unsigned long long)d.z_begin, (unsigned long long)d.z_end, 2 * R,
                        (unsigned long long)d.extended[0]);
    }
    if (d.extended[0] > (1u << 30) || d.extended[1] > (1u << 30) || d.extended[2] > (1u << 30))
        return fail(nullptr, FDW_EINVAL, "extent too large");

    c = new fdw_solver();
    c->d = d;
    if (c->d.check_interval == 0) c->d.check_interval = 100;
    if (c->d.world <= 1) {
        c->d.world = 1;
        c->d.rank = 0;
        c->d.z_begin = 0;
        c->d.z_end = d.ndim == 3 ? d.extended[0] : d.extended[0];
    }
    c->ndim = d.ndim;
    c->R = R;
    c->tsize = d.dtype_bytes;
    for (int a = 0; a < 3; ++a) c->P[a] = (long long)d.extended[a] + (a < d.ndim ? 2 * R : 0);
    if (d.ndim == 2) c->P[2] = 1;

    const long long EW = 128 / c->tsize;  // elements per 128 bytes
    const long long slack_cols = 64 + 16, slack_rows = 64;
    if (c->ndim == 3) {
        c->nzl = (long long)(c->d.z_end - c->d.z_begin);
        c->nxl = (long long)d.extended[1];
        c->nyl = (long long)d.extended[2];
        c->Lz = c->nzl + 2 * R;
        c->base = (long long)align_up(R, EW) - R;
        c->ld = (long long)align_up(c->base + c->P[2] + slack_cols, EW);
        c->rows_alloc = c->P[1] + slack_rows;
        c->plane = c->rows_alloc * c->ld;
        c->origin_pad = c->base;
        c->origin = c->base + (long long)R * c->plane + (long long)R * c->ld + R;
        c->level_elems = (size_t)(c->Lz + 1) * c->plane;
    } else {
        c->nzl = (long long)d.extended[0];
        c->nxl = (long long)d.extended[1];
        c->nyl = 1;
        c->Lz = 1;
        c->base = (long long)align_up(R, EW) - R;
        c->ld = (long long)align_up(c->base + c->P[1] + slack_cols, EW);
        c->rows_alloc = c->P[0] + slack_rows;
        c->plane = c->rows_alloc * c->ld;
        c->origin_pad = c->base;
        c->origin = c->base + (long long)R * c->ld + R;
        c->level_elems = (size_t)c->plane;
    }

    auto bail = [&](fdw_status s) {
        g_create_error = c->err;
        fdw_destroy(c);
        return s;
    };
    PhaseTimer pt("fdw_create");
    {
        cudaError_t e = cudaSetDevice(d.device);
        if (e != cudaSuccess) {
            fail(c, FDW_ECUDA, "cudaSetDevice(%d): %s", d.device, cudaGetErrorString(e));
            return bail(FDW_ECUDA);
        }
        // attribute queries, not cudaGetDeviceProperties (which is slow)
        int major = 0, minor = 0, sms = 0;
        cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, d.device);
        cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, d.device);
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d.device) == cudaSuccess && sms > 0)
            c->sm_count = sms;
        if (major < 10) {
            fail(c, FDW_ECUDA, "device %d is sm_%d%d; this library is built for sm_100a", d.device, major, minor);
            return bail(FDW_ECUDA);
        }
    }
    auto ck = [&](cudaError_t e, const char* what) -> bool {
        if (e == cudaSuccess) return true;
        fail(c, e == cudaErrorMemoryAllocation ? FDW_ENOMEM : FDW_ECUDA, "%s: %s", what, cudaGetErrorString(e));
        return false;
    };
    pt.lap("device");
    if (!ck(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "stream")) return bail(FDW_ECUDA);
    c->own_stream = true;
    if (!ck(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking), "side stream")) return bail(FDW_ECUDA);
    for (int k = 0; k < 2; ++k) {
        if (!ck(cudaEventCreateWithFlags(&c->fork_ev[k], cudaEventDisableTiming), "event")) return bail(FDW_ECUDA);
        if (!ck(cudaEventCreateWithFlags(&c->rec_ev[k], cudaEventDisableTiming), "event")) return bail(FDW_ECUDA);
    }
    pt.lap("stream");
    // The four field arrays come from the device's stream-ordered pool with an
    // unlimited release threshold: a process that builds one Solver after
    // another (the reference's one-run-per-Solver usage) reuses the
    // same physical pages instead of paying cudaMalloc/cudaFree each time.
    const size_t bytes = c->level_elems * c->tsize;
    {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, d.device) == cudaSuccess) {
            unsigned long long thr = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    }
    c->peer_mode = c->ndim == 3 && d.world > 1;
    c->no_pdl = std::getenv("FDW_NO_PDL") != nullptr;
    c->dbg_no_rot = std::getenv("FDW_DBG_NO_SEGROT") != nullptr;
    c->dbg_no_store = std::getenv("FDW_DBG_NO_HALO_STORE") != nullptr;
    c->dbg_fence_all = std::getenv("FDW_DBG_FENCE_ALL") != nullptr;
    c->dbg_fence_sc = std::getenv("FDW_DBG_FENCE_SC") != nullptr;
    if (!std::getenv("FDW_NO_PRIO")) {
        int lo = 0, hi = 0;
        if (cudaDeviceGetStreamPriorityRange(&lo, &hi) == cudaSuccess) {
            c->prio_lo = lo;
            c->prio_hi = hi;
        }
        cudaGetLastError();
    }
    c->guard_bytes = std::getenv("FDW_GUARD_CHECK") ? fdw_solver::GUARD : 0;
    for (void** p : {&c->lvl[0], &c->lvl[1], &c->c2dt2, &c->eta}) {
        // peer transport: the levels are mapped by the neighbours (cudaIpc
        // needs cudaMalloc memory, not the stream-ordered pool)
        const bool ipc = c->peer_mode && (p == &c->lvl[0] || p == &c->lvl[1]);
        const size_t nb = bytes + c->guard_bytes;
        if (!ck(ipc ? cudaMalloc(p, nb) : cudaMallocAsync(p, nb, c->stream), "cudaMalloc(level)"))
            return bail(FDW_ENOMEM);
        if (!ck(cudaMemsetAsync(*p, 0, bytes, c->stream), "memset")) return bail(FDW_ECUDA);
        if (c->guard_bytes &&
            !ck(cudaMemsetAsync(static_cast<char*>(*p) + bytes, 0xA5, c->guard_bytes, c->stream), "memset"))
            return bail(FDW_ECUDA);
    }
    if (c->peer_mode) {
        if (d.world > fdw::PEER_MAX_WORLD) {
            fail(c, FDW_EINVAL, "peer transport supports at most %d ranks", fdw::PEER_MAX_WORLD);
            return bail(FDW_EINVAL);
        }
        if (!ck(cudaMalloc(reinterpret_cast<void**>(&c->psync), sizeof(fdw::PeerSync)), "cudaMalloc(sync)"))
            return bail(FDW_ENOMEM);
        if (!ck(cudaMemsetAsync(c->psync, 0, sizeof(fdw::PeerSync), c->stream), "memset")) return bail(FDW_ECUDA);
        c->peer_sync[d.rank] = c->psync;
    }
    if (!ck(cudaMallocAsync(reinterpret_cast<void**>(&c->ctrl), sizeof(Ctrl), c->stream), "cudaMallocAsync(ctrl)"))
        return bail(FDW_ENOMEM);
    if (!ck(cudaMemsetAsync(c->ctrl, 0, sizeof(Ctrl), c->stream), "memset")) return bail(FDW_ECUDA);
    if (!(c->h_ctrl = pinned_ctrl_get())) {
        fail(c, FDW_ENOMEM, "cudaMallocHost(ctrl) failed");
        return bail(FDW_ENOMEM);
    }
    pt.lap("alloc");

    // kernel selection
    int variant = d.variant;
    if (variant == FDW_KERNEL_AUTO)
        variant = c->ndim == 2 ? FDW_KERNEL_FUSED2D
                               : (zmarch_supported(R) ? FDW_KERNEL_TMA : FDW_KERNEL_SIMPLE);
    if (variant == FDW_KERNEL_FUSED2D && c->ndim != 2) variant = FDW_KERNEL_SIMPLE;
    if (variant == FDW_KERNEL_FUSED2D) {
        const bool ex = d.math == FDW_MATH_EXACT;
        const void* f = c->tsize == 4 ? fused2d_kernel<float>(R, ex) : fused2d_kernel<double>(R, ex);
        int occ = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, f, 256, 0) != cudaSuccess || occ < 1) occ = 1;
        const long long need = (c->nzl * c->nxl + 255) / 256;
        c->fused_grid = (int)std::max<long long>(1, std::min<long long>(need, (long long)occ * c->sm_count));
        c->occupancy = occ;
        const size_t n = (size_t)(c->nzl * c->nxl) * sizeof(int);
        if (!ck(cudaMallocAsync(reinterpret_cast<void**>(&c->d_tmap), n, c->stream), "cudaMallocAsync(tmap)"))
            return bail(FDW_ENOMEM);
        if (!ck(cudaMemsetAsync(c->d_tmap, 0, n, c->stream), "memset(tmap)")) return bail(FDW_ECUDA);
        if (c->tsize == 4 ? res2d_configure<float>(c) : res2d_configure<double>(c)) {
            std::vector<long long> none;
            fdw_status rs = res2d_sources(c);
            if (!rs) rs = res2d_receivers(c, none);
            if (rs) return bail(rs);
        }
    }
    if ((variant == FDW_KERNEL_ZMARCH || variant == FDW_KERNEL_TMA) && (c->ndim != 3 || !zmarch_supported(R)))
        variant = FDW_KERNEL_SIMPLE;
    if (variant == FDW_KERNEL_TMA) {
        const bool ok = c->tsize == 4 ? make_maps_t<float>(c) : make_maps_t<double>(c);
        if (!ok) {
            fail(c, FDW_ECUDA, "cuTensorMapEncodeTiled failed (TMA descriptors)");
            return bail(FDW_ECUDA);
        }
    }
    c->variant = variant;
    pt.lap("variant");
    if (variant == FDW_KERNEL_ZMARCH || variant == FDW_KERNEL_TMA) {
        const bool ex = d.math == FDW_MATH_EXACT;
        int occ = 1;
        if (variant == FDW_KERNEL_ZMARCH) {
            occ = c->tsize == 4 ? zmarch_occupancy<float>(R, ex) : zmarch_occupancy<double>(R, ex);
        } else {
            // prefer 3 CTAs/SM (80-register cap) unless that build spills
            const char* env = std::getenv("FDW_TMA_MINB");
            int minb = env ? std::atoi(env) : 0;
            if (minb != 2 && minb != 3) {
                cudaFuncAttributes fa{};
                const void* f3 = c->tsize == 4 ? tma_kernel<float>(R, ex, 3) : tma_kernel<double>(R, ex, 3);
                // a few spilled bytes (FMA build) cost less than a third CTA per SM
                // buys (C4 FMA: 0.508 ms at 3 CTAs with 8 B of stack vs 0.578 at 2)
                minb = (cudaFuncGetAttributes(&fa, f3) == cudaSuccess && fa.localSizeBytes <= 8) ? 3 : 2;
            }
            c->tma_minb = minb;
            // split rings (2 planes in flight at 3 CTAs/SM): the default;
            // FDW_TMA_PD=0 restores the single ring (developed C4 field, same box:
            // sweep 528.6 -> 517.8 us, step 518.4 -> 516.7 us, profiles/r02/ab_pd.json;
            // fp64 C4 from rest: 1.043 -> 1.024 ms/step, 72 KB at 3 CTAs/SM)
            const char* pde = std::getenv("FDW_TMA_PD");
            const bool split = pde ? std::atoi(pde) > 0 : true;
            c->tma_pd = (split && minb == 3) ? TMA_PD : 0;
            const void* f = c->tsize == 4 ? tma_kernel<float>(R, ex, minb, c->tma_pd)
                                          : tma_kernel<double>(R, ex, minb, c->tma_pd);
            const int smem = c->tsize == 4 ? tma_smem<float>(R, false, c->tma_pd)
                                           : tma_smem<double>(R, false, c->tma_pd);
            if (!ck(raise_smem_limit(f, smem), "smem attr"))
                return bail(FDW_ECUDA);
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, f, 16 * TMA_BX, smem) != cudaSuccess || occ < 1)
                occ = 1;
        }
        c->occupancy = occ;
        c->zseg = d.z_segments > 0 ? d.z_segments : pick_zseg(c, occ);
        if (c->zseg > c->nzl) c->zseg = (int)c->nzl;
    }

    pt.lap("kernel_setup");
    if (!ck(cudaStreamSynchronize(c->stream), "sync")) return bail(FDW_ECUDA);
    pt.lap("sync");
    *out = c;
    return FDW_OK;
}

fdw_status fdw_destroy(fdw_solver* c) {
    NvtxRange nv("fdw_destroy");
    if (!c) return FDW_OK;
    PhaseTimer pt("fdw_destroy");
    auto lap = [&](const char* w) { pt.lap(w); };
    cudaSetDevice(c->d.device);
    if (c->copy_stream) cudaStreamSynchronize(c->copy_stream);
    if (c->stream) cudaStreamSynchronize(c->stream);
    lap("sync");
    for (int k = 0; k < fdw_solver::SNAP_SLOTS; ++k) {
        if (c->snap_dev[k]) cudaFreeAsync(c->snap_dev[k], c->stream);
        if (c->snap_host[k]) cudaFreeHost(c->snap_host[k]);
        if (c->snap_packed[k]) cudaEventDestroy(c->snap_packed[k]);
        if (c->snap_free[k]) cudaEventDestroy(c->snap_free[k]);
    }
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
    if (c->side) cudaStreamSynchronize(c->side);
    for (int k = 0; k < 2; ++k) {
        if (c->fork_ev[k]) cudaEventDestroy(c->fork_ev[k]);
        if (c->rec_ev[k]) cudaEventDestroy(c->rec_ev[k]);
    }
    if (c->side) cudaStreamDestroy(c->side);
    for (auto& kv : c->graphs) cudaGraphExecDestroy(kv.second);
    lap("graphs");
    peer_leave(c);
    for (void* p : c->ipc_mapped) cudaIpcCloseMemHandle(p);
    for (void* p : {c->loop_lvl[0], c->loop_lvl[1], (void*)c->loop_sync})
        if (p) cudaFree(p);
    if (c->peer_mode) {
        if (c->stream) cudaStreamSynchronize(c->stream);
        for (void* p : {c->lvl[0], c->lvl[1], (void*)c->psync})
            if (p) cudaFree(p);
        c->lvl[0] = c->lvl[1] = nullptr;
    }
    for (void* p : {c->lvl[0], c->lvl[1], c->c2dt2, c->eta, c->grad[0], c->grad[1], c->grad[2]})
        if (p) cudaFreeAsync(p, c->stream);
    for (void* p : c->vs_fields) cudaFreeAsync(p, c->stream);
    for (void* p : {c->d_vs_ptrs, c->d_vs_amp, (void*)c->d_vs_len})
        if (p) cudaFreeAsync(p, c->stream);
    for (void* p : {(void*)c->d_blk_toff, (void*)c->d_blk_tgt, (void*)c->d_blk_tpos, (void*)c->d_blk_roff,
                    (void*)c->d_blk_rpack, (void*)c->d_tap_ix, c->d_tapbuf})
        if (p) cudaFreeAsync(p, c->stream);
    if (c->d_res_hbuf) cudaFreeAsync(c->d_res_hbuf, c->stream);
    for (void* p : {(void*)c->d_sp_idx, (void*)c->d_sp_w, (void*)c->d_sp_prod})
        if (p) cudaFreeAsync(p, c->stream);
    for (void* p : {(void*)c->d_eidx, (void*)c->d_etab})
        if (p) cudaFreeAsync(p, c->stream);
    for (void* p : {(void*)c->d_ezr, (void*)c->ctrl, (void*)c->d_tgt, (void*)c->d_ent_off, (void*)c->d_ent_w, (void*)c->d_wavelet,
                    (void*)c->d_rec_idx, (void*)c->d_rec_off, (void*)c->d_rec_w, (void*)c->d_seis, (void*)c->d_tmap})
        if (p) cudaFreeAsync(p, c->stream);
    if (c->stream) cudaStreamSynchronize(c->stream);
    lap("free_async");
    if (c->h_ctrl) pinned_ctrl_put(c->h_ctrl);
    if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
    delete c;
    return FDW_OK;
}

fdw_status fdw_set_stream(fdw_solver* c, void* stream) {
    fdw_status s = enter(c);
    if (s) return s;
    CU(cudaStreamSynchronize(c->stream));
    for (auto& kv : c->graphs) cudaGraphExecDestroy(kv.second);
    c->graphs.clear();
    if (c->own_stream) cudaStreamDestroy(c->stream);
    if (stream) {
        c->stream = static_cast<cudaStream_t>(stream);
        c->own_stream = false;
    } else {
        CU(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        c->own_stream = true;
    }
    return FDW_OK;
}

// The damping table of the split-ring fp32 sweep (fdw_kernels.cuh eta_collect):
// distinct non-zero eta values on the device, indexed on the host in value
// order, (1 - eta dt, 1/(1 + eta dt)) formed in double exactly as
// kernel.hpp:284-287, then a 1-byte index per point.  More than 255 distinct
// values: no table (the sweep streams fp32 eta as before).
extern "C++" {
template <typename T>
fdw_status build_eta_table_t(fdw_solver* c) {
    using K = std::conditional_t<sizeof(T) == 4, unsigned, unsigned long long>;
    using T2 = typename fdw::EtabPair<T>::type;
    const K EMPTY = ~K(0);
    const unsigned long long n = c->level_elems;
    K* keys = nullptr;
    unsigned* overflow = nullptr;
    CU(cudaMallocAsync(reinterpret_cast<void**>(&keys), fdw::ETAB_CAP * sizeof(K) + sizeof(unsigned), c->stream));
    overflow = reinterpret_cast<unsigned*>(keys + fdw::ETAB_CAP);
    CU(cudaMemsetAsync(keys, 0xFF, fdw::ETAB_CAP * sizeof(K), c->stream));
    CU(cudaMemsetAsync(overflow, 0, sizeof(unsigned), c->stream));
    fdw::eta_collect<T><<<c->sm_count * 8, 256, 0, c->stream>>>(static_cast<const T*>(c->eta), n, keys, overflow);
    CHECK_LAUNCH();
    std::vector<K> h(fdw::ETAB_CAP);
    unsigned ovf = 0;
    CU(cudaMemcpyAsync(h.data(), keys, h.size() * sizeof(K), cudaMemcpyDeviceToHost, c->stream));
    CU(cudaMemcpyAsync(&ovf, overflow, sizeof(unsigned), cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    std::vector<T> vals;
    for (int k = 0; k < fdw::ETAB_CAP; ++k)
        if (h[k] != EMPTY) {
            T f;
            std::memcpy(&f, &h[k], sizeof(T));
            vals.push_back(f);
        }
    if (ovf || vals.size() > 255) {
        cudaFreeAsync(keys, c->stream);
        return FDW_OK;
    }
    std::sort(vals.begin(), vals.end());
    std::vector<T2> tab(256);
    tab[0].x = T(1);
    tab[0].y = T(1);
    std::vector<unsigned char> slot(fdw::ETAB_CAP, 0);
    for (size_t i = 0; i < vals.size(); ++i) {
        volatile double edt = static_cast<double>(vals[i]) * c->d.dt;  // no contraction: as damping_factors
        const double e = edt;
        tab[i + 1].x = static_cast<T>(1.0 - e);
        tab[i + 1].y = static_cast<T>(1.0 / (1.0 + e));
        K bits;
        std::memcpy(&bits, &vals[i], sizeof(T));
        for (int k = 0; k < fdw::ETAB_CAP; ++k)
            if (h[k] == bits) slot[k] = static_cast<unsigned char>(i + 1);
    }
    unsigned char* d_slot = nullptr;
    CU(cudaMallocAsync(reinterpret_cast<void**>(&d_slot), fdw::ETAB_CAP, c->stream));
    CU(cudaMemcpyAsync(d_slot, slot.data(), fdw::ETAB_CAP, cudaMemcpyHostToDevice, c->stream));
    if (!c->d_etab) CU(cudaMallocAsync(&c->d_etab, 256 * sizeof(T2), c->stream));
    CU(cudaMemcpyAsync(c->d_etab, tab.data(), 256 * sizeof(T2), cudaMemcpyHostToDevice, c->stream));
    if (!c->d_eidx) CU(cudaMallocAsync(reinterpret_cast<void**>(&c->d_eidx), n, c->stream));
    fdw::eta_index<T><<<c->sm_count * 8, 256, 0, c->stream>>>(static_cast<const T*>(c->eta), n, keys, d_slot,
                                                               c->d_eidx);
    CHECK_LAUNCH();
    cudaFreeAsync(keys, c->stream);
    cudaFreeAsync(d_slot, c->stream);
    // the index tile has the sweep's tile shape (TYW x BX points), 1 byte each
    if (!make_map(c, &c->tm_eb, c->d_eidx, fdw::TmaShape<T, 1, TMA_BX>::TYW, TMA_BX,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, 1))
        return fail(c, FDW_ECUDA, "cuTensorMapEncodeTiled failed (eta index map)");
    const bool ex = c->d.math == FDW_MATH_EXACT;
    const void* f = tma_kernel<T>(c->R, ex, 3, c->tma_pd, true);
    if (!f) return FDW_OK;
    CU(raise_smem_limit(f, tma_smem<T>(c->R, false, c->tma_pd)));
    c->n_etab = (int)vals.size() + 1;
    return FDW_OK;
}
}  // extern "C++"

static fdw_status build_eta_table(fdw_solver* c) {
    c->n_etab = 0;
    if (std::getenv("FDW_NO_ETAB") || c->variant != FDW_KERNEL_TMA || c->tma_pd == 0) return FDW_OK;
    return c->tsize == 4 ? build_eta_table_t<float>(c) : build_eta_table_t<double>(c);
}

fdw_status fdw_set_medium(fdw_solver* c, const void* velocity, const void* eta, int on_device) {
    NvtxRange nv("fdw_set_medium");
    fdw_status s = enter(c);
    if (s) return s;
    if (!velocity || !eta) return fail(c, FDW_EINVAL, "velocity and eta are required");
    PhaseTimer pt("fdw_set_medium");
    if ((s = copy_host_to_level(c, c->c2dt2, velocity, on_device))) return s;
    if ((s = copy_host_to_level(c, c->eta, eta, on_device))) return s;
    pt.lap("enqueue");
    const unsigned long long n = c->level_elems;
    const int tb = 256;
    if (c->tsize == 4)
        fdw::c2dt2_kernel<float><<<(unsigned)((n + tb - 1) / tb), tb, 0, c->stream>>>(static_cast<float*>(c->c2dt2), n, c->d.dt);
    else
        fdw::c2dt2_kernel<double><<<(unsigned)((n + tb - 1) / tb), tb, 0, c->stream>>>(static_cast<double*>(c->c2dt2), n, c->d.dt);
    CHECK_LAUNCH();
    if (c->variant == FDW_KERNEL_TMA && std::getenv("FDW_NO_ETA_SKIP") == nullptr) {
        // per TMA tile column: the planes whose eta tile is all zero
        const int tyw = c->tsize == 4 ? fdw::TmaShape<float, 1, TMA_BX>::TYW : fdw::TmaShape<double, 1, TMA_BX>::TYW;
        const int ncy = (int)((c->nyl + tyw - 1) / tyw), ncx = (int)((c->nxl + TMA_BX - 1) / TMA_BX);
        const size_t ncol = (size_t)ncy * ncx;
        if (!c->d_ezr) CU(cudaMallocAsync(reinterpret_cast<void**>(&c->d_ezr), ncol * sizeof(int2), c->stream));
        if (c->tsize == 4)
            fdw::eta_zero_ranges<float><<<(unsigned)ncol, 256, (size_t)c->nzl, c->stream>>>(
                static_cast<const float*>(c->eta), c->origin, c->plane, c->ld, (int)c->nzl, (int)c->nxl, (int)c->nyl,
                TMA_BX, tyw, c->d_ezr);
        else
            fdw::eta_zero_ranges<double><<<(unsigned)ncol, 256, (size_t)c->nzl, c->stream>>>(
                static_cast<const double*>(c->eta), c->origin, c->plane, c->ld, (int)c->nzl, (int)c->nxl,
                (int)c->nyl, TMA_BX, tyw, c->d_ezr);
        CHECK_LAUNCH();
    }
    if ((s = build_eta_table(c))) return s;
    for (auto& kv : c->graphs) cudaGraphExecDestroy(kv.second);  // a table may have appeared or gone
    c->graphs.clear();
    CU(cudaStreamSynchronize(c->stream));
    pt.lap("sync");
    c->medium_set = true;
    return FDW_OK;
}

fdw_status fdw_set_density(fdw_solver* c, const void* rho, int on_device) {
    fdw_status s = enter(c);
    if (s) return s;
    if (!rho) return fail(c, FDW_EINVAL, "density is required");
    for (int j = 0; j < c->R; ++j)
        if (!std::isfinite(c->d.coeffs1[j]) || (j == 0 && c->d.coeffs1[0] == 0.0))
            return fail(c, FDW_EINVAL, "desc.coeffs1 (first-derivative weights) must be set for variable density");
    const size_t bytes = c->level_elems * c->tsize;
    void* tmp = nullptr;
    CU(cudaMallocAsync(&tmp, bytes, c->stream));
    CU(cudaMemsetAsync(tmp, 0, bytes, c->stream));
    for (int ax = 0; ax < c->ndim; ++ax)
        if (!c->grad[ax]) {
            CU(cudaMallocAsync(&c->grad[ax], bytes, c->stream));
            CU(cudaMemsetAsync(c->grad[ax], 0, bytes, c->stream));
        }
    if ((s = copy_host_to_level(c, tmp, rho, on_device))) return s;
    s = c->tsize == 4 ? density_grad_t<float>(c, static_cast<const float*>(tmp))
                      : density_grad_t<double>(c, static_cast<const double*>(tmp));
    cudaFreeAsync(tmp, c->stream);
    if (s) return s;
    if (c->variant == FDW_KERNEL_TMA) {
        // the TMA sweep streams the three gradient tiles with the others
        const int pw = c->tsize == 4 ? fdw::TmaShape<float, 1, TMA_BX>::TYW : fdw::TmaShape<double, 1, TMA_BX>::TYW;
        for (int ax = 0; ax < 3; ++ax)
            if (!make_map(c, &c->tm_g[ax], c->grad[ax], pw, TMA_BX))
                return fail(c, FDW_ECUDA, "cuTensorMapEncodeTiled failed (density maps)");
        const bool ex = c->d.math == FDW_MATH_EXACT;
        const bool fast = c->tma_pd > 0 && c->n_etab > 0;  // as launch_tma chooses
        auto vd_fn = [&](bool fst) {
            return c->tsize == 4 ? tma_vd_kernel<float>(c->R, ex, fst) : tma_vd_kernel<double>(c->R, ex, fst);
        };
        auto vd_smem = [&](bool fst) {
            return c->tsize == 4 ? tma_smem<float>(c->R, true, fst ? TMA_PD : 0)
                                 : tma_smem<double>(c->R, true, fst ? TMA_PD : 0);
        };
        const void* f = vd_fn(fast);
        const int smem = vd_smem(fast);
        // both variants stay launchable: a later set_medium may build or drop the table
        CU(raise_smem_limit(vd_fn(false), vd_smem(false)));
        if (c->tma_pd > 0) CU(raise_smem_limit(vd_fn(true), vd_smem(true)));
        int occ = 1;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, f, 16 * TMA_BX, smem) != cudaSuccess || occ < 1)
            occ = 1;
        c->occupancy = occ;
        c->zseg = c->d.z_segments > 0 ? c->d.z_segments : pick_zseg(c, occ);
        if (c->zseg > c->nzl) c->zseg = (int)c->nzl;
    } else if (c->variant == FDW_KERNEL_FUSED2D && c->d.math == FDW_MATH_EXACT) {
        // the cooperative 2D kernel reads the two gradient fields beside
        // c2dt2/eta; its co-resident grid is re-sized for the VD build
        const void* f = c->tsize == 4 ? fused2d_kernel<float>(c->R, true, true) : fused2d_kernel<double>(c->R, true, true);
        int occ = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, f, 256, 0) != cudaSuccess || occ < 1) occ = 1;
        const long long need = (c->nzl * c->nxl + 255) / 256;
        c->fused_grid = (int)std::max<long long>(1, std::min<long long>(need, (long long)occ * c->sm_count));
        c->occupancy = occ;
    } else {
        // the other variants carry the density terms in the stored-ghost
        // element-wise sweep: move virtual-ghost levels to stored ghosts
        if ((s = settle_ghosts(c, 0))) return s;
        if ((s = settle_ghosts(c, 1))) return s;
        c->variant = FDW_KERNEL_SIMPLE;
    }
    c->vd = true;
    for (auto& kv : c->graphs) cudaGraphExecDestroy(kv.second);
    c->graphs.clear();
    CU(cudaStreamSynchronize(c->stream));
    return FDW_OK;
}

fdw_status fdw_add_volume_source(fdw_solver* c, const void* field, const double* amplitude, uint64_t n_amp,
                                 int on_device) {
    fdw_status s = enter(c);
    if (s) return s;
    if (!field || (!amplitude && n_amp)) return fail(c, FDW_EINVAL, "volume source field and amplitude required");
    if (n_amp < c->d.n_steps) return fail(c, FDW_EINVAL, "volume source amplitude shorter than run");
    const size_t bytes = c->level_elems * c->tsize;
    void* f = nullptr;
    CU(cudaMallocAsync(&f, bytes, c->stream));
    CU(cudaMemsetAsync(f, 0, bytes, c->stream));
    if ((s = copy_host_to_level(c, f, field, on_device))) {
        cudaFreeAsync(f, c->stream);
        return s;
    }
    // amplitude table [source][step] of T (the reference casts per step,
    // kernel.hpp:442), rows padded to the longest; per-source lengths gate the add
    auto& amps = c->vs_amps;
    amps.emplace_back(amplitude, amplitude + n_amp);
    c->vs_fields.push_back(f);
    unsigned long long L = 0;
    std::vector<unsigned long long> lens;
    for (auto& a : amps) {
        L = std::max<unsigned long long>(L, a.size());
        lens.push_back(a.size());
    }
    std::vector<unsigned char> tab(amps.size() * L * c->tsize, 0);
    for (size_t q = 0; q < amps.size(); ++q)
        for (unsigned long long j = 0; j < amps[q].size(); ++j) {
            if (c->tsize == 4)
                reinterpret_cast<float*>(tab.data())[q * L + j] = static_cast<float>(amps[q][j]);
            else
                reinterpret_cast<double*>(tab.data())[q * L + j] = amps[q][j];
        }
    CU(cudaStreamSynchronize(c->stream));  // the old tables may still be read by queued work
    for (void* p : {c->d_vs_amp, c->d_vs_ptrs, (void*)c->d_vs_len})
        if (p) cudaFreeAsync(p, c->stream);
    CU(cudaMallocAsync(&c->d_vs_amp, tab.size() ? tab.size() : 1, c->stream));
    if (tab.size()) CU(cudaMemcpyAsync(c->d_vs_amp, tab.data(), tab.size(), cudaMemcpyHostToDevice, c->stream));
    CU(cudaMallocAsync(&c->d_vs_ptrs, c->vs_fields.size() * sizeof(void*), c->stream));
    CU(cudaMemcpyAsync(c->d_vs_ptrs, c->vs_fields.data(), c->vs_fields.size() * sizeof(void*),
                       cudaMemcpyHostToDevice, c->stream));
    CU(cudaMallocAsync(&c->d_vs_len, lens.size() * sizeof(unsigned long long), c->stream));
    CU(cudaMemcpyAsync(c->d_vs_len, lens.data(), lens.size() * sizeof(unsigned long long), cudaMemcpyHostToDevice,
                       c->stream));
    c->vs_namp = L;
    // the cooperative 2D kernel fuses only point sources
    if (c->variant == FDW_KERNEL_FUSED2D) {
        if ((s = settle_ghosts(c, 0))) return s;
        if ((s = settle_ghosts(c, 1))) return s;
        c->variant = FDW_KERNEL_SIMPLE;
    }
    for (auto& kv : c->graphs) cudaGraphExecDestroy(kv.second);
    c->graphs.clear();
    CU(cudaStreamSynchronize(c->stream));
    return FDW_OK;
}

fdw_status fdw_set_sources(fdw_solver* c, uint64_t n_points, const uint64_t* off, const uint64_t* idx,
                           const double* w, const double* wavelet, uint64_t n_samples) {
    fdw_status s = enter(c);
    if (s) return s;
    if (n_points > 0 && n_samples < c->d.n_steps + 1)
        return fail(c, FDW_EINVAL, "wavelet shorter than the time axis");
    // merge entries per target index, keeping the reference's (point, entry) order
    std::unordered_map<long long, int> slot;
    std::vector<long long> tgt;
    std::vector<std::vector<double>> ws;
    for (uint64_t p = 0; p < n_points; ++p)
        for (uint64_t e = off[p]; e < off[p + 1]; ++e) {
            const long long o = remap(c, idx[e]);
            if (o < 0 || dropped_target(c, idx[e])) continue;
            auto it = slot.find(o);
            if (it == slot.end()) {
                it = slot.emplace(o, (int)tgt.size()).first;
                tgt.push_back(o);
                ws.emplace_back();
            }
            ws[it->second].push_back(w[e]);
        }
    std::vector<unsigned int> eo(1, 0);
    std::vector<double> ew;
    for (auto& v : ws) {
        ew.insert(ew.end(), v.begin(), v.end());
        eo.push_back((unsigned int)ew.size());
    }
    c->h_tgt = tgt;
    c->h_tw = ws;
    // a target in the first / last R owned planes is also a neighbour's ghost
    // cell: the point-source kernel mirrors it, and the step publishes after it
    c->mirror_tgt = false;
    if (c->ndim == 3 && c->d.world > 1)
        for (long long o : tgt) {
            const long long z = (o - c->origin) / c->plane;
            if ((c->d.rank > 0 && z < c->R) || (c->d.rank < c->d.world - 1 && z >= c->nzl - c->R))
                c->mirror_tgt = true;
        }
    if ((s = dev_upload(c, &c->d_tgt, tgt))) return s;
    if ((s = dev_upload(c, &c->d_ent_off, eo))) return s;
    if ((s = dev_upload(c, &c->d_ent_w, ew))) return s;
    std::vector<double> wv(wavelet, wavelet + (n_points ? n_samples : 0));
    if ((s = dev_upload(c, &c->d_wavelet, wv))) return s;
    c->n_wavelet = wv.size();
    c->n_tgt = (int)tgt.size();
    if (c->res2d && (s = res2d_sources(c))) return s;
    if (c->d_tmap) {  // FUSED2D: dense map extended point -> target index + 1
        std::vector<int> tm((size_t)(c->nzl * c->nxl), 0);
        for (size_t t = 0; t < tgt.size(); ++t) {
            const long long rem = tgt[t] - c->origin;
            const long long z = rem / c->ld, x = rem % c->ld;
            if (z >= 0 && z < c->nzl && x >= 0 && x < c->nxl) tm[(size_t)(z * c->nxl + x)] = (int)t + 1;
        }
        CU(cudaMemcpyAsync(c->d_tmap, tm.data(), tm.size() * sizeof(int), cudaMemcpyHostToDevice, c->stream));
        CU(cudaStreamSynchronize(c->stream));
    }
    for (auto& kv : c->graphs) cudaGraphExecDestroy(kv.second);
    c->graphs.clear();
    return FDW_OK;
}

fdw_status fdw_set_receivers(fdw_solver* c, uint64_t n_points, const uint64_t* off, const uint64_t* idx,
                             const double* w) {
    fdw_status s = enter(c);
    if (s) return s;
    std::vector<long long> ri, si;
    std::vector<unsigned int> ro(1, 0);
    std::vector<double> rw, sw;
    c->sp_rec.clear();
    c->sp_entry.clear();
    for (uint64_t p = 0; p < n_points; ++p) {
        uint64_t kept = 0;
        for (uint64_t e = off[p]; e < off[p + 1]; ++e) kept += remap(c, idx[e]) >= 0;
        // a receiver with taps on this and another slab: per-tap products
        const bool split = c->d.world > 1 && kept > 0 && kept < off[p + 1] - off[p];
        for (uint64_t e = off[p]; e < off[p + 1]; ++e) {
            const long long o = remap(c, idx[e]);
            if (o < 0) continue;
            if (split) {
                si.push_back(o);
                sw.push_back(w[e]);
                c->sp_rec.push_back(p);
                c->sp_entry.push_back(e - off[p]);
            } else {
                ri.push_back(o);
                rw.push_back(w[e]);
            }
        }
        ro.push_back((unsigned int)ri.size());
    }
    if ((s = dev_upload(c, &c->d_rec_idx, ri))) return s;
    if ((s = dev_upload(c, &c->d_rec_off, ro))) return s;
    if ((s = dev_upload(c, &c->d_rec_w, rw))) return s;
    if ((s = dev_upload(c, &c->d_sp_idx, si))) return s;
    if ((s = dev_upload(c, &c->d_sp_w, sw))) return s;
    c->n_split = (int)si.size();
    if (c->d_sp_prod) cudaFreeAsync(c->d_sp_prod, c->stream);
    c->d_sp_prod = nullptr;
    if (c->n_split) {
        const size_t bytes = (size_t)(c->d.n_steps + 1) * c->n_split * sizeof(double);
        CU(cudaMallocAsync(reinterpret_cast<void**>(&c->d_sp_prod), bytes, c->stream));
        CU(cudaMemsetAsync(c->d_sp_prod, 0, bytes, c->stream));
    }
    if (c->res2d && (s = res2d_receivers(c, ri))) return s;
    if (c->d_seis) cudaFreeAsync(c->d_seis, c->stream);
    c->d_seis = nullptr;
    c->n_rec = (int)n_points;
    c->seis_rows = c->d.n_steps + 1;
    if (n_points) {
        const size_t bytes = (size_t)c->seis_rows * n_points * sizeof(double);
        CU(cudaMallocAsync(reinterpret_cast<void**>(&c->d_seis), bytes, c->stream));
        CU(cudaMemsetAsync(c->d_seis, 0, bytes, c->stream));
        CU(cudaStreamSynchronize(c->stream));
    }
    for (auto& kv : c->graphs) cudaGraphExecDestroy(kv.second);
    c->graphs.clear();
    return FDW_OK;
}

fdw_status fdw_set_levels(fdw_solver* c, const void* prev, const void* curr) {
    NvtxRange nv("fdw_set_levels");
    fdw_status s = enter(c);
    if (s) return s;
    if (prev && (s = copy_host_to_level(c, c->lvl[1 - c->cur], prev, 0))) return s;
    if (curr && (s = copy_host_to_level(c, c->lvl[c->cur], curr, 0))) return s;
    if (prev) c->gstate[1 - c->cur] = 2;
    if (curr) c->gstate[c->cur] = 2;
    CU(cudaStreamSynchronize(c->stream));
    return FDW_OK;
}

fdw_status fdw_zero_levels(fdw_solver* c) {
    fdw_status s = enter(c);
    if (s) return s;
    const size_t bytes = c->level_elems * c->tsize;
    CU(cudaMemsetAsync(c->lvl[0], 0, bytes, c->stream));
    CU(cudaMemsetAsync(c->lvl[1], 0, bytes, c->stream));
    c->gstate[0] = c->gstate[1] = 0;  // all-zero levels satisfy every boundary condition
    return FDW_OK;
}

fdw_status fdw_get_levels(fdw_solver* c, void* prev, void* curr) {
    NvtxRange nv("fdw_get_levels");
    fdw_status s = enter(c);
    if (s) return s;
    if (prev && (s = settle_ghosts(c, 1 - c->cur))) return s;
    if (curr && (s = settle_ghosts(c, c->cur))) return s;
    if (prev && (s = copy_level_to_host(c, prev, c->lvl[1 - c->cur]))) return s;
    if (curr && (s = copy_level_to_host(c, curr, c->lvl[c->cur]))) return s;
    CU(cudaStreamSynchronize(c->stream));
    return FDW_OK;
}

fdw_status fdw_get_extended(fdw_solver* c, void* out) {
    fdw_status s = enter(c);
    if (s) return s;
    const char* src = static_cast<const char*>(c->lvl[c->cur]);
    const long long nz = c->nzl, nx = c->nxl, ny = c->ndim == 3 ? c->nyl : c->nxl;
    const long long bz = c->ndim == 3 ? nz : 1, bx = c->ndim == 3 ? nx : nz;  // 2D: one plane of Z rows
    const size_t bytes = (size_t)(bz * bx * ny) * c->tsize;
    void* tmp = nullptr;
    CU(cudaMallocAsync(&tmp, bytes, c->stream));
    s = launch_box_copy(c, tmp, bx * ny, ny, src + (size_t)c->origin * c->tsize, c->plane, c->ld, bz, bx, ny);
    if (!s) CU(cudaMemcpyAsync(out, tmp, bytes, cudaMemcpyDeviceToHost, c->stream));
    cudaFreeAsync(tmp, c->stream);
    if (s) return s;
    CU(cudaStreamSynchronize(c->stream));
    return FDW_OK;
}

fdw_status fdw_refresh_boundary(fdw_solver* c) {
    fdw_status s = enter(c);
    if (s) return s;
    if ((s = launch_boundary(c, c->cur, 0))) return s;
    if ((s = peer_exchange(c, c->cur))) return s;
    c->gstate[c->cur] = 0;
    CU(cudaStreamSynchronize(c->stream));
    return FDW_OK;
}

fdw_status fdw_record(fdw_solver* c) {
    fdw_status s = enter(c);
    if (s) return s;
    unsigned long long base = c->host_step;
    CU(cudaMemcpyAsync(&c->ctrl->row_base, &base, sizeof(base), cudaMemcpyHostToDevice, c->stream));
    if ((s = launch_receivers(c, c->cur, 0))) return s;
    CU(cudaStreamSynchronize(c->stream));
    return FDW_OK;
}

fdw_status fdw_advance(fdw_solver* c, uint64_t n, uint32_t flags, uint64_t* bad_step, double* bad_max) {
    fdw_status s = prologue(c);
    if (s) return s;
    if (!c->medium_set) return fail(c, FDW_ESTATE, "fdw_set_medium must be called before fdw_advance");
    const bool record = (flags & FDW_ADVANCE_RECORD) != 0;
    const unsigned long long ci = c->d.check_interval, total = c->d.n_steps;
    if (!c->pending) {
        c->pending = true;
        c->pend_start = c->host_step;
        c->pend_cur = c->cur;
    }
    unsigned long long st = c->host_step;
    const unsigned long long end = st + n;
    while (st < end) {
        unsigned long long nxt = (st / ci + 1) * ci;
        if (total > st) nxt = std::min(nxt, total);
        const unsigned long long e = std::min(end, nxt);
        const bool check = (e % ci == 0) || (e == total);
        if ((s = run_chunk(c, e - st, check, record))) return s;
        st = e;
    }
    if (flags & FDW_ADVANCE_ASYNC) return FDW_OK;
    return resolve_pending(c, bad_step, bad_max);
}

fdw_status fdw_wait(fdw_solver* c, uint64_t* bad_step, double* bad_max) {
    fdw_status s = prologue(c);
    if (s) return s;
    if (c->copy_stream) CU(cudaStreamSynchronize(c->copy_stream));
    CU(cudaStreamSynchronize(c->stream));
    return resolve_pending(c, bad_step, bad_max);
}

namespace {
void CUDART_CB snap_host_copy(void* p) {
    auto* j = static_cast<fdw_solver::SnapJob*>(p);
    std::memcpy(j->dst, j->src, j->bytes);
    delete j;
}
}  // namespace

fdw_status fdw_snapshot_async(fdw_solver* c, void* out) {
    NvtxRange nv("fdw_snapshot_async");
    fdw_status s = prologue(c);
    if (s) return s;
    if (!out) return fail(c, FDW_EINVAL, "null snapshot destination");
    const long long ny = c->ndim == 3 ? c->nyl : c->nxl;
    const long long bz = c->ndim == 3 ? c->nzl : 1, bx = c->ndim == 3 ? c->nxl : c->nzl;
    const size_t bytes = (size_t)(bz * bx * ny) * c->tsize;
    if (!c->copy_stream) {
        CU(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
        for (int k = 0; k < fdw_solver::SNAP_SLOTS; ++k) {
            CU(cudaEventCreateWithFlags(&c->snap_packed[k], cudaEventDisableTiming));
            CU(cudaEventCreateWithFlags(&c->snap_free[k], cudaEventDisableTiming));
            CU(cudaEventRecord(c->snap_free[k], c->copy_stream));
        }
    }
    const int k = c->snap_next;
    if (c->snap_bytes != bytes || !c->snap_dev[k]) {
        // (re)size every slot once; the copy stream is idle after the sync
        CU(cudaStreamSynchronize(c->copy_stream));
        CU(cudaStreamSynchronize(c->stream));
        for (int q = 0; q < fdw_solver::SNAP_SLOTS; ++q) {
            if (c->snap_dev[q]) cudaFreeAsync(c->snap_dev[q], c->stream);
            if (c->snap_host[q]) cudaFreeHost(c->snap_host[q]);
            c->snap_dev[q] = c->snap_host[q] = nullptr;
            CU(cudaMallocAsync(&c->snap_dev[q], bytes, c->stream));
        }
        c->snap_bytes = bytes;
    }
    // pack the extended box of the current level into the slot (compute
    // stream, after the slot's previous copy-out)
    CU(cudaStreamWaitEvent(c->stream, c->snap_free[k], 0));
    const char* src = static_cast<const char*>(c->lvl[c->cur]);
    if ((s = launch_box_copy(c, c->snap_dev[k], bx * ny, ny, src + (size_t)c->origin * c->tsize, c->plane, c->ld,
                             bz, bx, ny)))
        return s;
    CU(cudaEventRecord(c->snap_packed[k], c->stream));
    // copy-out on the copy stream: straight into pinned destinations, else
    // through a pinned bounce slot and a host-side memcpy
    CU(cudaStreamWaitEvent(c->copy_stream, c->snap_packed[k], 0));
    cudaPointerAttributes pa{};
    const bool pinned = cudaPointerGetAttributes(&pa, out) == cudaSuccess && pa.type == cudaMemoryTypeHost;
    cudaGetLastError();  // clear a benign error from an unregistered pointer
    if (pinned) {
        CU(cudaMemcpyAsync(out, c->snap_dev[k], bytes, cudaMemcpyDeviceToHost, c->copy_stream));
    } else {
        if (!c->snap_host[k]) CU(cudaMallocHost(&c->snap_host[k], bytes));
        CU(cudaMemcpyAsync(c->snap_host[k], c->snap_dev[k], bytes, cudaMemcpyDeviceToHost, c->copy_stream));
        // one job per snapshot (the callback frees it): a slot's previous job
        // may still be queued when the host reuses the slot
        auto* job = new fdw_solver::SnapJob{out, c->snap_host[k], bytes};
        cudaError_t e = cudaLaunchHostFunc(c->copy_stream, snap_host_copy, job);
        if (e != cudaSuccess) {
            delete job;
            return fail(c, FDW_ECUDA, "cudaLaunchHostFunc: %s", cudaGetErrorString(e));
        }
    }
    CU(cudaEventRecord(c->snap_free[k], c->copy_stream));
    c->snap_next = (k + 1) % fdw_solver::SNAP_SLOTS;
    return FDW_OK;
}

fdw_status fdw_step_index(fdw_solver* c, uint64_t* step) {
    if (!c || !step) return FDW_EINVAL;
    *step = c->host_step;
    return FDW_OK;
}

fdw_status fdw_set_step_index(fdw_solver* c, uint64_t step) {
    fdw_status s = enter(c);
    if (s) return s;
    unsigned long long v = step;
    CU(cudaMemcpyAsync(&c->ctrl->step, &v, sizeof(v), cudaMemcpyHostToDevice, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    c->host_step = step;
    return FDW_OK;
}

fdw_status fdw_max_abs(fdw_solver* c, double* out) {
    fdw_status s = enter(c);
    if (s) return s;
    if ((s = launch_health(c, c->cur, 0))) return s;
    if ((s = read_ctrl(c))) return s;
    if (c->h_ctrl->kind == 2)
        *out = std::numeric_limits<double>::quiet_NaN();
    else if (c->h_ctrl->kind == 1)
        *out = std::numeric_limits<double>::infinity();
    else {
        double m;
        std::memcpy(&m, &c->h_ctrl->max_bits, sizeof(m));
        *out = m;
    }
    return FDW_OK;
}

fdw_status fdw_download_seismogram_f64(fdw_solver* c, double* out, uint64_t rows) {
    fdw_status s = enter(c);
    if (s) return s;
    if (rows > c->seis_rows) return fail(c, FDW_EINVAL, "rows exceed the seismogram");
    if (c->n_rec == 0 || rows == 0) return FDW_OK;
    CU(cudaMemcpyAsync(out, c->d_seis, (size_t)rows * c->n_rec * sizeof(double), cudaMemcpyDeviceToHost,
                       c->stream));
    CU(cudaStreamSynchronize(c->stream));
    return FDW_OK;
}

fdw_status fdw_receiver_split_info(fdw_solver* c, uint64_t* n_slots, uint64_t* receiver, uint64_t* entry) {
    fdw_status s = prologue(c);
    if (s) return s;
    if (!n_slots) return fail(c, FDW_EINVAL, "null output");
    *n_slots = (uint64_t)c->n_split;
    if (receiver) std::copy(c->sp_rec.begin(), c->sp_rec.end(), receiver);
    if (entry) std::copy(c->sp_entry.begin(), c->sp_entry.end(), entry);
    return FDW_OK;
}

fdw_status fdw_download_receiver_products(fdw_solver* c, double* out, uint64_t rows) {
    fdw_status s = enter(c);
    if (s) return s;
    if (rows > c->seis_rows) return fail(c, FDW_EINVAL, "rows exceed the seismogram");
    if (c->n_split == 0 || rows == 0) return FDW_OK;
    if (c->side) CU(cudaStreamSynchronize(c->side));
    CU(cudaMemcpyAsync(out, c->d_sp_prod, (size_t)rows * c->n_split * sizeof(double), cudaMemcpyDeviceToHost,
                       c->stream));
    CU(cudaStreamSynchronize(c->stream));
    return FDW_OK;
}

fdw_status fdw_download_seismogram(fdw_solver* c, void* out, uint64_t rows) {
    fdw_status s = enter(c);
    if (s) return s;
    if (rows > c->seis_rows) return fail(c, FDW_EINVAL, "rows exceed the seismogram");
    const size_t n = (size_t)rows * c->n_rec;
    if (c->tsize == 8 || n == 0) return fdw_download_seismogram_f64(c, static_cast<double*>(out), rows);
    if (!c->d_seis) return fail(c, FDW_ESTATE, "no seismogram: set_receivers first");
    // fp32: rows rounded on the device, one D2H copy straight into `out`
    float* tmp = nullptr;
    CU(cudaMallocAsync(reinterpret_cast<void**>(&tmp), n * sizeof(float), c->stream));
    const unsigned blocks = (unsigned)std::min<size_t>((n + 255) / 256, (size_t)c->sm_count * 8);
    fdw::seis_to_float<<<blocks, 256, 0, c->stream>>>(c->d_seis, tmp, (unsigned long long)n);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(out, tmp, n * sizeof(float), cudaMemcpyDeviceToHost, c->stream);
    cudaFreeAsync(tmp, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) return fail(c, FDW_ECUDA, "fdw_download_seismogram: %s", cudaGetErrorString(e));
    return FDW_OK;
}

fdw_status fdw_synchronize(fdw_solver* c) {
    fdw_status s = prologue(c);
    if (s) return s;
    if (c->copy_stream) CU(cudaStreamSynchronize(c->copy_stream));
    CU(cudaStreamSynchronize(c->stream));
    return resolve_pending(c, nullptr, nullptr);
}

fdw_status fdw_profile_steps(fdw_solver* c, uint64_t n, double ms[6]) {
    fdw_status s = enter(c);
    if (s) return s;
    if (!c->medium_set) return fail(c, FDW_ESTATE, "fdw_set_medium must be called first");
    ProfileSink sink;
    c->prof = &sink;
    const unsigned long long ci = c->d.check_interval, total = c->d.n_steps;
    unsigned long long st = c->host_step;
    const unsigned long long end = st + n;
    while (st < end && s == FDW_OK) {
        unsigned long long nxt = (st / ci + 1) * ci;
        if (total > st) nxt = std::min(nxt, total);
        const unsigned long long e = std::min(end, nxt);
        s = run_chunk(c, e - st, (e % ci == 0) || (e == total), c->n_rec > 0);
        st = e;
    }
    c->prof = nullptr;
    cudaStreamSynchronize(c->stream);
    double sum[6] = {0, 0, 0, 0, 0, 0};
    int cnt[6] = {0, 0, 0, 0, 0, 0};
    for (auto& m : sink.marks) {
        float t = 0.f;
        cudaEventElapsedTime(&t, m.second.first, m.second.second);
        sum[m.first] += t;
        cnt[m.first] += 1;
        cudaEventDestroy(m.second.first);
        cudaEventDestroy(m.second.second);
    }
    for (int k = 0; k < 6; ++k) ms[k] = cnt[k] ? sum[k] / cnt[k] : 0.0;
    if (s) return s;
    if ((s = read_ctrl(c))) return s;
    return FDW_OK;
}

fdw_status fdw_launch_count(const fdw_solver* c, uint64_t* n) {
    if (!c || !n) return FDW_EINVAL;
    *n = c->launches;
    return FDW_OK;
}

fdw_status fdw_layout(const fdw_solver* c, uint64_t* ld, uint64_t* plane, uint64_t* base, uint64_t* planes,
                      int32_t* variant) {
    if (!c) return FDW_EINVAL;
    if (ld) *ld = (uint64_t)c->ld;
    if (plane) *plane = (uint64_t)c->plane;
    if (base) *base = (uint64_t)c->base;
    if (planes) *planes = (uint64_t)c->Lz;
    if (variant) *variant = c->variant | (c->zseg << 8) | (c->occupancy << 16) | (c->tma_pd << 24);
    return FDW_OK;
}

}  // extern "C"
