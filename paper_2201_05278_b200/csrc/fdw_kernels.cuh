// fdw_kernels.cuh -- sm_100a device code for the constant-density propagator.
//
// Every kernel restates one piece of fdwave::Solver<T>
// (/root/reference/proj/include/fdwave/kernel.hpp); the line range it replaces
// is in its comment.  Arithmetic follows the reference association exactly.
// With EXACT = true each operation is an explicitly rounded intrinsic
// (__fadd_rn/__fmul_rn/...), so no FMA contraction happens and the result is
// IEEE-identical to the reference's x86-64 build (which has no FMA: no -march,
// proj/CMakeLists.txt:7-19).  With EXACT = false the compiler may contract.
#pragma once

#include <cooperative_groups.h>
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

// Internal linkage: every translation unit that includes this header (fdw_api.cu,
// fdw_inst_*.cu) owns its copies; kernels cross TUs only as host stubs.
namespace fdw {
namespace {

// ---------------------------------------------------------------------------
// Device control block: step counter, abort latch, health-check scratch.
struct Ctrl {
    unsigned long long step;      // Solver::step_ (device authoritative)
    unsigned long long bad_step;  // step at which the health check tripped
    unsigned long long bad_idx;   // min global padded flat index of a non-finite value
    unsigned long long max_bits;  // max |u| over finite values, as double bits
    unsigned long long row_base;  // seismogram row 0 = this step (set by fdw_record)
    unsigned int abort;           // latched by the health check; every kernel no-ops
    unsigned int kind;            // 0 finite, 1 inf, 2 nan (|first non-finite|)
    unsigned int peer_err;        // peer transport: a wait for a neighbour timed out
};

// ---------------------------------------------------------------------------
// Peer transport for Z slabs (one GPU per rank on one NVLink/NVSwitch box).
// A rank's first / last R owned planes are the lower / upper neighbour's ghost
// planes; they are stored straight into the neighbour's level through mapped
// peer memory (by the sweep epilogue, by the point-source kernel for targets
// in those planes, or by peer_push).  No NCCL on the data path.
//
// Ordering is one halo epoch per collective operation (a step, a refresh, an
// upload): before an operation reads its ghost planes or stores into a
// neighbour's, it waits until both neighbours have PUBLISHED the epoch this
// rank is at (they finished the previous operation: their stores into this
// rank's ghost planes are visible, and they are done reading the buffer this
// rank writes into next); when its own boundary work is done it publishes
// epoch + 1.  In a TMA step both halves live inside the sweep: the CTAs that
// touch the first / last R planes wait at their start and the last of them to
// finish publishes, so no separate launch and no kernel-wide spin is needed.
template <typename T>
struct PeerMirror {
    T* lo = nullptr;             // lower neighbour's level (mapped), or null
    T* hi = nullptr;             // upper neighbour's level (mapped), or null
    long long lo_delta = 0, hi_delta = 0;  // neighbour element = local element + delta
    long long lo_end = 0;        // local elements [origin, lo_end) lie in the first R planes
    long long hi_begin = 0;      // local elements >= hi_begin lie in the last R planes
    __device__ __forceinline__ void store(long long i, T v) const {
        if (lo && i < lo_end) lo[i + lo_delta] = v;
        if (hi && i >= hi_begin) hi[i + hi_delta] = v;
    }
};

constexpr int PEER_MAX_WORLD = 8;
// Per-rank synchronisation block (device memory, IPC-exported).  Flags are
// written by the other ranks with st.release.sys and read with ld.acquire.sys.
struct PeerSync {
    unsigned long long halo_flag[PEER_MAX_WORLD];    // halo epoch last published by rank s
    unsigned long long health_flag[PEER_MAX_WORLD];  // health epoch last posted by rank s
    unsigned long long in_idx[2][PEER_MAX_WORLD];    // health inbox (epoch parity, source rank)
    unsigned long long in_max[2][PEER_MAX_WORLD];
    unsigned int in_kind[2][PEER_MAX_WORLD];
    unsigned long long halo_epoch;                   // this rank's own counters
    unsigned long long health_epoch;
    unsigned int bnd_done;                           // boundary CTAs of the running sweep that finished
    unsigned int abort_word;                         // sticky: some rank hit a peer failure (any rank may set it)
};

struct PeerArgs {
    PeerSync* self;
    PeerSync* peer[PEER_MAX_WORLD];  // mapped sync blocks of every rank (peer[rank] = self)
    int rank, world;
    Ctrl* ctrl;
};

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned int ld_volatile_u32(const unsigned int* p) {
    return *reinterpret_cast<const volatile unsigned int*>(p);
}
// Release/acquire fence at system scope (MEMBAR.ALL.SYS).  __threadfence_system()
// emits the sequentially consistent MEMBAR.SC.SYS, which the message-passing
// patterns here (stores, fence, flag) do not need and which costs far more.
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// A peer failure is made visible to EVERY rank: the sticky abort word is set in
// each rank's sync block, and every later wait on any rank sees it and latches
// its own abort (so no rank keeps stepping on frozen ghost planes).
__device__ void peer_fail(PeerSync* const* peer, int world, Ctrl* ctrl) {
    ctrl->peer_err = 1u;
    ctrl->abort = 1u;
    for (int s = 0; s < world; ++s)
        if (peer[s]) atomicExch_system(&peer[s]->abort_word, 1u);
    __threadfence_system();
}
__device__ __forceinline__ bool peer_aborted(const PeerSync* self, Ctrl* ctrl) {
    if (ld_volatile_u32(&self->abort_word) == 0u) return false;
    ctrl->peer_err = 1u;
    ctrl->abort = 1u;
    return true;
}

// Spins (one thread) until *flag >= want.  A failure anywhere (sticky word) or
// ~20 s without progress turns into peer_err + abort on every rank instead of
// a hung device.
__device__ bool peer_wait_flag(const unsigned long long* flag, unsigned long long want, PeerSync* const* peer,
                               int world, const PeerSync* self, Ctrl* ctrl) {
    if (peer_aborted(self, ctrl)) return false;
    if (ld_acquire_sys(flag) >= want) return true;
    const unsigned long long t0 = global_ns();
    unsigned int ns = 32;
    while (ld_acquire_sys(flag) < want) {
        __nanosleep(ns);
        if (ns < 1024) ns <<= 1;
        if (peer_aborted(self, ctrl)) return false;
        if (global_ns() - t0 > 20000000000ull) {
            peer_fail(peer, world, ctrl);
            return false;
        }
    }
    return true;
}

// Waits until both neighbours have published this rank's current halo epoch.
__device__ __forceinline__ bool peer_wait_neighbours(const PeerArgs& p) {
    const unsigned long long want = p.self->halo_epoch;
    if (p.rank > 0 && !peer_wait_flag(&p.self->halo_flag[p.rank - 1], want, p.peer, p.world, p.self, p.ctrl))
        return false;
    if (p.rank < p.world - 1 &&
        !peer_wait_flag(&p.self->halo_flag[p.rank + 1], want, p.peer, p.world, p.self, p.ctrl))
        return false;
    return true;
}
// Publishes epoch + 1 to both neighbours (after this rank's boundary work).
__device__ __forceinline__ void peer_publish(const PeerArgs& p) {
    const unsigned long long e = p.self->halo_epoch + 1;
    p.self->halo_epoch = e;
    fence_acq_rel_sys();
    if (p.rank > 0) st_release_sys(&p.peer[p.rank - 1]->halo_flag[p.rank], e);
    if (p.rank < p.world - 1) st_release_sys(&p.peer[p.rank + 1]->halo_flag[p.rank], e);
}

// ---------------------------------------------------------------------------
template <typename T, bool EXACT>
struct Ar;
template <>
struct Ar<float, true> {
    static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
    static __device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
    static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
};
template <>
struct Ar<float, false> {
    static __device__ __forceinline__ float add(float a, float b) { return a + b; }
    static __device__ __forceinline__ float sub(float a, float b) { return a - b; }
    static __device__ __forceinline__ float mul(float a, float b) { return a * b; }
};
template <>
struct Ar<double, true> {
    static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
    static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
    static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
};
template <>
struct Ar<double, false> {
    static __device__ __forceinline__ double add(double a, double b) { return a + b; }
    static __device__ __forceinline__ double sub(double a, double b) { return a - b; }
    static __device__ __forceinline__ double mul(double a, double b) { return a * b; }
};

// 1/(1 + eta dt) and (1 - eta dt) exactly as kernel.hpp:284-287 forms them:
// double arithmetic on double(eta) * dt, then cast to T.
// Packed fp32 pairs (sm_100 FADD2 / FFMA2), IEEE round-to-nearest per lane.
// The exact product is fma(a, b, nz) with nz a RUNTIME -0: ptxas contracts a
// plain mul.rn.f32x2 + add.rn.f32x2 into FFMA2 even under -fmad=false, and
// a*b + (-0) is exactly RN(a*b) (signed zeros included).
__device__ __forceinline__ unsigned long long f2u(float2 v) { return *reinterpret_cast<unsigned long long*>(&v); }
__device__ __forceinline__ float2 u2f(unsigned long long v) { return *reinterpret_cast<float2*>(&v); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
    unsigned long long r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)));
    return u2f(r);
}
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
    unsigned long long r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)));
    return u2f(r);
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
    unsigned long long r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)), "l"(f2u(c)));
    return u2f(r);
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b, float2 nz) {
    unsigned long long r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)), "l"(f2u(nz)));
    return u2f(r);
}

template <typename T>
__device__ __forceinline__ void damping_factors(T eta, double dt, T& om, T& iop) {
    const double edt = __dmul_rn(static_cast<double>(eta), dt);
    om = static_cast<T>(__dsub_rn(1.0, edt));
    iop = static_cast<T>(__ddiv_rn(1.0, __dadd_rn(1.0, edt)));
}

// kernel.hpp:418-420:  (c2dt2*rhs + 2u - om*prev) * iop.  eta == 0 gives
// om = iop = 1 exactly, and the multiplications by 1 are identities.
template <typename T, bool EXACT>
__device__ __forceinline__ T time_update(T rhs, T uc, T c2, T prev, T eta, double dt) {
    using A = Ar<T, EXACT>;
    const T t = A::add(A::mul(c2, rhs), A::mul(T(2), uc));
    if (eta == T(0)) return A::sub(t, prev);
    T om, iop;
    damping_factors(eta, dt, om, iop);
    return A::mul(A::sub(t, A::mul(om, prev)), iop);
}

// (1 - eta dt, 1/(1 + eta dt)) pairs of the damping table, in T
template <typename T>
struct EtabPair;
template <>
struct EtabPair<float> {
    using type = float2;
};
template <>
struct EtabPair<double> {
    using type = double2;
};

template <typename T>
struct SweepArgs {
    const T* __restrict__ u;      // current level
    T* out;                       // previous level, overwritten with the next one
    const T* __restrict__ c2dt2;  // c^2 dt^2
    const T* __restrict__ eta;    // damping eta (1/s)
    T v[11];                      // v_0..v_r cast to T (kernel.hpp:293)
    T ih[3];                      // T(1/h^2) per axis (kernel.hpp:290)
    double dt;
    long long ld, plane, origin;  // element strides; offset of extended (0,0,0)
    int nz, nx, ny;               // extended extents (local Z for slabs; 2D: rows nz, cols nx)
    // virtual ghosts (FDW_KERNEL_TMA): mirror factor per face (-1 Dirichlet,
    // +1 Neumann, 0 none) and whether the face is physical on this rank
    int gf[3][2];
    int gact[3][2];
    // variable density (simple kernels): grad(rho)/rho per axis, w_1..w_r, 1/(2h)
    const T* grad[3];
    T w1[10];
    T i2h[3];
    int vd;
    // TMA sweep: per tile column, the Z range [x, y) of planes whose eta tile
    // is all zero (those planes skip the eta stream); null: none
    const int2* ezr;
    // split-ring sweep with a damping table: (1 - eta dt, 1/(1 + eta dt)) per
    // index, index 0 = undamped; the eta map then streams 1-byte indices
    const typename EtabPair<T>::type* etab;
    int n_etab;
    // TMA sweep Z segments: CTA z-index b sweeps segment (b + seg_rot) mod
    // gridDim.z; a slab rotates its boundary segments (S-1, 0) into the first
    // wave so the halo stores and the epoch publish happen early in the step.
    int seg_rot;
    // peer transport (Z slabs over NVLink peer memory): the TMA sweep also
    // stores its first / last R planes into the lower / upper neighbour's ghost
    // planes of the same level, at element (local index + delta); null: none.
    // The CTAs that touch those planes wait for the neighbours' epoch first;
    // the last of the n_bnd of them publishes the next epoch (publish = 1).
    T* peer_lo;
    T* peer_hi;
    long long peer_lo_delta, peer_hi_delta;
    PeerArgs peer;
    unsigned int n_bnd;
    int publish;
    int halo_store;  // 0: skip the halo stores (fdw_peer_loopback timing experiments only)
    int fence_all;   // A/B of the one-fence-per-CTA release: 1 every thread fences (SC), 2 thread 0 SC
    T negz;  // -0 (runtime value for the packed exact products)
    const Ctrl* ctrl;
};

// ---------------------------------------------------------------------------
// sweep_3d<false>, kernel.hpp:381-424 -- one thread per point, cache-fed.
template <typename T, int R, bool EXACT>
__global__ void __launch_bounds__(256) sweep3d_simple(SweepArgs<T> a) {
    using A = Ar<T, EXACT>;
    if (a.ctrl->abort) return;
    const int iy = blockIdx.x * 32 + threadIdx.x;
    const int ix = blockIdx.y * 8 + threadIdx.y;
    const int iz = blockIdx.z;
    if (iy >= a.ny || ix >= a.nx) return;
    const long long i = a.origin + (long long)iz * a.plane + (long long)ix * a.ld + iy;
    const T* u = a.u;
    const T uc = __ldg(u + i);
    T lz = A::mul(a.v[0], uc), lx = A::mul(a.v[0], uc), ly = A::mul(a.v[0], uc);
#pragma unroll
    for (int j = 1; j <= R; ++j) {
        lz = A::add(lz, A::mul(a.v[j], A::add(__ldg(u + i + j * a.plane), __ldg(u + i - j * a.plane))));
        lx = A::add(lx, A::mul(a.v[j], A::add(__ldg(u + i + j * a.ld), __ldg(u + i - j * a.ld))));
        ly = A::add(ly, A::mul(a.v[j], A::add(__ldg(u + i + j), __ldg(u + i - j))));
    }
    T rhs = A::add(A::add(A::mul(lz, a.ih[0]), A::mul(lx, a.ih[1])), A::mul(ly, a.ih[2]));
    if (a.vd) {  // kernel.hpp:407-417
        T dz = T(0), dx = T(0), dy = T(0);
#pragma unroll
        for (int j = 1; j <= R; ++j) {
            dz = A::add(dz, A::mul(a.w1[j - 1], A::sub(__ldg(u + i + j * a.plane), __ldg(u + i - j * a.plane))));
            dx = A::add(dx, A::mul(a.w1[j - 1], A::sub(__ldg(u + i + j * a.ld), __ldg(u + i - j * a.ld))));
            dy = A::add(dy, A::mul(a.w1[j - 1], A::sub(__ldg(u + i + j), __ldg(u + i - j))));
        }
        rhs = A::sub(rhs, A::add(A::add(A::mul(A::mul(__ldg(a.grad[0] + i), dz), a.i2h[0]),
                                        A::mul(A::mul(__ldg(a.grad[1] + i), dx), a.i2h[1])),
                                 A::mul(A::mul(__ldg(a.grad[2] + i), dy), a.i2h[2])));
    }
    a.out[i] = time_update<T, EXACT>(rhs, uc, __ldg(a.c2dt2 + i), a.out[i], __ldg(a.eta + i), a.dt);
}

// sweep_2d<false>, kernel.hpp:344-379 -- rows are Z, the fast axis is X.
template <typename T, int R, bool EXACT>
__global__ void __launch_bounds__(256) sweep2d_simple(SweepArgs<T> a) {
    using A = Ar<T, EXACT>;
    if (a.ctrl->abort) return;
    const int ix = blockIdx.x * blockDim.x + threadIdx.x;
    const int iz = blockIdx.y * blockDim.y + threadIdx.y;
    if (ix >= a.nx || iz >= a.nz) return;
    const long long i = a.origin + (long long)iz * a.ld + ix;
    const T* u = a.u;
    const T uc = __ldg(u + i);
    T lz = A::mul(a.v[0], uc), lx = A::mul(a.v[0], uc);
#pragma unroll
    for (int j = 1; j <= R; ++j) {
        lz = A::add(lz, A::mul(a.v[j], A::add(__ldg(u + i + j * a.ld), __ldg(u + i - j * a.ld))));
        lx = A::add(lx, A::mul(a.v[j], A::add(__ldg(u + i + j), __ldg(u + i - j))));
    }
    T rhs = A::add(A::mul(lz, a.ih[0]), A::mul(lx, a.ih[1]));
    if (a.vd) {  // kernel.hpp:365-373
        T dz = T(0), dx = T(0);
#pragma unroll
        for (int j = 1; j <= R; ++j) {
            dz = A::add(dz, A::mul(a.w1[j - 1], A::sub(__ldg(u + i + j * a.ld), __ldg(u + i - j * a.ld))));
            dx = A::add(dx, A::mul(a.w1[j - 1], A::sub(__ldg(u + i + j), __ldg(u + i - j))));
        }
        rhs = A::sub(rhs, A::add(A::mul(A::mul(__ldg(a.grad[0] + i), dz), a.i2h[0]),
                                 A::mul(A::mul(__ldg(a.grad[1] + i), dx), a.i2h[1])));
    }
    a.out[i] = time_update<T, EXACT>(rhs, uc, __ldg(a.c2dt2 + i), a.out[i], __ldg(a.eta + i), a.dt);
}

// ---------------------------------------------------------------------------
// 16-byte vectors along the fast (Y) axis.
template <typename T, int V>
struct __align__(16) Vec {
    T e[V];
};

__device__ __forceinline__ Vec<float, 4> ldg16(const float* p) {
    const float4 t = __ldg(reinterpret_cast<const float4*>(p));
    return {{t.x, t.y, t.z, t.w}};
}
__device__ __forceinline__ Vec<double, 2> ldg16(const double* p) {
    const double2 t = __ldg(reinterpret_cast<const double2*>(p));
    return {{t.x, t.y}};
}
// streaming (evict-first) load for data read exactly once per step
__device__ __forceinline__ Vec<float, 4> ldcs16(const float* p) {
    const float4 t = __ldcs(reinterpret_cast<const float4*>(p));
    return {{t.x, t.y, t.z, t.w}};
}
__device__ __forceinline__ Vec<double, 2> ldcs16(const double* p) {
    const double2 t = __ldcs(reinterpret_cast<const double2*>(p));
    return {{t.x, t.y}};
}
__device__ __forceinline__ void st16(float* p, const Vec<float, 4>& v) {
    *reinterpret_cast<float4*>(p) = make_float4(v.e[0], v.e[1], v.e[2], v.e[3]);
}
__device__ __forceinline__ void st16(double* p, const Vec<double, 2>& v) {
    *reinterpret_cast<double2*>(p) = make_double2(v.e[0], v.e[1]);
}

template <typename T, int BX>
struct ZMarchShape {
    static constexpr int V = 16 / sizeof(T);  // elements per 16-byte vector
    static constexpr int NTY = 16;            // threads along Y
    static constexpr int TYW = NTY * V;       // tile width along Y (elements)
    static constexpr int THREADS = NTY * BX;
};

// sweep_3d<false>, kernel.hpp:381-424 -- 2.5D blocking.  A CTA owns a BX x TYW
// column of (X, Y) outputs and marches a Z segment.  The current u plane
// (tile + radius-R halos in X and Y) is staged in double-buffered shared
// memory; the Z neighbours of each thread's V outputs live in a register queue
// of 2R+1 vectors.  Loads for plane z+1 (queue head, halos, prev, c2dt2, eta)
// are issued before plane z is computed.  One __syncthreads per plane.
template <typename T, int R, int BX, bool EXACT>
__global__ void __launch_bounds__(ZMarchShape<T, BX>::THREADS)
    sweep3d_zmarch(SweepArgs<T> a) {
    using A = Ar<T, EXACT>;
    using S = ZMarchShape<T, BX>;
    constexpr int V = S::V, NTY = S::NTY, TYW = S::TYW;
    constexpr int HY = ((R + V - 1) / V) * V;  // Y halo, whole vectors
    constexpr int HYV = HY / V;
    constexpr int SP = TYW + 2 * HY;           // smem row pitch (elements)
    constexpr int SR = BX + 2 * R;             // smem rows
    using VT = Vec<T, V>;
    __shared__ __align__(16) T sm[2][SR][SP];

    if (a.ctrl->abort) return;
    const int ty = threadIdx.x, tx = threadIdx.y, tid = tx * NTY + ty;
    const int ty0 = blockIdx.x * TYW;  // tile origin (extended Y)
    const int tx0 = blockIdx.y * BX;   // tile origin (extended X)
    const int y0 = ty0 + ty * V;
    const int x = tx0 + tx;
    const int zs = (int)((long long)a.nz * blockIdx.z / gridDim.z);
    const int ze = (int)((long long)a.nz * (blockIdx.z + 1) / gridDim.z);
    const long long ld = a.ld, plane = a.plane;
    const long long col0 = a.origin + (long long)x * ld + y0;

    // X halo: 2R rows x NTY vectors (rows above, then rows below the tile)
    const bool hx_act = tid < 2 * R * NTY;
    const int hx_r = tid / NTY, hx_c = tid % NTY;
    const int hx_gx = hx_r < R ? tx0 - R + hx_r : tx0 + BX + (hx_r - R);
    const int hx_sr = hx_r < R ? hx_r : BX + R + (hx_r - R);
    const long long hx_off = a.origin + (long long)hx_gx * ld + ty0 + hx_c * V;
    // Y halo: BX rows x 2 sides x HYV vectors
    const bool hy_act = tid < BX * 2 * HYV;
    const int hy_r = tid / (2 * HYV), hy_k = tid % (2 * HYV);
    const int hy_side = hy_k / HYV, hy_kv = hy_k % HYV;
    const int hy_sc = hy_side == 0 ? hy_kv * V : HY + TYW + hy_kv * V;
    const int hy_gy = hy_side == 0 ? ty0 - HY + hy_kv * V : ty0 + TYW + hy_kv * V;
    const long long hy_off = a.origin + (long long)(tx0 + hy_r) * ld + hy_gy;

    const T* u = a.u;
    VT q[2 * R + 1];
#pragma unroll
    for (int k = 0; k < 2 * R; ++k) q[k] = ldg16(u + col0 + (long long)(zs - R + k) * plane);
    VT qn = ldg16(u + col0 + (long long)(zs + R) * plane);
    VT pv = ldcs16(a.out + col0 + (long long)zs * plane);
    VT cv = ldcs16(a.c2dt2 + col0 + (long long)zs * plane);
    VT ev = ldcs16(a.eta + col0 + (long long)zs * plane);
    VT hxv, hyv;
    if (hx_act) hxv = ldg16(u + hx_off + (long long)zs * plane);
    if (hy_act) hyv = ldg16(u + hy_off + (long long)zs * plane);

    const bool xin = x < a.nx;
    for (int z = zs; z < ze; ++z) {
        const int b = (z - zs) & 1;
        *reinterpret_cast<VT*>(&sm[b][R + tx][HY + ty * V]) = q[R];
        if (hx_act) *reinterpret_cast<VT*>(&sm[b][hx_sr][HY + hx_c * V]) = hxv;
        if (hy_act) *reinterpret_cast<VT*>(&sm[b][R + hy_r][hy_sc]) = hyv;
        q[2 * R] = qn;
        const VT pc = pv, cc = cv, ec = ev;
        if (z + 1 < ze) {
            const long long zo = (long long)(z + 1) * plane;
            qn = ldg16(u + col0 + zo + (long long)R * plane);
            pv = ldcs16(a.out + col0 + zo);
            cv = ldcs16(a.c2dt2 + col0 + zo);
            ev = ldcs16(a.eta + col0 + zo);
            if (hx_act) hxv = ldg16(u + hx_off + zo);
            if (hy_act) hyv = ldg16(u + hy_off + zo);
        }
        __syncthreads();

        T lz[V], lx[V], ly[V];
#pragma unroll
        for (int e = 0; e < V; ++e) {
            const T uc = q[R].e[e];
            lz[e] = A::mul(a.v[0], uc);
            lx[e] = lz[e];
            ly[e] = lz[e];
        }
        // Y window: smem row R+tx, columns [ty*V, ty*V + 2HY + V)
        T w[2 * HY + V];
#pragma unroll
        for (int k = 0; k < 2 * HYV + 1; ++k) {
            const VT t = *reinterpret_cast<const VT*>(&sm[b][R + tx][ty * V + k * V]);
#pragma unroll
            for (int e = 0; e < V; ++e) w[k * V + e] = t.e[e];
        }
#pragma unroll
        for (int j = 1; j <= R; ++j) {
            const VT xp = *reinterpret_cast<const VT*>(&sm[b][R + tx + j][HY + ty * V]);
            const VT xm = *reinterpret_cast<const VT*>(&sm[b][R + tx - j][HY + ty * V]);
            const T vj = a.v[j];
#pragma unroll
            for (int e = 0; e < V; ++e) {
                lz[e] = A::add(lz[e], A::mul(vj, A::add(q[R + j].e[e], q[R - j].e[e])));
                lx[e] = A::add(lx[e], A::mul(vj, A::add(xp.e[e], xm.e[e])));
                ly[e] = A::add(ly[e], A::mul(vj, A::add(w[HY + e + j], w[HY + e - j])));
            }
        }
        VT res;
#pragma unroll
        for (int e = 0; e < V; ++e) {
            const T rhs = A::add(A::add(A::mul(lz[e], a.ih[0]), A::mul(lx[e], a.ih[1])),
                                 A::mul(ly[e], a.ih[2]));
            res.e[e] = time_update<T, EXACT>(rhs, q[R].e[e], cc.e[e], pc.e[e], ec.e[e], a.dt);
        }
        if (xin) {
            T* o = a.out + col0 + (long long)z * plane;
            if (y0 + V <= a.ny) {
                st16(o, res);
            } else {
#pragma unroll
                for (int e = 0; e < V; ++e)
                    if (y0 + e < a.ny) o[e] = res.e[e];
            }
        }
#pragma unroll
        for (int k = 0; k < 2 * R; ++k) q[k] = q[k + 1];
    }
}


// ---------------------------------------------------------------------------
// Programmatic dependent launch.  A kernel launched with the programmatic
// stream-serialisation attribute may start before its predecessor on the
// stream has finished; pdl_wait() blocks until that predecessor has completed
// and its writes are visible.  Both are no-ops for an ordinary launch.  Every
// PDL-aware kernel calls pdl_wait() in every thread before its first read of
// data the predecessor writes and before any exit, so completion of a kernel
// still implies completion of everything before it on the stream.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ---------------------------------------------------------------------------
// TMA + mbarrier helpers (inline PTX, sm_90+/sm_100a)
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "FDW_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra FDW_WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

// PD = 0: one u ring of full tiles, the head plane z+R loaded one plane
// ahead and kept until it is the centre.  PD > 0 (split rings): the full
// centre tile and the head's interior tile are separate TMA loads, each PD
// planes ahead, so the same shared memory holds PD planes in flight at 3
// CTAs/SM (the centre tiles are L2 hits: their interiors arrived as heads).
template <typename T, int R, int BX, int NPA = 3, int PD = 0>
struct TmaShape {
    static constexpr int V = 16 / sizeof(T);
    static constexpr int NTY = 16;
    static constexpr int TYW = NTY * V;                  // tile width (elements)
    static constexpr int HY = ((R + V - 1) / V) * V;     // Y halo, whole vectors
    static constexpr int UW = TYW + 2 * HY;              // U tile row (elements)
    static constexpr int UH = BX + 2 * R;                // U tile rows
    static constexpr bool SPLIT = PD > 0;
    static constexpr int NU = SPLIT ? PD + 1 : R + 2;    // U ring: planes z .. z+R, +1 in flight (split: centres)
    static constexpr int NH = SPLIT ? PD + 1 : 0;        // split: head interior tiles
    static constexpr int NP = SPLIT ? PD + 1 : 2;        // prev/c2dt2/eta[/grad x3] ring
    static constexpr int U_BOX = UW * UH * (int)sizeof(T);
    static constexpr int P_BOX = TYW * BX * (int)sizeof(T);
    static constexpr int U_STRIDE = (U_BOX + 127) / 128 * 128;
    static constexpr int P_STRIDE = (P_BOX + 127) / 128 * 128;
    static constexpr int H_OFF = NU * U_STRIDE;
    static constexpr int P_OFF = H_OFF + NH * P_STRIDE;
    static constexpr int BAR_OFF = P_OFF + NP * NPA * P_STRIDE;
    static constexpr int SMEM = BAR_OFF + (NU + NH + NP) * 8;
    static constexpr int THREADS = NTY * BX;
};

// sweep_3d<false>, kernel.hpp:381-424 -- TMA-fed 2.5D Z-march.  Per CTA a
// BX x TYW (X, Y) column, one Z segment.  One elected thread streams, per
// plane, the u tile with its radius-R X/Y halos and the prev/c2dt2/eta tiles
// into shared-memory rings with cp.async.bulk.tensor (completion on
// mbarriers); the 2R+1 Z neighbours of each thread's V outputs live in a
// register queue fed from the ring (head = plane z+R).  No per-thread global
// loads on the hot path; one __syncthreads per plane recycles ring stages.
// VD (sweep_3d<true>, kernel.hpp:407-417): three more tiles per plane
// (grad(rho)/rho per axis) and the first-derivative taps on the same operands.
template <typename T, int R, int BX, bool EXACT, int MINB, bool VD = false, int PD = 0, bool ETAB = false>
__global__ void __launch_bounds__(TmaShape<T, R, BX, VD ? 6 : 3, PD>::THREADS, MINB)
    sweep3d_tma(SweepArgs<T> a, const __grid_constant__ CUtensorMap tu, const __grid_constant__ CUtensorMap tp,
                const __grid_constant__ CUtensorMap tc, const __grid_constant__ CUtensorMap te,
                const __grid_constant__ CUtensorMap tg0, const __grid_constant__ CUtensorMap tg1,
                const __grid_constant__ CUtensorMap tg2, const __grid_constant__ CUtensorMap th, int col_base) {
    using A = Ar<T, EXACT>;
    constexpr int NPA = VD ? 6 : 3;
    using S = TmaShape<T, R, BX, NPA, PD>;
    constexpr bool SPLIT = S::SPLIT;
    constexpr int V = S::V, NTY = S::NTY, TYW = S::TYW, HY = S::HY, HYV = HY / V, UW = S::UW, NU = S::NU;
    constexpr int NH = S::NH, NP = S::NP;
    constexpr int THREADS = S::THREADS;
    static_assert(!ETAB || ((std::is_same<T, float>::value && V == 4) || (std::is_same<T, double>::value && V == 2)),
                  "damping table: fp32 or fp64");
    using T2 = typename EtabPair<T>::type;
    constexpr int E_BOX = ETAB ? TYW * BX : S::P_BOX;  // bytes of the eta (or eta index) tile
    using VT = Vec<T, V>;
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned long long* barU = reinterpret_cast<unsigned long long*>(smem + S::BAR_OFF);
    unsigned long long* barH = barU + NU;
    unsigned long long* barP = barH + NH;

    // the next kernel (point sources) may launch once our last wave is placed
    pdl_launch_dependents();
    const int ty = threadIdx.x, tx = threadIdx.y, tid = tx * NTY + ty;
    const int ty0 = blockIdx.x * TYW;
    const int tx0 = blockIdx.y * BX;
    const int y0 = ty0 + ty * V;
    const int x = tx0 + tx;
    const int nz = a.nz, nx = a.nx, ny = a.ny;
    const int nseg = (int)gridDim.z;
    const int seg = ((int)blockIdx.z + a.seg_rot) % nseg;
    const int zs = (int)((long long)nz * seg / nseg);
    const int ze = (int)((long long)nz * (seg + 1) / nseg);
    const long long plane = a.plane;
    const long long col0 = a.origin + (long long)x * a.ld + y0;

    // Virtual Z ghosts on physical Z faces: plane p outside [0, nz) reads its
    // mirror plane scaled by the face factor (apply_boundary, kernel.hpp:84-97).
    const bool zlo = a.gact[0][0], zhi = a.gact[0][1];
    auto zsrc = [&](int p) {
        if (p < 0 && zlo) return -p;
        if (p >= nz && zhi) return 2 * (nz - 1) - p;
        return p;
    };
    auto mir = [](int f, T v) { return f == 0 ? T(0) : (f < 0 ? -v : v); };
    // planes [ez0, ez1) of this column have an all-zero eta tile: no eta
    // stream there, and the undamped update (om = iop = 1, exact identities)
    int ez0 = 0, ez1 = 0;
    if (a.ezr) {
        const int2 r = a.ezr[blockIdx.y * gridDim.x + blockIdx.x];
        ez0 = r.x;
        ez1 = r.y;
    }

    auto u_stage = [&](int k) { return reinterpret_cast<T*>(smem + (k % NU) * S::U_STRIDE); };
    auto h_stage = [&](int k) { return reinterpret_cast<T*>(smem + S::H_OFF + (k % (NH ? NH : 1)) * S::P_STRIDE); };
    auto p_stage = [&](int k, int which) {
        return reinterpret_cast<T*>(smem + S::P_OFF + ((k % NP) * NPA + which) * S::P_STRIDE);
    };
    auto issue_u = [&](int k) {  // tile of plane zs + k (mirrored plane beyond a physical Z face)
        unsigned long long* b = &barU[k % NU];
        mbar_expect_tx(b, S::U_BOX);
        tma_load_3d(u_stage(k), &tu, col_base + ty0 - HY, tx0, zsrc(zs + k) + R, b);
    };
    auto issue_h = [&](int k) {  // split rings: interior tile of the head plane zs + k + R
        unsigned long long* b = &barH[k % (NH ? NH : 1)];
        mbar_expect_tx(b, S::P_BOX);
        tma_load_3d(h_stage(k), &th, col_base + ty0, tx0 + R, zsrc(zs + k + R) + R, b);
    };
    auto issue_p = [&](int k) {
        unsigned long long* b = &barP[k % NP];
        const bool skip_e = zs + k >= ez0 && zs + k < ez1;
        mbar_expect_tx(b, (NPA - 1) * S::P_BOX + (skip_e ? 0 : E_BOX));
        const int c0 = col_base + ty0, c1 = tx0 + R, c2 = zs + k + R;
        tma_load_3d(p_stage(k, 0), &tp, c0, c1, c2, b);
        tma_load_3d(p_stage(k, 1), &tc, c0, c1, c2, b);
        if (!skip_e) tma_load_3d(p_stage(k, 2), &te, c0, c1, c2, b);
        if constexpr (VD) {
            tma_load_3d(p_stage(k, 3), &tg0, c0, c1, c2, b);
            tma_load_3d(p_stage(k, 4), &tg1, c0, c1, c2, b);
            tma_load_3d(p_stage(k, 5), &tg2, c0, c1, c2, b);
        }
    };

    if (tid == 0) {
        for (int k = 0; k < NU + NH + NP; ++k) mbar_init(&barU[k], 1);  // barU, barH, barP are contiguous
        mbar_fence_init();
    }
    __shared__ T2 s_etab[ETAB ? 256 : 1];
    if constexpr (ETAB)
        for (int k = tid; k < a.n_etab; k += THREADS) s_etab[k] = a.etab[k];
    __syncthreads();
    // everything above touches shared memory and setup-time data only
    pdl_wait();
    if (a.ctrl->abort) return;
    // peer transport: this CTA reads ghost planes written by a neighbour and
    // stores into the neighbour's -> the neighbours must have published this
    // rank's epoch (they finished the previous step)
    const bool plo = a.peer_lo && zs < R, phi = a.peer_hi && ze > nz - R;
    auto issue_first = [&]() {
        if constexpr (SPLIT) {
            for (int k = 0; k < PD; ++k) {  // PD planes in flight
                issue_u(k);
                issue_h(k);
                issue_p(k);
            }
        } else {
            for (int k = 0; k <= R; ++k) issue_u(k);  // planes zs .. zs+R
            issue_p(0);
        }
    };
    if (plo || phi) {
        // The first TMA loads read owned planes only (unless the segment is
        // thinner than its head reach): issue them while another warp waits
        // for the neighbours, so the wait overlaps the load latency.
        const bool early = !phi || zs + R + (SPLIT ? PD - 1 : 0) < nz;
        if (tid == 0 && early) issue_first();
        __shared__ int peer_ok;
        if (tid == 32) peer_ok = peer_wait_neighbours(a.peer) ? 1 : 0;
        __syncthreads();
        if (!peer_ok) {
            if (tid == 0 && early) {  // no bulk copy may outlive the CTA
                if constexpr (SPLIT) {
                    for (int k = 0; k < PD; ++k) {
                        mbar_wait(&barU[k], 0);
                        mbar_wait(&barH[k], 0);
                        mbar_wait(&barP[k], 0);
                    }
                } else {
                    for (int k = 0; k <= R; ++k) mbar_wait(&barU[k], 0);
                    mbar_wait(&barP[0], 0);
                }
            }
            return;
        }
        if (tid == 0 && !early) issue_first();
    } else if (tid == 0) {
        issue_first();
    }
    VT qq[2 * R + 4];
#pragma unroll
    for (int k = 0; k < 2 * R; ++k) {
        const int p = zs - R + k;
        qq[k] = ldg16(a.u + col0 + (long long)zsrc(p) * plane);
        if ((p < 0 && zlo) || (p >= nz && zhi)) {
            const int f = p < 0 ? a.gf[0][0] : a.gf[0][1];
#pragma unroll
            for (int e = 0; e < V; ++e) qq[k].e[e] = mir(f, qq[k].e[e]);
        }
    }

    // Virtual X/Y ghosts: CTAs whose halo crosses a physical X/Y face patch
    // the halo rows/columns of the staged tile from their mirror images
    // (one extra __syncthreads per plane, edge CTAs only).
    const bool pxl = a.gact[1][0] && tx0 == 0;
    const bool pxh = a.gact[1][1] && tx0 + BX + R > nx;
    const bool pyl = a.gact[2][0] && ty0 == 0;
    const bool pyh = a.gact[2][1] && ty0 + TYW + HY > ny;
    const bool edge_tile = pxl || pxh || pyl || pyh;
    auto patch = [&](T* U) {
        if (pxl) {  // rows x = -k <- row k
            const int f = a.gf[1][0];
            for (int i = tid; i < R * TYW; i += THREADS) {
                const int k = i / TYW + 1, c = HY + i % TYW;
                U[(R - k) * UW + c] = mir(f, U[(R + k) * UW + c]);
            }
        }
        if (pxh) {  // rows x in [nx, nx+R) inside the tile
            const int f = a.gf[1][1];
            for (int i = tid; i < R * TYW; i += THREADS) {
                const int xg = nx + i / TYW, c = HY + i % TYW;
                const int r = xg - tx0 + R;
                if (r < BX + 2 * R) U[r * UW + c] = mir(f, U[(2 * (nx - 1) - xg - tx0 + R) * UW + c]);
            }
        }
        if (pyl) {  // columns y = -k <- column k
            const int f = a.gf[2][0];
            for (int i = tid; i < R * BX; i += THREADS) {
                const int k = i % R + 1, r = R + i / R;
                U[r * UW + HY - k] = mir(f, U[r * UW + HY + k]);
            }
        }
        if (pyh) {  // columns y in [ny, ny+R) inside the tile
            const int f = a.gf[2][1];
            for (int i = tid; i < R * BX; i += THREADS) {
                const int yg = ny + i % R, r = R + i / R;
                const int c = yg - ty0 + HY;
                if (c < UW) U[r * UW + c] = mir(f, U[r * UW + (2 * (ny - 1) - yg - ty0 + HY)]);
            }
        }
    };

    const bool xin = x < nx;
    const int nit = ze - zs;
    // one plane; the Z queue window is qq[S .. S+2R] for the S-th plane of an
    // unrolled group, so consecutive planes rename registers instead of moving
    // the queue (one 4-slot shift per group of 4 planes)
    auto do_plane = [&](const int it, auto S) {
        VT* q = qq + decltype(S)::value;
        const int z = zs + it;
        if (it > 0) __syncthreads();  // stages of plane z-1 are free
        if constexpr (SPLIT) {
            if (tid == 0 && it + PD < nit) {
                issue_u(it + PD);
                issue_h(it + PD);
                issue_p(it + PD);
            }
            mbar_wait(&barH[it % NH], (it / NH) & 1);
            q[2 * R] = *reinterpret_cast<const VT*>(h_stage(it) + tx * TYW + ty * V);
        } else {
            if (tid == 0 && it + 1 < nit) {
                issue_u(it + 1 + R);
                issue_p(it + 1);
            }
            const int kh = it + R;
            mbar_wait(&barU[kh % NU], (kh / NU) & 1);
            q[2 * R] = *reinterpret_cast<const VT*>(u_stage(kh) + (R + tx) * UW + HY + ty * V);
        }
        if (zhi && z + R >= nz) {  // head is a mirrored plane (uniform branch)
#pragma unroll
            for (int e = 0; e < V; ++e) q[2 * R].e[e] = mir(a.gf[0][1], q[2 * R].e[e]);
        }
        mbar_wait(&barU[it % NU], (it / NU) & 1);
        mbar_wait(&barP[it % NP], (it / NP) & 1);
        T* U0 = u_stage(it);
        if (edge_tile) {
            patch(U0);
            __syncthreads();
        }

        constexpr bool PACK = std::is_same<T, float>::value && !VD && V == 4;
        VT res;
        if constexpr (PACK) {
            // the same operations in the same order, two lanes per instruction
            // (FMA mode: each multiply-add contracted into FFMA2)
            const float2 nz2 = make_float2(a.negz, a.negz);
            auto mac2 = [&](float2 acc, float2 x, float2 y) {
                if constexpr (EXACT)
                    return add2(acc, mul2(x, y, nz2));
                else
                    return fma2(x, y, acc);
            };
            auto pr = [](const VT& v, int p) { return p ? make_float2(v.e[2], v.e[3]) : make_float2(v.e[0], v.e[1]); };
            float2 lz2[2], lx2[2];
            T ly[V];
            const float2 v02 = make_float2(a.v[0], a.v[0]);
#pragma unroll
            for (int p = 0; p < 2; ++p) {
                lz2[p] = mul2(v02, pr(q[R], p), nz2);
                lx2[p] = lz2[p];
                ly[2 * p] = lz2[p].x;
                ly[2 * p + 1] = lz2[p].y;
            }
            T w[2 * HY + V];
#pragma unroll
            for (int k = 0; k < 2 * HYV + 1; ++k) {
                const VT t = *reinterpret_cast<const VT*>(U0 + (R + tx) * UW + ty * V + k * V);
#pragma unroll
                for (int e = 0; e < V; ++e) w[k * V + e] = t.e[e];
            }
#pragma unroll
            for (int j = 1; j <= R; ++j) {
                const VT xp = *reinterpret_cast<const VT*>(U0 + (R + tx + j) * UW + HY + ty * V);
                const VT xm = *reinterpret_cast<const VT*>(U0 + (R + tx - j) * UW + HY + ty * V);
                const float2 vj2 = make_float2(a.v[j], a.v[j]);
#pragma unroll
                for (int p = 0; p < 2; ++p) {
                    lz2[p] = mac2(lz2[p], vj2, add2(pr(q[R + j], p), pr(q[R - j], p)));
                    lx2[p] = mac2(lx2[p], vj2, add2(pr(xp, p), pr(xm, p)));
                }
                // ly stays scalar: odd-j Y pairs straddle register pairs (measured slower packed)
#pragma unroll
                for (int e = 0; e < V; ++e)
                    ly[e] = A::add(ly[e], A::mul(a.v[j], A::add(w[HY + e + j], w[HY + e - j])));
            }
            const int po = tx * TYW + ty * V;
            const VT pc = *reinterpret_cast<const VT*>(p_stage(it, 0) + po);
            const VT cc = *reinterpret_cast<const VT*>(p_stage(it, 1) + po);
            const float2 ih0 = make_float2(a.ih[0], a.ih[0]), ih1 = make_float2(a.ih[1], a.ih[1]);
            const float2 ih2 = make_float2(a.ih[2], a.ih[2]), two = make_float2(2.f, 2.f);
            float2 rhs2[2];
#pragma unroll
            for (int p = 0; p < 2; ++p)
                rhs2[p] = mac2(mac2(mul2(lz2[p], ih0, nz2), lx2[p], ih1), make_float2(ly[2 * p], ly[2 * p + 1]), ih2);
            if (z >= ez0 && z < ez1) {  // eta == 0: time_update's undamped form
#pragma unroll
                for (int p = 0; p < 2; ++p) {
                    const float2 r2 = sub2(mac2(mul2(two, pr(q[R], p), nz2), pr(cc, p), rhs2[p]), pr(pc, p));
                    res.e[2 * p] = r2.x;
                    res.e[2 * p + 1] = r2.y;
                }
            } else if constexpr (ETAB) {
                // time_update with the tabled factors, two lanes per instruction.
                // Index 0 (eta == 0) holds (1, 1): x * 1 == x exactly (signed
                // zeros, subnormals, NaN), so the damped form reproduces the
                // undamped (t - prev) bit for bit and no lane branches.
                const uchar4 ib = *reinterpret_cast<const uchar4*>(
                    reinterpret_cast<const unsigned char*>(p_stage(it, 2)) + po);
                const float2 f0 = s_etab[ib.x], f1 = s_etab[ib.y], f2 = s_etab[ib.z], f3 = s_etab[ib.w];
                const float2 om[2] = {make_float2(f0.x, f1.x), make_float2(f2.x, f3.x)};
                const float2 io[2] = {make_float2(f0.y, f1.y), make_float2(f2.y, f3.y)};
#pragma unroll
                for (int p = 0; p < 2; ++p) {
                    const float2 t2 = mac2(mul2(two, pr(q[R], p), nz2), pr(cc, p), rhs2[p]);
                    const float2 r2 = mul2(sub2(t2, mul2(om[p], pr(pc, p), nz2)), io[p], nz2);
                    res.e[2 * p] = r2.x;
                    res.e[2 * p + 1] = r2.y;
                }
            } else {
                const VT ec = *reinterpret_cast<const VT*>(p_stage(it, 2) + po);
#pragma unroll
                for (int p = 0; p < 2; ++p) {
                    res.e[2 * p] = time_update<T, EXACT>(rhs2[p].x, q[R].e[2 * p], cc.e[2 * p], pc.e[2 * p],
                                                         ec.e[2 * p], a.dt);
                    res.e[2 * p + 1] = time_update<T, EXACT>(rhs2[p].y, q[R].e[2 * p + 1], cc.e[2 * p + 1],
                                                             pc.e[2 * p + 1], ec.e[2 * p + 1], a.dt);
                }
            }
        } else {
            T lz[V], lx[V], ly[V];
            T dz[VD ? V : 1], dx[VD ? V : 1], dy[VD ? V : 1];
            (void)dz, (void)dx, (void)dy;
    #pragma unroll
            for (int e = 0; e < V; ++e) {
                lz[e] = A::mul(a.v[0], q[R].e[e]);
                lx[e] = lz[e];
                ly[e] = lz[e];
                if constexpr (VD) dz[e] = dx[e] = dy[e] = T(0);
            }
            T w[2 * HY + V];
    #pragma unroll
            for (int k = 0; k < 2 * HYV + 1; ++k) {
                const VT t = *reinterpret_cast<const VT*>(U0 + (R + tx) * UW + ty * V + k * V);
    #pragma unroll
                for (int e = 0; e < V; ++e) w[k * V + e] = t.e[e];
            }
    #pragma unroll
            for (int j = 1; j <= R; ++j) {
                const VT xp = *reinterpret_cast<const VT*>(U0 + (R + tx + j) * UW + HY + ty * V);
                const VT xm = *reinterpret_cast<const VT*>(U0 + (R + tx - j) * UW + HY + ty * V);
                const T vj = a.v[j];
    #pragma unroll
                for (int e = 0; e < V; ++e) {
                    lz[e] = A::add(lz[e], A::mul(vj, A::add(q[R + j].e[e], q[R - j].e[e])));
                    lx[e] = A::add(lx[e], A::mul(vj, A::add(xp.e[e], xm.e[e])));
                    ly[e] = A::add(ly[e], A::mul(vj, A::add(w[HY + e + j], w[HY + e - j])));
                }
                if constexpr (VD) {  // each accumulator sees the reference's order
                    const T wj = a.w1[j - 1];
    #pragma unroll
                    for (int e = 0; e < V; ++e) {
                        dz[e] = A::add(dz[e], A::mul(wj, A::sub(q[R + j].e[e], q[R - j].e[e])));
                        dx[e] = A::add(dx[e], A::mul(wj, A::sub(xp.e[e], xm.e[e])));
                        dy[e] = A::add(dy[e], A::mul(wj, A::sub(w[HY + e + j], w[HY + e - j])));
                    }
                }
            }
            const int po = tx * TYW + ty * V;
            const VT pc = *reinterpret_cast<const VT*>(p_stage(it, 0) + po);
            const VT cc = *reinterpret_cast<const VT*>(p_stage(it, 1) + po);
            auto rhs_of = [&](int e) {
                T rhs = A::add(A::add(A::mul(lz[e], a.ih[0]), A::mul(lx[e], a.ih[1])), A::mul(ly[e], a.ih[2]));
                if constexpr (VD) {
                    const T g0 = p_stage(it, 3)[po + e], g1 = p_stage(it, 4)[po + e], g2 = p_stage(it, 5)[po + e];
                    rhs = A::sub(rhs, A::add(A::add(A::mul(A::mul(g0, dz[e]), a.i2h[0]),
                                                    A::mul(A::mul(g1, dx[e]), a.i2h[1])),
                                             A::mul(A::mul(g2, dy[e]), a.i2h[2])));
                }
                return rhs;
            };
            if (z >= ez0 && z < ez1) {  // eta == 0: time_update's undamped form
    #pragma unroll
                for (int e = 0; e < V; ++e)
                    res.e[e] = A::sub(A::add(A::mul(cc.e[e], rhs_of(e)), A::mul(T(2), q[R].e[e])), pc.e[e]);
            } else if constexpr (ETAB) {  // tabled factors; index 0 = (1, 1) is exact
                const unsigned char* ibp = reinterpret_cast<const unsigned char*>(p_stage(it, 2)) + po;
                unsigned ix[V];
                if constexpr (V == 4) {
                    const uchar4 ib = *reinterpret_cast<const uchar4*>(ibp);
                    ix[0] = ib.x, ix[1] = ib.y, ix[2] = ib.z, ix[3] = ib.w;
                } else {
                    const uchar2 ib = *reinterpret_cast<const uchar2*>(ibp);
                    ix[0] = ib.x, ix[1] = ib.y;
                }
    #pragma unroll
                for (int e = 0; e < V; ++e) {
                    const T2 f = s_etab[ix[e]];
                    const T t = A::add(A::mul(cc.e[e], rhs_of(e)), A::mul(T(2), q[R].e[e]));
                    res.e[e] = A::mul(A::sub(t, A::mul(f.x, pc.e[e])), f.y);
                }
            } else {
                const VT ec = *reinterpret_cast<const VT*>(p_stage(it, 2) + po);
    #pragma unroll
                for (int e = 0; e < V; ++e)
                    res.e[e] = time_update<T, EXACT>(rhs_of(e), q[R].e[e], cc.e[e], pc.e[e], ec.e[e], a.dt);
            }
        }
        // null-Dirichlet face nodes are forced to +0 (kernel.hpp:87-88)
        if ((zlo && z == 0 && a.gf[0][0] < 0) || (zhi && z == nz - 1 && a.gf[0][1] < 0)) {
#pragma unroll
            for (int e = 0; e < V; ++e) res.e[e] = T(0);
        }
        if (edge_tile) {
            const bool dx = (pxl && x == 0 && a.gf[1][0] < 0) || (pxh && x == nx - 1 && a.gf[1][1] < 0);
#pragma unroll
            for (int e = 0; e < V; ++e) {
                const int yy = y0 + e;
                if (dx || (pyl && yy == 0 && a.gf[2][0] < 0) || (pyh && yy == ny - 1 && a.gf[2][1] < 0))
                    res.e[e] = T(0);
            }
        }
        if (xin) {
            T* o = a.out + col0 + (long long)z * plane;
            if (y0 + V <= ny) {
                st16(o, res);
            } else {
#pragma unroll
                for (int e = 0; e < V; ++e)
                    if (y0 + e < ny) o[e] = res.e[e];
            }
        }
    };
    int it0 = 0;
    if constexpr (!VD) {
        for (; it0 + 3 < nit; it0 += 4) {  // 4 planes per trip: measured best (3: -1.6%, 5+: I-cache)
            do_plane(it0, std::integral_constant<int, 0>{});
            do_plane(it0 + 1, std::integral_constant<int, 1>{});
            do_plane(it0 + 2, std::integral_constant<int, 2>{});
            do_plane(it0 + 3, std::integral_constant<int, 3>{});
#pragma unroll
            for (int k = 0; k < 2 * R; ++k) qq[k] = qq[k + 4];
        }
    }
    for (; it0 < nit; ++it0) {  // (VD: the larger body keeps the rolled loop)
        do_plane(it0, std::integral_constant<int, 0>{});
#pragma unroll
        for (int k = 0; k < 2 * R; ++k) qq[k] = qq[k + 1];
    }
    // peer transport: this column's share of the first / last R planes goes
    // straight into the neighbour's ghost planes over NVLink (each thread
    // re-reads its own just-written outputs; outside the plane loop, so the
    // hot loop's registers are untouched), performed system-wide before the
    // grid ends
    if ((plo || phi) && xin && a.halo_store) {
        auto copy_plane = [&](T* peer, long long delta, int z) {
            const T* o = a.out + col0 + (long long)z * plane;
            T* po = peer + (col0 + (long long)z * plane + delta);
            if (y0 + V <= ny) {
                st16(po, *reinterpret_cast<const VT*>(o));
            } else {
                for (int e = 0; e < V; ++e)
                    if (y0 + e < ny) po[e] = o[e];
            }
        };
        if (plo)
            for (int z = zs; z < min(ze, R); ++z) copy_plane(a.peer_lo, a.peer_lo_delta, z);
        if (phi)
            for (int z = max(zs, nz - R); z < ze; ++z) copy_plane(a.peer_hi, a.peer_hi_delta, z);
    }
    if (plo || phi) {
        // release: the CTA's halo stores (ordered before thread 0 by the
        // barrier, fence cumulativity) are made visible system-wide by one
        // fence; the last boundary CTA of the step publishes the next epoch
        if (a.fence_all == 1) __threadfence_system();
        __syncthreads();
        if (tid == 0) {
            if (a.fence_all == 2)
                __threadfence_system();  // A/B: the sequentially consistent fence of round 2
            else
                fence_acq_rel_sys();
            if (a.publish && atomicAdd(&a.peer.self->bnd_done, 1u) == a.n_bnd - 1) {
                a.peer.self->bnd_done = 0u;
                peer_publish(a.peer);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// 2D: one persistent cooperative kernel runs a whole chunk of time steps
// (FDW_KERNEL_FUSED2D).  The 2D working set (C2: 3 MB per field) lives in L2,
// so a step is launch/latency-bound; here a step is one grid-wide barrier:
//   phase k: sweep of step k (virtual ghosts, Dirichlet faces forced to +0,
//            point-source injection fused per target point) + the receiver
//            row of step k-1 (its level is read-only during step k)
//   grid.sync()
// Loads of data written inside the launch use ld.global.cg (L2, no stale L1).
template <typename T>
struct Fused2DArgs {
    T* lvl[2];
    const T* __restrict__ c2dt2;
    const T* __restrict__ eta;
    T v[11];
    T ih[3];
    double dt;
    long long ld, origin;
    int nz, nx;
    int gf[2][2];                // mirror factor per face: -1 Dirichlet, +1 Neumann, 0 none
    const int* tmap;             // [nz*nx] injection target index + 1, 0 if none
    const long long* tgt;        // unused here (offsets of targets)
    const unsigned* ent_off;
    const double* ent_w;
    const double* wavelet;
    unsigned long long n_wavelet;
    const long long* ridx;       // receivers (device offsets), CSR
    const unsigned* roff;
    const double* rw;
    double* seis;
    int n_rec;
    unsigned long long n_rows;
    int dbg;                     // development: bit0 skip sweep, bit1 skip receivers
    Ctrl* ctrl;
    const T* grad[2];            // variable density: grad(rho)/rho per axis
    T w1[10];                    // first-derivative weights w_1..w_r
    T i2h[2];                    // 1/(2h) per axis
};

__device__ __forceinline__ Vec<float, 4> ldcg16(const float* p) {
    const float4 v = __ldcg(reinterpret_cast<const float4*>(p));
    return Vec<float, 4>{{v.x, v.y, v.z, v.w}};
}
__device__ __forceinline__ Vec<double, 2> ldcg16(const double* p) {
    const double2 v = __ldcg(reinterpret_cast<const double2*>(p));
    return Vec<double, 2>{{v.x, v.y}};
}

template <typename T>
__device__ __forceinline__ T ldcg(const T* p) {
    return __ldcg(p);
}

// Receiver rows inside the fused kernel: a warp per receiver, lanes form the
// products into shared memory, lane 0 sums them in entry order (exact).
constexpr int F2D_CHUNK = 128;
template <typename T>
__device__ void fused2d_receivers(const Fused2DArgs<T>& a, const T* u, unsigned long long row, int gwarp, int nwarps,
                                  int lane, double* prod) {
    if (row >= a.n_rows) return;
    for (int r = gwarp; r < a.n_rec; r += nwarps) {
        const unsigned b = a.roff[r], e = a.roff[r + 1];
        double acc = 0.0;
        for (unsigned base = b; base < e; base += F2D_CHUNK) {
            const int m = (int)min((unsigned)F2D_CHUNK, e - base);
#pragma unroll
            for (int q = 0; q < F2D_CHUNK / 32; ++q) {
                const int k = q * 32 + lane;
                if (k < m) prod[k] = __dmul_rn(a.rw[base + k], static_cast<double>(u[a.ridx[base + k]]));
            }
            __syncwarp();
            if (lane == 0) {
#pragma unroll 8
                for (int k = 0; k < m; ++k) acc = __dadd_rn(acc, prod[k]);
            }
            __syncwarp();
        }
        if (lane == 0) a.seis[row * (unsigned long long)a.n_rec + r] = acc;
    }
}

template <typename T, int R, bool EXACT, bool VD = false>
__global__ void __launch_bounds__(256) step2d_fused(Fused2DArgs<T> a, int L, int cur0, int record, int k0) {
    using A = Ar<T, EXACT>;
    constexpr int V = 16 / sizeof(T);
    constexpr int HY = ((R + V - 1) / V) * V;  // X window halo, whole vectors
    constexpr int HV = HY / V;
    using VT = Vec<T, V>;
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    if (a.ctrl->abort) return;  // same value in every block: nothing here writes it
    // k0: steps of this chunk already taken before the launch (host-side split)
    const unsigned long long base = a.ctrl->step + (unsigned long long)k0, row_base = a.ctrl->row_base;
    const int nz = a.nz, nx = a.nx;
    const int nxv = (nx + V - 1) / V;  // vectors per row
    const int nitems = nz * nxv;
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    const int nth = gridDim.x * blockDim.x;
    const int lane = threadIdx.x & 31, gwarp = tid >> 5, nwarps = nth >> 5;
    const long long ld = a.ld;
    __shared__ double rec_prod[8][F2D_CHUNK];  // per warp (256 threads)
    double* prod = rec_prod[threadIdx.x >> 5];
    // Ghost cells are STORED: the thread that produces a point within R of a
    // face also writes its mirror copies into the new level (apply_boundary,
    // kernel.hpp:84-97: Dirichlet -u, Neumann +u, none 0), so every item reads
    // plain 16-byte vectors.  grid.sync() ends with an L1 invalidate
    // (CCTL.IVALL): cached loads never see a stale line of an earlier step.
    for (int k = 0; k < L; ++k) {
        const T* u = a.lvl[cur0 ^ (k & 1)];
        T* out = a.lvl[1 ^ cur0 ^ (k & 1)];
        const unsigned long long n = base + (unsigned long long)k;
        for (int item = tid; item < ((a.dbg & 1) ? 0 : nitems); item += nth) {
            const int z = item / nxv;
            const int x0 = (item - z * nxv) * V;
            const long long i0 = a.origin + (long long)z * ld + x0;
            const VT c = *reinterpret_cast<const VT*>(u + i0);
            T lz[V], lx[V], res[V];
            T dz[VD ? V : 1], dx[VD ? V : 1];
#pragma unroll
            for (int e = 0; e < V; ++e) {
                lz[e] = lx[e] = A::mul(a.v[0], c.e[e]);
                if constexpr (VD) dz[e] = dx[e] = T(0);
            }
            T w[2 * HY + V];
#pragma unroll
            for (int q = 0; q < 2 * HV + 1; ++q) {
                const VT t = *reinterpret_cast<const VT*>(u + i0 - HY + q * V);
#pragma unroll
                for (int e = 0; e < V; ++e) w[q * V + e] = t.e[e];
            }
#pragma unroll
            for (int j = 1; j <= R; ++j) {
                const VT zp = *reinterpret_cast<const VT*>(u + i0 + j * ld);
                const VT zm = *reinterpret_cast<const VT*>(u + i0 - j * ld);
#pragma unroll
                for (int e = 0; e < V; ++e) {
                    lz[e] = A::add(lz[e], A::mul(a.v[j], A::add(zp.e[e], zm.e[e])));
                    lx[e] = A::add(lx[e], A::mul(a.v[j], A::add(w[HY + e + j], w[HY + e - j])));
                }
                if constexpr (VD) {  // sweep_2d<true>, kernel.hpp:365-373
#pragma unroll
                    for (int e = 0; e < V; ++e) {
                        dz[e] = A::add(dz[e], A::mul(a.w1[j - 1], A::sub(zp.e[e], zm.e[e])));
                        dx[e] = A::add(dx[e], A::mul(a.w1[j - 1], A::sub(w[HY + e + j], w[HY + e - j])));
                    }
                }
            }
            const VT pv = *reinterpret_cast<const VT*>(out + i0);
            const VT cv = ldg16(a.c2dt2 + i0);
            const VT ev = ldg16(a.eta + i0);
            VT g0v, g1v;
            if constexpr (VD) {
                g0v = ldg16(a.grad[0] + i0);
                g1v = ldg16(a.grad[1] + i0);
            }
#pragma unroll
            for (int e = 0; e < V; ++e) {
                T rhs = A::add(A::mul(lz[e], a.ih[0]), A::mul(lx[e], a.ih[1]));
                if constexpr (VD)
                    rhs = A::sub(rhs, A::add(A::mul(A::mul(g0v.e[e], dz[e]), a.i2h[0]),
                                             A::mul(A::mul(g1v.e[e], dx[e]), a.i2h[1])));
                res[e] = time_update<T, EXACT>(rhs, c.e[e], cv.e[e], pv.e[e], ev.e[e], a.dt);
            }
            const bool near = z <= R || z >= nz - 1 - R || x0 <= R || x0 + V - 1 >= nx - 1 - R;
#pragma unroll
            for (int e = 0; e < V; ++e) {
                const int x = x0 + e;
                if (x >= nx) break;
                const int t = a.tmap[z * nx + x];
                if (t) {  // inject, kernel.hpp:429-438 (entries in the reference's order)
                    using AX = Ar<T, true>;
                    const double amp = n < a.n_wavelet ? a.wavelet[n] : 0.0;
                    T om, iop = T(1);
                    if (ev.e[e] != T(0)) damping_factors(ev.e[e], a.dt, om, iop);
                    for (unsigned q = a.ent_off[t - 1]; q < a.ent_off[t]; ++q)
                        res[e] = AX::add(res[e], AX::mul(AX::mul(cv.e[e], static_cast<T>(__dmul_rn(a.ent_w[q], amp))), iop));
                }
                if (near) {
                    if ((z == 0 && a.gf[0][0] < 0) || (z == nz - 1 && a.gf[0][1] < 0) || (x == 0 && a.gf[1][0] < 0) ||
                        (x == nx - 1 && a.gf[1][1] < 0))
                        res[e] = T(0);
                    auto put = [&](int zz, int xx, int f) {
                        out[a.origin + (long long)zz * ld + xx] = f == 0 ? T(0) : (f < 0 ? -res[e] : res[e]);
                    };
                    if (z >= 1 && z <= R) put(-z, x, a.gf[0][0]);
                    if (z >= nz - 1 - R && z <= nz - 2) put(2 * (nz - 1) - z, x, a.gf[0][1]);
                    if (x >= 1 && x <= R) put(z, -x, a.gf[1][0]);
                    if (x >= nx - 1 - R && x <= nx - 2) put(z, 2 * (nx - 1) - x, a.gf[1][1]);
                }
            }
            if (x0 + V <= nx) {
                VT rv;
#pragma unroll
                for (int e = 0; e < V; ++e) rv.e[e] = res[e];
                st16(out + i0, rv);
            } else {
                for (int e = 0; e < V && x0 + e < nx; ++e) out[i0 + e] = res[e];
            }
        }
        if (record && k > 0 && !(a.dbg & 2))
            fused2d_receivers(a, u, base + (unsigned long long)k - row_base, gwarp, nwarps, lane, prod);
        grid.sync();
    }
    if (record)
        fused2d_receivers(a, a.lvl[cur0 ^ (L & 1)], base + (unsigned long long)L - row_base, gwarp, nwarps, lane, prod);
}

// ---------------------------------------------------------------------------
// 2D, shared-memory resident (FDW_KERNEL_FUSED2D, constant density): one
// persistent cooperative launch per chunk; every CTA keeps ONE block of the
// grid -- both levels with a radius-R halo, c2dt2 and the two damping factors
// -- in shared memory for the whole chunk.  Per step only the block's boundary
// strips go through global memory (L2): the owner stores them into the
// level's natural positions, and after the grid barrier each neighbour loads
// them as its halo; physical faces are mirrored from the block itself
// (apply_boundary, kernel.hpp:67-102).  Point sources of the block are
// applied in smem (kernel.hpp:429-438); receiver taps are copied to a tap
// buffer and summed in entry order after the barrier (acquisition.hpp:
// 150-161).  At the chunk's end the block (and its face ghosts) goes back to
// global, so the level arrays hold exactly what the step-by-step kernels
// leave.  Same arithmetic and association as sweep_2d (kernel.hpp:344-379).
template <typename T>
struct Res2DArgs {
    T* lvl[2];
    const T* __restrict__ c2dt2;
    const T* __restrict__ eta;
    T v[11];
    T ih[2];
    double dt;
    long long ld, origin;
    int nz, nx;
    int gf[2][2];        // mirror factor per face: -1 Dirichlet, +1 Neumann, 0 none
    int BZ, xb;          // block rows; blocks per grid row (block b = zb_idx * xb + xb_idx)
    // point sources: per-block CSR over the merged targets: target index and
    // res2d_pack(rr, cc) block-local coordinates (bit 22: inside the block;
    // otherwise in its R-wide ring, used by the two-step kernel)
    const int* blk_toff;
    const int* blk_tgt;
    const int* blk_tpos;
    const unsigned* ent_off;
    const double* ent_w;
    const double* wavelet;
    unsigned long long n_wavelet;
    // receivers: per-block CSR of taps, packed (res2d_pack(rr, cc) << 2 | factor + 1);
    // tap q of the concatenated lists goes to tapbuf[q]; entry e reads tap_ix[e]
    const int* blk_roff;
    const int* blk_rpack;
    const int* tap_ix;
    int tapcap;          // taps cached in shared memory per block (0: read the list from global)
    T* tapbuf;           // [2][n_ent]
    int n_ent;
    const unsigned* roff;
    const double* rw;
    double* seis;
    int n_rec;
    unsigned long long n_rows;
    Ctrl* ctrl;
    // two-step kernel only: strip / halo exchange buffers (level-shaped, same
    // origin and pitch as the levels), alternated by pair parity
    T* hbuf[2];
};

// block-local coordinates (rr, cc in [-512, 1536)) packed into 22 bits
__host__ __device__ __forceinline__ int res2d_pack(int rr, int cc) { return ((rr + 512) << 11) | (cc + 512); }
__host__ __device__ __forceinline__ int res2d_rr(int pk) { return ((pk >> 11) & 2047) - 512; }
__host__ __device__ __forceinline__ int res2d_cc(int pk) { return (pk & 2047) - 512; }
constexpr int RES2D_IN_BLOCK = 1 << 22;

template <typename T, int R>
struct Res2DShape {
    static constexpr int V = 16 / (int)sizeof(T);
    static constexpr int TX = 16 * V;                      // block columns
    static constexpr int HY = ((R + V - 1) / V) * V;       // X halo, whole vectors
    static constexpr int UW = TX + 2 * HY;                 // smem row pitch of a level
    static __host__ __device__ constexpr int rows(int BZ) { return BZ + 2 * R; }
    static __host__ __device__ constexpr size_t smem(int BZ, int tapcap = 0) {
        return (size_t)(2 * rows(BZ) * UW + 3 * BZ * TX) * sizeof(T) + 8 * F2D_CHUNK * sizeof(double) +
               (size_t)tapcap * sizeof(int);
    }
};

template <typename T, int R, bool EXACT>
__global__ void __launch_bounds__(256) step2d_resident(Res2DArgs<T> a, int L, int cur0, int record, int k0) {
    using A = Ar<T, EXACT>;
    using S = Res2DShape<T, R>;
    constexpr int V = S::V, TX = S::TX, HY = S::HY, UW = S::UW, HV = HY / V;
    using VT = Vec<T, V>;
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    if (a.ctrl->abort) return;  // same value in every block: nothing here writes it
    extern __shared__ __align__(16) unsigned char sm_raw[];
    const int BZ = a.BZ, ROWS = S::rows(BZ);
    T* const su0 = reinterpret_cast<T*>(sm_raw);
    T* const su1 = su0 + ROWS * UW;
    T* sc = su1 + ROWS * UW;  // c2dt2, om, iop: BZ x TX
    T* som = sc + BZ * TX;
    T* siop = som + BZ * TX;
    double* prod = reinterpret_cast<double*>(siop + BZ * TX) + (threadIdx.x >> 5) * F2D_CHUNK;
    int* stap = reinterpret_cast<int*>(reinterpret_cast<double*>(siop + BZ * TX) + 8 * F2D_CHUNK);

    const int nz = a.nz, nx = a.nx;
    const long long ld = a.ld;
    const int bzi = blockIdx.x / a.xb, bxi = blockIdx.x % a.xb;
    const int z0 = bzi * BZ, x0 = bxi * TX;
    const int bz = min(BZ, nz - z0), bx = min(TX, nx - x0);  // valid rows / columns
    const int tid = threadIdx.x, tcv = tid & 15, trow = tid >> 4;
    // k0: steps of this chunk already taken by an earlier launch (two-step kernel)
    const unsigned long long base = a.ctrl->step + (unsigned long long)k0, row_base = a.ctrl->row_base;
    auto gidx = [&](int z, int x) { return a.origin + (long long)z * ld + x; };
    auto sidx = [&](int z, int x) { return (z - z0 + R) * UW + (x - x0 + HY); };  // smem offset of (z, x)
    const bool top = z0 == 0, bot = z0 + bz == nz, lef = x0 == 0, rig = x0 + bx == nx;
    auto mir = [](int f, T v) { return f == 0 ? T(0) : (f < 0 ? -v : v); };

    // ---- chunk start: both levels' valid region, the current level's halo
    // (stored ghosts on faces: a caller-uploaded level's ghosts are used as
    // given, kernel.hpp:344-379 reads them), and the constant fields ----
    for (int i = tid; i < ROWS * UW; i += 256) {
        const int r = i / UW, cc = i % UW;
        const int z = z0 - R + r, x = x0 - HY + cc;
        const bool inz = z >= -R && z < nz + R, inx = x >= -HY && x < nx + HY;
        T c = T(0), p = T(0);
        const bool valid = z >= z0 && z < z0 + bz && x >= x0 && x < x0 + bx;
        const bool halo = (z >= z0 && z < z0 + bz && ((x >= x0 - HY && x < x0) || (x >= x0 + bx && x < x0 + bx + HY))) ||
                          (x >= x0 && x < x0 + bx && ((z >= z0 - R && z < z0) || (z >= z0 + bz && z < z0 + bz + R)));
        if (inz && inx && (valid || halo)) c = a.lvl[cur0][gidx(z, x)];
        if (valid) p = a.lvl[cur0 ^ 1][gidx(z, x)];
        su0[i] = c;
        su1[i] = p;
    }
    for (int i = tid; i < BZ * TX; i += 256) {
        const int r = i / TX, cc = i % TX;
        T c2 = T(0), om = T(1), iop = T(1);
        if (r < bz && cc < bx) {
            const long long g = gidx(z0 + r, x0 + cc);
            c2 = a.c2dt2[g];
            const T e = a.eta[g];
            if (e != T(0)) damping_factors(e, a.dt, om, iop);
        }
        sc[i] = c2;
        som[i] = om;
        siop[i] = iop;
    }
    __syncthreads();

    const int nt0 = a.blk_toff[blockIdx.x], nt1 = a.blk_toff[blockIdx.x + 1];
    const int nr0 = a.blk_roff[blockIdx.x], nr1 = a.blk_roff[blockIdx.x + 1];
    const bool tap_cached = record && nr1 - nr0 <= a.tapcap;
    if (tap_cached)
        for (int q = nr0 + tid; q < nr1; q += 256) stap[q - nr0] = a.blk_rpack[q];
    const int lane = tid & 31, wib = tid >> 5;
    // Receivers (acquisition.hpp:150-161): receiver r belongs to CTA r % grid,
    // warp r / grid, so every CTA carries an equal share.  The taps of row k
    // are loaded at the start of step k+1 and summed after its compute, so the
    // L2 latency hides behind the sweep; lane 0 sums in entry order (double,
    // no FMA), exactly the reference's association.
    constexpr int TPL = F2D_CHUNK / 32;  // taps per lane on the fast path
    const int r_fast = (int)blockIdx.x + (int)gridDim.x * wib;
    const bool has_fast = record && r_fast < a.n_rec;
    unsigned rb = 0, re = 0;
    double wv[TPL];
    int ti[TPL];
    if (has_fast) {
        rb = a.roff[r_fast];
        re = a.roff[r_fast + 1];
#pragma unroll
        for (int q = 0; q < TPL; ++q) {
            const unsigned kk = rb + (unsigned)(q * 32 + lane);
            wv[q] = kk < re ? a.rw[kk] : 0.0;
            ti[q] = kk < re ? a.tap_ix[kk] : 0;
        }
    }
    const bool fast_ok = re - rb <= (unsigned)F2D_CHUNK;
    auto rec_slow = [&](int rcv, const T* tb, unsigned long long row) {  // any tap count, global loads
        const unsigned b0 = a.roff[rcv], e = a.roff[rcv + 1];
        double acc = 0.0;
        for (unsigned c0 = b0; c0 < e; c0 += F2D_CHUNK) {
            const int m = (int)min((unsigned)F2D_CHUNK, e - c0);
#pragma unroll
            for (int q = 0; q < TPL; ++q) {
                const int kk = q * 32 + lane;
                if (kk < m) prod[kk] = __dmul_rn(a.rw[c0 + kk], static_cast<double>(__ldcg(tb + a.tap_ix[c0 + kk])));
            }
            __syncwarp();
            if (lane == 0) {
#pragma unroll 8
                for (int kk = 0; kk < m; ++kk) acc = __dadd_rn(acc, prod[kk]);
            }
            __syncwarp();
        }
        if (lane == 0) a.seis[row * (unsigned long long)a.n_rec + rcv] = acc;
    };
    // row of the state after step kk of this chunk
    auto rec_row = [&](int kk) { return base + (unsigned long long)kk + 1 - row_base; };

    for (int k = 0; k < L; ++k) {
        const T* U = (k & 1) ? su1 : su0;
        T* O = (k & 1) ? su0 : su1;
        T* gout = a.lvl[cur0 ^ (k & 1) ^ 1];
        const unsigned long long n = base + (unsigned long long)k;
        // ---- taps of the previous step's row, in flight during the sweep ----
        T tv[TPL];
        const bool rec_prev = record && k > 0 && rec_row(k - 1) < a.n_rows;
        if (rec_prev && has_fast && fast_ok) {
            const T* tb = a.tapbuf + (size_t)((k - 1) & 1) * a.n_ent;
#pragma unroll
            for (int q = 0; q < TPL; ++q) {
                const unsigned kk = rb + (unsigned)(q * 32 + lane);
                tv[q] = kk < re ? __ldcg(tb + ti[q]) : T(0);
            }
        }
        // ---- sweep of the block (valid points only) ----
        for (int r = trow; r < bz; r += 16) {
            const int xc = tcv * V;
            if (xc >= bx) continue;
            const int o = (r + R) * UW + HY + xc;
            const VT c = *reinterpret_cast<const VT*>(U + o);
            T lz[V], lx[V], res[V];
#pragma unroll
            for (int e = 0; e < V; ++e) lz[e] = lx[e] = A::mul(a.v[0], c.e[e]);
            T w[2 * HY + V];
#pragma unroll
            for (int q = 0; q < 2 * HV + 1; ++q) {
                const VT t = *reinterpret_cast<const VT*>(U + o - HY + q * V);
#pragma unroll
                for (int e = 0; e < V; ++e) w[q * V + e] = t.e[e];
            }
#pragma unroll
            for (int j = 1; j <= R; ++j) {
                const VT zp = *reinterpret_cast<const VT*>(U + o + j * UW);
                const VT zm = *reinterpret_cast<const VT*>(U + o - j * UW);
#pragma unroll
                for (int e = 0; e < V; ++e) {
                    lz[e] = A::add(lz[e], A::mul(a.v[j], A::add(zp.e[e], zm.e[e])));
                    lx[e] = A::add(lx[e], A::mul(a.v[j], A::add(w[HY + e + j], w[HY + e - j])));
                }
            }
            const int po = r * TX + xc;
            const VT pv = *reinterpret_cast<const VT*>(O + o);
            const VT cv = *reinterpret_cast<const VT*>(sc + po);
            const VT omv = *reinterpret_cast<const VT*>(som + po);
            const VT iov = *reinterpret_cast<const VT*>(siop + po);
            const int z = z0 + r;
#pragma unroll
            for (int e = 0; e < V; ++e) {
                const T rhs = A::add(A::mul(lz[e], a.ih[0]), A::mul(lx[e], a.ih[1]));
                const T t = A::add(A::mul(cv.e[e], rhs), A::mul(T(2), c.e[e]));
                // time_update (kernel.hpp:418-420): om = iop = 1 where eta = 0, exact identities
                res[e] = A::mul(A::sub(t, A::mul(omv.e[e], pv.e[e])), iov.e[e]);
                const int x = x0 + xc + e;
                if ((z == 0 && a.gf[0][0] < 0) || (z == nz - 1 && a.gf[0][1] < 0) || (x == 0 && a.gf[1][0] < 0) ||
                    (x == nx - 1 && a.gf[1][1] < 0))
                    res[e] = T(0);  // null-Dirichlet face nodes (kernel.hpp:87-88)
            }
            if (xc + V <= bx) {
                VT rv;
#pragma unroll
                for (int e = 0; e < V; ++e) rv.e[e] = res[e];
                *reinterpret_cast<VT*>(O + o) = rv;
            } else {
                for (int e = 0; e < V && xc + e < bx; ++e) O[o + e] = res[e];
            }
        }
        __syncthreads();
        // ---- point sources of the block, entries in the reference's order ----
        if (nt1 > nt0) {
            if (n < a.n_wavelet) {
                using AX = Ar<T, true>;
                const double amp = a.wavelet[n];
                for (int q = nt0 + tid; q < nt1; q += 256) {
                    const int t = a.blk_tgt[q], pk = a.blk_tpos[q];
                    if (!(pk & RES2D_IN_BLOCK)) continue;  // ring target (two-step kernel only)
                    const int r = res2d_rr(pk), cc = res2d_cc(pk), so = (r + R) * UW + (cc + HY);
                    const T c2 = sc[r * TX + cc], iop = siop[r * TX + cc];
                    T val = O[so];
                    for (unsigned e = a.ent_off[t]; e < a.ent_off[t + 1]; ++e)
                        val = AX::add(val, AX::mul(AX::mul(c2, static_cast<T>(__dmul_rn(a.ent_w[e], amp))), iop));
                    O[so] = val;
                }
            }
            __syncthreads();
        }
        // ---- boundary strips to global (the neighbours' halos), receiver taps ----
        {
            // top / bottom R rows (valid columns), if a neighbour reads them
            for (int i = tid; i < R * TX; i += 256) {
                const int rr = i / TX, cc = i % TX;
                if (cc >= bx) continue;
                if (!top) gout[gidx(z0 + rr, x0 + cc)] = O[sidx(z0 + rr, x0 + cc)];
                if (!bot) gout[gidx(z0 + bz - R + rr, x0 + cc)] = O[sidx(z0 + bz - R + rr, x0 + cc)];
            }
            // left / right HY columns (valid rows), whole vectors
            for (int i = tid; i < 2 * HV * BZ; i += 256) {
                const int side = i / (HV * BZ), rem = i % (HV * BZ), rr = rem / HV, q = rem % HV;
                if (rr >= bz || (side == 0 && lef) || (side == 1 && rig)) continue;
                const int z = z0 + rr, x = side == 0 ? x0 + q * V : x0 + TX - HY + q * V;
                *reinterpret_cast<VT*>(gout + gidx(z, x)) = *reinterpret_cast<const VT*>(O + sidx(z, x));
            }
            if (record) {
                T* tb = a.tapbuf + (size_t)(k & 1) * a.n_ent;
#pragma unroll 4
                for (int q = nr0 + tid; q < nr1; q += 256) {
                    const int pk = tap_cached ? stap[q - nr0] : a.blk_rpack[q];
                    const int c = pk >> 2;
                    tb[q] = mir((pk & 3) - 1, O[(res2d_rr(c) + R) * UW + res2d_cc(c) + HY]);
                }
            }
        }
        // ---- the previous step's row (its taps were loaded before the sweep) ----
        if (rec_prev) {
            const unsigned long long row = rec_row(k - 1);
            const T* tb = a.tapbuf + (size_t)((k - 1) & 1) * a.n_ent;
            if (has_fast && fast_ok) {
                const int m = (int)(re - rb);
#pragma unroll
                for (int q = 0; q < TPL; ++q) {
                    const int kk = q * 32 + lane;
                    if (kk < m) prod[kk] = __dmul_rn(wv[q], static_cast<double>(tv[q]));
                }
                __syncwarp();
                if (lane == 0) {
                    double acc = 0.0;
#pragma unroll 8
                    for (int kk = 0; kk < m; ++kk) acc = __dadd_rn(acc, prod[kk]);
                    a.seis[row * (unsigned long long)a.n_rec + r_fast] = acc;
                }
                __syncwarp();
            } else if (has_fast) {
                rec_slow(r_fast, tb, row);
            }
            for (int rcv = r_fast + (int)gridDim.x * 8; rcv < a.n_rec; rcv += (int)gridDim.x * 8)
                rec_slow(rcv, tb, row);
        }
        grid.sync();
        // ---- halo of the new level: neighbours' strips from global ----
        for (int i = tid; i < R * TX; i += 256) {
            const int rr = i / TX, cc = i % TX;
            if (cc >= bx) continue;
            T a0 = T(0), a1 = T(0);
            if (!top) a0 = __ldcg(gout + gidx(z0 - R + rr, x0 + cc));
            if (!bot) a1 = __ldcg(gout + gidx(z0 + bz + rr, x0 + cc));
            if (!top) O[sidx(z0 - R + rr, x0 + cc)] = a0;
            if (!bot) O[sidx(z0 + bz + rr, x0 + cc)] = a1;
        }
        for (int i = tid; i < HV * BZ; i += 256) {
            const int rr = i / HV, q = i % HV;
            if (rr >= bz) continue;
            const int z = z0 + rr;
            // left: whole vectors of the left neighbour's strip; right: this
            // block is full width (bx == TX) whenever a right neighbour exists
            VT l, r;
            if (!lef) l = ldcg16(gout + gidx(z, x0 - HY + q * V));
            if (!rig) r = ldcg16(gout + gidx(z, x0 + TX + q * V));
            if (!lef) *reinterpret_cast<VT*>(O + sidx(z, x0 - HY + q * V)) = l;
            if (!rig) *reinterpret_cast<VT*>(O + sidx(z, x0 + TX + q * V)) = r;
        }
        __syncthreads();
        // ---- physical faces: the new level's ghosts mirror the block
        // (apply_boundary, kernel.hpp:84-97; Z then X; corners never read) ----
        if (top || bot)
            for (int i = tid; i < R * TX; i += 256) {
                const int kk = i / TX + 1, cc = i % TX;
                if (cc >= bx) continue;
                if (top) O[sidx(-kk, x0 + cc)] = mir(a.gf[0][0], O[sidx(kk, x0 + cc)]);
                if (bot) O[sidx(nz - 1 + kk, x0 + cc)] = mir(a.gf[0][1], O[sidx(nz - 1 - kk, x0 + cc)]);
            }
        if (lef || rig)
            for (int i = tid; i < R * BZ; i += 256) {
                const int kk = i % R + 1, rr = i / R;
                if (rr >= bz) continue;
                const int z = z0 + rr;
                if (lef) O[sidx(z, -kk)] = mir(a.gf[1][0], O[sidx(z, kk)]);
                if (rig) O[sidx(z, nx - 1 + kk)] = mir(a.gf[1][1], O[sidx(z, nx - 1 - kk)]);
            }
        __syncthreads();
    }
    // ---- the last step's row (its taps are complete after the last barrier) ----
    if (record && L > 0 && rec_row(L - 1) < a.n_rows) {
        const T* tb = a.tapbuf + (size_t)((L - 1) & 1) * a.n_ent;
        for (int rcv = r_fast; rcv < a.n_rec; rcv += (int)gridDim.x * 8) rec_slow(rcv, tb, rec_row(L - 1));
    }
    // ---- chunk end: both levels' valid region and face ghosts back to global ----
    for (int s2 = 0; s2 < 2; ++s2) {
        T* g = a.lvl[cur0 ^ s2];
        const T* Ls = s2 ? su1 : su0;
        for (int i = tid; i < bz * bx; i += 256) {
            const int z = z0 + i / bx, x = x0 + i % bx;
            g[gidx(z, x)] = Ls[sidx(z, x)];
        }
        if (top || bot)
            for (int i = tid; i < 2 * R * bx; i += 256) {
                const int side = i / (R * bx), rem = i % (R * bx), kk = rem / bx + 1, x = x0 + rem % bx;
                if (side == 0 && top) g[gidx(-kk, x)] = Ls[sidx(-kk, x)];
                if (side == 1 && bot) g[gidx(nz - 1 + kk, x)] = Ls[sidx(nz - 1 + kk, x)];
            }
        if (lef || rig)
            for (int i = tid; i < 2 * R * bz; i += 256) {
                const int side = i / (R * bz), rem = i % (R * bz), kk = rem / bz + 1, z = z0 + rem % bz;
                if (side == 0 && lef) g[gidx(z, -kk)] = Ls[sidx(z, -kk)];
                if (side == 1 && rig) g[gidx(z, nx - 1 + kk)] = Ls[sidx(z, nx - 1 + kk)];
            }
    }
}

// ---------------------------------------------------------------------------
// Two steps per grid barrier (step2d_resident2): each block also computes the
// first step of a pair on an R-wide ring around itself (the neighbours'
// points, recomputed with the same operations and inputs, so bit-identical),
// which lets the second step run without an exchange.  Per pair the blocks
// exchange a 2R-wide halo of the newest level (corners included) and keep the
// ring of the intermediate level as the next pair's "previous" level.
// Odd chunk lengths finish with one step2d_resident launch.
template <typename T, int R>
struct Res2DShape2 {
    static constexpr int V = 16 / (int)sizeof(T);
    static constexpr int TX = 16 * V;
    static constexpr int H1 = ((R + V - 1) / V) * V;      // ring columns, whole vectors
    static constexpr int H2 = ((2 * R + V - 1) / V) * V;  // halo columns of the level slots
    static constexpr int UW = TX + 2 * H2;                // slot row pitch
    static constexpr int CW = TX + 2 * H1;                // coefficient row pitch (block + ring)
    static constexpr int NV1 = CW / V;                    // vectors per ring row
    static __host__ __device__ constexpr size_t smem(int BZ, int tapcap = 0) {
        return (size_t)(2 * (BZ + 4 * R) * UW + 3 * (BZ + 2 * R) * CW) * sizeof(T) +
               8 * F2D_CHUNK * sizeof(double) + (size_t)tapcap * sizeof(int);
    }
};

template <typename T, int R, bool EXACT>
__global__ void __launch_bounds__(256, 2) step2d_resident2(Res2DArgs<T> a, int L, int cur0, int record) {
    using A = Ar<T, EXACT>;
    using S = Res2DShape2<T, R>;
    constexpr int V = S::V, TX = S::TX, H1 = S::H1, H2 = S::H2, UW = S::UW, CW = S::CW;
    constexpr int HV = ((R + V - 1) / V);  // x-window vectors each side for the stencil
    constexpr int HW = HV * V;
    using VT = Vec<T, V>;
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    if (a.ctrl->abort) return;
    extern __shared__ __align__(16) unsigned char sm_raw[];
    const int BZ = a.BZ, ROWS = BZ + 4 * R, CROWS = BZ + 2 * R;
    T* const sU = reinterpret_cast<T*>(sm_raw);  // current level (2R halo)
    T* const sO = sU + ROWS * UW;                // previous / intermediate level (R ring)
    T* const sc = sO + ROWS * UW;                // c2dt2, om, iop on the block + ring
    T* const som = sc + CROWS * CW;
    T* const siop = som + CROWS * CW;
    double* prod = reinterpret_cast<double*>(siop + CROWS * CW) + (threadIdx.x >> 5) * F2D_CHUNK;
    int* stap = reinterpret_cast<int*>(reinterpret_cast<double*>(siop + CROWS * CW) + 8 * F2D_CHUNK);

    const int nz = a.nz, nx = a.nx;
    const long long ld = a.ld;
    const int bzi = blockIdx.x / a.xb, bxi = blockIdx.x % a.xb;
    const int z0 = bzi * BZ, x0 = bxi * TX;
    const int bz = min(BZ, nz - z0), bx = min(TX, nx - x0);
    const int tid = threadIdx.x;
    const unsigned long long base = a.ctrl->step, row_base = a.ctrl->row_base;
    auto gidx = [&](int z, int x) { return a.origin + (long long)z * ld + x; };
    auto sidx = [&](int z, int x) { return (z - z0 + 2 * R) * UW + (x - x0 + H2); };
    auto cidx = [&](int z, int x) { return (z - z0 + R) * CW + (x - x0 + H1); };
    const bool top = z0 == 0, bot = z0 + bz == nz, lef = x0 == 0, rig = x0 + bx == nx;
    auto mir = [](int f, T v) { return f == 0 ? T(0) : (f < 0 ? -v : v); };
    // ring extent inside the grid
    const int rz0 = max(z0 - R, 0), rz1 = min(z0 + bz + R, nz);
    const int rx0 = max(x0 - R, 0), rx1 = min(x0 + bx + R, nx);

    // ---- chunk start: current level with its 2R halo (stored ghosts on the
    // faces), previous level and the coefficients on the block + ring ----
    for (int i = tid; i < ROWS * UW; i += 256) {
        const int z = z0 - 2 * R + i / UW, x = x0 - H2 + i % UW;
        T c = T(0), p = T(0);
        if (z >= -R && z < nz + R && x >= -H2 && x < nx + H2) c = a.lvl[cur0][gidx(z, x)];
        if (z >= rz0 && z < rz1 && x >= rx0 && x < rx1) p = a.lvl[cur0 ^ 1][gidx(z, x)];
        sU[i] = c;
        sO[i] = p;
    }
    for (int i = tid; i < CROWS * CW; i += 256) {
        const int z = z0 - R + i / CW, x = x0 - H1 + i % CW;
        T c2 = T(0), om = T(1), iop = T(1);
        if (z >= 0 && z < nz && x >= 0 && x < nx) {
            const long long g = gidx(z, x);
            c2 = a.c2dt2[g];
            const T e = a.eta[g];
            if (e != T(0)) damping_factors(e, a.dt, om, iop);
        }
        sc[i] = c2;
        som[i] = om;
        siop[i] = iop;
    }
    const int nt0 = a.blk_toff[blockIdx.x], nt1 = a.blk_toff[blockIdx.x + 1];
    const int nr0 = a.blk_roff[blockIdx.x], nr1 = a.blk_roff[blockIdx.x + 1];
    const bool tap_cached = record && nr1 - nr0 <= a.tapcap;
    if (tap_cached)
        for (int q = nr0 + tid; q < nr1; q += 256) stap[q - nr0] = a.blk_rpack[q];
    __syncthreads();

    const int lane = tid & 31, wib = tid >> 5;
    constexpr int TPL = F2D_CHUNK / 32;
    const int r_fast = (int)blockIdx.x + (int)gridDim.x * wib;
    const bool has_fast = record && r_fast < a.n_rec;
    unsigned rb = 0, re = 0;
    double wv[TPL];
    int ti[TPL];
    if (has_fast) {
        rb = a.roff[r_fast];
        re = a.roff[r_fast + 1];
#pragma unroll
        for (int q = 0; q < TPL; ++q) {
            const unsigned kk = rb + (unsigned)(q * 32 + lane);
            wv[q] = kk < re ? a.rw[kk] : 0.0;
            ti[q] = kk < re ? a.tap_ix[kk] : 0;
        }
    }
    const bool fast_ok = re - rb <= (unsigned)F2D_CHUNK;
    auto rec_slow = [&](int rcv, const T* tb, unsigned long long row) {
        const unsigned b0 = a.roff[rcv], e = a.roff[rcv + 1];
        double acc = 0.0;
        for (unsigned c0 = b0; c0 < e; c0 += F2D_CHUNK) {
            const int m = (int)min((unsigned)F2D_CHUNK, e - c0);
#pragma unroll
            for (int q = 0; q < TPL; ++q) {
                const int kk = q * 32 + lane;
                if (kk < m) prod[kk] = __dmul_rn(a.rw[c0 + kk], static_cast<double>(__ldcg(tb + a.tap_ix[c0 + kk])));
            }
            __syncwarp();
            if (lane == 0) {
#pragma unroll 8
                for (int kk = 0; kk < m; ++kk) acc = __dadd_rn(acc, prod[kk]);
            }
            __syncwarp();
        }
        if (lane == 0) a.seis[row * (unsigned long long)a.n_rec + rcv] = acc;
    };
    auto rec_fast = [&](const T (&tv)[TPL], unsigned long long row) {
        const int m = (int)(re - rb);
#pragma unroll
        for (int q = 0; q < TPL; ++q) {
            const int kk = q * 32 + lane;
            if (kk < m) prod[kk] = __dmul_rn(wv[q], static_cast<double>(tv[q]));
        }
        __syncwarp();
        if (lane == 0) {
            double acc = 0.0;
#pragma unroll 8
            for (int kk = 0; kk < m; ++kk) acc = __dadd_rn(acc, prod[kk]);
            a.seis[row * (unsigned long long)a.n_rec + r_fast] = acc;
        }
        __syncwarp();
    };
    auto rec_row = [&](int kk) { return base + (unsigned long long)kk + 1 - row_base; };
    // 8 rows in flight: a pair's receiver sums run after the grid barrier
    // (beside the halo loads), so slot kk is free again only two pairs later
    auto tslot = [&](int kk) { return a.tapbuf + (size_t)(kk & 7) * a.n_ent; };

    // one step on the region [zA, zB) x vectors [vx0, vx1) (block-local vector
    // index, 0 = column x0 - H1): out <- in / prev, coefficient arrays at cidx
    auto sweep = [&](const T* In, T* Out, int zA, int zB, int vx0, int vx1, int xlo, int xhi) {
        const int nvr = vx1 - vx0;
        // (row, vector) of this thread's items, stepped without a division per item
        const int dz = 256 / nvr, dv = 256 % nvr;
        int zi = tid / nvr, vi = tid % nvr;
        for (int it = tid; it < (zB - zA) * nvr; it += 256) {
            const int z = zA + zi, xv = x0 - H1 + (vx0 + vi) * V;
            zi += dz;
            vi += dv;
            if (vi >= nvr) {
                vi -= nvr;
                ++zi;
            }
            if (xv + V <= xlo || xv >= xhi) continue;
            const int o = sidx(z, xv);
            const VT c = *reinterpret_cast<const VT*>(In + o);
            T lz[V], lx[V], res[V];
#pragma unroll
            for (int e = 0; e < V; ++e) lz[e] = lx[e] = A::mul(a.v[0], c.e[e]);
            T w[2 * HW + V];
#pragma unroll
            for (int q = 0; q < 2 * HV + 1; ++q) {
                const VT t = *reinterpret_cast<const VT*>(In + o - HW + q * V);
#pragma unroll
                for (int e = 0; e < V; ++e) w[q * V + e] = t.e[e];
            }
#pragma unroll
            for (int j = 1; j <= R; ++j) {
                const VT zp = *reinterpret_cast<const VT*>(In + o + j * UW);
                const VT zm = *reinterpret_cast<const VT*>(In + o - j * UW);
#pragma unroll
                for (int e = 0; e < V; ++e) {
                    lz[e] = A::add(lz[e], A::mul(a.v[j], A::add(zp.e[e], zm.e[e])));
                    lx[e] = A::add(lx[e], A::mul(a.v[j], A::add(w[HW + e + j], w[HW + e - j])));
                }
            }
            const int po = cidx(z, xv);
            const VT pv = *reinterpret_cast<const VT*>(Out + o);
            const VT cv = *reinterpret_cast<const VT*>(sc + po);
            const VT omv = *reinterpret_cast<const VT*>(som + po);
            const VT iov = *reinterpret_cast<const VT*>(siop + po);
#pragma unroll
            for (int e = 0; e < V; ++e) {
                const T rhs = A::add(A::mul(lz[e], a.ih[0]), A::mul(lx[e], a.ih[1]));
                const T t = A::add(A::mul(cv.e[e], rhs), A::mul(T(2), c.e[e]));
                res[e] = A::mul(A::sub(t, A::mul(omv.e[e], pv.e[e])), iov.e[e]);
                const int x = xv + e;
                if ((z == 0 && a.gf[0][0] < 0) || (z == nz - 1 && a.gf[0][1] < 0) || (x == 0 && a.gf[1][0] < 0) ||
                    (x == nx - 1 && a.gf[1][1] < 0))
                    res[e] = T(0);
            }
            if (xv >= xlo && xv + V <= xhi) {
                VT rv;
#pragma unroll
                for (int e = 0; e < V; ++e) rv.e[e] = res[e];
                *reinterpret_cast<VT*>(Out + o) = rv;
            } else {
                for (int e = 0; e < V; ++e)
                    if (xv + e >= xlo && xv + e < xhi) Out[o + e] = res[e];
            }
        }
    };
    // point sources: ring targets too when `ring` (entries in reference order)
    auto inject = [&](T* Out, unsigned long long n, bool ring) {
        if (nt1 > nt0) {
            if (n < a.n_wavelet) {
                using AX = Ar<T, true>;
                const double amp = a.wavelet[n];
                for (int q = nt0 + tid; q < nt1; q += 256) {
                    const int t = a.blk_tgt[q], pk = a.blk_tpos[q];
                    if (!ring && !(pk & RES2D_IN_BLOCK)) continue;
                    const int z = z0 + res2d_rr(pk), x = x0 + res2d_cc(pk);
                    const T c2 = sc[cidx(z, x)], iop = siop[cidx(z, x)];
                    T val = Out[sidx(z, x)];
                    for (unsigned e = a.ent_off[t]; e < a.ent_off[t + 1]; ++e)
                        val = AX::add(val, AX::mul(AX::mul(c2, static_cast<T>(__dmul_rn(a.ent_w[e], amp))), iop));
                    Out[sidx(z, x)] = val;
                }
            }
            __syncthreads();
        }
    };
    // physical faces: R-deep ghosts mirror the level over columns [cA, cB) /
    // rows [rA, rB) (apply_boundary, kernel.hpp:84-97)
    auto mirror = [&](T* F, int cA, int cB, int rA, int rB) {
        if (top || bot)
            for (int i = tid; i < R * (cB - cA); i += 256) {
                const int kk = i / (cB - cA) + 1, x = cA + i % (cB - cA);
                if (top) F[sidx(-kk, x)] = mir(a.gf[0][0], F[sidx(kk, x)]);
                if (bot) F[sidx(nz - 1 + kk, x)] = mir(a.gf[0][1], F[sidx(nz - 1 - kk, x)]);
            }
        if (lef || rig)
            for (int i = tid; i < R * (rB - rA); i += 256) {
                const int kk = i % R + 1, z = rA + i / R;
                if (lef) F[sidx(z, -kk)] = mir(a.gf[1][0], F[sidx(z, kk)]);
                if (rig) F[sidx(z, nx - 1 + kk)] = mir(a.gf[1][1], F[sidx(z, nx - 1 - kk)]);
            }
    };
    const int vr0 = (rx0 - (x0 - H1)) / V, vr1 = (rx1 - (x0 - H1) + V - 1) / V;  // ring vectors
    const int vb0 = H1 / V, vb1 = (H1 + bx + V - 1) / V;                         // block vectors

    for (int k = 0; k < L; k += 2) {  // L is even
        const unsigned long long n1 = base + (unsigned long long)k;
        // taps of the previous pair's two rows, in flight during the sweeps
        T tv0[TPL], tv1[TPL];
        const bool rec_prev = record && k > 0;
        if (rec_prev && has_fast && fast_ok) {
            const T* t0 = tslot(k - 2);
            const T* t1 = tslot(k - 1);
#pragma unroll
            for (int q = 0; q < TPL; ++q) {
                const unsigned kk = rb + (unsigned)(q * 32 + lane);
                tv0[q] = kk < re ? __ldcg(t0 + ti[q]) : T(0);
                tv1[q] = kk < re ? __ldcg(t1 + ti[q]) : T(0);
            }
        }
        // step 1 on block + ring: O <- (U, prev O)
        sweep(sU, sO, rz0, rz1, vr0, vr1, rx0, rx1);
        __syncthreads();
        inject(sO, n1, true);
        mirror(sO, x0, x0 + bx, z0, z0 + bz);
        __syncthreads();
        // step 2 on the block: U <- (O, prev U)
        sweep(sO, sU, z0, z0 + bz, vb0, vb1, x0, x0 + bx);
        __syncthreads();
        inject(sU, n1 + 1, false);
        // 2R-wide strips of the newest level; receiver taps of both rows
        // The strips go to a buffer the chunk-start loads never read, and pair j
        // uses buffer j & 1: a block overwrites pair j's strips only in pair
        // j + 2, after the barrier its neighbours reach once they loaded them.
        {
            T* g = a.hbuf[(k >> 1) & 1];
            for (int i = tid; i < 2 * R * TX; i += 256) {
                const int rr = i / TX, cc = i % TX;
                if (cc >= bx) continue;
                if (!top) g[gidx(z0 + rr, x0 + cc)] = sU[sidx(z0 + rr, x0 + cc)];
                if (!bot) g[gidx(z0 + bz - 2 * R + rr, x0 + cc)] = sU[sidx(z0 + bz - 2 * R + rr, x0 + cc)];
            }
            constexpr int H2V = H2 / V;
            for (int i = tid; i < 2 * H2V * BZ; i += 256) {
                const int side = i / (H2V * BZ), rem = i % (H2V * BZ), rr = rem / H2V, q = rem % H2V;
                if (rr >= bz || (side == 0 && lef) || (side == 1 && rig)) continue;
                const int z = z0 + rr, x = side == 0 ? x0 + q * V : x0 + TX - H2 + q * V;
                *reinterpret_cast<VT*>(g + gidx(z, x)) = *reinterpret_cast<const VT*>(sU + sidx(z, x));
            }
            if (record) {
                T* t0 = tslot(k);
                T* t1 = tslot(k + 1);
                for (int q = nr0 + tid; q < nr1; q += 256) {
                    const int pk = tap_cached ? stap[q - nr0] : a.blk_rpack[q];
                    const int c = pk >> 2, f = (pk & 3) - 1;
                    const int so = sidx(z0 + res2d_rr(c), x0 + res2d_cc(c));
                    t0[q] = mir(f, sO[so]);
                    t1[q] = mir(f, sU[so]);
                }
            }
        }
        // the previous pair's rows (taps loaded before the sweeps); run while
        // the halo loads after the grid barrier are in flight
        auto recv_prev = [&]() {
        if (rec_prev) {
            if (has_fast && fast_ok && re - rb <= (unsigned)(F2D_CHUNK / 2) && rec_row(k - 1) < a.n_rows) {
                // both rows at once: products in the two halves of the warp's
                // buffer, lanes 0 and 16 run the two sequential sums side by side
                const int m = (int)(re - rb);
#pragma unroll
                for (int q = 0; q < TPL; ++q) {
                    const int kk = q * 32 + lane;
                    if (kk < m) {
                        prod[kk] = __dmul_rn(wv[q], static_cast<double>(tv0[q]));
                        prod[F2D_CHUNK / 2 + kk] = __dmul_rn(wv[q], static_cast<double>(tv1[q]));
                    }
                }
                __syncwarp();
                if (lane == 0 || lane == 16) {
                    const double* pp = prod + (lane ? F2D_CHUNK / 2 : 0);
                    double acc = 0.0;
#pragma unroll 8
                    for (int kk = 0; kk < m; ++kk) acc = __dadd_rn(acc, pp[kk]);
                    a.seis[rec_row(k - (lane ? 1 : 2)) * (unsigned long long)a.n_rec + r_fast] = acc;
                }
                __syncwarp();
            } else if (has_fast && fast_ok) {
                if (rec_row(k - 2) < a.n_rows) rec_fast(tv0, rec_row(k - 2));
                if (rec_row(k - 1) < a.n_rows) rec_fast(tv1, rec_row(k - 1));
            } else if (has_fast) {
                if (rec_row(k - 2) < a.n_rows) rec_slow(r_fast, tslot(k - 2), rec_row(k - 2));
                if (rec_row(k - 1) < a.n_rows) rec_slow(r_fast, tslot(k - 1), rec_row(k - 1));
            }
            for (int rcv = r_fast + (int)gridDim.x * 8; rcv < a.n_rec; rcv += (int)gridDim.x * 8) {
                if (rec_row(k - 2) < a.n_rows) rec_slow(rcv, tslot(k - 2), rec_row(k - 2));
                if (rec_row(k - 1) < a.n_rows) rec_slow(rcv, tslot(k - 1), rec_row(k - 1));
            }
        }
        };
        grid.sync();
        // 2R halo of the newest level (corners too): neighbours' strips.  Only
        // the halo is enumerated (2R rows above and below over the slot width,
        // H2 columns left and right of the block rows); each thread issues its
        // L2 loads in batches before storing any of them, and the first batch
        // is in flight during the previous pair's receiver sums.
        {
            const T* g = a.hbuf[(k >> 1) & 1];
            constexpr int UWV = UW / V, H2V = H2 / V, B = 2;
            const int n_rows = 2 * R * UWV, n_tot = 2 * n_rows + bz * 2 * H2V;
            for (int i0 = 0; i0 < n_tot; i0 += B * 256) {
                VT hv[B];
                int ho[B];
#pragma unroll
                for (int u = 0; u < B; ++u) {
                    const int i = i0 + u * 256 + tid;
                    ho[u] = -1;
                    if (i >= n_tot) continue;
                    int z, x;
                    if (i < 2 * n_rows) {  // rows above, then rows below the block
                        const int j = i < n_rows ? i : i - n_rows;
                        z = (i < n_rows ? z0 - 2 * R : z0 + bz) + j / UWV;
                        x = x0 - H2 + (j % UWV) * V;
                    } else {  // left / right columns of the block rows
                        const int j = i - 2 * n_rows, q = j % (2 * H2V);
                        z = z0 + j / (2 * H2V);
                        x = q < H2V ? x0 - H2 + q * V : x0 + TX + (q - H2V) * V;
                    }
                    // own block (incl. its columns past nx), ghost rows / columns: skipped
                    if ((z >= z0 && z < z0 + bz && x >= x0 && x < x0 + TX) || z < 0 || z >= nz || x < 0 ||
                        x + V > nx)
                        continue;
                    hv[u] = ldcg16(g + gidx(z, x));
                    ho[u] = sidx(z, x);
                }
                if (i0 == 0) recv_prev();
#pragma unroll
                for (int u = 0; u < B; ++u)
                    if (ho[u] >= 0) *reinterpret_cast<VT*>(sU + ho[u]) = hv[u];
            }
            if (n_tot <= 0) recv_prev();
        }
        __syncthreads();
        // faces of the newest level, over the block + ring (the next step 1 reads them there)
        mirror(sU, rx0, rx1, rz0, rz1);
        __syncthreads();
    }
    // the last pair's rows
    if (record && L >= 2) {
        for (int rcv = r_fast; rcv < a.n_rec; rcv += (int)gridDim.x * 8) {
            if (rec_row(L - 2) < a.n_rows) rec_slow(rcv, tslot(L - 2), rec_row(L - 2));
            if (rec_row(L - 1) < a.n_rows) rec_slow(rcv, tslot(L - 1), rec_row(L - 1));
        }
    }
    // chunk end: both levels' block and face ghosts back to global
    for (int s2 = 0; s2 < 2; ++s2) {
        T* g = a.lvl[cur0 ^ s2];
        const T* F = s2 ? sO : sU;
        for (int i = tid; i < bz * TX; i += 256) {
            const int z = z0 + i / TX, x = x0 + i % TX;
            if (x < x0 + bx) g[gidx(z, x)] = F[sidx(z, x)];
        }
        if (top || bot)
            for (int i = tid; i < R * TX; i += 256) {
                const int kk = i / TX + 1, x = x0 + i % TX;
                if (x >= x0 + bx) continue;
                if (top) g[gidx(-kk, x)] = F[sidx(-kk, x)];
                if (bot) g[gidx(nz - 1 + kk, x)] = F[sidx(nz - 1 + kk, x)];
            }
        if (lef || rig)
            for (int i = tid; i < R * BZ; i += 256) {
                const int kk = i % R + 1, z = z0 + i / R;
                if (z >= z0 + bz) continue;
                if (lef) g[gidx(z, -kk)] = F[sidx(z, -kk)];
                if (rig) g[gidx(z, nx - 1 + kk)] = F[sidx(z, nx - 1 + kk)];
            }
    }
}

// ---------------------------------------------------------------------------
// apply_boundary, kernel.hpp:67-102, as ONE launch per step.  Threads cover
// every ghost cell of the level (global Z faces only for slabs; internal ghost
// planes arrive by halo exchange) plus every node of an active null-Dirichlet
// face.  A ghost cell takes prod(f_a) * u(m): m mirrors each ghost coordinate
// about its face (f = -1 Dirichlet, +1 Neumann), 0 if any side is "none" or if
// m lies on a Dirichlet face (that node is zeroed in the same pass).  This is
// the closed form of the reference's axis-by-axis passes (values equal; only
// the sign of a zero may differ in ghost cells, which never reaches an
// extended point).
struct BoxRegion {
    int p0[3];      // first padded coordinate (z, x, y)
    int n[3];       // extent
    int zero_face;  // 1: Dirichlet face nodes (write 0); 0: ghost cells
};

struct BoundaryArgs {
    int nd;
    int h;
    int ext[3];            // extended extents (local Z)
    signed char f[3][2];   // -1 Dirichlet, +1 Neumann, 0 none
    unsigned char act[3][2];
    long long s[3];        // strides (plane, ld, 1) / 2D (ld, 1, 0)
    long long origin_pad;  // offset of padded (0,0,0)
    int n_regions;
    BoxRegion reg[12];
    long long start[13];   // prefix sums of region sizes
};

template <typename T>
__global__ void __launch_bounds__(256) boundary_kernel(T* f, BoundaryArgs b, const Ctrl* ctrl) {
    // blockIdx.y selects the region; blocks past its size exit
    if (ctrl && ctrl->abort) return;
    const BoxRegion& R = b.reg[blockIdx.y];
    const int size = R.n[0] * R.n[1] * R.n[2];
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= size) return;
    const int k2 = q % R.n[2];
    const int r12 = q / R.n[2];
    const int k1 = r12 % R.n[1];
    const int k0 = r12 / R.n[1];
    const int p0 = R.p0[0] + k0, p1 = R.p0[1] + k1, p2 = R.p0[2] + k2;
    T* dst = f + b.origin_pad + (long long)p0 * b.s[0] + (long long)p1 * b.s[1] + (long long)p2 * b.s[2];
    if (R.zero_face) {
        *dst = T(0);
        return;
    }
    int fac = 1;
    bool on_dir = false;
    long long src = b.origin_pad;
    const int p[3] = {p0, p1, p2};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        if (a < b.nd) {
            const int e = p[a] - b.h;  // extended coordinate
            int m = e;
            if (e < 0) {
                m = -e;
                fac *= b.f[a][0];
            } else if (e >= b.ext[a]) {
                m = 2 * (b.ext[a] - 1) - e;
                fac *= b.f[a][1];
            }
            on_dir |= (b.act[a][0] && b.f[a][0] < 0 && m == 0) ||
                      (b.act[a][1] && b.f[a][1] < 0 && m == b.ext[a] - 1);
            src += (long long)(m + b.h) * b.s[a];
        }
    }
    if (fac == 0 || on_dir) {
        *dst = T(0);
    } else {
        const T v = f[src];
        *dst = fac < 0 ? -v : v;
    }
}

// density_log_gradient, kernel.hpp:104-136, one axis: over extended points
// g = T(acc * inv2h / double(rho)), acc = sum_j w_j (double(rho+) - double(rho-)).
template <typename T>
__global__ void density_grad_kernel(const T* __restrict__ rho, T* __restrict__ g, long long origin, long long ld,
                                    long long plane, int nz, int nx, int ny, long long stride, int R, double w0,
                                    double w1, double w2, double w3, double w4, double w5, double w6, double w7,
                                    double w8, double w9, double inv2h) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long n = (long long)nz * nx * ny;
    if (t >= n) return;
    const int y = (int)(t % ny);
    const long long r2 = t / ny;
    const int x = (int)(r2 % nx), z = (int)(r2 / nx);
    const long long i = origin + (long long)z * plane + (long long)x * ld + y;
    const double w[10] = {w0, w1, w2, w3, w4, w5, w6, w7, w8, w9};
    double acc = 0.0;
    for (int j = 1; j <= R; ++j)
        acc = __dadd_rn(acc, __dmul_rn(w[j - 1], __dsub_rn(static_cast<double>(rho[i + j * stride]),
                                                           static_cast<double>(rho[i - j * stride]))));
    g[i] = static_cast<T>(__ddiv_rn(__dmul_rn(acc, inv2h), static_cast<double>(rho[i])));
}

// Halo epoch halves as separate launches, for operations whose kernels do not
// wait / publish themselves (stored-ghost and non-TMA sweeps, uploads,
// refresh_boundary, point sources mirrored into a neighbour).
__global__ void peer_wait_kernel(PeerArgs p, int honor_abort) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (honor_abort && p.ctrl->abort) return;
    peer_wait_neighbours(p);
}
__global__ void peer_publish_kernel(PeerArgs p, int honor_abort) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (honor_abort && p.ctrl->abort) return;
    peer_publish(p);
}

// Teardown handshake: before a rank frees the memory its neighbours map, it
// waits (bounded; no abort latched) until every rank has finished the halo and
// health epochs this rank went through, so no neighbour store is in flight.
__global__ void peer_quiesce(PeerArgs p, unsigned long long timeout_ns) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const unsigned long long t0 = global_ns();
    auto reach = [&](const unsigned long long* f, unsigned long long want) {
        while (ld_acquire_sys(f) < want) {
            if (ld_volatile_u32(&p.self->abort_word) || global_ns() - t0 > timeout_ns) return false;
            __nanosleep(1024);
        }
        return true;
    };
    for (int s = 0; s < p.world; ++s) {
        if (s == p.rank) continue;
        if ((s == p.rank - 1 || s == p.rank + 1) && !reach(&p.self->halo_flag[s], p.self->halo_epoch)) return;
        if (!reach(&p.self->health_flag[s], p.self->health_epoch)) return;
    }
}

// Health reduction across ranks (kernel.hpp:456-458 over all slabs): every
// rank posts its (first non-finite index, max |u| bits, kind) into each other
// rank's inbox slot (double-buffered by epoch parity) and signals; the reduce
// half waits for all ranks and combines locally.  Two launches so that a
// host-ordered group can put its cross-rank event between them.
__global__ void peer_health_post(PeerArgs p, int honor_abort) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (honor_abort && p.ctrl->abort) return;
    const unsigned long long e = p.self->health_epoch + 1;
    const int slot = (int)(e & 1);
    const unsigned long long idx = p.ctrl->bad_idx, mx = p.ctrl->max_bits;
    const unsigned int kind = p.ctrl->kind;
    for (int s = 0; s < p.world; ++s) {
        if (s == p.rank) continue;
        PeerSync* d = p.peer[s];
        d->in_idx[slot][p.rank] = idx;
        d->in_max[slot][p.rank] = mx;
        d->in_kind[slot][p.rank] = kind;
    }
    __threadfence_system();
    for (int s = 0; s < p.world; ++s)
        if (s != p.rank) st_release_sys(&p.peer[s]->health_flag[p.rank], e);
}
__global__ void peer_health_reduce(PeerArgs p, int honor_abort) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (honor_abort && p.ctrl->abort) return;
    const unsigned long long e = p.self->health_epoch + 1;
    p.self->health_epoch = e;
    const int slot = (int)(e & 1);
    unsigned long long r_idx = p.ctrl->bad_idx, r_max = p.ctrl->max_bits;
    unsigned int r_kind = p.ctrl->kind;
    for (int s = 0; s < p.world; ++s) {
        if (s == p.rank) continue;
        if (!peer_wait_flag(&p.self->health_flag[s], e, p.peer, p.world, p.self, p.ctrl)) return;
        r_idx = min(r_idx, p.self->in_idx[slot][s]);
        r_max = max(r_max, p.self->in_max[slot][s]);
        r_kind = max(r_kind, p.self->in_kind[slot][s]);
    }
    p.ctrl->bad_idx = r_idx;
    p.ctrl->max_bits = r_max;
    p.ctrl->kind = r_kind;
    peer_aborted(p.self, p.ctrl);  // a failure on any rank surfaces at every check
}

// Copies this rank's first / last R owned planes (full padded planes,
// contiguous) into the neighbours' ghost planes: used where the producing
// kernel did not store them itself (refresh_boundary, uploads, stored-ghost
// and non-TMA sweeps, volume sources).  16-byte vectors.
template <typename T>
__global__ void peer_push(const T* __restrict__ lvl, T* lo, T* hi, long long lo_src, long long lo_delta,
                          long long hi_src, long long hi_delta, long long n) {
    using VT = Vec<T, 16 / sizeof(T)>;
    constexpr int V = 16 / sizeof(T);
    const long long nv = n / V;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < nv;
         t += (long long)gridDim.x * blockDim.x) {
        const long long o = t * V;
        if (lo) *reinterpret_cast<VT*>(lo + lo_src + o + lo_delta) = *reinterpret_cast<const VT*>(lvl + lo_src + o);
        if (hi) *reinterpret_cast<VT*>(hi + hi_src + o + hi_delta) = *reinterpret_cast<const VT*>(lvl + hi_src + o);
    }
    __threadfence_system();
}

// ---------------------------------------------------------------------------
// inject, kernel.hpp:429-438.  One thread per distinct target index; its
// entries are applied in the reference's (point, entry) order.
template <typename T, bool EXACT>
__global__ void inject_kernel(T* out, const T* __restrict__ c2dt2, const T* __restrict__ eta,
                              double dt, const long long* __restrict__ tgt,
                              const unsigned int* __restrict__ ent_off,
                              const double* __restrict__ ent_w, const double* __restrict__ wavelet,
                              unsigned long long n_wavelet, int n_tgt, int k, const Ctrl* ctrl,
                              PeerMirror<T> pm) {
    using A = Ar<T, true>;  // the reference's scalar order; never contracted
    // Under PDL this runs while the sweep's last wave drains: everything but
    // out[i] is setup-time data (ctrl->step is advanced only between chunks,
    // by an ordinary launch), so it is loaded before pdl_wait().
    pdl_launch_dependents();
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const unsigned long long n = ctrl->step + (unsigned long long)k;
    const bool act = t < n_tgt && n < n_wavelet;
    const double amp = act ? wavelet[n] : 0.0;
    const long long i = act ? tgt[t] : 0;
    const T c2 = act ? c2dt2[i] : T(0);
    const T e = act ? eta[i] : T(0);
    pdl_wait();
    if (ctrl->abort || !act) return;
    T om, iop = T(1);
    if (e != T(0)) damping_factors(e, dt, om, iop);
    T val = out[i];
    for (unsigned int q = ent_off[t]; q < ent_off[t + 1]; ++q)
        val = A::add(val, A::mul(A::mul(c2, static_cast<T>(__dmul_rn(ent_w[q], amp))), iop));
    out[i] = val;
    pm.store(i, val);
}

// Dense modulated sources, kernel.hpp:439-452: after the point sources, for
// each source in insertion order, out[i] += c2dt2[i]*field[i]*T(amp[n])*iop[i]
// over every extended point.  One thread per point, sources looped in order.
template <typename T>
__global__ void volume_source_kernel(T* out, const T* __restrict__ c2dt2, const T* __restrict__ eta, double dt,
                                     const T* const* __restrict__ fields, const T* __restrict__ amps,
                                     const unsigned long long* __restrict__ amp_len, int n_src,
                                     unsigned long long n_amp, long long origin, long long plane, long long ld,
                                     int nz, int nx, int ny, int dface, int k, const Ctrl* ctrl) {
    using A = Ar<T, true>;
    if (ctrl->abort) return;
    const unsigned long long n = ctrl->step + (unsigned long long)k;
    if (n >= n_amp) return;  // n_amp: the longest amplitude vector
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (long long)nz * nx * ny) return;
    const int y = (int)(t % ny);
    const long long r2 = t / ny;
    const int x = (int)(r2 % nx), z = (int)(r2 / nx);
    // null-Dirichlet face points are zeroed by apply_boundary right after
    // (kernel.hpp:87-88): skipping them is exact, and the virtual-ghost
    // kernels rely on the stored face staying zero
    if (((dface & 1) && z == 0) || ((dface & 2) && z == nz - 1) || ((dface & 4) && x == 0) ||
        ((dface & 8) && x == nx - 1) || ((dface & 16) && y == 0) || ((dface & 32) && y == ny - 1))
        return;
    const long long i = origin + (long long)z * plane + (long long)x * ld + y;
    const T c2 = c2dt2[i];
    const T e = eta[i];
    T om, iop = T(1);
    if (e != T(0)) damping_factors(e, dt, om, iop);
    T val = out[i];
    for (int q = 0; q < n_src; ++q)
        if (n < amp_len[q])
            val = A::add(val, A::mul(A::mul(A::mul(c2, fields[q][i]), amps[(unsigned long long)q * n_amp + n]), iop));
    out[i] = val;
}

// apply_boundary, kernel.hpp:67-102, one axis per launch (the reference's axis
// order is kept by launching axis 0, 1, 2 in sequence).  One thread per line.
// mode: 0 always, 1 skip when aborted, 2 only when a non-finite value was found
template <typename T>
__global__ void ghost_lines(T* f, long long origin_pad, long long sa, int n_ext, int h,
                            long long s1, int n1, long long s2, int n2, int bc_lo, int bc_hi,
                            int do_lo, int do_hi, const Ctrl* ctrl, int mode) {
    if (mode == 1 && ctrl->abort) return;
    if (mode == 2 && ctrl->bad_idx == ~0ull) return;
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (long long)n1 * n2) return;
    const int i2 = (int)(t % n2), i1 = (int)(t / n2);
    T* line = f + origin_pad + (long long)i1 * s1 + (long long)i2 * s2;
#pragma unroll 1
    for (int side = 0; side < 2; ++side) {
        if (side == 0 ? !do_lo : !do_hi) continue;
        const int bc = side == 0 ? bc_lo : bc_hi;
        const long long face = side == 0 ? h : h + n_ext - 1;
        const long long o = side == 0 ? -1 : 1;
        T* fp = line + face * sa;
        if (bc == 0) {  // null Dirichlet
            *fp = T(0);
            for (int k = 1; k <= h; ++k) fp[o * k * sa] = -fp[-o * k * sa];
        } else if (bc == 1) {  // null Neumann
            for (int k = 1; k <= h; ++k) fp[o * k * sa] = fp[-o * k * sa];
        } else {
            for (int k = 1; k <= h; ++k) fp[o * k * sa] = T(0);
        }
    }
}

// record -> sample_receivers, kernel.hpp:299-304 / acquisition.hpp:150-161.
// One warp per receiver: the lanes form the products w_e * double(u[idx_e]) in
// parallel into shared memory, then lane 0 sums them in entry order (double,
// no FMA) -- the reference's exact association.
constexpr int REC_WARPS = 4;
constexpr int REC_CHUNK = 512;
template <typename T>
__global__ void __launch_bounds__(32 * REC_WARPS)
    receivers_kernel(const T* __restrict__ u, const long long* __restrict__ idx,
                     const unsigned int* __restrict__ off, const double* __restrict__ w, double* seis,
                     int n_rec, unsigned long long n_rows, int row_add, const Ctrl* ctrl) {
    __shared__ double prod[REC_WARPS][REC_CHUNK];
    if (ctrl->abort) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int r = blockIdx.x * REC_WARPS + warp;
    const unsigned long long row = ctrl->step + (unsigned long long)row_add - ctrl->row_base;
    if (r >= n_rec || row >= n_rows) return;
    const unsigned int b = off[r], e = off[r + 1];
    double acc = 0.0;
    constexpr int BATCH = 8;  // gathers in flight per lane
    for (unsigned int base = b; base < e; base += REC_CHUNK) {
        const int m = (int)min((unsigned int)REC_CHUNK, e - base);
        for (int k0 = 0; k0 < m; k0 += 32 * BATCH) {
            long long ix[BATCH];
            double wt[BATCH];
            T uv[BATCH];
#pragma unroll
            for (int j = 0; j < BATCH; ++j) {
                const int k = k0 + j * 32 + lane;
                ix[j] = k < m ? idx[base + k] : idx[base];
                wt[j] = k < m ? w[base + k] : 0.0;
            }
#pragma unroll
            for (int j = 0; j < BATCH; ++j) uv[j] = u[ix[j]];
#pragma unroll
            for (int j = 0; j < BATCH; ++j) {
                const int k = k0 + j * 32 + lane;
                if (k < m) prod[warp][k] = __dmul_rn(wt[j], static_cast<double>(uv[j]));
            }
        }
        __syncwarp();
        if (lane == 0) {
#pragma unroll 8
            for (int k = 0; k < m; ++k) acc = __dadd_rn(acc, prod[warp][k]);
        }
        __syncwarp();
    }
    if (lane == 0) seis[row * (unsigned long long)n_rec + r] = acc;
}

// Receivers whose taps straddle a slab face (Z slabs): the reference sums a
// receiver's products in entry order in ONE sequential double accumulation
// (acquisition.hpp:155-158), which per-slab partial sums cannot reproduce.
// For those taps each rank stores the products themselves, row by row; the
// host merges the ranks' products in entry order and sums them sequentially,
// so the seismogram stays bit-identical to the reference at any slab count.
template <typename T>
__global__ void receiver_products_kernel(const T* __restrict__ u, const long long* __restrict__ idx,
                                         const double* __restrict__ w, double* prod, int n_slots,
                                         unsigned long long n_rows, int row_add, const Ctrl* ctrl) {
    if (ctrl->abort) return;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const unsigned long long row = ctrl->step + (unsigned long long)row_add - ctrl->row_base;
    if (j >= n_slots || row >= n_rows) return;
    prod[row * (unsigned long long)n_slots + j] = __dmul_rn(w[j], static_cast<double>(u[idx[j]]));
}

// max_abs / check_health, kernel.hpp:265-273 and :456-458.  max |u| over
// finite values plus the smallest global padded flat index holding a
// non-finite value (the reference returns the first one in flat order).
// Scans the box [p0, p0+n_planes) x [r0, r0+n_rows) x [c0, c0+n_cols) of padded
// local coordinates; flat indices are GLOBAL padded (gplane0 = global padded
// plane of local plane 0).  only_if_bad: run only after a non-finite was seen.
template <typename T>
__global__ void health_kernel(const T* __restrict__ u, long long origin_pad, long long ld,
                              long long plane, int p0, int n_planes, int r0, int n_rows, int c0,
                              int n_cols, unsigned long long gplane0, unsigned long long P1,
                              unsigned long long P2, int is3d, Ctrl* ctrl, int honor_abort,
                              int only_if_bad) {
    if (honor_abort && ctrl->abort) return;
    if (only_if_bad && ctrl->bad_idx == ~0ull) return;
    double m = 0.0;
    unsigned long long bad = ~0ull;
    const long long total = (long long)n_planes * n_rows;
    for (long long pr = blockIdx.x; pr < total; pr += gridDim.x) {
        const int p = p0 + (int)(pr / n_rows), r = r0 + (int)(pr % n_rows);
        const T* row = u + origin_pad + (long long)p * plane + (long long)r * ld;
        for (int c = c0 + threadIdx.x; c < c0 + n_cols; c += blockDim.x) {
            const double av = fabs(static_cast<double>(row[c]));
            if (!isfinite(av)) {
                const unsigned long long flat =
                    is3d ? ((gplane0 + p) * P1 + r) * P2 + c : (unsigned long long)r * P1 + c;
                bad = flat < bad ? flat : bad;
            } else {
                m = av > m ? av : m;
            }
        }
    }
    // warp then block reduction
    for (int o = 16; o > 0; o >>= 1) {
        const double mo = __shfl_down_sync(0xffffffffu, m, o);
        const unsigned long long bo = __shfl_down_sync(0xffffffffu, bad, o);
        m = mo > m ? mo : m;
        bad = bo < bad ? bo : bad;
    }
    __shared__ double sm_m[32];
    __shared__ unsigned long long sm_b[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) {
        sm_m[wid] = m;
        sm_b[wid] = bad;
    }
    __syncthreads();
    if (wid == 0) {
        const int nw = (blockDim.x + 31) >> 5;
        m = lane < nw ? sm_m[lane] : 0.0;
        bad = lane < nw ? sm_b[lane] : ~0ull;
        for (int o = 16; o > 0; o >>= 1) {
            const double mo = __shfl_down_sync(0xffffffffu, m, o);
            const unsigned long long bo = __shfl_down_sync(0xffffffffu, bad, o);
            m = mo > m ? mo : m;
            bad = bo < bad ? bo : bad;
        }
        if (lane == 0) {
            atomicMax(&ctrl->max_bits, (unsigned long long)__double_as_longlong(m));
            if (bad != ~0ull) atomicMin(&ctrl->bad_idx, bad);
        }
    }
}

// Extended-point scan of check_health (kernel.hpp:456-467 / max_abs :265-273)
// as a streaming pass: 16-byte loads (the extended row start is 128-byte
// aligned), independent loads in flight, max |u| in T (exactly the maximum
// of the doubles), the first non-finite flat GLOBAL padded index.
template <typename T>
__global__ void __launch_bounds__(256) health_scan_ext(const T* __restrict__ u, long long origin, long long ld,
                                                       long long plane, int nz, int nx, int ny, int h,
                                                       unsigned long long gplane0, unsigned long long P1,
                                                       unsigned long long P2, int is3d, Ctrl* ctrl, int honor_abort) {
    constexpr int V = 16 / sizeof(T);
    using VT = Vec<T, V>;
    if (honor_abort && ctrl->abort) return;
    T m = T(0);
    unsigned long long bad = ~0ull;
    auto visit = [&](T val, int z, int x, int y) {
        const T av = fabs(val);
        if (!isfinite(av)) {
            const unsigned long long flat =
                is3d ? ((gplane0 + (unsigned long long)(z + h)) * P1 + (unsigned long long)(x + h)) * P2 + (y + h)
                     : (unsigned long long)(x + h) * P1 + (y + h);
            bad = flat < bad ? flat : bad;
        } else {
            m = av > m ? av : m;
        }
    };
    // a warp per extended row, lanes over its 16-byte vectors; each lane
    // issues up to NB independent loads before visiting any of them
    constexpr int NB = 8;
    const int lane0 = threadIdx.x & 31;
    const int nrows = nz * nx;
    const int nfull = ny / V;  // whole vectors; the ragged tail is visited scalar
    for (int row = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5); row < nrows;
         row += (int)((gridDim.x * blockDim.x) >> 5)) {
        const int z = row / nx, x = row - z * nx;
        const T* p = u + origin + (long long)z * plane + (long long)x * ld;
        for (int b = 0; b < nfull; b += 32 * NB) {
            VT t[NB];
#pragma unroll
            for (int j = 0; j < NB; ++j) {
                const int v = b + j * 32 + lane0;
                if (v < nfull) t[j] = ldg16(p + v * V);
            }
#pragma unroll
            for (int j = 0; j < NB; ++j) {
                const int v = b + j * 32 + lane0;
                if (v < nfull) {
#pragma unroll
                    for (int e = 0; e < V; ++e) visit(t[j].e[e], z, x, v * V + e);
                }
            }
        }
        for (int y = nfull * V + lane0; y < ny; y += 32) visit(p[y], z, x, y);
    }
    double md = static_cast<double>(m);
    for (int o = 16; o > 0; o >>= 1) {
        const double mo = __shfl_down_sync(0xffffffffu, md, o);
        const unsigned long long bo = __shfl_down_sync(0xffffffffu, bad, o);
        md = mo > md ? mo : md;
        bad = bo < bad ? bo : bad;
    }
    __shared__ double sm_m[8];
    __shared__ unsigned long long sm_b[8];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) {
        sm_m[wid] = md;
        sm_b[wid] = bad;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
            md = sm_m[w] > md ? sm_m[w] : md;
            bad = sm_b[w] < bad ? sm_b[w] : bad;
        }
        atomicMax(&ctrl->max_bits, (unsigned long long)__double_as_longlong(md));
        if (bad != ~0ull) atomicMin(&ctrl->bad_idx, bad);
    }
}

// Debug guard check (FDW_GUARD_CHECK=1, fdw_debug_check_guards): the bytes
// past each allocation hold a pattern, and in a wavefield level every element
// outside the padded box (row / column slack, the spare plane) must still be
// zero -- no kernel may write there.  Counts the violations.
__global__ void guard_scan(const unsigned int* __restrict__ a, unsigned long long n_words,
                           unsigned long long body_words, int check_slack, long long ld, long long plane,
                           long long base, long long nrows, long long ncols, long long nplanes, int tsize,
                           unsigned long long* bad) {
    unsigned long long cnt = 0;
    for (unsigned long long w = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; w < n_words;
         w += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned int v = a[w];
        if (w >= body_words) {
            cnt += v != 0xA5A5A5A5u;
        } else if (check_slack && v != 0u) {
            const long long e = (long long)(w * 4 / tsize);
            const long long p = e / plane, rem = e % plane, r = rem / ld, col = rem % ld;
            cnt += !(p < nplanes && r < nrows && col >= base && col < base + ncols);
        }
    }
    if (cnt) atomicAdd(bad, cnt);
}

__global__ void health_reset(Ctrl* ctrl, int honor_abort) {
    if (honor_abort && ctrl->abort) return;
    ctrl->bad_idx = ~0ull;
    ctrl->max_bits = 0ull;
    ctrl->kind = 0u;
}

// Classifies the first non-finite value if this rank owns it (kind 1 inf, 2 nan).
template <typename T>
__global__ void health_classify(const T* u, Ctrl* ctrl, long long origin_pad, long long ld,
                                long long plane, unsigned long long gplane_lo,
                                unsigned long long gplane_hi, unsigned long long P1,
                                unsigned long long P2, int is3d, int honor_abort) {
    if (honor_abort && ctrl->abort) return;
    const unsigned long long f = ctrl->bad_idx;
    if (f == ~0ull) return;
    long long off;
    if (is3d) {
        const unsigned long long gp = f / (P1 * P2), rem = f % (P1 * P2);
        if (gp < gplane_lo || gp >= gplane_hi) return;
        off = origin_pad + (long long)(gp - gplane_lo) * plane + (long long)(rem / P2) * ld +
              (long long)(rem % P2);
    } else {
        off = origin_pad + (long long)(f / P1) * ld + (long long)(f % P1);
    }
    const double av = fabs(static_cast<double>(u[off]));
    ctrl->kind = isnan(av) ? 2u : 1u;
}

// Latches the abort flag after a failed check (kernel.hpp:458 throw).
__global__ void health_latch(Ctrl* ctrl) {
    if (ctrl->abort) return;
    if (ctrl->kind != 0u) {
        ctrl->abort = 1u;
        ctrl->bad_step = ctrl->step;
    }
}

__global__ void step_advance(Ctrl* ctrl, unsigned long long n) {
    if (!ctrl->abort) ctrl->step += n;
}

// precompute, kernel.hpp:282-285: c2dt2 = T(c * c * dt * dt) in double, in place
// over the whole allocation (zero padding stays zero).
// Eta-zero Z ranges per TMA tile column (BX x TYW outputs): flags[z] = 1 when
// the column's eta tile on plane z is all zero; thread 0 then keeps the
// longest run of such planes.  One block per column.
template <typename T>
__global__ void eta_zero_ranges(const T* __restrict__ eta, long long origin, long long plane, long long ld, int nz,
                                int nx, int ny, int bx, int tyw, int2* __restrict__ out) {
    extern __shared__ unsigned char zflag[];
    const int col = blockIdx.x;  // = blockIdx.y * gridDim.x + blockIdx.x of the sweep grid
    const int ncy = (ny + tyw - 1) / tyw;
    const int x0 = (col / ncy) * bx, y0 = (col % ncy) * tyw;
    const int w = min(tyw, ny - y0), h = min(bx, nx - x0);
    for (int z = 0; z < nz; ++z) {
        int nzv = 0;
        for (int t = threadIdx.x; t < w * h; t += blockDim.x) {
            const int xx = x0 + t / w, yy = y0 + t % w;
            nzv |= eta[origin + (long long)z * plane + (long long)xx * ld + yy] != T(0);
        }
        nzv = __syncthreads_or(nzv);
        if (threadIdx.x == 0) zflag[z] = nzv ? 0 : 1;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int best0 = 0, best1 = 0, run0 = 0;
        for (int z = 0; z <= nz; ++z) {
            if (z < nz && zflag[z]) continue;
            if (z - run0 > best1 - best0) best0 = run0, best1 = z;
            run0 = z + 1;
        }
        out[col] = make_int2(best0, best1);
    }
}

// Damping table (fp32 TMA sweep): when the damping field takes at most 255
// distinct non-zero values -- damping_field (model.hpp:141-186) gives a few
// dozen: eta depends only on the distance to the physical box -- the sweep
// streams a 1-byte index per point instead of the 4-byte eta, and reads
// (1 - eta dt, 1 / (1 + eta dt)) from a table formed on the host in double
// exactly as kernel.hpp:284-287 (bit-identical to forming them per point).
// Pass 1: distinct non-zero bit patterns into an open-addressing set.
constexpr int ETAB_CAP = 1024;  // set slots (power of two)
// Set keys are the bit patterns of T(eta): 32-bit for float, 64-bit for double;
// the all-ones pattern (a NaN) marks an empty slot.
template <typename T>
struct EtaKey;
template <>
struct EtaKey<float> {
    using type = unsigned;
    static __device__ __forceinline__ type bits(float f) { return __float_as_uint(f); }
};
template <>
struct EtaKey<double> {
    using type = unsigned long long;
    static __device__ __forceinline__ type bits(double f) { return (unsigned long long)__double_as_longlong(f); }
};
__device__ __forceinline__ unsigned etab_hash(unsigned long long w) {
    unsigned v = (unsigned)(w ^ (w >> 32));
    v ^= v >> 16;
    v *= 0x7feb352du;
    v ^= v >> 15;
    return v & (ETAB_CAP - 1);
}
template <typename T>
__global__ void eta_collect(const T* __restrict__ eta, unsigned long long n, typename EtaKey<T>::type* keys,
                            unsigned* overflow) {
    using K = typename EtaKey<T>::type;
    constexpr K EMPTY = ~K(0);
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const T f = eta[i];
        if (f == T(0)) continue;
        const K v = EtaKey<T>::bits(f);
        unsigned h = etab_hash(v);
        for (int probe = 0;; ++probe) {
            const K k = *reinterpret_cast<volatile K*>(&keys[h]);
            if (k == v) break;
            if (k == EMPTY) {
                const K old = atomicCAS(&keys[h], EMPTY, v);
                if (old == EMPTY || old == v) break;
            }
            if (probe >= ETAB_CAP) {
                atomicOr(overflow, 1u);
                break;
            }
            h = (h + 1) & (ETAB_CAP - 1);
        }
    }
}
// Pass 2: the index of every point (0: eta == 0, undamped).
template <typename T>
__global__ void eta_index(const T* __restrict__ eta, unsigned long long n,
                          const typename EtaKey<T>::type* __restrict__ keys,
                          const unsigned char* __restrict__ slot_index, unsigned char* __restrict__ out) {
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const T f = eta[i];
        unsigned char ix = 0;
        if (f != T(0)) {
            const typename EtaKey<T>::type v = EtaKey<T>::bits(f);
            unsigned h = etab_hash(v);
            while (keys[h] != v) h = (h + 1) & (ETAB_CAP - 1);
            ix = slot_index[h];
        }
        out[i] = ix;
    }
}

// Box copy between the caller's dense layout and the pitched device layout
// (either direction): nz x nx x ny elements, per-side plane/row strides.
// Grid-stride; used so host transfers are single contiguous DMA copies.
template <typename T>
__global__ void box_copy(T* __restrict__ dst, long long d_plane, long long d_row, const T* __restrict__ src,
                         long long s_plane, long long s_row, int nz, int nx, int ny) {
    const long long total = (long long)nz * nx * ny;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int y = (int)(t % ny);
        const long long r = t / ny;
        const int x = (int)(r % nx), z = (int)(r / nx);
        dst[z * d_plane + x * d_row + y] = src[z * s_plane + x * s_row + y];
    }
}

// Seismogram rows to T (Seismogram<T> holds T(sum), acquisition.hpp:158):
// double -> float rounds to nearest, as static_cast<float> does on the host.
__global__ void seis_to_float(const double* __restrict__ in, float* __restrict__ out, unsigned long long n) {
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x)
        out[i] = __double2float_rn(in[i]);
}

template <typename T>
__global__ void c2dt2_kernel(T* f, unsigned long long n, double dt) {
    const unsigned long long t = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const double cv = static_cast<double>(f[t]);
    f[t] = static_cast<T>(__dmul_rn(__dmul_rn(__dmul_rn(cv, cv), dt), dt));
}

}  // namespace
}  // namespace fdw
