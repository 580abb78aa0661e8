/*
 * fdwave_cuda.h -- C-ABI of libfdwave_cuda.so, the sm_100a (B200) engine behind
 * fdwave::Solver<T> (constant-density acoustic propagator of arXiv 2201.05278).
 *
 * The reference has no plugin registry: its seam is the Solver<T> class
 * template, /root/reference/proj/include/fdwave/kernel.hpp:170-495.  Each entry
 * point below replaces one piece of that class; the reference file:line is given
 * beside it.  include/fdwave/kernel.hpp (the drop-in C++ header) and
 * paper_2201_05278_b200/kernel.py (the Python mirror) are thin hosts over this
 * ABI; INTEGRATION.md shows the bindings.
 *
 * Conventions
 *  - extern "C", plain pointers and sizes; no exceptions cross the boundary.
 *  - Every call returns an fdw_status; fdw_last_error(ctx) (or NULL ctx for
 *    fdw_create failures) gives the message.
 *  - Scalars of the field type T are passed as void* with desc.dtype_bytes 4
 *    (float) or 8 (double).
 *  - Host arrays use the reference padded layout (field.hpp:10-23, grid.hpp:
 *    37-42): row-major Z,X[,Y], last index fastest, extended grid + halo on each
 *    side.  For a Z-slab context (world > 1) the host arrays are the LOCAL padded
 *    slab: global padded Z planes [z_begin, z_end + 2*halo).
 *  - Flat indices in source/receiver maps are GLOBAL padded flat indices exactly
 *    as InterpolationMap::Entry::index holds them (acquisition.hpp:79-85).
 *  - One host thread per context; calls are serialised by the caller
 *    ("one run per Solver").
 */
#ifndef FDWAVE_CUDA_H
#define FDWAVE_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FDW_ABI_VERSION 3

typedef enum fdw_status {
    FDW_OK = 0,
    FDW_EINVAL = 1,     /* maps to std::invalid_argument */
    FDW_ECUDA = 2,      /* CUDA runtime error -> std::runtime_error */
    FDW_EPEER = 3,      /* peer transport: a slab rank failed / timed out -> std::runtime_error */
    FDW_EINSTABLE = 4,  /* non-finite wavefield -> fdwave::instability_error */
    FDW_ENOMEM = 5,
    FDW_ESTATE = 6      /* call order violated (e.g. advance before set_medium) */
} fdw_status;

/* BoundaryCondition, kernel.hpp:27 (same enumerator order). */
enum { FDW_BC_NULL_DIRICHLET = 0, FDW_BC_NULL_NEUMANN = 1, FDW_BC_NONE = 2 };

/* Stencil kernel variants (fdw_desc.variant). */
enum {
    FDW_KERNEL_AUTO = 0,   /* best registered kernel for (ndim, order, dtype) */
    FDW_KERNEL_SIMPLE = 1, /* one thread per point, cache-fed (parity baseline) */
    FDW_KERNEL_ZMARCH = 2, /* 3D: 2.5D Z-march, smem X-Y plane + register Z queue (LDG-fed) */
    FDW_KERNEL_TMA = 3,    /* 3D: Z-march fed by cp.async.bulk.tensor (TMA) + mbarrier rings */
    FDW_KERNEL_FUSED2D = 4 /* 2D: persistent cooperative kernel, one grid barrier per time step */
};

/* Arithmetic mode (fdw_desc.math). */
enum {
    FDW_MATH_EXACT = 0, /* reference association, no FMA contraction: IEEE-identical
                           to the reference's own x86-64 build (kernel.hpp:398-420) */
    FDW_MATH_FMA = 1    /* same association, FMA contraction allowed */
};

/* Advance flags. */
enum {
    FDW_ADVANCE_RECORD = 1, /* sample receivers after every step (forward()) */
    FDW_ADVANCE_ASYNC = 2   /* enqueue only: no host sync; an instability is reported
                               by the next fdw_wait / state-reading call */
};

typedef struct fdw_desc {
    int32_t abi_version;     /* FDW_ABI_VERSION */
    int32_t ndim;            /* 2 or 3                         grid.hpp:19 */
    int32_t space_order;     /* even, 2..20                    grid.hpp:26 */
    int32_t dtype_bytes;     /* 4 (float) or 8 (double)        Solver<T> */
    uint64_t extended[3];    /* Grid::extended_shape (2D: [2] = 1) grid.hpp:28 */
    double spacing[3];       /* Grid::spacing                  grid.hpp:21 */
    double coeffs[11];       /* StencilCoeffs::second, v_0..v_r  stencil.hpp:95 */
    int32_t bc[3][2];        /* BoundarySpec::face             kernel.hpp:37-45 */
    double dt;               /* TimeAxis::dt                   time_axis.hpp:18 */
    uint64_t n_steps;        /* TimeAxis::n_steps (health check at the last step) */
    uint64_t check_interval; /* kernel.hpp:491 (0 -> 100) */
    int32_t device;          /* CUDA device ordinal */
    int32_t variant;         /* FDW_KERNEL_* */
    int32_t math;            /* FDW_MATH_* */
    /* Z-slab decomposition (3D only; world == 1 for a single GPU). */
    int32_t rank;
    int32_t world;
    int32_t z_segments;      /* ZMARCH: Z segments per column (0 -> auto) */
    uint64_t z_begin;        /* first extended Z plane owned by this rank */
    uint64_t z_end;          /* one past the last owned plane */
    double coeffs1[10];      /* StencilCoeffs::first, w_1..w_r (variable density) stencil.hpp:96 */
} fdw_desc;

typedef struct fdw_solver fdw_solver;

/* Fills *desc with defaults (abi_version, check_interval 100, world 1, AUTO, EXACT). */
void fdw_desc_init(fdw_desc* desc);

/* Solver<T>::Solver, kernel.hpp:173-186: validates the descriptor and allocates
 * the device wavefield ring (two levels) and coefficient arrays. */
fdw_status fdw_create(const fdw_desc* desc, fdw_solver** out);
fdw_status fdw_destroy(fdw_solver* ctx);
const char* fdw_last_error(const fdw_solver* ctx);
const char* fdw_status_string(fdw_status s);

/* Optional: run on a caller stream (cudaStream_t as void*; NULL = own stream). */
fdw_status fdw_set_stream(fdw_solver* ctx, void* cuda_stream);

/* Solver<T>::precompute, kernel.hpp:276-297: c^2 dt^2 from the velocity in
 * double (bit-identical to the reference), eta kept as given; the damping
 * factors (1 - eta dt) and 1/(1 + eta dt) are formed in double inside the
 * stencil exactly as the reference precomputes them.  Arrays are host (or, with
 * on_device = 1, device) padded slabs of T. */
fdw_status fdw_set_medium(fdw_solver* ctx, const void* velocity, const void* eta,
                          int on_device);

/* MaterialModel::density present -> the VariableDensity = true sweep
 * (kernel.hpp:365-373 / :407-417).  grad(rho)/rho is formed on the device in
 * double exactly as density_log_gradient (kernel.hpp:104-136); needs
 * desc.coeffs1.  Padded slab of T (host, or device with on_device = 1). */
fdw_status fdw_set_density(fdw_solver* ctx, const void* rho, int on_device);

/* Solver<T>::add_volume_source, kernel.hpp:199-203 (ModulatedField, :140-144;
 * applied in inject, :439-452): a padded forcing field of T (host, or device
 * with on_device = 1) and one double amplitude per step (n_amp >= n_steps,
 * else FDW_EINVAL).  Sources accumulate in call order. */
fdw_status fdw_add_volume_source(fdw_solver* ctx, const void* field, const double* amplitude, uint64_t n_amp,
                                 int on_device);

/* Solver<T>::set_sources, kernel.hpp:188-193: CSR view of an InterpolationMap
 * (offsets[n_points+1], idx/w[offsets[n_points]]) plus the wavelet (double,
 * >= n_steps + 1 samples when n_points > 0).  Entries outside this rank's slab
 * are dropped; overlapping windows are merged per index on the host and applied
 * in the reference's sequential order (kernel.hpp:426-438). */
fdw_status fdw_set_sources(fdw_solver* ctx, uint64_t n_points, const uint64_t* offsets,
                           const uint64_t* idx, const double* w, const double* wavelet,
                           uint64_t n_samples);

/* Solver<T>::set_receivers, kernel.hpp:194-198 (coordinates stay on the host).
 * Allocates the device seismogram: n_steps + 1 rows of n_points doubles
 * (per-rank partial sums, acquisition.hpp:150-161). */
fdw_status fdw_set_receivers(fdw_solver* ctx, uint64_t n_points, const uint64_t* offsets,
                             const uint64_t* idx, const double* w);

/* current_level()/previous_level() host mirror, kernel.hpp:217-218: upload /
 * download both levels (local padded slab of T; either pointer may be NULL).
 * Downloads include the halo exactly as apply_boundary left it. */
fdw_status fdw_set_levels(fdw_solver* ctx, const void* prev, const void* curr);
fdw_status fdw_get_levels(fdw_solver* ctx, void* prev, void* curr);
/* Both levels back to the quiescent zero state of a fresh Solver (field.hpp:23). */
fdw_status fdw_zero_levels(fdw_solver* ctx);
/* extract_extended, kernel.hpp:313-323: halo-stripped current level (local slab). */
fdw_status fdw_get_extended(fdw_solver* ctx, void* out);

/* refresh_boundary, kernel.hpp:223 (+ Z-halo exchange between slabs). */
fdw_status fdw_refresh_boundary(fdw_solver* ctx);

/* record, kernel.hpp:299-304: starts a recording -- seismogram row 0 = the
 * current level; FDW_ADVANCE_RECORD then writes row (step - step at this call). */
fdw_status fdw_record(fdw_solver* ctx);

/* n x step(), kernel.hpp:226-233 (sweep -> inject -> swap -> apply_boundary ->
 * health check when step % check_interval == 0 or step == n_steps), optionally
 * recording the seismogram row after each step (forward(), kernel.hpp:255-258).
 * Launched as CUDA-graph chunks; returns FDW_EINSTABLE with *bad_step /
 * *bad_max (instability_error::step/max_abs) and leaves the state at that step. */
fdw_status fdw_advance(fdw_solver* ctx, uint64_t n, uint32_t flags, uint64_t* bad_step,
                       double* bad_max);

/* Waits for the context's compute and copy streams and checks asynchronous
 * advances: FDW_EINSTABLE with *bad_step / *bad_max as fdw_advance. */
fdw_status fdw_wait(fdw_solver* ctx, uint64_t* bad_step, double* bad_max);

/* forward()'s strided snapshots, kernel.hpp:305-310 / extract_extended
 * :313-323, streamed: enqueues a halo-stripped copy of the current level into
 * out (host, extended shape of this rank) behind the queued steps and returns.
 * The device copy goes to a ring slot; the host copy runs on a separate copy
 * stream (pinned destinations directly, others through a pinned bounce slot),
 * overlapping the following steps.  out is valid after fdw_wait. */
fdw_status fdw_snapshot_async(fdw_solver* ctx, void* out);

/* Device step counter (Solver<T>::step_index, kernel.hpp:219). */
fdw_status fdw_step_index(fdw_solver* ctx, uint64_t* step);
/* Resets the step counter (a fresh forward on the same medium). */
fdw_status fdw_set_step_index(fdw_solver* ctx, uint64_t step);

/* max_abs, kernel.hpp:265-273 over this rank's slab (first non-finite wins). */
fdw_status fdw_max_abs(fdw_solver* ctx, double* out);

/* Seismogram rows [0, rows) as T (this rank's partial sums cast to T; for
 * world > 1 use fdw_download_seismogram_f64 and reduce in rank order). */
fdw_status fdw_download_seismogram(fdw_solver* ctx, void* out, uint64_t rows);
fdw_status fdw_download_seismogram_f64(fdw_solver* ctx, double* out, uint64_t rows);

/* Z slabs: receivers whose taps straddle a slab face keep per-tap products
 * instead of a partial sum (their seismogram entries stay 0 on every rank), so
 * the host can merge the ranks' products in entry order and sum them
 * sequentially -- bit-identical to the reference's single accumulation
 * (acquisition.hpp:155-158).  split_info: the number of product slots on this
 * rank and, per slot, the receiver and the entry position within its
 * InterpolationMap point (either array may be NULL).  products: rows x slots. */
fdw_status fdw_receiver_split_info(fdw_solver* ctx, uint64_t* n_slots, uint64_t* receiver, uint64_t* entry);
fdw_status fdw_download_receiver_products(fdw_solver* ctx, double* out, uint64_t rows);

/* Waits for all work queued on the context (compute + copy streams); reports a
 * pending asynchronous instability like fdw_wait (without the step details). */
fdw_status fdw_synchronize(fdw_solver* ctx);

/* Profiling: runs n steps with direct launches and CUDA events around every
 * kernel; ms[k] = mean device ms per launch of kernel class k
 * (0 sweep, 1 inject, 2 boundary, 3 receivers, 4 health, 5 halo exchange). */
fdw_status fdw_profile_steps(fdw_solver* ctx, uint64_t n, double ms[6]);

/* Number of kernels this context has launched (CUDA-graph nodes included). */
fdw_status fdw_launch_count(const fdw_solver* ctx, uint64_t* n);

/* Introspection: device layout of one level (elements): row pitch, plane pitch,
 * column base, stored planes, selected kernel variant | z_segments << 8 |
 * resident CTAs per SM << 16 | TMA planes in flight (split rings, 0: one) << 24. */
fdw_status fdw_layout(const fdw_solver* ctx, uint64_t* ld, uint64_t* plane,
                      uint64_t* base, uint64_t* planes, int32_t* variant);

/* ---- peer transport (Z slabs over NVLink / NVSwitch peer memory) ----
 * Replaces the reference's only parallelism, the OpenMP loop over Z planes
 * (kernel.hpp:392-393), with one GPU per Z slab.  A slab context (world > 1)
 * exchanges no messages: each step's TMA sweep stores its first / last R owned
 * planes straight into the neighbours' ghost planes through mapped peer memory
 * (the point-source kernel does the same for targets in those planes; other
 * paths copy the planes with a push kernel).  Ordering is one halo epoch per
 * collective operation: the sweep's boundary CTAs wait until both neighbours
 * have published this rank's epoch, and the last of them publishes the next
 * one (release / acquire at system scope).  The health reduction
 * (kernel.hpp:456-458 across slabs) goes through the same per-rank sync blocks.
 * Every collective call (advance, refresh_boundary, max_abs) must be made on
 * all ranks.  A rank that fails or does not signal within 20 s raises a sticky
 * abort word in every rank's sync block: every rank then returns FDW_EPEER
 * instead of hanging or stepping on stale ghost planes.
 *
 * Ranks linked in ONE process whose GPUs coincide (one GPU emulating several
 * slabs) are host-ordered: at each cross-rank point the rank threads meet at a
 * host barrier and order their streams with events, so no kernel ever waits
 * on a flag that another launch on the same GPU sets (they run as direct
 * launches instead of graphs).  IPC-imported neighbours on the same GPU are
 * refused at the first collective call (FDW_ESTATE).
 *
 * Teardown: fdw_destroy waits (bounded) until the neighbours have finished the
 * epochs this rank went through before it frees the mapped memory; callers
 * should still destroy all ranks after the same collective calls. */
#define FDW_PEER_BLOB_BYTES 512
/* IPC handles of this rank's levels and sync block plus its slab geometry. */
fdw_status fdw_peer_export(fdw_solver* ctx, unsigned char out[FDW_PEER_BLOB_BYTES]);
/* One process per GPU: every rank's export blob in rank order (world x
 * FDW_PEER_BLOB_BYTES bytes); maps the neighbours' levels and all sync blocks. */
fdw_status fdw_peer_import(fdw_solver* ctx, const unsigned char* blobs, int32_t world);
/* One process driving every rank (one thread per context): all[r] = rank r. */
fdw_status fdw_peer_link(fdw_solver* ctx, fdw_solver* const* all, int32_t world);

/* Debug: with FDW_GUARD_CHECK=1 set when the context is created, every field
 * allocation carries a patterned guard zone after its end.  Counts the guard
 * words that changed, plus every non-zero element OUTSIDE the padded box of
 * the two wavefield levels (row / column slack, spare plane), where no kernel
 * may write.  (Out-of-bounds store detection of our own: compute-sanitizer is
 * not available on the GPU pool this was built on.) */
fdw_status fdw_debug_check_guards(fdw_solver* ctx, uint64_t* n_bad);

/* Profiling hook: emulated neighbours for a slab context on ONE GPU.  The
 * halo planes this rank stores go to scratch levels on its own GPU, and the
 * neighbours' halo epochs and health posts are pre-satisfied, so the step runs
 * the complete multi-GPU path (boundary-first Z segments, in-sweep epoch waits
 * and publish, fused halo stores, cross-rank health reduction) without
 * another rank; only the NVLink transfer itself is absent.  Instead of
 * fdw_peer_import / fdw_peer_link.  The wavefield is not a valid slab
 * solution (its ghost planes are never refreshed): for timing only. */
fdw_status fdw_peer_loopback(fdw_solver* ctx);

/* ---- host-only helpers (no GPU needed) ---- */

/* Z-slab split of n_ext planes over `world` ranks: [*z_begin, *z_end). */
fdw_status fdw_slab_range(uint64_t n_ext, int32_t world, int32_t rank, uint64_t* z_begin,
                          uint64_t* z_end);
/* Owner rank of global padded flat index (3D slabs; -1 if not an extended point). */
int32_t fdw_owner_of(uint64_t flat_idx, const uint64_t extended[3], int32_t halo,
                     int32_t world);

#ifdef __cplusplus
}
#endif
#endif /* FDWAVE_CUDA_H */
