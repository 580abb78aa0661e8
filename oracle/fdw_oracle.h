/*
 * fdw_oracle.h -- CPU restatement of the fdwave constant-density hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the checker for the CUDA path:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it.  The product (libfdwave_cuda.so and paper_2201_05278_b200/) never
 * links, imports or calls anything under oracle/.
 *
 * Every function restates one reference function; the reference file:line it
 * follows is given beside it (paths relative to /root/reference/proj/include/
 * fdwave/).  Arithmetic is written in the reference's association and the file
 * is compiled with -ffp-contract=off and without -ffast-math, so on x86-64 the
 * results are IEEE-identical to the reference's own Release build (checked
 * against oracle/_ref, the reference compiled in place, by
 * tests/test_oracle_vs_reference.py and the committed golden fixtures).
 */
#ifndef FDW_ORACLE_H
#define FDW_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { FDWO_DIRICHLET = 0, FDWO_NEUMANN = 1, FDWO_NONE = 2 };
enum { FDWO_OK = 0, FDWO_EINVAL = 1, FDWO_EINSTABLE = 4, FDWO_ENOMEM = 5 };

/* grid.hpp:18-48 Grid (geometry only; precision is carried by the solver). */
typedef struct fdwo_grid {
    int32_t ndim;
    int32_t halo;
    int32_t space_order;
    int32_t _pad;
    double bbox[3][2];
    double spacing[3];
    uint64_t interior[3];
    uint64_t damping_cells[3][2];
    double damping_length[3][2];
    uint64_t extended[3];
    uint64_t padded[3];
} fdwo_grid;

/* stencil.hpp:55-72 */
int fdwo_second_derivative_coefficients(int order, double* v_out /* r+1 */);
/* stencil.hpp:77-90 */
int fdwo_first_derivative_coefficients(int order, double* w_out /* r */);
/* stencil.hpp:113-129 */
double fdwo_stable_dt(double c_max, const double* spacing, int n_spacing, int order,
                      int ndim);
/* time_axis.hpp:31-50 (n_steps only; dt <= 0 selects the stable bound) */
uint64_t fdwo_n_steps(double tf, double dt);

/* grid.hpp:50-80 + grid.hpp:85-104 (lengths: Zlo,Zhi,Xlo,Xhi[,Ylo,Yhi]) */
int fdwo_build_grid(int ndim, const double* bbox, const double* spacing, int space_order,
                    const double* damping_lengths, fdwo_grid* out);

/* model.hpp:34-106, result cast to float (dtype 4) or double (dtype 8) */
int fdwo_resample_model(const fdwo_grid* g, const double* raw, const uint64_t* raw_shape,
                        int dtype, void* out_padded);
/* model.hpp:148-186 */
int fdwo_damping_field(const fdwo_grid* g, double alpha, double power, int dtype,
                       void* out_padded);

/* special.hpp:49-71 / :113-118 and acquisition.hpp:21-59 */
double fdwo_bessel_i0(double x);
double fdwo_sinc(double x);
double fdwo_kaiser_window(double x, int radius, double b);
double fdwo_default_kaiser_b(int radius);
/* acquisition.hpp:89-147.  CSR output: offsets[n+1], idx/w[offsets[n]].
 * Returns the total entry count (also when cap is too small; nothing past cap
 * is written), or -1 on invalid input. */
int64_t fdwo_build_injection_map(const fdwo_grid* g, const double* coords /* n x 3 */,
                                 uint64_t n, int radius, double kaiser_b,
                                 uint64_t* offsets, uint64_t* idx, double* w, uint64_t cap);
/* acquisition.hpp:165-177 */
void fdwo_ricker_samples(uint64_t count, double dt, double f, double* out);

/* kernel.hpp:67-102 on a padded field */
void fdwo_apply_boundary(const fdwo_grid* g, const int32_t bc[3][2], int dtype, void* f);

/* ---- Solver<T> (kernel.hpp:170-495), constant density only ---- */
typedef struct fdwo_solver fdwo_solver;

int fdwo_solver_create(const fdwo_grid* g, int dtype, const double* coeffs /* v_0..v_r */,
                       double dt, uint64_t n_steps, const int32_t bc[3][2],
                       const void* velocity_padded, const void* eta_padded,
                       fdwo_solver** out);
void fdwo_solver_destroy(fdwo_solver* s);
/* VariableDensity = true (kernel.hpp:104-136 density_log_gradient; sweep terms
 * :365-373 / :407-417): rho is the padded density field of T. */
int fdwo_solver_set_density(fdwo_solver* s, const void* rho_padded);
/* density_log_gradient alone: grad[axis] padded fields of T (3 x padded size). */
int fdwo_density_log_gradient(const fdwo_grid* g, int dtype, const void* rho_padded, void* grad_out);
/* kernel.hpp:199-203 add_volume_source: padded field of T, amplitude per step
 * (n_amp >= n_steps), applied after the point sources (:439-452). */
int fdwo_solver_add_volume_source(fdwo_solver* s, const void* field_padded, const double* amplitude,
                                  uint64_t n_amp);
void fdwo_solver_set_threads(fdwo_solver* s, int threads); /* 0: all, 1: serial */
int fdwo_solver_set_sources(fdwo_solver* s, uint64_t n_points, const uint64_t* offsets,
                            const uint64_t* idx, const double* w, const double* wavelet,
                            uint64_t n_samples);
int fdwo_solver_set_receivers(fdwo_solver* s, uint64_t n_points, const uint64_t* offsets,
                              const uint64_t* idx, const double* w);
void* fdwo_solver_current(fdwo_solver* s);
void* fdwo_solver_previous(fdwo_solver* s);
uint64_t fdwo_solver_step_index(const fdwo_solver* s);
void fdwo_solver_refresh_boundary(fdwo_solver* s);
/* kernel.hpp:226-233.  On instability returns FDWO_EINSTABLE and fills
 * *bad_step / *bad_max (instability_error::step / max_abs). */
int fdwo_solver_step(fdwo_solver* s, uint64_t* bad_step, double* bad_max);
/* kernel.hpp:265-273 */
double fdwo_solver_max_abs(const fdwo_solver* s);
/* kernel.hpp:150-161 sample_receivers on the current level: one T per point */
void fdwo_solver_sample(const fdwo_solver* s, void* row_out);
/* kernel.hpp:237-263 with saving_stride 0: seismogram (n_steps+1) x n_rec of T,
 * final extended level (halo stripped) of T (may be NULL), kernel seconds. */
int fdwo_solver_forward(fdwo_solver* s, void* seismogram, void* final_extended,
                        double* kernel_seconds, uint64_t* bad_step, double* bad_max);

#ifdef __cplusplus
}
#endif
#endif
