/*
 * fdw_oracle.c -- CPU restatement of the fdwave hot path (TEST INFRASTRUCTURE).
 * See fdw_oracle.h.  Build: oracle/Makefile (gcc -O3 -fopenmp -ffp-contract=off).
 */
#define _GNU_SOURCE
#include "fdw_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

/* ------------------------------------------------------------------ */
/* stencil.hpp:17-44 detail::solve_dense -- partial pivoting, same op order */
static int solve_dense(int n, double* a /* n*n row-major */, double* b, double* x) {
    for (int col = 0; col < n; ++col) {
        int pivot = col;
        for (int row = col + 1; row < n; ++row)
            if (fabs(a[row * n + col]) > fabs(a[pivot * n + col])) pivot = row;
        if (pivot != col) {
            for (int k = 0; k < n; ++k) {
                double t = a[col * n + k];
                a[col * n + k] = a[pivot * n + k];
                a[pivot * n + k] = t;
            }
            double t = b[col];
            b[col] = b[pivot];
            b[pivot] = t;
        }
        if (a[col * n + col] == 0.0) return FDWO_EINVAL;
        for (int row = col + 1; row < n; ++row) {
            const double f = a[row * n + col] / a[col * n + col];
            if (f == 0.0) continue;
            for (int k = col; k < n; ++k) a[row * n + k] -= f * a[col * n + k];
            b[row] -= f * b[col];
        }
    }
    for (int row = n; row-- > 0;) {
        double s = b[row];
        for (int k = row + 1; k < n; ++k) s -= a[row * n + k] * x[k];
        x[row] = s / a[row * n + row];
    }
    return FDWO_OK;
}

static int bad_order(int order) { return order < 2 || order > 20 || order % 2 != 0; }

/* stencil.hpp:55-72 */
int fdwo_second_derivative_coefficients(int order, double* v_out) {
    if (bad_order(order)) return FDWO_EINVAL;
    const int r = order / 2;
    double a[100], rhs[10], x[10];
    for (int m = 1; m <= r; ++m) {
        double inv_fact = 1.0;
        for (int k = 2; k <= 2 * m; ++k) inv_fact /= (double)k;
        for (int j = 1; j <= r; ++j) a[(m - 1) * r + (j - 1)] = pow((double)j, (double)(2 * m)) * inv_fact;
        rhs[m - 1] = (m == 1) ? inv_fact : 0.0;
    }
    if (solve_dense(r, a, rhs, x) != FDWO_OK) return FDWO_EINVAL;
    double sum = 0.0;
    for (int j = 0; j < r; ++j) sum += x[j];
    v_out[0] = -2.0 * sum;
    for (int j = 0; j < r; ++j) v_out[j + 1] = x[j];
    return FDWO_OK;
}

/* stencil.hpp:77-90 */
int fdwo_first_derivative_coefficients(int order, double* w_out) {
    if (bad_order(order)) return FDWO_EINVAL;
    const int r = order / 2;
    double a[100], rhs[10];
    for (int m = 1; m <= r; ++m) {
        double inv_fact = 1.0;
        for (int k = 2; k <= 2 * m - 1; ++k) inv_fact /= (double)k;
        for (int j = 1; j <= r; ++j) a[(m - 1) * r + (j - 1)] = pow((double)j, (double)(2 * m - 1)) * inv_fact;
        rhs[m - 1] = (m == 1) ? inv_fact : 0.0;
    }
    return solve_dense(r, a, rhs, w_out);
}

/* stencil.hpp:113-129 */
double fdwo_stable_dt(double c_max, const double* spacing, int n_spacing, int order, int ndim) {
    if (c_max <= 0.0 || (ndim != 2 && ndim != 3) || n_spacing < 1 || bad_order(order)) return -1.0;
    double dx_min = spacing[0];
    for (int i = 0; i < n_spacing; ++i) {
        if (spacing[i] <= 0.0) return -1.0;
        dx_min = spacing[i] < dx_min ? spacing[i] : dx_min;
    }
    double v[11];
    fdwo_second_derivative_coefficients(order, v);
    double abs_sum = fabs(v[0]);
    for (int j = 1; j <= order / 2; ++j) abs_sum += 2.0 * fabs(v[j]);
    const double a = (double)ndim * abs_sum;
    return 2.0 * dx_min / (c_max * sqrt(a));
}

/* time_axis.hpp:45-47 */
uint64_t fdwo_n_steps(double tf, double dt) {
    uint64_t n = (uint64_t)ceil(tf / dt * (1.0 - 1e-12));
    return n == 0 ? 1 : n;
}

/* grid.hpp:50-104 */
int fdwo_build_grid(int ndim, const double* bbox, const double* spacing, int space_order,
                    const double* damping_lengths, fdwo_grid* g) {
    if ((ndim != 2 && ndim != 3) || bad_order(space_order)) return FDWO_EINVAL;
    memset(g, 0, sizeof(*g));
    g->ndim = ndim;
    g->space_order = space_order;
    g->halo = space_order / 2;
    for (int a = 0; a < 3; ++a) {
        g->spacing[a] = 1.0;
        g->interior[a] = g->extended[a] = g->padded[a] = 1;
    }
    for (int a = 0; a < ndim; ++a) {
        const double lo = bbox[2 * a], hi = bbox[2 * a + 1];
        if (!(hi > lo) || !(spacing[a] > 0.0)) return FDWO_EINVAL;
        g->bbox[a][0] = lo;
        g->bbox[a][1] = hi;
        g->spacing[a] = spacing[a];
        g->interior[a] = (uint64_t)llround((hi - lo) / spacing[a]) + 1;
    }
    for (int a = 0; a < ndim; ++a) {
        for (int side = 0; side < 2; ++side) {
            const double len = damping_lengths ? damping_lengths[2 * a + side] : 0.0;
            if (len < 0.0) return FDWO_EINVAL;
            g->damping_length[a][side] = len;
            g->damping_cells[a][side] = (uint64_t)llround(len / g->spacing[a]);
        }
        g->extended[a] = g->interior[a] + g->damping_cells[a][0] + g->damping_cells[a][1];
        g->padded[a] = g->extended[a] + 2 * (uint64_t)g->halo;
    }
    return FDWO_OK;
}

/* model.hpp:21-26 detail::axis_weights */
static void axis_weights(double coord, double lo, double hi, uint64_t raw_n, uint64_t* i0,
                         double* w) {
    const double pos = (coord - lo) / (hi - lo) * (double)(raw_n - 1);
    double clamped = pos < 0.0 ? 0.0 : pos;
    if ((double)(raw_n - 1) < clamped) clamped = (double)(raw_n - 1);
    uint64_t i = (uint64_t)clamped;
    if (raw_n - 2 < i) i = raw_n - 2;
    *i0 = i;
    *w = clamped - (double)i;
}

static uint64_t clampu(uint64_t v, uint64_t lo, uint64_t hi) { return v < lo ? lo : (hi < v ? hi : v); }

/* model.hpp:34-106 */
int fdwo_resample_model(const fdwo_grid* g, const double* raw, const uint64_t* raw_shape,
                        int dtype, void* out_padded) {
    if (dtype != 4 && dtype != 8) return FDWO_EINVAL;
    for (int a = 0; a < g->ndim; ++a)
        if (raw_shape[a] < 2) return FDWO_EINVAL;
    const uint64_t h = (uint64_t)g->halo;
    uint64_t lo[3] = {0, 0, 0}, n_int[3] = {1, 1, 1};
    for (int a = 0; a < g->ndim; ++a) {
        lo[a] = h + g->damping_cells[a][0];
        n_int[a] = g->interior[a];
    }
    const int is3d = g->ndim == 3;
    const uint64_t rsz = is3d ? raw_shape[2] : 1;
    const uint64_t rsx = raw_shape[1];
#define RAW(iz, ix, iy) raw[((iz) * rsx + (ix)) * rsz + (iy)]
    const uint64_t P0 = g->padded[0], P1 = g->padded[1], P2 = g->padded[2];
#pragma omp parallel for schedule(static)
    for (uint64_t pz = 0; pz < P0; ++pz) {
        const uint64_t cz = clampu(pz, lo[0], lo[0] + n_int[0] - 1) - lo[0];
        uint64_t z0;
        double wz;
        axis_weights(g->bbox[0][0] + (double)cz * g->spacing[0], g->bbox[0][0], g->bbox[0][1],
                     raw_shape[0], &z0, &wz);
        for (uint64_t px = 0; px < P1; ++px) {
            const uint64_t cx = clampu(px, lo[1], lo[1] + n_int[1] - 1) - lo[1];
            uint64_t x0;
            double wx;
            axis_weights(g->bbox[1][0] + (double)cx * g->spacing[1], g->bbox[1][0],
                         g->bbox[1][1], raw_shape[1], &x0, &wx);
            for (uint64_t py = 0; py < P2; ++py) {
                double value;
                if (!is3d) {
                    value = (1 - wz) * ((1 - wx) * RAW(z0, x0, 0) + wx * RAW(z0, x0 + 1, 0)) +
                            wz * ((1 - wx) * RAW(z0 + 1, x0, 0) + wx * RAW(z0 + 1, x0 + 1, 0));
                } else {
                    const uint64_t cy = clampu(py, lo[2], lo[2] + n_int[2] - 1) - lo[2];
                    uint64_t y0;
                    double wy;
                    axis_weights(g->bbox[2][0] + (double)cy * g->spacing[2], g->bbox[2][0],
                                 g->bbox[2][1], raw_shape[2], &y0, &wy);
                    double c00 = (1 - wy) * RAW(z0, x0, y0) + wy * RAW(z0, x0, y0 + 1);
                    double c01 = (1 - wy) * RAW(z0, x0 + 1, y0) + wy * RAW(z0, x0 + 1, y0 + 1);
                    double c10 = (1 - wy) * RAW(z0 + 1, x0, y0) + wy * RAW(z0 + 1, x0, y0 + 1);
                    double c11 = (1 - wy) * RAW(z0 + 1, x0 + 1, y0) + wy * RAW(z0 + 1, x0 + 1, y0 + 1);
                    value = (1 - wz) * ((1 - wx) * c00 + wx * c01) + wz * ((1 - wx) * c10 + wx * c11);
                }
                const uint64_t i = (pz * P1 + px) * P2 + py;
                if (dtype == 4)
                    ((float*)out_padded)[i] = (float)value;
                else
                    ((double*)out_padded)[i] = value;
            }
        }
    }
#undef RAW
    return FDWO_OK;
}

/* model.hpp:162-170 excess distance */
static double excess(const fdwo_grid* g, int axis, uint64_t p) {
    const int64_t rel = (int64_t)p - (int64_t)g->halo - (int64_t)g->damping_cells[axis][0];
    if (rel < 0) return (double)(-rel) * g->spacing[axis];
    const int64_t n = (int64_t)g->interior[axis];
    if (rel >= n) return (double)(rel - n + 1) * g->spacing[axis];
    return 0.0;
}

/* model.hpp:148-186 */
int fdwo_damping_field(const fdwo_grid* g, double alpha, double power, int dtype, void* out) {
    if (alpha < 0.0 || power < 0.0 || (dtype != 4 && dtype != 8)) return FDWO_EINVAL;
    const uint64_t P0 = g->padded[0], P1 = g->padded[1], P2 = g->padded[2];
#pragma omp parallel for schedule(static)
    for (uint64_t pz = 0; pz < P0; ++pz) {
        const double dz = excess(g, 0, pz);
        for (uint64_t px = 0; px < P1; ++px) {
            const double dx = excess(g, 1, px);
            for (uint64_t py = 0; py < P2; ++py) {
                const double dy = g->ndim == 3 ? excess(g, 2, py) : 0.0;
                const double d = sqrt(dz * dz + dx * dx + dy * dy);
                const uint64_t i = (pz * P1 + px) * P2 + py;
                if (dtype == 4)
                    ((float*)out)[i] = d > 0.0 ? (float)(alpha * pow(d, power)) : 0.0f;
                else
                    ((double*)out)[i] = d > 0.0 ? (double)(alpha * pow(d, power)) : 0.0;
            }
        }
    }
    return FDWO_OK;
}

/* special.hpp:49-71 */
double fdwo_bessel_i0(double x) {
    x = fabs(x);
    if (x < 100.0) {
        const double q = 0.25 * x * x;
        double term = 1.0, sum = 1.0;
        for (int k = 1; k < 200; ++k) {
            term *= q / ((double)k * k);
            sum += term;
            if (term < sum * 1e-17) break;
        }
        return sum;
    }
    double term = 1.0, sum = 1.0;
    for (int k = 1; k < 30; ++k) {
        const double odd = 2.0 * k - 1.0;
        term *= odd * odd / (8.0 * k * x);
        sum += term;
        if (fabs(term) < sum * 1e-17) break;
    }
    return exp(x) / sqrt(2.0 * M_PI * x) * sum;
}

/* special.hpp:113-118 */
double fdwo_sinc(double x) {
    if (x == nearbyint(x)) return x == 0.0 ? 1.0 : 0.0;
    const double px = M_PI * x;
    if (fabs(px) < 1e-4) return 1.0 - px * px / 6.0;
    return sin(px) / px;
}

/* acquisition.hpp:21-27 */
double fdwo_kaiser_window(double x, int radius, double b) {
    if (radius < 1 || !(b > 0.0)) return NAN;
    const double u = x / (double)radius;
    if (fabs(u) > 1.0) return 0.0;
    return fdwo_bessel_i0(b * sqrt(1.0 - u * u)) / fdwo_bessel_i0(b);
}

/* acquisition.hpp:31-37 */
double fdwo_default_kaiser_b(int radius) {
    static const double table[10] = {1.24, 2.94, 4.53, 6.31, 7.91, 9.42, 10.88, 12.33, 13.80, 14.93};
    if (radius < 1 || radius > 10) return NAN;
    return table[radius - 1];
}

/* acquisition.hpp:47-59 */
typedef struct {
    int n_min;
    int n;
    double w[32];
} hicks_w;

static void hicks_weights_1d(double alpha, int radius, double b, hicks_w* hw) {
    const double r = (double)radius;
    const int n_lo = (int)ceil(-r - alpha);
    const int n_hi = (int)floor(r - alpha);
    hw->n_min = n_lo;
    hw->n = 0;
    for (int n = n_lo; n <= n_hi; ++n) {
        const double x = (double)n + alpha;
        hw->w[hw->n++] = fdwo_kaiser_window(x, radius, b) * fdwo_sinc(x);
    }
}

/* acquisition.hpp:89-147 */
int64_t fdwo_build_injection_map(const fdwo_grid* g, const double* coords, uint64_t n,
                                 int radius, double kaiser_b, uint64_t* offsets, uint64_t* idx,
                                 double* w, uint64_t cap) {
    if (radius < 1 || radius > 10) return -1;
    const uint64_t s0 = g->padded[1] * g->padded[2], s1 = g->padded[2];
    const int64_t h = g->halo;
    uint64_t total = 0;
    if (offsets) offsets[0] = 0;
    for (uint64_t p = 0; p < n; ++p) {
        const double* coord = coords + 3 * p;
        hicks_w aw[3];
        int64_t nearest[3] = {0, 0, 0};
        for (int a = 0; a < g->ndim; ++a) {
            if (coord[a] < g->bbox[a][0] - 1e-9 || coord[a] > g->bbox[a][1] + 1e-9) return -1;
            const double pos = (coord[a] - g->bbox[a][0]) / g->spacing[a] + (double)g->damping_cells[a][0];
            nearest[a] = (int64_t)floor(pos + 0.5);
            const double alpha = (double)nearest[a] - pos;
            hicks_weights_1d(alpha, radius, kaiser_b, &aw[a]);
        }
        if (g->ndim == 2) {
            aw[2].n_min = 0;
            aw[2].n = 1;
            aw[2].w[0] = 1.0;
            nearest[2] = 0;
        }
        for (int kz = 0; kz < aw[0].n; ++kz) {
            const int64_t iz = nearest[0] + aw[0].n_min + kz;
            if (!(iz >= 0 && iz < (int64_t)g->extended[0])) continue;
            for (int kx = 0; kx < aw[1].n; ++kx) {
                const int64_t ix = nearest[1] + aw[1].n_min + kx;
                if (!(ix >= 0 && ix < (int64_t)g->extended[1])) continue;
                for (int ky = 0; ky < aw[2].n; ++ky) {
                    const int64_t iy = g->ndim == 3 ? nearest[2] + aw[2].n_min + ky : 0;
                    if (g->ndim == 3 && !(iy >= 0 && iy < (int64_t)g->extended[2])) continue;
                    const double wt = aw[0].w[kz] * aw[1].w[kx] * aw[2].w[ky];
                    if (wt == 0.0) continue;
                    const uint64_t flat = (uint64_t)(iz + h) * s0 + (uint64_t)(ix + h) * s1 +
                                          (uint64_t)(iy + (g->ndim == 3 ? h : 0));
                    if (total < cap) {
                        idx[total] = flat;
                        w[total] = wt;
                    }
                    ++total;
                }
            }
        }
        if (offsets) offsets[p + 1] = total;
    }
    return (int64_t)total;
}

/* acquisition.hpp:165-177 */
void fdwo_ricker_samples(uint64_t count, double dt, double f, double* s) {
    const double t0 = 1.0 / f;
    for (uint64_t n = 0; n < count; ++n) {
        const double tau = (double)n * dt - t0;
        const double q = M_PI * M_PI * f * f * tau * tau;
        s[n] = (1.0 - 2.0 * q) * exp(-q);
    }
}

/* ------------------------------------------------------------------ */
/* Solver<T>: generic body instantiated for float and double.          */

struct fdwo_solver {
    fdwo_grid g;
    int dtype;
    int threads;
    int32_t bc[3][2];
    double dt;
    uint64_t n_steps;
    uint64_t step;
    int r;
    double v[11];
    void* prev;
    void* curr;
    void* c2dt2;
    void* om;
    void* iop;
    void* grad[3]; /* grad(rho)/rho per axis when variable density */
    double w[10];  /* first-derivative coefficients w_1..w_r */
    /* sources / receivers: CSR */
    uint64_t n_src, n_rec;
    uint64_t *src_off, *src_idx, *rec_off, *rec_idx;
    double *src_w, *rec_w, *wavelet;
    uint64_t n_wavelet;
    /* volume sources (ModulatedField, kernel.hpp:140-144), insertion order */
    uint64_t n_vol;
    void** vol_field;    /* padded fields of T */
    double** vol_amp;    /* per-step amplitudes */
    uint64_t* vol_namp;
};

#define T float
#define SFX f32
#include "fdw_oracle_solver.inc"
#undef T
#undef SFX
#define T double
#define SFX f64
#include "fdw_oracle_solver.inc"
#undef T
#undef SFX

void fdwo_apply_boundary(const fdwo_grid* g, const int32_t bc[3][2], int dtype, void* f) {
    if (dtype == 4)
        apply_boundary_f32(g, bc, (float*)f);
    else
        apply_boundary_f64(g, bc, (double*)f);
}

int fdwo_solver_create(const fdwo_grid* g, int dtype, const double* coeffs, double dt,
                       uint64_t n_steps, const int32_t bc[3][2], const void* velocity,
                       const void* eta, fdwo_solver** out) {
    if (dtype != 4 && dtype != 8) return FDWO_EINVAL;
    fdwo_solver* s = (fdwo_solver*)calloc(1, sizeof(fdwo_solver));
    if (!s) return FDWO_ENOMEM;
    s->g = *g;
    s->dtype = dtype;
    s->threads = 0;
    memcpy(s->bc, bc, sizeof(s->bc));
    s->dt = dt;
    s->n_steps = n_steps;
    s->r = g->space_order / 2;
    for (int j = 0; j <= s->r; ++j) s->v[j] = coeffs[j];
    const uint64_t n = g->padded[0] * g->padded[1] * g->padded[2];
    s->prev = calloc(n, dtype);
    s->curr = calloc(n, dtype);
    s->c2dt2 = malloc(n * dtype);
    s->om = malloc(n * dtype);
    s->iop = malloc(n * dtype);
    if (!s->prev || !s->curr || !s->c2dt2 || !s->om || !s->iop) {
        fdwo_solver_destroy(s);
        return FDWO_ENOMEM;
    }
    if (dtype == 4)
        precompute_f32(s, (const float*)velocity, (const float*)eta);
    else
        precompute_f64(s, (const double*)velocity, (const double*)eta);
    *out = s;
    return FDWO_OK;
}

void fdwo_solver_destroy(fdwo_solver* s) {
    if (!s) return;
    for (int a = 0; a < 3; ++a) free(s->grad[a]);
    free(s->prev);
    free(s->curr);
    free(s->c2dt2);
    free(s->om);
    free(s->iop);
    free(s->src_off);
    free(s->src_idx);
    free(s->src_w);
    free(s->rec_off);
    free(s->rec_idx);
    free(s->rec_w);
    free(s->wavelet);
    for (uint64_t q = 0; q < s->n_vol; ++q) {
        free(s->vol_field[q]);
        free(s->vol_amp[q]);
    }
    free(s->vol_field);
    free(s->vol_amp);
    free(s->vol_namp);
    free(s);
}

void fdwo_solver_set_threads(fdwo_solver* s, int threads) { s->threads = threads; }

int fdwo_density_log_gradient(const fdwo_grid* g, int dtype, const void* rho, void* grad) {
    double w[10];
    if (fdwo_first_derivative_coefficients(g->space_order, w)) return FDWO_EINVAL;
    const uint64_t n = g->padded[0] * g->padded[1] * g->padded[2];
    memset(grad, 0, 3 * n * dtype);
    if (dtype == 4)
        density_log_gradient_f32(g, w, (const float*)rho, (float*)grad);
    else
        density_log_gradient_f64(g, w, (const double*)rho, (double*)grad);
    return FDWO_OK;
}

int fdwo_solver_set_density(fdwo_solver* s, const void* rho) {
    const uint64_t n = s->g.padded[0] * s->g.padded[1] * s->g.padded[2];
    void* buf = calloc(3 * n, s->dtype);
    if (!buf) return FDWO_ENOMEM;
    int rc = fdwo_density_log_gradient(&s->g, s->dtype, rho, buf);
    if (rc) {
        free(buf);
        return rc;
    }
    for (int a = 0; a < 3; ++a) {
        free(s->grad[a]);
        s->grad[a] = malloc(n * s->dtype);
        memcpy(s->grad[a], (char*)buf + a * n * s->dtype, n * s->dtype);
    }
    free(buf);
    fdwo_first_derivative_coefficients(s->g.space_order, s->w);
    return FDWO_OK;
}

/* kernel.hpp:199-203 add_volume_source */
int fdwo_solver_add_volume_source(fdwo_solver* s, const void* field, const double* amp, uint64_t n_amp) {
    if (n_amp < s->n_steps) return FDWO_EINVAL;
    const uint64_t n = s->g.padded[0] * s->g.padded[1] * s->g.padded[2];
    const uint64_t q = s->n_vol;
    void** vf = (void**)realloc(s->vol_field, (q + 1) * sizeof(void*));
    if (!vf) return FDWO_ENOMEM;
    s->vol_field = vf;
    double** va = (double**)realloc(s->vol_amp, (q + 1) * sizeof(double*));
    if (!va) return FDWO_ENOMEM;
    s->vol_amp = va;
    uint64_t* vn = (uint64_t*)realloc(s->vol_namp, (q + 1) * sizeof(uint64_t));
    if (!vn) return FDWO_ENOMEM;
    s->vol_namp = vn;
    s->vol_field[q] = malloc(n * s->dtype);
    s->vol_amp[q] = (double*)malloc((n_amp ? n_amp : 1) * sizeof(double));
    if (!s->vol_field[q] || !s->vol_amp[q]) return FDWO_ENOMEM;
    memcpy(s->vol_field[q], field, n * s->dtype);
    if (n_amp) memcpy(s->vol_amp[q], amp, n_amp * sizeof(double));
    s->vol_namp[q] = n_amp;
    s->n_vol = q + 1;
    return FDWO_OK;
}

static int copy_csr(uint64_t n, const uint64_t* off, const uint64_t* idx, const double* w,
                    uint64_t** o_off, uint64_t** o_idx, double** o_w) {
    free(*o_off);
    free(*o_idx);
    free(*o_w);
    const uint64_t m = off[n];
    *o_off = (uint64_t*)malloc((n + 1) * sizeof(uint64_t));
    *o_idx = (uint64_t*)malloc((m ? m : 1) * sizeof(uint64_t));
    *o_w = (double*)malloc((m ? m : 1) * sizeof(double));
    if (!*o_off || !*o_idx || !*o_w) return FDWO_ENOMEM;
    memcpy(*o_off, off, (n + 1) * sizeof(uint64_t));
    if (m) {
        memcpy(*o_idx, idx, m * sizeof(uint64_t));
        memcpy(*o_w, w, m * sizeof(double));
    }
    return FDWO_OK;
}

/* kernel.hpp:188-193 */
int fdwo_solver_set_sources(fdwo_solver* s, uint64_t n_points, const uint64_t* offsets,
                            const uint64_t* idx, const double* w, const double* wavelet,
                            uint64_t n_samples) {
    if (n_points > 0 && n_samples < s->n_steps + 1) return FDWO_EINVAL;
    int rc = copy_csr(n_points, offsets, idx, w, &s->src_off, &s->src_idx, &s->src_w);
    if (rc) return rc;
    s->n_src = n_points;
    free(s->wavelet);
    s->wavelet = (double*)malloc((n_samples ? n_samples : 1) * sizeof(double));
    if (n_samples) memcpy(s->wavelet, wavelet, n_samples * sizeof(double));
    s->n_wavelet = n_samples;
    return FDWO_OK;
}

/* kernel.hpp:194-198 */
int fdwo_solver_set_receivers(fdwo_solver* s, uint64_t n_points, const uint64_t* offsets,
                              const uint64_t* idx, const double* w) {
    int rc = copy_csr(n_points, offsets, idx, w, &s->rec_off, &s->rec_idx, &s->rec_w);
    if (rc) return rc;
    s->n_rec = n_points;
    return FDWO_OK;
}

void* fdwo_solver_current(fdwo_solver* s) { return s->curr; }
void* fdwo_solver_previous(fdwo_solver* s) { return s->prev; }
uint64_t fdwo_solver_step_index(const fdwo_solver* s) { return s->step; }

void fdwo_solver_refresh_boundary(fdwo_solver* s) {
    fdwo_apply_boundary(&s->g, (const int32_t(*)[2])s->bc, s->dtype, s->curr);
}

int fdwo_solver_step(fdwo_solver* s, uint64_t* bad_step, double* bad_max) {
    return s->dtype == 4 ? step_f32(s, bad_step, bad_max) : step_f64(s, bad_step, bad_max);
}

double fdwo_solver_max_abs(const fdwo_solver* s) {
    return s->dtype == 4 ? max_abs_f32(s) : max_abs_f64(s);
}

void fdwo_solver_sample(const fdwo_solver* s, void* row) {
    if (s->dtype == 4)
        sample_f32(s, (float*)row);
    else
        sample_f64(s, (double*)row);
}

int fdwo_solver_forward(fdwo_solver* s, void* seis, void* final_ext, double* kernel_seconds,
                        uint64_t* bad_step, double* bad_max) {
    return s->dtype == 4 ? forward_f32(s, seis, final_ext, kernel_seconds, bad_step, bad_max)
                         : forward_f64(s, seis, final_ext, kernel_seconds, bad_step, bad_max);
}
