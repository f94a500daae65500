/* TEST INFRASTRUCTURE ONLY — the CPU checker (see tpflow_oracle.h).
 *
 * Plain-C restatement of the reference (paths relative to /root/reference/proj).
 * Every function cites the reference lines it restates and keeps their
 * expression trees (parenthesisation, std::max/std::min operand order), so with
 * -ffp-contract=off the results are bitwise those of the reference build.
 *
 * Parity pin: tests/test_oracle_cpu.py compares this port with the unmodified
 * reference compiled in place (oracle/_ref) bit for bit — geometry, every step
 * piece, trajectories, audits and error messages — and with the SPEC.md
 * known-answer values.
 *
 * State layout: the reference's (padded, j-major, nx = ncols+6).  A context can
 * own a row slab [row0, row1) of the interior; its padded array then has
 * (row1-row0)+6 rows whose outer three rows are the physical ghosts (at the
 * domain's south/north edges) or halo rows filled from the neighbour.
 * The step keeps two buffers: A = u^n (the reference's u0_ and, after the step,
 * u_) and B = u* (the reference's u_ between the stages, solver.cpp:497-543).
 */
#include "tpflow_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define KG 3 /* kGhost, solver.hpp:14 */

/* std::max / std::min with the reference's operand order (NaN/±0 semantics) */
static inline double smax(double a, double b) { return (a < b) ? b : a; }
static inline double smin(double a, double b) { return (b < a) ? b : a; }

enum { NX_ = 0, NY_, NZ_, JB_, A11_, A12_, A21_, A22_, DNXX_, DNYX_, DNZX_, DNXY_, DNYY_, DNZY_ };

struct orc_ctx {
    char err[512];
    orc_params p;
    int ncols, nrows_g, row0, row1, nrows, nx, ny;
    int has_south, has_north;
    double dxi, deta, eps, t_unit, v_unit, eps_chi, tan_d;
    double* geo[14];
    double* A[6];
    double* B[6];
    double* rhs[6];
    double* f[6];
    double* g[6];
    double *vxs, *vys, *vxf, *vyf, *pjb, *bvx, *bvy, *bvxy;
    int n_cells, n_samples;
    int* ci;
    int* cj;
    char* side;
    double* samples; /* [n][4] */
    double audit[10];
    int adv_only;
    int ghosts_in_B;
    /* split-step scalars */
    double t, t_next, t_end, dt;
    int hit;
    double lam_cur;
    int err_code;
};

static size_t NN(const orc_ctx* c) { return (size_t)c->nx * c->ny; }
#define AT(c, i, j) ((size_t)(j) * (c)->nx + (i))

static double* alloc0(size_t n) {
    double* p = (double*)calloc(n, sizeof(double));
    if (!p) abort();
    return p;
}

static int fail(orc_ctx* c, int code, const char* fmt, ...) __attribute__((format(printf, 3, 4)));
#include <stdarg.h>
static int fail(orc_ctx* c, int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(c->err, sizeof(c->err), fmt, ap);
    va_end(ap);
    c->err_code = code;
    return code;
}

/* ---- terrain.cpp:23-45: second-order slopes --------------------------------- */
static double deriv(double m1, double p1, double spacing) { return (p1 - m1) / (2.0 * spacing); }
static double deriv_low(double f0, double f1, double f2, double spacing) {
    return (-3.0 * f0 + 4.0 * f1 - f2) / (2.0 * spacing);
}
static double deriv_high(double f0, double f1, double f2, double spacing) {
    return (3.0 * f0 - 4.0 * f1 + f2) / (2.0 * spacing);
}
static double diff_x(const double* f, int nx, int i, int j, double d) {
    const double* r = f + (size_t)j * nx;
    if (i == 0) return deriv_low(r[0], r[1], r[2], d);
    if (i == nx - 1) return deriv_high(r[nx - 1], r[nx - 2], r[nx - 3], d);
    return deriv(r[i - 1], r[i + 1], d);
}
static double diff_y(const double* f, int nx, int ny, int i, int j, double d) {
    if (j == 0) return deriv_low(f[i], f[(size_t)nx + i], f[2 * (size_t)nx + i], d);
    if (j == ny - 1)
        return deriv_high(f[(size_t)(ny - 1) * nx + i], f[(size_t)(ny - 2) * nx + i],
                          f[(size_t)(ny - 3) * nx + i], d);
    return deriv(f[(size_t)(j - 1) * nx + i], f[(size_t)(j + 1) * nx + i], d);
}

/* ---- terrain.cpp:113-145 extend_grid + :157-215 compute_geometry (whole grid) --- */
static void build_geometry(const double* z, int ncols, int nrows, double cellsize, double L,
                           double** G /* 14 fields, (ncols+6)*(nrows+6) */) {
    const int W = ncols + 2 * KG, H = nrows + 2 * KG;
    double* e = alloc0((size_t)W * H);
#define Z(i, j) e[(size_t)(j) * W + (i)]
    for (int j = 0; j < nrows; ++j)
        for (int i = 0; i < ncols; ++i) Z(i + KG, j + KG) = z[(size_t)j * ncols + i];
    for (int j = KG; j < KG + nrows; ++j) {
        for (int g = 1; g <= KG; ++g) {
            Z(KG - g, j) = Z(KG, j) + g * (Z(KG, j) - Z(KG + 1, j));
            int ee = KG + ncols - 1;
            Z(ee + g, j) = Z(ee, j) + g * (Z(ee, j) - Z(ee - 1, j));
        }
    }
    for (int i = 0; i < W; ++i) {
        for (int g = 1; g <= KG; ++g) {
            Z(i, KG - g) = Z(i, KG) + g * (Z(i, KG) - Z(i, KG + 1));
            int n = KG + nrows - 1;
            Z(i, n + g) = Z(i, n) + g * (Z(i, n) - Z(i, n - 1));
        }
    }
#undef Z
    const double dxi = cellsize / L, deta = cellsize / L;
    double* b = alloc0((size_t)W * H);
    for (size_t k = 0; k < (size_t)W * H; ++k) b[k] = e[k] / L;
    for (int j = 0; j < H; ++j) {
        for (int i = 0; i < W; ++i) {
            size_t k = (size_t)j * W + i;
            double bx = diff_x(b, W, i, j, dxi);
            double by = diff_y(b, W, H, i, j, deta);
            double norm = sqrt(1.0 + (bx * bx + by * by));
            G[NX_][k] = -bx / norm;
            G[NY_][k] = -by / norm;
            G[NZ_][k] = 1.0 / norm;
            /* basal_transform, terrain.cpp:147-155 */
            double bn = sqrt(1.0 + (bx * bx + by * by));
            double m[3][3] = {{1.0, 0.0, -bx / bn}, {0.0, 1.0, -by / bn}, {bx, by, 1.0 / bn}};
            double det = norm;
            G[JB_][k] = det;
            G[A11_][k] = (m[1][1] * m[2][2] - m[1][2] * m[2][1]) / det;
            G[A12_][k] = (m[0][2] * m[2][1] - m[0][1] * m[2][2]) / det;
            G[A21_][k] = (m[1][2] * m[2][0] - m[1][0] * m[2][2]) / det;
            G[A22_][k] = (m[0][0] * m[2][2] - m[0][2] * m[2][0]) / det;
        }
    }
    for (int j = 0; j < H; ++j) {
        for (int i = 0; i < W; ++i) {
            size_t k = (size_t)j * W + i;
            G[DNXX_][k] = diff_x(G[NX_], W, i, j, dxi);
            G[DNYX_][k] = diff_x(G[NY_], W, i, j, dxi);
            G[DNZX_][k] = diff_x(G[NZ_], W, i, j, dxi);
            G[DNXY_][k] = diff_y(G[NX_], W, H, i, j, deta);
            G[DNYY_][k] = diff_y(G[NY_], W, H, i, j, deta);
            G[DNZY_][k] = diff_y(G[NZ_], W, H, i, j, deta);
        }
    }
    free(e);
    free(b);
}

static int validate(orc_ctx* c, const orc_params* p) {
    /* params.hpp:40-50, :21-25, config.hpp:31-40 (messages verbatim) */
    if (!(p->delta_b >= 0.0 && p->delta_b < 90.0)) return fail(c, 2, "params: delta_b must be in [0, 90) degrees");
    if (!(p->C_d >= 0.0)) return fail(c, 2, "params: C_d must be >= 0");
    if (!(p->N_R > 0.0)) return fail(c, 2, "params: N_R must be > 0");
    if (!(p->theta_b >= 0.0)) return fail(c, 2, "params: theta_b must be >= 0");
    if (!(p->phi_s0 >= 0.0 && p->phi_s0 <= 1.0)) return fail(c, 2, "params: phi_s0 must be in [0, 1]");
    if (!(p->alpha_rho > 0.0 && p->alpha_rho <= 1.0)) return fail(c, 2, "params: alpha_rho must be in (0, 1]");
    if (!(p->L > 0.0)) return fail(c, 2, "scaling: L must be > 0");
    if (!(p->H > 0.0)) return fail(c, 2, "scaling: H must be > 0");
    if (!(p->g > 0.0)) return fail(c, 2, "scaling: g must be > 0");
    if (!(p->cfl > 0.0 && p->cfl <= 0.125)) return fail(c, 2, "config: cfl must be in (0, 0.125], got %f", p->cfl);
    if (!(p->t_end > 0.0)) return fail(c, 2, "config: t_end must be > 0");
    if (!(p->dt_out > 0.0)) return fail(c, 2, "config: dt_out must be > 0");
    if (!(p->h_dry > 0.0)) return fail(c, 2, "config: h_dry must be > 0");
    if (!(p->eps_h > 0.0)) return fail(c, 2, "config: eps_h must be > 0");
    return 0;
}

int orc_create_slab(const orc_params* p, int ncols, int nrows, double cellsize, double xll, double yll,
                    const double* z, int row0, int row1, orc_ctx** out) {
    (void)xll;
    (void)yll;
    orc_ctx* c = (orc_ctx*)calloc(1, sizeof(orc_ctx));
    *out = c;
    int rc = validate(c, p);
    if (rc) return rc;
    if (row0 < 0 || row1 > nrows || row1 - row0 < 2) return fail(c, 2, "slab rows out of range");
    c->p = *p;
#ifdef _OPENMP
    omp_set_num_threads(p->lanes > 1 ? p->lanes : 1);
#endif
    c->ncols = ncols;
    c->nrows_g = nrows;
    c->row0 = row0;
    c->row1 = row1;
    c->nrows = row1 - row0;
    c->nx = ncols + 2 * KG;
    c->ny = c->nrows + 2 * KG;
    c->has_south = row0 == 0;
    c->has_north = row1 == nrows;
    c->dxi = cellsize / p->L;
    c->deta = cellsize / p->L;
    c->eps = p->H / p->L;              /* ScalingConfig::epsilon */
    c->t_unit = sqrt(p->L / p->g);     /* ScalingConfig::t_unit */
    c->v_unit = sqrt(p->g * p->L);     /* ScalingConfig::v_unit */
    c->eps_chi = pow(c->eps, p->chi);  /* physics.hpp:60 */
    c->tan_d = tan(p->delta_b * M_PI / 180.0); /* params.hpp:38 */
    /* whole-grid geometry, then our rows (solver.cpp:16) */
    const int Wg = ncols + 2 * KG, Hg = nrows + 2 * KG;
    double* Gfull[14];
    for (int k = 0; k < 14; ++k) Gfull[k] = alloc0((size_t)Wg * Hg);
    build_geometry(z, ncols, nrows, cellsize, p->L, Gfull);
    for (int k = 0; k < 14; ++k) {
        c->geo[k] = alloc0(NN(c));
        memcpy(c->geo[k], Gfull[k] + (size_t)row0 * Wg, sizeof(double) * NN(c));
        free(Gfull[k]);
    }
    for (int k = 0; k < 6; ++k) {
        c->A[k] = alloc0(NN(c));
        c->B[k] = alloc0(NN(c));
        c->rhs[k] = alloc0(NN(c));
        c->f[k] = alloc0(NN(c));
        c->g[k] = alloc0(NN(c));
    }
    c->vxs = alloc0(NN(c));
    c->vys = alloc0(NN(c));
    c->vxf = alloc0(NN(c));
    c->vyf = alloc0(NN(c));
    c->pjb = alloc0(NN(c));
    c->bvx = alloc0(NN(c));
    c->bvy = alloc0(NN(c));
    c->bvxy = alloc0(NN(c));
    return 0;
}

int orc_create(const orc_params* p, int ncols, int nrows, double cellsize, double xll, double yll,
               const double* z, orc_ctx** out) {
    return orc_create_slab(p, ncols, nrows, cellsize, xll, yll, z, 0, nrows, out);
}

void orc_destroy(orc_ctx* c) {
    if (!c) return;
    for (int k = 0; k < 14; ++k) free(c->geo[k]);
    for (int k = 0; k < 6; ++k) {
        free(c->A[k]);
        free(c->B[k]);
        free(c->rhs[k]);
        free(c->f[k]);
        free(c->g[k]);
    }
    free(c->vxs); free(c->vys); free(c->vxf); free(c->vyf); free(c->pjb);
    free(c->bvx); free(c->bvy); free(c->bvxy);
    free(c->ci); free(c->cj); free(c->side); free(c->samples);
    free(c);
}

const char* orc_last_error(orc_ctx* c) { return c->err; }

void orc_dims(orc_ctx* c, int* nx, int* ny, double* dxi, double* deta) {
    *nx = c->nx; *ny = c->ny; *dxi = c->dxi; *deta = c->deta;
}

static void sync_ghosts(orc_ctx* c);

/* solver.cpp:35-57 */
int orc_set_initial_thickness(orc_ctx* c, const double* h) {
    sync_ghosts(c);
    double phi = c->p.phi_s0;
    for (int j = 0; j < c->nrows_g; ++j) {
        for (int i = 0; i < c->ncols; ++i) {
            double hm = h[(size_t)j * c->ncols + i];
            if (hm < 0.0)
                return fail(c, 2, "initial state: negative thickness at column %d, row %d", i, j);
            if (j < c->row0 || j >= c->row1) continue;
            double h_scaled = hm / c->p.H;
            size_t k = AT(c, i + KG, j - c->row0 + KG);
            double jb = c->geo[JB_][k];
            c->A[0][k] = jb * h_scaled * phi;
            c->A[1][k] = jb * h_scaled * (1.0 - phi);
            c->A[2][k] = 0.0; c->A[3][k] = 0.0; c->A[4][k] = 0.0; c->A[5][k] = 0.0;
        }
    }
    return 0;
}

/* solver.cpp:59-76 */
int orc_set_initial_velocity(orc_ctx* c, const double* vx, const double* vy) {
    sync_ghosts(c);
    double vu = c->v_unit;
    for (int j = c->row0; j < c->row1; ++j) {
        for (int i = 0; i < c->ncols; ++i) {
            size_t k = AT(c, i + KG, j - c->row0 + KG);
            double jb = c->geo[JB_][k];
            double hs = c->A[0][k] / jb;
            double hf = c->A[1][k] / jb;
            double ux = vx[(size_t)j * c->ncols + i] / vu, uy = vy[(size_t)j * c->ncols + i] / vu;
            c->A[2][k] = jb * hs * ux;
            c->A[3][k] = jb * hs * uy;
            c->A[4][k] = jb * hf * ux;
            c->A[5][k] = jb * hf * uy;
        }
    }
    return 0;
}

/* hydrograph.hpp:49-77 + solver.cpp:78-81 */
int orc_set_hydrograph(orc_ctx* c, int n_cells, const int* ci, const int* cj, const char* side,
                       int n_samples, const double* t, const double* h, const double* phi,
                       const double* speed) {
    for (int k = 1; k < n_samples; ++k)
        if (!(t[k] > t[k - 1]))
            return fail(c, 2, "hydrograph: sample times must be strictly increasing (t=%f after t=%f)",
                        t[k], t[k - 1]);
    for (int k = 0; k < n_samples; ++k) {
        if (h[k] < 0.0) return fail(c, 2, "hydrograph: negative thickness");
        if (speed[k] < 0.0) return fail(c, 2, "hydrograph: negative speed");
        if (phi[k] < 0.0 || phi[k] > 1.0) return fail(c, 2, "hydrograph: phi_s out of [0, 1]");
    }
    for (int k = 0; k < n_cells; ++k) {
        int ok = 0;
        switch (side[k]) {
            case 'N': ok = cj[k] == c->nrows_g - 1; break;
            case 'S': ok = cj[k] == 0; break;
            case 'E': ok = ci[k] == c->ncols - 1; break;
            case 'W': ok = ci[k] == 0; break;
            default: return fail(c, 2, "hydrograph: unknown side '%c'", side[k]);
        }
        if (ci[k] < 0 || ci[k] >= c->ncols || cj[k] < 0 || cj[k] >= c->nrows_g) ok = 0;
        if (!ok)
            return fail(c, 2, "hydrograph: cell (%d, %d) is not on the boundary ring of side %c", ci[k],
                        cj[k], side[k]);
    }
    free(c->ci); free(c->cj); free(c->side); free(c->samples);
    c->n_cells = n_cells;
    c->n_samples = n_samples;
    c->ci = (int*)malloc(sizeof(int) * (n_cells + 1));
    c->cj = (int*)malloc(sizeof(int) * (n_cells + 1));
    c->side = (char*)malloc(n_cells + 1);
    c->samples = (double*)malloc(sizeof(double) * 4 * (n_samples + 1));
    for (int k = 0; k < n_cells; ++k) { c->ci[k] = ci[k]; c->cj[k] = cj[k]; c->side[k] = side[k]; }
    for (int k = 0; k < n_samples; ++k) {
        c->samples[4 * k] = t[k]; c->samples[4 * k + 1] = h[k];
        c->samples[4 * k + 2] = phi[k]; c->samples[4 * k + 3] = speed[k];
    }
    return 0;
}

static void ghost_copy(orc_ctx* c, double** dst, double** src);

static void sync_ghosts(orc_ctx* c) {
    if (c->ghosts_in_B) {
        ghost_copy(c, c->A, c->B);
        c->ghosts_in_B = 0;
    }
}

void orc_get_state(orc_ctx* c, double* out) {
    sync_ghosts(c);
    for (int k = 0; k < 6; ++k) memcpy(out + k * NN(c), c->A[k], sizeof(double) * NN(c));
}
void orc_set_state(orc_ctx* c, const double* in) {
    for (int k = 0; k < 6; ++k) memcpy(c->A[k], in + k * NN(c), sizeof(double) * NN(c));
    c->ghosts_in_B = 0;
}
void orc_get_geometry(orc_ctx* c, double* out) {
    for (int k = 0; k < 14; ++k) memcpy(out + k * NN(c), c->geo[k], sizeof(double) * NN(c));
}

/* ---- hydrograph.hpp:31-45 ------------------------------------------------------- */
static void hydro_at(const orc_ctx* c, double t, double* h, double* phi, double* speed) {
    const double* s = c->samples;
    int n = c->n_samples;
    if (n == 0 || t > s[4 * (n - 1)]) { *h = *phi = *speed = 0.0; return; }
    if (t <= s[0]) { *h = s[1]; *phi = s[2]; *speed = s[3]; return; }
    for (int k = 1; k < n; ++k) {
        if (t <= s[4 * k]) {
            const double* a = s + 4 * (k - 1);
            const double* b = s + 4 * k;
            double w = (t - a[0]) / (b[0] - a[0]);
            *h = a[1] + w * (b[1] - a[1]);
            *phi = a[2] + w * (b[2] - a[2]);
            *speed = a[3] + w * (b[3] - a[3]);
            return;
        }
    }
    *h = s[4 * (n - 1) + 1]; *phi = s[4 * (n - 1) + 2]; *speed = s[4 * (n - 1) + 3];
}

/* ---- solver.cpp:83-137 apply_boundaries (slab-aware) ------------------------------ */
static void apply_bc(orc_ctx* c, double** s, double t_scaled) {
    const int nx = c->nx, ny = c->ny;
    for (int k = 0; k < 6; ++k) {
        double* f = s[k];
        for (int j = KG; j < ny - KG; ++j) {
            double w = f[AT(c, KG, j)];
            double e = f[AT(c, nx - KG - 1, j)];
            for (int g = 0; g < KG; ++g) {
                f[AT(c, g, j)] = w;
                f[AT(c, nx - 1 - g, j)] = e;
            }
        }
        for (int i = 0; i < nx; ++i) {
            double so = f[AT(c, i, KG)];
            double no = f[AT(c, i, ny - KG - 1)];
            for (int g = 0; g < KG; ++g) {
                if (c->has_south) f[AT(c, i, g)] = so;
                if (c->has_north) f[AT(c, i, ny - 1 - g)] = no;
            }
        }
    }
    if (c->p.mode == 1 && c->n_samples > 0) {
        double t_seconds = t_scaled * c->t_unit;
        double sh, sphi, sspeed;
        hydro_at(c, t_seconds, &sh, &sphi, &sspeed);
        double h = sh / c->p.H;
        double speed = sspeed / c->v_unit;
        double hs = h * sphi;
        double hf = h * (1.0 - sphi);
        for (int q = 0; q < c->n_cells; ++q) {
            int pi = c->ci[q] + KG, pj = c->cj[q] + KG - c->row0;
            double vx = 0.0, vy = 0.0;
            int di = 0, dj = 0;
            switch (c->side[q]) {
                case 'E': vx = -speed; di = 1; break;
                case 'W': vx = speed; di = -1; break;
                case 'N': vy = -speed; dj = 1; break;
                case 'S': vy = speed; dj = -1; break;
            }
            for (int g = 1; g <= KG; ++g) {
                int gi = pi + di * g, gj = pj + dj * g;
                if (gj < 0 || gj >= ny) continue;
                /* rows we do not own (halo rows) belong to the neighbour's BC */
                if (dj == 0 && (gj < KG || gj >= ny - KG)) continue;
                if (dj != 0 && ((dj < 0 && !c->has_south) || (dj > 0 && !c->has_north))) continue;
                size_t k = AT(c, gi, gj);
                double jb = c->geo[JB_][k];
                s[0][k] = jb * hs;
                s[1][k] = jb * hf;
                s[2][k] = jb * hs * vx;
                s[3][k] = jb * hs * vy;
                s[4][k] = jb * hf * vx;
                s[5][k] = jb * hf * vy;
            }
        }
    }
}

static void ghost_copy(orc_ctx* c, double** dst, double** src) {
    const int nx = c->nx, ny = c->ny;
    for (int k = 0; k < 6; ++k)
        for (int j = 0; j < ny; ++j)
            for (int i = 0; i < nx; ++i) {
                int ghost = i < KG || i >= nx - KG || (c->has_south && j < KG) || (c->has_north && j >= ny - KG);
                if (ghost) dst[k][AT(c, i, j)] = src[k][AT(c, i, j)];
            }
}

/* ---- solver.cpp:139-166 regularize ----------------------------------------------------- */
static int regularize(orc_ctx* c, double** s) {
    double cell_area = c->dxi * c->deta;
    for (int j = KG; j < c->ny - KG; ++j) {
        for (int i = KG; i < c->nx - KG; ++i) {
            size_t k = AT(c, i, j);
            double jb = c->geo[JB_][k];
            for (int ph = 0; ph < 2; ++ph) {
                double* w = s[ph];
                double hp = w[k] / jb;
                if (hp < 0.0) {
                    if (hp < -1e-12) {
                        char num[64];
                        snprintf(num, sizeof(num), "%f", hp);
                        return fail(c, 4, "negative %s thickness %s at cell (%d, %d)", ph == 0 ? "solid" : "fluid",
                                    num, i - KG, j - KG + c->row0);
                    }
                    c->audit[5 * ph + 4] += -w[k] * cell_area;
                    w[k] = 0.0;
                    hp = 0.0;
                }
                if (hp < c->p.h_dry) {
                    s[2 + 2 * ph][k] = 0.0;
                    s[3 + 2 * ph][k] = 0.0;
                }
            }
        }
    }
    return 0;
}

/* ---- physics.hpp ------------------------------------------------------------------- */
static inline double desing(double q, double jb, double h_phase, double eps_h) { /* :33-37 */
    double hm = smax(h_phase, eps_h);
    double denom = h_phase * h_phase + hm * hm;
    return (q / jb) * (2.0 * h_phase / denom);
}
static inline double curvature(const orc_ctx* c, size_t k, double vx, double vy) { /* :40-52 */
    double vz = -(c->geo[NX_][k] * vx + c->geo[NY_][k] * vy) / c->geo[NZ_][k];
    double along_xi = (vx * c->geo[DNXX_][k] + vy * c->geo[DNYX_][k]) + vz * c->geo[DNZX_][k];
    double along_eta = (vx * c->geo[DNXY_][k] + vy * c->geo[DNYY_][k]) + vz * c->geo[DNZY_][k];
    return along_xi * vx + along_eta * vy;
}
static inline double limited_slope(double a, double b) { /* solver.hpp:17-21 */
    if (a > 0.0 && b > 0.0) return smin(a, b);
    if (a < 0.0 && b < 0.0) return smax(a, b);
    return 0.0;
}

/* ---- solver.cpp:168-208 compute_cell_fields ------------------------------------------- */
static void cell_fields(orc_ctx* c, double** s) {
    const size_t n = NN(c);
    const double eps_h = c->p.eps_h;
#pragma omp parallel for schedule(static)
    for (size_t k = 0; k < n; ++k) {
        double jb = c->geo[JB_][k];
        double hs = s[0][k] / jb;
        double hf = s[1][k] / jb;
        double h = hs + hf;
        c->vxs[k] = desing(s[2][k], jb, hs, eps_h);
        c->vys[k] = desing(s[3][k], jb, hs, eps_h);
        c->vxf[k] = desing(s[4][k], jb, hf, eps_h);
        c->vyf[k] = desing(s[5][k], jb, hf, eps_h);
        c->pjb[k] = jb * h * (c->geo[NZ_][k] * h / 2.0);
    }
    if (c->adv_only) return;
    const int nx = c->nx, ny = c->ny;
#pragma omp parallel for schedule(static)
    for (int j = 1; j < ny - 1; ++j) {
        for (int i = 1; i < nx - 1; ++i) {
            size_t k = AT(c, i, j);
            double jb = c->geo[JB_][k];
            double h = (s[0][k] + s[1][k]) / jb;
            double gux = (c->vxf[k + 1] - c->vxf[k - 1]) / (2.0 * c->dxi);
            double guy = (c->vxf[k + nx] - c->vxf[k - nx]) / (2.0 * c->deta);
            double gwx = (c->vyf[k + 1] - c->vyf[k - 1]) / (2.0 * c->dxi);
            double gwy = (c->vyf[k + nx] - c->vyf[k - nx]) / (2.0 * c->deta);
            /* physics::viscous_brackets, physics.hpp:166-174 */
            double jh = jb * h;
            double a11 = c->geo[A11_][k], a12 = c->geo[A12_][k], a21 = c->geo[A21_][k], a22 = c->geo[A22_][k];
            c->bvx[k] = jh * (a11 * gux + a21 * guy);
            c->bvy[k] = jh * (a12 * gwx + a22 * gwy);
            c->bvxy[k] = jh * ((a12 * gux + a22 * guy) + (a11 * gwx + a21 * gwy));
        }
    }
}

/* ---- solver.cpp:220-350 compute_face_fluxes ------------------------------------------ */
static inline double edge(const double* f, size_t k, long d, double sign) { /* :229-235 */
    double um = f[k - d];
    double uc = f[k];
    double up = f[k + d];
    double slope = limited_slope(uc - um, up - uc);
    return uc + sign * 0.5 * slope;
}

static void face_flux(orc_ctx* c, double** s, size_t k, long d, double ann_l, double ann_r, double ant_l,
                      double ant_r, double** out, int normal_is_x) { /* :239-316 */
    const double eps = c->eps, eps_h = c->p.eps_h, h_dry = c->p.h_dry, alpha = c->p.alpha_rho;
    size_t kp = k + d;
    double jbf = 0.5 * (c->geo[JB_][k] + c->geo[JB_][kp]);
    double cf = 0.5 * (c->geo[NZ_][k] + c->geo[NZ_][kp]);
    double ann = 0.5 * (ann_l + ann_r);
    double ant = 0.5 * (ant_l + ant_r);
    double Lw[2], Rw[2], Lqn[2], Lqt[2], Rqn[2], Rqt[2];
    for (int p = 0; p < 2; ++p) {
        Lw[p] = edge(s[p], k, d, +1.0);
        Rw[p] = edge(s[p], kp, d, -1.0);
        double qxl = edge(s[2 + 2 * p], k, d, +1.0);
        double qxr = edge(s[2 + 2 * p], kp, d, -1.0);
        double qyl = edge(s[3 + 2 * p], k, d, +1.0);
        double qyr = edge(s[3 + 2 * p], kp, d, -1.0);
        Lqn[p] = normal_is_x ? qxl : qyl;
        Lqt[p] = normal_is_x ? qyl : qxl;
        Rqn[p] = normal_is_x ? qxr : qyr;
        Rqt[p] = normal_is_x ? qyr : qxr;
    }
    double hL[2], hR[2];
    for (int p = 0; p < 2; ++p) {
        hL[p] = Lw[p] / jbf;
        hR[p] = Rw[p] / jbf;
    }
    double htL = hL[0] + hL[1];
    double htR = hR[0] + hR[1];
    if (htL < h_dry && htR < h_dry) {
        for (int q = 0; q < 6; ++q) out[q][k] = 0.0;
        return;
    }
    double vnL[2], vnR[2];
    double a = 0.0;
    double celL = sqrt(eps * cf * smax(htL, 0.0));
    double celR = sqrt(eps * cf * smax(htR, 0.0));
    for (int p = 0; p < 2; ++p) {
        vnL[p] = desing(Lqn[p], jbf, smax(hL[p], 0.0), eps_h);
        vnR[p] = desing(Rqn[p], jbf, smax(hR[p], 0.0), eps_h);
        a = smax(a, smax(fabs(vnL[p]) + celL, fabs(vnR[p]) + celR));
    }
    double prL[2], prR[2];
    if (c->adv_only) {
        prL[0] = prL[1] = prR[0] = prR[1] = 0.0;
    } else {
        prL[0] = cf * (1.0 - alpha) * hL[0] / 2.0;
        prR[0] = cf * (1.0 - alpha) * hR[0] / 2.0;
        prL[1] = cf * htL / 2.0;
        prR[1] = cf * htR / 2.0;
    }
    for (int p = 0; p < 2; ++p) {
        /* physics::directional_flux, physics.hpp:84-95 */
        double flm = Lw[p] * vnL[p];
        double fln = Lqn[p] * vnL[p] + eps * jbf * htL * ann * prL[p];
        double flt = Lqt[p] * vnL[p] + eps * jbf * htL * ant * prL[p];
        double frm = Rw[p] * vnR[p];
        double frn = Rqn[p] * vnR[p] + eps * jbf * htR * ann * prR[p];
        double frt = Rqt[p] * vnR[p] + eps * jbf * htR * ant * prR[p];
        double mass = 0.5 * (flm + frm) - 0.5 * a * (Rw[p] - Lw[p]);
        double momn = 0.5 * (fln + frn) - 0.5 * a * (Rqn[p] - Lqn[p]);
        double momt = 0.5 * (flt + frt) - 0.5 * a * (Rqt[p] - Lqt[p]);
        out[p][k] = mass;
        out[2 + 2 * p][k] = normal_is_x ? momn : momt;
        out[3 + 2 * p][k] = normal_is_x ? momt : momn;
    }
}

static void face_fluxes(orc_ctx* c, double** s) {
    const int nx = c->nx, ny = c->ny;
#pragma omp parallel for schedule(static)
    for (int j = KG; j < ny - KG; ++j)
        for (int i = KG - 1; i < nx - KG; ++i) {
            size_t k = AT(c, i, j);
            face_flux(c, s, k, 1, c->geo[A11_][k], c->geo[A11_][k + 1], c->geo[A12_][k], c->geo[A12_][k + 1],
                      c->f, 1);
        }
#pragma omp parallel for schedule(static)
    for (int j = KG - 1; j < ny - KG; ++j)
        for (int i = KG; i < nx - KG; ++i) {
            size_t k = AT(c, i, j);
            face_flux(c, s, k, nx, c->geo[A22_][k], c->geo[A22_][k + nx], c->geo[A21_][k],
                      c->geo[A21_][k + nx], c->g, 0);
        }
}

/* ---- solver.cpp:352-376 accumulate_boundary_fluxes (physical edges of the slab) ------ */
static void tally(orc_ctx* c, double weight_dt) {
    for (int ph = 0; ph < 2; ++ph) {
        const double* fx = c->f[ph];
        const double* fy = c->g[ph];
        double in = 0.0, out = 0.0;
#define ADD(v)                       \
    do {                             \
        double o_ = (v);             \
        if (o_ >= 0.0) out += o_;    \
        else in += -o_;              \
    } while (0)
        int iw = KG - 1, ie = c->nx - KG - 1;
        for (int j = KG; j < c->ny - KG; ++j) {
            ADD(-fx[AT(c, iw, j)] * c->deta * weight_dt);
            ADD(fx[AT(c, ie, j)] * c->deta * weight_dt);
        }
        int js = KG - 1, jn = c->ny - KG - 1;
        for (int i = KG; i < c->nx - KG; ++i) {
            if (c->has_south) ADD(-fy[AT(c, i, js)] * c->dxi * weight_dt);
            if (c->has_north) ADD(fy[AT(c, i, jn)] * c->dxi * weight_dt);
        }
#undef ADD
        c->audit[5 * ph + 2] += in;
        c->audit[5 * ph + 3] += out;
    }
}

/* ---- solver.cpp:378-448 residual ----------------------------------------------------- */
static void residual(orc_ctx* c, double** s, double flux_weight_dt) {
    cell_fields(c, s);
    face_fluxes(c, s);
    tally(c, flux_weight_dt);
    const double eps = c->eps, h_dry = c->p.h_dry;
    const int nx = c->nx, ny = c->ny;
#pragma omp parallel for schedule(static)
    for (int j = KG; j < ny - KG; ++j) {
        for (int i = KG; i < nx - KG; ++i) {
            size_t k = AT(c, i, j);
            double div[6];
            for (int q = 0; q < 6; ++q)
                div[q] = (-(c->f[q][k] - c->f[q][k - 1]) / c->dxi) + (-(c->g[q][k] - c->g[q][k - nx]) / c->deta);
            if (c->adv_only) {
                for (int q = 0; q < 6; ++q) c->rhs[q][k] = div[q];
                continue;
            }
            double jb = c->geo[JB_][k], nX = c->geo[NX_][k], nY = c->geo[NY_][k], cc = c->geo[NZ_][k];
            double a11 = c->geo[A11_][k], a12 = c->geo[A12_][k], a21 = c->geo[A21_][k], a22 = c->geo[A22_][k];
            double hs = s[0][k] / jb;
            double hf = s[1][k] / jb;
            double h = hs + hf;
            double phi_s = h < h_dry ? 0.0 : hs / h;
            double phi_f = h < h_dry ? 0.0 : hf / h;
            double vsx = c->vxs[k], vsy = c->vys[k], vfx = c->vxf[k], vfy = c->vyf[k];
            double kappa_s = curvature(c, k, vsx, vsy);
            double kappa_f = curvature(c, k, vfx, vfy);
            /* physics::hydrostatic_terms, physics.hpp:56-69 */
            double p_b_s = smax(0.0, hs * (cc * (1.0 - c->p.alpha_rho) - c->eps_chi * kappa_s));
            double p_b_f = smax(0.0, hf * (cc - c->eps_chi * kappa_f));
            double gPx = (c->pjb[k + 1] - c->pjb[k - 1]) / (2.0 * c->dxi);
            double gPy = (c->pjb[k + nx] - c->pjb[k - nx]) / (2.0 * c->deta);
            /* physics.hpp:98-155 */
            double sn_sx = jb * p_b_s * nX, sn_sy = jb * p_b_s * nY;
            double Avx = a11 * gPx + a21 * gPy, Avy = a12 * gPx + a22 * gPy;
            double fsp = -eps * c->p.alpha_rho * phi_s;
            double sf_sx = fsp * Avx, sf_sy = fsp * Avy;
            double sv_sx = 0.0, sv_sy = 0.0, sv_fx = 0.0, sv_fy = 0.0;
            if (!(h <= 0.0)) {
                double common = jb * c->p.C_d * (hs * hf / h);
                double cx = common * (vfx - vsx);
                double cy = common * (vfy - vsy);
                sv_sx = c->p.alpha_rho * cx;
                sv_sy = c->p.alpha_rho * cy;
                sv_fx = -cx;
                sv_fy = -cy;
            }
            double sn_fx = jb * p_b_f * nX, sn_fy = jb * p_b_f * nY;
            double coeff = jb * hf * c->p.theta_b / (eps * c->p.N_R);
            double sd_fx = -coeff * vfx, sd_fy = -coeff * vfy;
            double sf_fx = eps * phi_f * Avx, sf_fy = eps * phi_f * Avy;
            double visc = eps * phi_f / c->p.N_R;
            double svis_x = visc * (2.0 * (c->bvx[k + 1] - c->bvx[k - 1]) / (2.0 * c->dxi) +
                                    (c->bvxy[k + nx] - c->bvxy[k - nx]) / (2.0 * c->deta));
            double svis_y = visc * (2.0 * (c->bvy[k + nx] - c->bvy[k - nx]) / (2.0 * c->deta) +
                                    (c->bvxy[k + 1] - c->bvxy[k - 1]) / (2.0 * c->dxi));
            c->rhs[0][k] = div[0];
            c->rhs[1][k] = div[1];
            c->rhs[2][k] = div[2] + (sn_sx + sf_sx + sv_sx);
            c->rhs[3][k] = div[3] + (sn_sy + sf_sy + sv_sy);
            c->rhs[4][k] = div[4] + (sn_fx + sd_fx + sf_fx + sv_fx + svis_x);
            c->rhs[5][k] = div[5] + (sn_fy + sd_fy + sf_fy + sv_fy + svis_y);
        }
    }
}

/* ---- solver.cpp:450-480 apply_coulomb_cap ----------------------------------------------- */
static void coulomb_cap(orc_ctx* c, double** s, double dt) {
    if (c->adv_only || c->tan_d == 0.0) return;
    const int nx = c->nx, ny = c->ny;
#pragma omp parallel for schedule(static)
    for (int j = KG; j < ny - KG; ++j) {
        for (int i = KG; i < nx - KG; ++i) {
            size_t k = AT(c, i, j);
            double qx = s[2][k], qy = s[3][k];
            if (qx == 0.0 && qy == 0.0) continue;
            double jb = c->geo[JB_][k];
            double hs = s[0][k] / jb;
            if (hs < c->p.h_dry) continue;
            double vsx = desing(qx, jb, hs, c->p.eps_h);
            double vsy = desing(qy, jb, hs, c->p.eps_h);
            double kappa_s = curvature(c, k, vsx, vsy);
            double p_b_s = smax(0.0, hs * (c->geo[NZ_][k] * (1.0 - c->p.alpha_rho) - c->eps_chi * kappa_s));
            double rate = jb * p_b_s * c->tan_d;
            double qnorm = sqrt(qx * qx + qy * qy);
            double factor = smax(0.0, 1.0 - dt * rate / qnorm);
            s[2][k] = qx * factor;
            s[3][k] = qy * factor;
        }
    }
}

/* ---- solver.cpp:482-494 check_finite ----------------------------------------------------- */
static int check_finite(orc_ctx* c, double** s) {
    static const char* names[6] = {"ws", "wf", "qsx", "qsy", "qfx", "qfy"};
    for (int q = 0; q < 6; ++q)
        for (int j = KG; j < c->ny - KG; ++j)
            for (int i = KG; i < c->nx - KG; ++i)
                if (!isfinite(s[q][AT(c, i, j)]))
                    return fail(c, 4, "non-finite value in field '%s' at cell (%d, %d) during advance_step", names[q],
                                i - KG, j - KG + c->row0);
    return 0;
}

/* ---- the two Heun stages of solver.cpp:496-545 on the A/B buffers ------------------------ */
static int stage(orc_ctx* c, int corrector, double dt) {
    const int nx = c->nx, ny = c->ny;
    if (!corrector) {
        /* u* = u0 + dt R(u0); cap; regularize   (:512-522) */
        residual(c, c->A, dt / 2.0);
        for (int q = 0; q < 6; ++q)
            for (int j = KG; j < ny - KG; ++j)
                for (int i = KG; i < nx - KG; ++i) {
                    size_t k = AT(c, i, j);
                    c->B[q][k] = c->A[q][k] + dt * c->rhs[q][k];
                }
        coulomb_cap(c, c->B, dt);
        return regularize(c, c->B);
    }
    /* u** = u* + dt R(u*); cap; u = (u0 + u**)/2; regularize; check_finite   (:526-544) */
    residual(c, c->B, dt / 2.0);
    for (int q = 0; q < 6; ++q)
        for (int j = KG; j < ny - KG; ++j)
            for (int i = KG; i < nx - KG; ++i) {
                size_t k = AT(c, i, j);
                c->B[q][k] += dt * c->rhs[q][k];
            }
    coulomb_cap(c, c->B, dt);
    for (int q = 0; q < 6; ++q)
        for (int j = KG; j < ny - KG; ++j)
            for (int i = KG; i < nx - KG; ++i) {
                size_t k = AT(c, i, j);
                c->A[q][k] = 0.5 * (c->A[q][k] + c->B[q][k]);
            }
    int rc = regularize(c, c->A);
    if (rc) return rc;
    return check_finite(c, c->A);
}

int orc_apply_boundaries(orc_ctx* c, double t) {
    c->ghosts_in_B = 0;
    apply_bc(c, c->A, t);
    return 0;
}

/* solver.cpp:547-580 (lambda of the interior, exact max) */
static double lambda_local(orc_ctx* c) {
    const double eps_h = c->p.eps_h, h_dry = c->p.h_dry, eps = c->eps;
    double lam_max = 0.0; /* the reference's lambda_ ghosts are 0.0 (lambda_.fill(0)) */
    for (int j = KG; j < c->ny - KG; ++j) {
        for (int i = KG; i < c->nx - KG; ++i) {
            size_t k = AT(c, i, j);
            double jb = c->geo[JB_][k];
            double hs = c->A[0][k] / jb;
            double hf = c->A[1][k] / jb;
            double h = hs + hf;
            double vsx = desing(c->A[2][k], jb, hs, eps_h);
            double vsy = desing(c->A[3][k], jb, hs, eps_h);
            double vfx = desing(c->A[4][k], jb, hf, eps_h);
            double vfy = desing(c->A[5][k], jb, hf, eps_h);
            double lx, ly;
            if (h < h_dry) {
                lx = ly = 0.0;
            } else {
                double cel = sqrt(eps * c->geo[NZ_][k] * h);
                lx = smax(fabs(vsx), fabs(vfx)) + cel;
                ly = smax(fabs(vsy), fabs(vfy)) + cel;
            }
            lam_max = smax(lam_max, smax(lx, ly));
        }
    }
    return lam_max;
}

static double dt_from(const orc_ctx* c, double lam_max, double t, double t_next) {
    double remaining = t_next - t;
    if (lam_max <= 0.0) return remaining;
    double dt = c->p.cfl * smin(c->dxi, c->deta) / lam_max;
    return smin(dt, remaining);
}

int orc_compute_dt(orc_ctx* c, double t, double t_next, double* dt) {
    *dt = dt_from(c, lambda_local(c), t, t_next);
    return 0;
}

int orc_advance_step(orc_ctx* c, double dt, double t) {
    sync_ghosts(c);
    int rc = stage(c, 0, dt);
    if (rc) return rc;
    apply_bc(c, c->B, t + dt);
    rc = stage(c, 1, dt);
    c->ghosts_in_B = 1;
    return rc;
}

int orc_regularize(orc_ctx* c) {
    sync_ghosts(c);
    return regularize(c, c->A);
}

void orc_set_advection_only(orc_ctx* c, int on) { c->adv_only = on != 0; }
void orc_get_audit(orc_ctx* c, double* a) { memcpy(a, c->audit, sizeof(c->audit)); }
void orc_reset_audit(orc_ctx* c) { memset(c->audit, 0, sizeof(c->audit)); }

/* solver.cpp:582-588 (KahanSum, field.hpp:46-59) */
static double interior_mass(orc_ctx* c, const double* w) {
    double sum = 0.0, comp = 0.0;
    for (int j = KG; j < c->ny - KG; ++j)
        for (int i = KG; i < c->nx - KG; ++i) {
            double y = w[AT(c, i, j)] - comp;
            double t = sum + y;
            comp = (t - sum) - y;
            sum = t;
        }
    return sum * c->dxi * c->deta;
}

void orc_interior_mass(orc_ctx* c, double* ms, double* mf) {
    *ms = interior_mass(c, c->A[0]);
    *mf = interior_mass(c, c->A[1]);
}

/* the body of Simulator::run's loop, solver.cpp:637-649 */
int orc_steps(orc_ctx* c, double t_next, double t_end, long max_steps, double* t, long* steps, int* hit,
              double* dts) {
    *steps = 0;
    *hit = 0;
    while (*t < t_end && *steps < max_steps) {
        orc_apply_boundaries(c, *t);
        double dt;
        orc_compute_dt(c, *t, t_next, &dt);
        int exact_hit = dt == t_next - *t;
        int rc = orc_advance_step(c, dt, *t);
        if (rc) return rc;
        if (dts) dts[*steps] = dt;
        ++*steps;
        *t = exact_hit ? t_next : *t + dt;
        *hit = exact_hit;
        if (exact_hit) break;
    }
    return 0;
}

/* Simulator::snapshot, solver.cpp:590-617 */
void orc_snapshot(orc_ctx* c, double t, double* out) {
    (void)t;
    sync_ghosts(c);
    size_t m = (size_t)c->ncols * c->nrows;
    memset(out, 0, sizeof(double) * 6 * m);
    for (int j = 0; j < c->nrows; ++j) {
        for (int i = 0; i < c->ncols; ++i) {
            size_t k = AT(c, i + KG, j + KG), o = (size_t)j * c->ncols + i;
            double jb = c->geo[JB_][k];
            double hs = c->A[0][k] / jb;
            double hf = c->A[1][k] / jb;
            double h = hs + hf;
            out[o] = h * c->p.H;
            if (h < c->p.h_dry) continue;
            out[m + o] = hs / h;
            out[2 * m + o] = desing(c->A[2][k], jb, hs, c->p.eps_h) * c->v_unit;
            out[3 * m + o] = desing(c->A[3][k], jb, hs, c->p.eps_h) * c->v_unit;
            out[4 * m + o] = desing(c->A[4][k], jb, hf, c->p.eps_h) * c->v_unit;
            out[5 * m + o] = desing(c->A[5][k], jb, hf, c->p.eps_h) * c->v_unit;
        }
    }
}

/* Simulator::run, solver.cpp:619-659 (wall time not measured here) */
int orc_run(orc_ctx* c, double* report, double* snap_times, int max_snaps, int* n_snaps) {
    memset(c->audit, 0, sizeof(c->audit));
    int rc = orc_regularize(c);
    if (rc) return rc;
    orc_interior_mass(c, &c->audit[0], &c->audit[5]);
    double t_end = c->p.t_end / c->t_unit;
    double dt_out = c->p.dt_out / c->t_unit;
    double t = 0.0;
    long steps = 0;
    *n_snaps = 0;
    if (*n_snaps < max_snaps) snap_times[*n_snaps] = t * c->t_unit;
    ++*n_snaps;
    double next_out = dt_out;
    while (t < t_end) {
        double t_next = smin(next_out, t_end);
        long n;
        int hit;
        rc = orc_steps(c, t_next, t_end, 1, &t, &n, &hit, NULL);
        if (rc) return rc;
        steps += n;
        if (hit) {
            if (*n_snaps < max_snaps) snap_times[*n_snaps] = t * c->t_unit;
            ++*n_snaps;
            if (t_next == next_out) next_out += dt_out;
        }
    }
    orc_interior_mass(c, &c->audit[1], &c->audit[6]);
    report[0] = (double)steps;
    report[1] = 0.0;
    memcpy(report + 2, c->audit, sizeof(c->audit));
    return 0;
}

/* Backend::reduce_max, parallel.cpp:109-132 (serial shape; the max is exact anyway) */
int orc_reduce_max(int lanes, const double* v, long n, double* out) {
    (void)lanes;
    if (n <= 0) return 4;
    double m = v[0];
    for (long i = 1; i < n; ++i) m = smax(m, v[i]);
    *out = m;
    return 0;
}

/* ---- split step on a slab --------------------------------------------------------------- */
long orc_halo_doubles(orc_ctx* c) { return 2L * 6L * c->nx; }

void orc_halo_pack(orc_ctx* c, int buf, int side, double* dst) {
    if (buf == 0) sync_ghosts(c);
    double** s = buf ? c->B : c->A;
    int row = side == 0 ? KG : c->ny - KG - 2;
    for (int q = 0; q < 6; ++q) memcpy(dst + 2L * q * c->nx, s[q] + (size_t)row * c->nx, sizeof(double) * 2 * c->nx);
}

void orc_halo_unpack(orc_ctx* c, int buf, int side, const double* src) {
    double** s = buf ? c->B : c->A;
    int row = side == 0 ? KG - 2 : c->ny - KG;
    for (int q = 0; q < 6; ++q) memcpy(s[q] + (size_t)row * c->nx, src + 2L * q * c->nx, sizeof(double) * 2 * c->nx);
}

void orc_step_begin(orc_ctx* c, double t, double t_next, double t_end) {
    c->t = t;
    c->t_next = t_next;
    c->t_end = t_end;
}

void orc_bc(orc_ctx* c, int buf) {
    if (buf == 0) {
        c->ghosts_in_B = 0;
        apply_bc(c, c->A, c->t);
    } else {
        apply_bc(c, c->B, c->t + c->dt);
    }
}

double orc_lambda_local(orc_ctx* c) { return lambda_local(c); }

void orc_dt_from(orc_ctx* c, double lam) {
    c->dt = dt_from(c, lam, c->t, c->t_next);
    c->hit = c->dt == c->t_next - c->t;
}

int orc_stage(orc_ctx* c, int corrector) {
    int rc = stage(c, corrector, c->dt);
    if (corrector) c->ghosts_in_B = 1;
    return rc;
}

int orc_step_end(orc_ctx* c, double* t, int* hit, double* dt) {
    *dt = c->dt;
    *hit = c->hit;
    c->t = c->hit ? c->t_next : c->t + c->dt;
    *t = c->t;
    return 0;
}
