/* TEST INFRASTRUCTURE ONLY — CPU checker, never part of the product path.
 *
 * Plain-C restatement of the reference time-stepping core
 * (/root/reference/proj/src/solver.cpp:83-580, include/tpflow/physics.hpp:33-189,
 * src/terrain.cpp:113-215, include/tpflow/hydrograph.hpp:31-45), expression by
 * expression, built with -ffp-contract=off so it is bit-identical to the
 * reference build (checked by tests/test_oracle_cpu.py against oracle/_ref).
 *
 * Entry points mirror oracle/ref_harness.cpp (prefix orc_ instead of ref_), plus
 * row-slab contexts and the split-step API used by the multi-rank tests
 * (same shape as the tp_* slab API of include/tpflow_b200.h).
 */
#ifndef TPFLOW_ORACLE_H
#define TPFLOW_ORACLE_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_params {
    double delta_b, C_d, N_R, theta_b, phi_s0, alpha_rho, chi;
    double L, H, g;
    double t_end, dt_out, cfl, h_dry, eps_h;
    int mode;  /* 0 = FiniteRelease, 1 = InflowHydrograph */
    int lanes; /* OpenMP threads for the per-cell loops (0/1 = serial) */
} orc_params;

typedef struct orc_ctx orc_ctx;

int orc_create(const orc_params* p, int ncols, int nrows, double cellsize, double xll, double yll,
               const double* z, orc_ctx** out);
int orc_create_slab(const orc_params* p, int ncols, int nrows, double cellsize, double xll, double yll,
                    const double* z, int row0, int row1, orc_ctx** out);
void orc_destroy(orc_ctx* c);
const char* orc_last_error(orc_ctx* c);
void orc_dims(orc_ctx* c, int* nx, int* ny, double* dxi, double* deta);
int orc_set_initial_thickness(orc_ctx* c, const double* h);
int orc_set_initial_velocity(orc_ctx* c, const double* vx, const double* vy);
int orc_set_hydrograph(orc_ctx* c, int n_cells, const int* ci, const int* cj, const char* side,
                       int n_samples, const double* t, const double* h, const double* phi,
                       const double* speed);
void orc_get_state(orc_ctx* c, double* out);
void orc_set_state(orc_ctx* c, const double* in);
void orc_get_geometry(orc_ctx* c, double* out);
int orc_apply_boundaries(orc_ctx* c, double t);
int orc_compute_dt(orc_ctx* c, double t, double t_next, double* dt);
int orc_advance_step(orc_ctx* c, double dt, double t);
int orc_regularize(orc_ctx* c);
void orc_set_advection_only(orc_ctx* c, int on);
void orc_get_audit(orc_ctx* c, double* a);
void orc_reset_audit(orc_ctx* c);
void orc_interior_mass(orc_ctx* c, double* ms, double* mf);
int orc_steps(orc_ctx* c, double t_next, double t_end, long max_steps, double* t, long* steps,
              int* hit, double* dts);
int orc_run(orc_ctx* c, double* report, double* snap_times, int max_snaps, int* n_snaps);
void orc_snapshot(orc_ctx* c, double t, double* out);
int orc_reduce_max(int lanes, const double* v, long n, double* out);

/* split step on a slab (buf 0 = u^n, buf 1 = u*; side 0 = south, 1 = north) */
long orc_halo_doubles(orc_ctx* c);
void orc_halo_pack(orc_ctx* c, int buf, int side, double* dst);
void orc_halo_unpack(orc_ctx* c, int buf, int side, const double* src);
void orc_step_begin(orc_ctx* c, double t, double t_next, double t_end);
void orc_bc(orc_ctx* c, int buf);
double orc_lambda_local(orc_ctx* c);
void orc_dt_from(orc_ctx* c, double lam);
int orc_stage(orc_ctx* c, int corrector);
int orc_step_end(orc_ctx* c, double* t, int* hit, double* dt);

#ifdef __cplusplus
}
#endif
#endif
