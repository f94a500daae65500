// TEST INFRASTRUCTURE ONLY — never linked into or called by the product path.
//
// extern "C" shim around the UNMODIFIED reference `tpflow::Simulator`
// (/root/reference/proj/src/*.cpp, compiled in place by oracle/Makefile into
// oracle/_ref/libtpflow_ref.so).  It exists so the Python tests, the bench's
// `--impl reference` arm and the C restatement's self-check can drive the
// reference's own step API (solver.hpp:41-47) on arrays we generate.
//
// Every entry point maps 1:1 onto a reference call:
//   ref_create            -> Simulator::Simulator        solver.cpp:13-33
//   ref_set_initial_*     -> set_initial_thickness/velocity solver.cpp:35-76
//   ref_set_hydrograph    -> set_hydrograph             solver.cpp:78-81
//   ref_apply_boundaries  -> apply_boundaries           solver.cpp:83-137
//   ref_compute_dt        -> compute_dt                 solver.cpp:547-580
//   ref_advance_step      -> advance_step               solver.cpp:496-545
//   ref_regularize        -> regularize                 solver.cpp:139-166
//   ref_steps             -> the body of Simulator::run's while loop, solver.cpp:637-649
//   ref_run               -> Simulator::run             solver.cpp:619-659
// Exceptions are mapped to the reference exit codes (errors.hpp:8-21).
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "tpflow/config.hpp"
#include "tpflow/errors.hpp"
#include "tpflow/hydrograph.hpp"
#include "tpflow/parallel.hpp"
#include "tpflow/solver.hpp"
#include "tpflow/terrain.hpp"

using namespace tpflow;

extern "C" {

// Mirrors the scalar part of SimConfig (config.hpp:12-30) + ModelParams + ScalingConfig.
struct ref_params {
    double delta_b, C_d, N_R, theta_b, phi_s0, alpha_rho, chi;
    double L, H, g;
    double t_end, dt_out, cfl, h_dry, eps_h;
    int mode;  // 0 = FiniteRelease, 1 = InflowHydrograph
    int lanes; // 0 = BackendConfig::serial(), >0 = BackendConfig::parallel(lanes)
};

struct ref_ctx {
    std::unique_ptr<Backend> backend;
    std::unique_ptr<Simulator> sim;
    ElevationGrid dem;
    std::string err;
};

static int fail(ref_ctx* c, int code, const char* what) {
    if (c) c->err = what;
    return code;
}

#define REF_TRY(ctx, ...)                                                      \
    try {                                                                      \
        __VA_ARGS__;                                                               \
        return 0;                                                              \
    } catch (const ConfigError& e) { return fail(ctx, 2, e.what()); }          \
    catch (const IoError& e) { return fail(ctx, 3, e.what()); }                \
    catch (const NumericsError& e) { return fail(ctx, 4, e.what()); }          \
    catch (const std::exception& e) { return fail(ctx, 1, e.what()); }

static SimConfig to_config(const ref_params* p) {
    SimConfig cfg;
    cfg.params.delta_b = p->delta_b;
    cfg.params.C_d = p->C_d;
    cfg.params.N_R = p->N_R;
    cfg.params.theta_b = p->theta_b;
    cfg.params.phi_s0 = p->phi_s0;
    cfg.params.alpha_rho = p->alpha_rho;
    cfg.params.chi = p->chi;
    cfg.scaling.L = p->L;
    cfg.scaling.H = p->H;
    cfg.scaling.g = p->g;
    cfg.mode = p->mode ? SimConfig::Mode::InflowHydrograph : SimConfig::Mode::FiniteRelease;
    cfg.t_end = p->t_end;
    cfg.dt_out = p->dt_out;
    cfg.cfl = p->cfl;
    cfg.h_dry = p->h_dry;
    cfg.eps_h = p->eps_h;
    cfg.dem_path = "<memory>";
    cfg.init_path = "<memory>";
    cfg.hydrograph_path = "<memory>";
    return cfg;
}

// z: ncols*nrows elevations, j-major, j=0 is the SOUTH row (terrain.hpp:12-14).
int ref_create(const ref_params* p, int ncols, int nrows, double cellsize, double xll, double yll,
               const double* z, ref_ctx** out) {
    auto* c = new ref_ctx();
    *out = c;
    REF_TRY(c, {
        c->dem.ncols = ncols;
        c->dem.nrows = nrows;
        c->dem.cellsize = cellsize;
        c->dem.xll = xll;
        c->dem.yll = yll;
        c->dem.z = Field(ncols, nrows);
        std::memcpy(c->dem.z.data(), z, sizeof(double) * ncols * nrows);
        BackendConfig bc = p->lanes > 0 ? BackendConfig::parallel(p->lanes) : BackendConfig::serial();
        c->backend = std::make_unique<Backend>(bc);
        c->sim = std::make_unique<Simulator>(to_config(p), c->dem, *c->backend);
    })
}

void ref_destroy(ref_ctx* c) { delete c; }

const char* ref_last_error(ref_ctx* c) { return c->err.c_str(); }

void ref_dims(ref_ctx* c, int* nx, int* ny, double* dxi, double* deta) {
    const auto& g = c->sim->geometry();
    *nx = g.nx; *ny = g.ny; *dxi = g.dxi; *deta = g.deta;
}

int ref_set_initial_thickness(ref_ctx* c, const double* h) {
    REF_TRY(c, {
        Field f(c->dem.ncols, c->dem.nrows);
        std::memcpy(f.data(), h, sizeof(double) * f.size());
        c->sim->set_initial_thickness(f);
    })
}

int ref_set_initial_velocity(ref_ctx* c, const double* vx, const double* vy) {
    REF_TRY(c, {
        Field fx(c->dem.ncols, c->dem.nrows), fy(c->dem.ncols, c->dem.nrows);
        std::memcpy(fx.data(), vx, sizeof(double) * fx.size());
        std::memcpy(fy.data(), vy, sizeof(double) * fy.size());
        c->sim->set_initial_velocity(fx, fy);
    })
}

int ref_set_hydrograph(ref_ctx* c, int n_cells, const int* ci, const int* cj, const char* side,
                       int n_samples, const double* t, const double* h, const double* phi,
                       const double* speed) {
    REF_TRY(c, {
        Hydrograph hg;
        for (int k = 0; k < n_cells; ++k) hg.cells.push_back({ci[k], cj[k], side[k]});
        for (int k = 0; k < n_samples; ++k) hg.samples.push_back({t[k], h[k], phi[k], speed[k]});
        c->sim->set_hydrograph(std::move(hg));
    })
}

// 6 padded fields in MixtureState order (state.hpp:29), each nx*ny, j-major.
void ref_get_state(ref_ctx* c, double* out) {
    auto f = c->sim->state().fields();
    std::size_t n = f[0]->size();
    for (int k = 0; k < 6; ++k) std::memcpy(out + k * n, f[k]->data(), sizeof(double) * n);
}

void ref_set_state(ref_ctx* c, const double* in) {
    auto f = c->sim->state().fields();
    std::size_t n = f[0]->size();
    for (int k = 0; k < 6; ++k) std::memcpy(f[k]->data(), in + k * n, sizeof(double) * n);
}

// 14 padded geometry fields in TerrainGeometry declaration order (terrain.hpp:59-63).
void ref_get_geometry(ref_ctx* c, double* out) {
    const auto& g = c->sim->geometry();
    const Field* f[14] = {&g.nX, &g.nY, &g.nZ, &g.jb, &g.a11, &g.a12, &g.a21, &g.a22,
                          &g.dnX_dxi, &g.dnY_dxi, &g.dnZ_dxi, &g.dnX_deta, &g.dnY_deta, &g.dnZ_deta};
    std::size_t n = g.jb.size();
    for (int k = 0; k < 14; ++k) std::memcpy(out + k * n, f[k]->data(), sizeof(double) * n);
}

int ref_apply_boundaries(ref_ctx* c, double t) {
    REF_TRY(c, c->sim->apply_boundaries(c->sim->state(), t))
}

int ref_compute_dt(ref_ctx* c, double t, double t_next, double* dt) {
    REF_TRY(c, *dt = c->sim->compute_dt(t, t_next))
}

int ref_advance_step(ref_ctx* c, double dt, double t) {
    REF_TRY(c, c->sim->advance_step(dt, t))
}

int ref_regularize(ref_ctx* c) {
    REF_TRY(c, c->sim->regularize(c->sim->state()))
}

void ref_set_advection_only(ref_ctx* c, int on) { c->sim->set_advection_only(on != 0); }

// audit[0..4] = solid {initial, final, injected, outflow, clipped}, [5..9] = fluid.
void ref_get_audit(ref_ctx* c, double* a) {
    const MassAudit* m[2] = {&c->sim->solid_audit(), &c->sim->fluid_audit()};
    for (int p = 0; p < 2; ++p) {
        a[5 * p + 0] = m[p]->initial;
        a[5 * p + 1] = m[p]->final_mass;
        a[5 * p + 2] = m[p]->injected;
        a[5 * p + 3] = m[p]->outflow;
        a[5 * p + 4] = m[p]->clipped;
    }
}

void ref_reset_audit(ref_ctx* c) {
    c->sim->solid_audit() = MassAudit{};
    c->sim->fluid_audit() = MassAudit{};
}

void ref_interior_mass(ref_ctx* c, double* ms, double* mf) {
    *ms = c->sim->interior_mass_solid();
    *mf = c->sim->interior_mass_fluid();
}

// The body of Simulator::run's loop (solver.cpp:637-649), without snapshots:
// from *t, step while t < t_end until the exact hit of t_next (or max_steps).
// Records every accepted dt; *hit = exact_hit of the last step.
int ref_steps(ref_ctx* c, double t_next, double t_end, long max_steps, double* t, long* steps,
              int* hit, double* dts) {
    *steps = 0;
    *hit = 0;
    REF_TRY(c, {
        while (*t < t_end && *steps < max_steps) {
            c->sim->apply_boundaries(c->sim->state(), *t);
            double dt = c->sim->compute_dt(*t, t_next);
            bool exact_hit = dt == t_next - *t;
            c->sim->advance_step(dt, *t);
            if (dts) dts[*steps] = dt;
            ++*steps;
            *t = exact_hit ? t_next : *t + dt;
            *hit = exact_hit ? 1 : 0;
            if (exact_hit) break;
        }
    })
}

// Full Simulator::run (solver.cpp:619-659).  report = {steps, wall_seconds,
// 10 audit values as ref_get_audit}; snap_times receives each snapshot time
// (seconds) up to max_snaps.
int ref_run(ref_ctx* c, double* report, double* snap_times, int max_snaps, int* n_snaps) {
    *n_snaps = 0;
    REF_TRY(c, {
        RunReport r = c->sim->run([&](const SimSnapshot& s) {
            if (*n_snaps < max_snaps) snap_times[*n_snaps] = s.t;
            ++*n_snaps;
        });
        report[0] = static_cast<double>(r.steps);
        report[1] = r.wall_seconds;
        ref_get_audit(c, report + 2);
    })
}

// Simulator::snapshot (solver.cpp:590-617): 6 interior fields, each ncols*nrows.
void ref_snapshot(ref_ctx* c, double t, double* out) {
    SimSnapshot s = c->sim->snapshot(t, 0);
    const Field* f[6] = {&s.h_total, &s.phi_s, &s.vX_s, &s.vY_s, &s.vX_f, &s.vY_f};
    std::size_t n = s.h_total.size();
    for (int k = 0; k < 6; ++k) std::memcpy(out + k * n, f[k]->data(), sizeof(double) * n);
}

// Backend::reduce_max (parallel.cpp:109-132) on an arbitrary array.
int ref_reduce_max(int lanes, const double* v, long n, double* out) {
    try {
        Backend b(lanes > 0 ? BackendConfig::parallel(lanes) : BackendConfig::serial());
        *out = b.reduce_max(std::span<const double>(v, static_cast<std::size_t>(n)));
        return 0;
    } catch (const NumericsError&) { return 4; }
    catch (...) { return 1; }
}

}  // extern "C"
