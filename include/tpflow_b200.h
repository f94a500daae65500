/*
 * tpflow_b200 — C ABI of the B200-native MoSES_2PDF time-stepping core.
 *
 * This is the drop-in boundary for the reference's host/device split: the
 * step API of `tpflow::Simulator` (/root/reference/proj/include/tpflow/solver.hpp:28-62),
 * which the reference's own run loop (solver.cpp:619-659) and tests drive.
 * Plain C types only (no torch, no C++); every call returns an int status using the
 * reference's error taxonomy (errors.hpp:8-21): 0 ok, 2 ConfigError, 3 IoError,
 * 4 NumericsError, plus 1 internal / 5 CUDA.  tp_last_error() returns the message,
 * which for 2/3/4 is the reference's message text.
 *
 * All state is device-resident (FP64 SoA, padded grid of nx = ncols+6 by
 * ny = nrows+6 cells, j-major, field order ws,wf,qsx,qsy,qfx,qfy — state.hpp:29).
 * Host arrays are borrowed for the duration of a call and copied.  Scaled times
 * everywhere except hydrograph samples (seconds), as in the reference.
 * One host thread per context; calls are not re-entrant.
 */
#ifndef TPFLOW_B200_H
#define TPFLOW_B200_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tp_ctx tp_ctx;

enum {
    TP_OK = 0,
    TP_ERR_INTERNAL = 1,
    TP_ERR_CONFIG = 2,   /* tpflow::ConfigError   */
    TP_ERR_IO = 3,       /* tpflow::IoError       */
    TP_ERR_NUMERICS = 4, /* tpflow::NumericsError */
    TP_ERR_CUDA = 5
};

/* SimConfig numerics + ModelParams + ScalingConfig (config.hpp:12-30, params.hpp:12-51). */
typedef struct tp_params {
    double delta_b, C_d, N_R, theta_b, phi_s0, alpha_rho, chi;
    double L, H, g;
    double t_end, dt_out, cfl, h_dry, eps_h;
    int mode;   /* 0 = FiniteRelease (Mode-I), 1 = InflowHydrograph (Mode-II) */
    int device; /* CUDA device ordinal */
} tp_params;

/* ElevationGrid (terrain.hpp:15-29): interior elevations in metres, ncols*nrows,
 * j-major with row 0 the SOUTH row. */
typedef struct tp_dem {
    int ncols, nrows;
    double xll, yll, cellsize;
    const double* z;
} tp_dem;

/* Simulator::Simulator (solver.cpp:13-33): validates the config, builds the
 * terrain geometry (terrain.cpp:113-215, bit-identical), allocates device state. */
int tp_create(const tp_params* p, const tp_dem* dem, tp_ctx** out);
/* Same, for the row block [row0, row1) of the interior (multi-GPU slab). */
int tp_create_slab(const tp_params* p, const tp_dem* dem, int row0, int row1, tp_ctx** out);
void tp_destroy(tp_ctx* c);
const char* tp_last_error(const tp_ctx* c);

/* Host-only utility (no device needed): the padded terrain geometry of a DEM,
 * extend_grid + compute_geometry (terrain.cpp:113-215), 14*(ncols+6)*(nrows+6) doubles. */
int tp_geometry(const tp_dem* dem, double L, double* out14);

/* padded dims of this context and the scaled spacings */
int tp_dims(const tp_ctx* c, int* nx, int* ny, double* dxi, double* deta);
/* options: "fastdiv" (0/1, default 1), "skip_dry" (0/1, default 1), "graph_steps" (steps per
 * CUDA graph, default 16), "wide_tiles" (replay the graphs with one 512-thread stage CTA per SM
 * while the last tile lists held <= this many tiles; default -1 = the SM count, 0 = never) */
int tp_set_option(tp_ctx* c, const char* key, long value);

/* Simulator::set_initial_thickness / set_initial_velocity / set_hydrograph
 * (solver.cpp:35-81).  Interior grids ncols*nrows (whole DEM even for a slab). */
int tp_set_initial_thickness(tp_ctx* c, const double* h_m);
int tp_set_initial_velocity(tp_ctx* c, const double* vx, const double* vy);
int tp_set_hydrograph(tp_ctx* c, int n_cells, const int* ci, const int* cj, const char* side,
                      int n_samples, const double* t, const double* h, const double* phi_s,
                      const double* speed);

/* whole padded state, 6 * nx * ny doubles (dense, no pitch) */
int tp_get_state(tp_ctx* c, double* out);
int tp_set_state(tp_ctx* c, const double* in);
/* the 14 geometry fields (terrain.hpp:59-63 order), 14 * nx * ny doubles */
int tp_get_geometry(tp_ctx* c, double* out);

/* The step pieces "exposed for tests and diagnostics" (solver.hpp:41-47). */
int tp_apply_boundaries(tp_ctx* c, double t_scaled);
int tp_compute_dt(tp_ctx* c, double t_scaled, double t_next_scaled, double* dt);
int tp_advance_step(tp_ctx* c, double dt_scaled, double t_scaled);
int tp_regularize(tp_ctx* c);
int tp_set_advection_only(tp_ctx* c, int on);

/* Device-resident run loop: from *t, repeat the body of Simulator::run's loop
 * (solver.cpp:637-649) — apply_boundaries(t); dt = compute_dt(t, t_next);
 * advance_step(dt, t); t = exact_hit ? t_next : t + dt — while t < t_end, until
 * the exact hit of t_next or max_steps steps; *hit = exact_hit of the last step.
 * dts (optional, max_steps long)
 * receives every accepted dt.  The host synchronises once per CUDA graph. */
int tp_steps(tp_ctx* c, double t_next, double t_end, long max_steps, double* t, long* steps,
             int* hit, double* dts);
/* tp_steps replaying a one-step graph that records CUDA events (external event nodes on the
 * context stream) right around the predictor and corrector kernels; *pred_ms / *corr_ms =
 * the summed device time of those kernels over the steps taken (measurement hook) */
int tp_steps_timed(tp_ctx* c, double t_next, double t_end, long max_steps, double* t, long* steps, int* hit,
                   float* pred_ms, float* corr_ms);
/* tiles the predictor / corrector launches processed, summed over the steps of the last
 * tp_steps_timed call (the roofline's processed bytes, bench.py) */
int tp_timed_tiles(tp_ctx* c, long long* pred_tiles, long long* corr_tiles);

/* audit[0..4] = solid {initial, final, injected, outflow, clipped}, [5..9] fluid
 * (MassAudit, config.hpp:60-75); initial/final are host-owned (see tp_set_audit). */
int tp_get_audit(tp_ctx* c, double* audit10);
int tp_set_audit(tp_ctx* c, const double* audit10);
/* Simulator::interior_mass (solver.cpp:582-588), Kahan-summed in the reference order */
int tp_interior_mass(tp_ctx* c, double* mass_solid, double* mass_fluid);
/* Simulator::snapshot (solver.cpp:590-617): h, phi_s, vXs, vYs, vXf, vYf on the
 * interior (6 * ncols * nrows_local), physical units */
/* interior masses reduced on the device (deterministic, compensated; within ~1 ulp of the
 * exact sum, not bit-identical to the reference's serial KahanSum, which tp_interior_mass
 * keeps): the fast conservation check for large grids */
int tp_interior_mass_device(tp_ctx* c, double* ms, double* mf);
int tp_snapshot(tp_ctx* c, double* out6);

/* ---- multi-GPU slab plumbing (row-block decomposition) ---------
 * buf: 0 = the current state u^n, 1 = the predictor state u*.
 * side: 0 = south neighbour, 1 = north neighbour.  Halo = 2 rows x 6 fields x nx,
 * tp_halo_bytes() bytes, packed/unpacked on the context's stream to/from a
 * caller-owned DEVICE buffer (e.g. a torch tensor used by NCCL send/recv). */
long tp_halo_bytes(const tp_ctx* c);
int tp_halo_pack(tp_ctx* c, int buf, int side, void* dst_device);
int tp_halo_unpack(tp_ctx* c, int buf, int side, const void* src_device);
/* one step split at its exchange points; t/dt live on the device */
int tp_step_begin(tp_ctx* c, double t, double t_next, double t_end);      /* sets scalars */
int tp_bc(tp_ctx* c, int buf);                         /* buf 0 at t, buf 1 at t + dt */
int tp_lambda_local(tp_ctx* c, void* dst_device);      /* local lambda_max (1 double) -> dst */
int tp_dt_from(tp_ctx* c, const void* lam_device);     /* dt from an all-reduced lambda */
int tp_stage(tp_ctx* c, int corrector);                /* predictor u^n -> u*, corrector */
/* tp_stage with CUDA events recorded on the context stream right around the stage
 * kernel (after its tile-list kernel); *ms = that kernel's device time */
int tp_stage_timed(tp_ctx* c, int corrector, float* ms);
int tp_step_end(tp_ctx* c, double* t, int* hit, double* dt); /* fold audit, advance t, sync */

/* interop: the CUDA stream the context launches on (default: its own stream) */
int tp_set_stream(tp_ctx* c, void* cuda_stream);
int tp_synchronize(tp_ctx* c);
/* device pointer of a state buffer (buf 0/1), row pitch and field stride in doubles */
int tp_device_state(tp_ctx* c, int buf, void** ptr, long* pitch, long* field_stride);
/* diagnostic: checks the FASTDIV division identity on n random operand pairs on
 * `device`; *mismatches = number of quotients differing from IEEE a/b (expect 0) */
int tp_selftest_division(int device, long n, unsigned long long seed, unsigned long long* mismatches);
/* diagnostic: out[k] = the device minmod limited_slope(a[k], b[k]) (solver.hpp:17-21)
 * for n host operand pairs, so tests can compare it with the reference bit for bit */
int tp_selftest_minmod(int device, long n, const double* a, const double* b, double* out);
/* tiles listed by the last predictor / corrector launch (dry tiles whose stage is a
 * bitwise no-op are skipped) and the number of tiles of the grid */
int tp_active_tiles(tp_ctx* c, int* pred, int* corr, int* total);
/* how many tiles of the last corrector list were "safe" (every value their box reads is
 * +-0 or of magnitude in [2^-200, 2^200): FASTDIV window tests compiled out) */
int tp_safe_tiles(tp_ctx* c, int* corr);
/* peer-joined slabs: how many tiles listed only because their box reads halo rows were
 * skipped because the neighbour's pushed rows were +0.0 there (cumulative) */
int tp_cond_skipped_tiles(tp_ctx* c, unsigned long long* n);
/* development probe: per-phase warp cycles of the stage kernels [2][19] (pred, corr;
 * slot 16 counts warps, 17/18 sum warp lifetimes in cycles / ns); all zero unless the library was built with `make timing` */
int tp_debug_phase_cycles(unsigned long long* out, int reset);
/* ---- device-resident row-slab exchange over peer memory (tp_peer.cu) ----------------
 * Slabs (tp_create_slab) connected here run tp_steps with the halo rows stored straight
 * into the neighbours' buffers and the lambda all-reduce done in device memory: no host
 * round trip per step (replaces the host-driven tp_halo_pack / tp_lambda_local path).
 * One rank per GPU: every rank calls tp_peer_export, the blobs are all-gathered (any
 * transport), every rank calls tp_peer_connect with all nranks blobs in rank order, and
 * every rank then calls tp_steps with identical arguments.  Contexts of one process:
 * tp_peer_connect_local, then tp_steps_group. */
#define TP_PEER_BLOB_BYTES 256
int tp_peer_export(tp_ctx* c, void* blob /* TP_PEER_BLOB_BYTES */);
int tp_peer_connect(tp_ctx* c, int rank, int nranks, const void* blobs /* nranks * TP_PEER_BLOB_BYTES */);
int tp_peer_connect_local(tp_ctx* c, int rank, int nranks, tp_ctx* const* all);
int tp_steps_group(tp_ctx* const* cs, int n, double t_next, double t_end, long max_steps, double* t,
                   long* steps, int* hit);
/* number of kernels launched by the last tp_steps call (graph replays included) */
long tp_kernel_launches(const tp_ctx* c);

#ifdef __cplusplus
}
#endif
#endif /* TPFLOW_B200_H */
