// C ABI of the B200-native time-stepping core (include/tpflow_b200.h).
//
// A tp_ctx is the device-resident counterpart of one tpflow::Simulator
// (/root/reference/proj/include/tpflow/solver.hpp:26-98): it owns two FP64 SoA
// state buffers (A = u^n / u^{n+1}, B = u*), the 14 geometry fields, the device
// step scalars and the per-tile boundary tallies, and drives the kernels of
// tp_kernels.cu on one CUDA stream.  tp_steps runs Simulator::run's loop body
// (solver.cpp:637-649) entirely on the device, replayed from a CUDA graph; the
// host synchronises once per graph (graph_steps steps).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstddef>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/tpflow_b200.h"
#include "tp_host.hpp"
#include "tp_types.h"

namespace tpb {
size_t stage_smem_bytes();
cudaError_t launch_stage(const StageArgs& a, bool fastdiv, bool corr, bool peer, bool wide, cudaStream_t st);
cudaError_t launch_bc(const BcArgs& a, cudaStream_t st);
cudaError_t launch_ghost_copy(const GridDesc& g, const double* src, double* dst, cudaStream_t st);
cudaError_t launch_lambda(const GridDesc& g, const Phys& P, const double* s, const double* geo,
                          DevScalars* sc, bool fastdiv, cudaStream_t st);
cudaError_t launch_dt(const Phys& P, DevScalars* sc, int loop, cudaStream_t st);
cudaError_t launch_post(const PostArgs& a, cudaStream_t st);
cudaError_t launch_prepost(const PrePostArgs& a, cudaStream_t st);
cudaError_t launch_regularize(const GridDesc& g, const Phys& P, double* s, const double* geo,
                              DevScalars* sc, bool fastdiv, cudaStream_t st);
cudaError_t init_kernels();
cudaError_t launch_tiles(const TileArgs& a, cudaStream_t st);
cudaError_t build_geometry_device(const double* dem_h, int ncols, int nrows, double L, double cellsize, int row0,
                                  int ny, const GridDesc& g, double* geo, cudaStream_t st);
cudaError_t launch_init_thickness(const GridDesc& g, const double* geo, const double* h, int ncols, int nrows,
                                  double H, double phi, double* s, cudaStream_t st);
cudaError_t launch_init_velocity(const GridDesc& g, const double* geo, const double* vx, const double* vy,
                                 int ncols, int nrows, double vu, double* s, cudaStream_t st);
cudaError_t launch_geo_check(const GridDesc& g, const double* geo, int* ok, cudaStream_t st);
cudaError_t launch_peer_lambda(const PeerLink& L, DevScalars* sc, cudaStream_t st);
cudaError_t launch_peer_halo(const PeerLink& L, const GridDesc& g, const double* s, int buf, DevScalars* sc,
                             cudaStream_t st);
cudaError_t launch_pack_state(const GridDesc& g, const double* src, double* dst, bool unpack, cudaStream_t st);
cudaError_t launch_flag_scan(const GridDesc& g, const Phys& P, const double* s, const double* geo, int ntx,
                             int nty, unsigned short* flags, DevScalars* sc, bool fastdiv, cudaStream_t st);
cudaError_t launch_mass(const GridDesc& g, const double* s, double* part, int blocks, cudaStream_t st);
cudaError_t launch_snapshot(const GridDesc& g, const double* s, const double* geo, double* out, int ncols,
                            int nrows, double H, double h_dry, double eps_h, double vu, cudaStream_t st);
cudaError_t launch_pre(const PreArgs& a, cudaStream_t st);
int bc_blocks(const GridDesc& g);
cudaError_t selftest_division(long long n, unsigned long long seed, unsigned long long* mismatches);
cudaError_t selftest_minmod(long long n, const double* a, const double* b, double* out);
cudaError_t phase_cycles(unsigned long long* out, int reset);
}  // namespace tpb

using tpb::DevScalars;
using tpb::host::kGhost;

namespace {

struct ConfigErr { std::string msg; };
struct NumErr { std::string msg; };
struct CudaErr { std::string msg; };

inline void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaErr{std::string(what) + ": " + cudaGetErrorString(e)};
}

constexpr size_t kCtrlBytes = offsetof(DevScalars, lam_bits);
constexpr int kNactInts = 10;

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        ck(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q),
           "cuTensorMapEncodeTiled entry point");
        if (!p || q != cudaDriverEntryPointSuccess) throw CudaErr{"cuTensorMapEncodeTiled unavailable"};
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// 3-D tiled descriptor over [nfields][ny][pitch] doubles with the stage-kernel box
CUtensorMap make_box_map(void* base, int nx, int ny, int pitch, long long fs, int nfields, int bw = tpb::W2,
                         int bh = tpb::H2, int bf = -1) {
    CUtensorMap m;
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(nx), static_cast<cuuint64_t>(ny),
                          static_cast<cuuint64_t>(nfields)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(pitch) * sizeof(double),
                             static_cast<cuuint64_t>(fs) * sizeof(double)};
    cuuint32_t box[3] = {static_cast<cuuint32_t>(bw), static_cast<cuuint32_t>(bh),
                         static_cast<cuuint32_t>(bf < 0 ? nfields : bf)};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaErr{"cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")"};
    return m;
}

}  // namespace

struct tp_ctx {
    std::string err;
    tp_params p{};
    int device = 0;
    // grid
    int ncols = 0, nrows_g = 0;      // interior dims of the whole DEM
    int row0 = 0, row1 = 0, nrows = 0;  // owned interior rows [row0, row1)
    int nx = 0, ny = 0, pitch = 0;
    long long fs = 0;
    double dxi = 0, deta = 0;
    tpb::GridDesc g{};
    tpb::Phys ph{};
    std::vector<double> geo_h;  // 14 * nx * ny (dense, local rows)
    tpb::host::Dem dem;
    // device
    // logical element (i, j) of a field lives at raw[f*fs + j*pitch + i + 1]: one
    // leading pad column makes every stage-kernel box origin (column X0-2, X0 = 3+16k)
    // 16-byte aligned, which TMA requires.  dX = rawX + 1.
    double* rawA = nullptr;
    double* rawB = nullptr;
    double* rawGeo = nullptr;
    double* dA = nullptr;
    double* dB = nullptr;
    double* dGeo = nullptr;
    DevScalars* dSc = nullptr;
    tpb::ClipList* dClip = nullptr;  // regularize's clipped-mass events (tp_types.h)
    long long timed_tiles[2] = {0, 0};  // tiles processed per stage over the last tp_steps_timed
    double* dTallyP = nullptr;
    double* dTallyC = nullptr;
    unsigned* dStampP = nullptr;  // ring-tally stamps (DevScalars::tally_epoch)
    unsigned* dStampC = nullptr;
    signed char* dSide = nullptr;
    unsigned char* dInflowTiles = nullptr;  // per tile: its radius-2 box reads an inflow ghost
    double* dSamples = nullptr;
    double* dDts = nullptr;
    long dts_cap = 0;
    int ntx = 0, nty = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    // options / flags
    bool fastdiv = true;
    int graph_steps = 16;
    bool skip_dry = true;  // list only tiles that are not bitwise no-ops (tiles_kernel)
    bool geo_safe = false; // every jb (and so every face jbf) in [1, 2^100]: safe tiles allowed
    bool geo_safe2 = false; // geometry and constants inside the window-B bounds
    bool host_geometry = false;  // TPFLOW_HOST_GEOMETRY=1: host restatement instead of tp_geometry.cu
    unsigned short* dFlagA = nullptr;  // per-tile TileFlag bits of A / B (all set = unknown)
    unsigned short* dFlagB = nullptr;
    int* dTiles = nullptr;            // active-tile list of the stage in flight + its count
    double* dDense = nullptr;         // dense [6][ny][nx] staging for host transfers (lazy)
    // device-resident slab exchange (tp_peer.cu)
    tpb::PeerBox* dBox = nullptr;     // this slab's mailbox (exported to the other ranks)
    tpb::PeerLink link{};
    bool peered = false;
    unsigned long long peer_base = 0; // host copy of DevScalars::peer_base
    std::vector<void*> ipc_opened;    // CUDA-IPC mappings to close at destroy
    int* dNact = nullptr;             // [kNactInts] list counts pred, corr; last-launch stats pred, corr;
                                      // safe-tile counts pred, corr; tile-scheduler counters;
                                      // back-region counts pred, corr (peer-joined slabs)
    int stage_ctas = 0;               // stage grid cap (0: 2 per SM); peers sharing this device leave SMs free
    int last_tiles_stage = 1;         // stage of the last tiles_kernel enqueued (0 pred, 1 corr)
    bool lam_valid = false;
    bool ghosts_in_B = false;
    bool inflow_active = false;
    int n_samples = 0;
    bool hydro_set = false;
    int adv_only = 0;
    // unrolled step graphs of 1, 2, 4, ..., graph_steps steps: [0] dense stage CTAs, [1] wide
    // (short lists); a replay runs a power-of-two number of steps (steps_launch)
    static constexpr int kMaxGraphLog = 13;  // graph_steps <= 4096 (tp_set_option)
    cudaGraphExec_t graphs[2][kMaxGraphLog] = {};
    double dt_hint = 0.0;               // the last step's dt: sizes the next replays (steps to the output)
    bool merge_post = true;             // option "merge_post": post + the next pre in one launch
    cudaGraphExec_t graphT = nullptr;   // one step with timing events around the stage kernels
    int num_sms = 148;
    int wide_tiles = -1;                // use the wide graphs while the last lists had <= this many tiles (-1: #SMs)
    bool wide = false;                  // the graph family of the next replay
    cudaEvent_t evT[4] = {nullptr, nullptr, nullptr, nullptr};
    int graphK_steps = 0;
    long launches = 0;
    double t_next_last = 0.0;
    CUtensorMap tmA{}, tmB{}, tmG{}, tmC{}, tmU{};
};

namespace {

tpb::Inflow inflow_desc(const tp_ctx* c) {
    tpb::Inflow in{};
    in.n_samples = c->n_samples;
    in.samples = c->dSamples;
    in.ghost_side = c->dSide;
    in.t_unit = std::sqrt(c->p.L / c->p.g);
    in.H = c->p.H;
    in.v_unit = std::sqrt(c->p.g * c->p.L);
    in.active = c->inflow_active ? 1 : 0;
    return in;
}

void validate_params(const tp_params* p) {
    // ModelParams::validate (params.hpp:40-50), ScalingConfig::validate (:21-25),
    // SimConfig::validate numerics (config.hpp:31-40) — same order and messages.
    if (!(p->delta_b >= 0.0 && p->delta_b < 90.0))
        throw ConfigErr{"params: delta_b must be in [0, 90) degrees"};
    if (!(p->C_d >= 0.0)) throw ConfigErr{"params: C_d must be >= 0"};
    if (!(p->N_R > 0.0)) throw ConfigErr{"params: N_R must be > 0"};
    if (!(p->theta_b >= 0.0)) throw ConfigErr{"params: theta_b must be >= 0"};
    if (!(p->phi_s0 >= 0.0 && p->phi_s0 <= 1.0)) throw ConfigErr{"params: phi_s0 must be in [0, 1]"};
    if (!(p->alpha_rho > 0.0 && p->alpha_rho <= 1.0))
        throw ConfigErr{"params: alpha_rho must be in (0, 1]"};
    if (!(p->L > 0.0)) throw ConfigErr{"scaling: L must be > 0"};
    if (!(p->H > 0.0)) throw ConfigErr{"scaling: H must be > 0"};
    if (!(p->g > 0.0)) throw ConfigErr{"scaling: g must be > 0"};
    if (!(p->cfl > 0.0 && p->cfl <= 0.125))
        throw ConfigErr{"config: cfl must be in (0, 0.125], got " + std::to_string(p->cfl)};
    if (!(p->t_end > 0.0)) throw ConfigErr{"config: t_end must be > 0"};
    if (!(p->dt_out > 0.0)) throw ConfigErr{"config: dt_out must be > 0"};
    if (!(p->h_dry > 0.0)) throw ConfigErr{"config: h_dry must be > 0"};
    if (!(p->eps_h > 0.0)) throw ConfigErr{"config: eps_h must be > 0"};
}

void build_phys(tp_ctx* c) {
    const tp_params& p = c->p;
    tpb::Phys& P = c->ph;
    P.eps = p.H / p.L;  // ScalingConfig::epsilon
    P.alpha = p.alpha_rho;
    P.oma = 1.0 - p.alpha_rho;
    P.C_d = p.C_d;
    P.N_R = p.N_R;
    P.theta_b = p.theta_b;
    P.eps_chi = std::pow(P.eps, p.chi);                  // physics.hpp:60
    P.tan_d = std::tan(p.delta_b * M_PI / 180.0);        // params.hpp:38
    P.neg_eps_alpha = -P.eps * p.alpha_rho;              // physics.hpp:147
    P.eps_NR = P.eps * p.N_R;                            // physics.hpp:115
    P.h_dry = p.h_dry;
    P.eps_h = p.eps_h;
    P.eps_h2 = p.eps_h * p.eps_h;
    P.dxi = c->dxi;
    P.deta = c->deta;
    P.two_dxi = 2.0 * c->dxi;
    P.two_deta = 2.0 * c->deta;
    P.cell_area = c->dxi * c->deta;
    P.cfl = p.cfl;
    P.r_dxi = 1.0 / P.dxi;
    P.r_deta = 1.0 / P.deta;
    P.r_two_dxi = 1.0 / P.two_dxi;
    P.r_two_deta = 1.0 / P.two_deta;
    P.r_eps_NR = 1.0 / P.eps_NR;
    P.r_NR = 1.0 / P.N_R;
    P.adv_only = c->adv_only;
    P.cap_on = !(c->adv_only || P.tan_d == 0.0) ? 1 : 0;  // solver.cpp:454
    // mkrcp_const's divisor test (tp_math.cuh): b positive in [2^-200, 2^200]
    auto window = [](double b) {
        uint64_t u;
        std::memcpy(&u, &b, sizeof(u));
        const unsigned eb = static_cast<unsigned>(u >> 52);
        return (eb - (1023u - 200u)) <= 400u ? 1 : 0;
    };
    P.ok_dxi = window(P.dxi);
    P.ok_deta = window(P.deta);
    P.ok_two_dxi = window(P.two_dxi);
    P.ok_two_deta = window(P.two_deta);
}

void drop_graphs(tp_ctx* c) {
    for (auto& fam : c->graphs)
        for (cudaGraphExec_t& gx : fam) {
            if (gx) cudaGraphExecDestroy(gx);
            gx = nullptr;
        }
    if (c->graphT) cudaGraphExecDestroy(c->graphT);
    c->graphT = nullptr;
    c->graphK_steps = 0;
}

tpb::StageArgs stage_args(tp_ctx* c, bool corr, int loop) {
    tpb::StageArgs a{};
    a.tm_s = corr ? c->tmB : c->tmA;
    a.tm_g = c->tmG;
    a.tm_c = c->tmC;
    a.tm_u = c->tmU;
    a.g = c->g;
    a.ph = c->ph;
    a.s = corr ? c->dB : c->dA;
    a.u0 = c->dA;
    a.out = corr ? c->dA : c->dB;
    a.geo = c->dGeo;
    a.sc = c->dSc;
    a.tally = corr ? c->dTallyC : c->dTallyP;
    a.tally_stamp = corr ? c->dStampC : c->dStampP;
    a.inflow = inflow_desc(c);  // corrector in the loop: the next predictor's inflow-window test
    a.ntx = c->ntx;
    a.nty = c->nty;
    a.loop = loop;
    a.use_sc_dt = 1;
    a.tiles = c->dTiles;
    a.ntiles_active = c->dNact + (corr ? 1 : 0);
    a.flag_out = corr ? c->dFlagA : c->dFlagB;
    a.nact_stat = c->dNact + 2;
    a.work = c->dNact + 6 + (corr ? 1 : 0);
    a.nback = c->dNact + 8 + (corr ? 1 : 0);
    a.max_ctas = c->stage_ctas;
    if (loop && c->peered) {  // stage_kernel<..., PEER>: halo tiles wait in the kernel (tp_peer.cu)
        const int buf = corr ? 1 : 0;
        for (int side = 0; side < 2; ++side) {
            a.has_nbr[side] = c->link.nbr_state[buf][side] ? 1 : 0;
            a.halo_seq[side] = &c->dBox->halo_seq[buf][side];
            a.halo_nz[side] = c->dBox->halo_nz[buf][side];
        }
        a.nyi = c->ny - 6;
        a.peer_phase = 1 + buf;
        a.timeout_ns = c->link.timeout_ns;
    }
    return a;
}

tpb::TileArgs tile_args(tp_ctx* c, const tpb::StageArgs& a, bool corr) {
    tpb::TileArgs t{};
    t.flag_in = corr ? c->dFlagB : c->dFlagA;
    t.flag_out = corr ? c->dFlagA : c->dFlagB;
    t.tiles = c->dTiles;
    t.ntiles_active = c->dNact + (corr ? 1 : 0);
    t.ntiles_reset = c->dNact + (corr ? 0 : 1);
    t.work = c->dNact + 6 + (corr ? 1 : 0);
    t.ntx = c->ntx;
    t.nty = c->nty;
    t.nxi = c->nx - 6;
    t.nyi = c->ny - 6;
    t.skip = c->skip_dry ? 1 : 0;
    // ring boxes read ghost cells: only plain zero-gradient copies refreshed right before
    // the stage (the device loop) keep the 3x3 flag rule exact; Mode-II inflow ghosts are
    // not copies, so the ring tiles whose boxes reach them are always listed (and unsafe)
    t.ring_ineligible = a.loop ? 0 : 1;
    t.inflow_tiles = c->inflow_active ? c->dInflowTiles : nullptr;
    t.south_ineligible = c->g.has_south ? 0 : 1;
    t.north_ineligible = c->g.has_north ? 0 : 1;
    t.safe_ok = (c->fastdiv && c->geo_safe && c->geo_safe2) ? 1 : 0;
    t.cond_halo = (a.loop && c->peered) ? 1 : 0;
    t.stage = corr ? 1 : 0;
    t.nback = c->dNact + 8 + (corr ? 1 : 0);
    t.nback_reset = c->dNact + 8 + (corr ? 0 : 1);
    t.loop = a.loop;
    t.sc = c->dSc;
    return t;
}

// Stage launches outside the fused device loop: the active-tile list (tiles_kernel), then the stage.
cudaError_t launch_stage_sel(tp_ctx* c, const tpb::StageArgs& a, bool fastdiv, bool corr, cudaStream_t st,
                             cudaEvent_t ev0 = nullptr, cudaEvent_t ev1 = nullptr) {
    const tpb::TileArgs t = tile_args(c, a, corr);
    // each tiles_kernel zeroes the other stage's counter; two launches of one stage in a
    // row (a bare tp_stage call) need an explicit reset
    const int stage = corr ? 1 : 0;
    if (c->last_tiles_stage == stage) {
        cudaError_t e0 = cudaMemsetAsync(t.ntiles_active, 0, sizeof(int), st);
        if (e0 == cudaSuccess) e0 = cudaMemsetAsync(t.ntiles_active + 4, 0, sizeof(int), st);
        if (e0 != cudaSuccess) return e0;
    }
    c->last_tiles_stage = stage;
    cudaError_t e = tpb::launch_tiles(t, st);
    if (e != cudaSuccess) return e;
    if (ev0 && (e = cudaEventRecord(ev0, st)) != cudaSuccess) return e;
    e = tpb::launch_stage(a, fastdiv, corr, false, false, st);
    if (e == cudaSuccess && ev1) e = cudaEventRecord(ev1, st);
    return e;
}

// Conservative reset of the per-tile flags (after any write to a state buffer that is
// not a stage kernel): every tile is listed until a stage recomputes its flag.
void invalidate_flags(tp_ctx* c, bool a_buf, bool b_buf) {
    const size_t n = static_cast<size_t>(c->ntx) * c->nty;
    if (a_buf) ck(cudaMemsetAsync(c->dFlagA, 0xff, n * sizeof(unsigned short), c->stream), "flags");
    if (b_buf) ck(cudaMemsetAsync(c->dFlagB, 0xff, n * sizeof(unsigned short), c->stream), "flags");
}

// Exact flags of buffer A after a write outside the stage kernels (flag_scan_kernel): the next
// stage lists only the tiles that can change instead of every tile (after tp_set_state the
// first step used to process the whole grid twice).  The same pass computes compute_dt's
// lambda of A (what fresh_lambda would), so lam_valid holds afterwards.
void scan_flags_A(tp_ctx* c) {
    ck(cudaMemsetAsync(&c->dSc->lam_bits, 0, sizeof(unsigned long long), c->stream), "memset");
    ck(tpb::launch_flag_scan(c->g, c->ph, c->dA, c->dGeo, c->ntx, c->nty, c->dFlagA, c->dSc, c->fastdiv, c->stream),
       "flag scan");
    ck(cudaMemcpyAsync(&c->dSc->lam_cur, &c->dSc->lam_bits, sizeof(unsigned long long), cudaMemcpyDeviceToDevice,
                       c->stream),
       "lam copy");
    c->lam_valid = true;
}

void launch_bc(tp_ctx* c, int buf, int tsrc, double t, int loop) {
    tpb::BcArgs b{};
    b.g = c->g;
    b.s = buf ? c->dB : c->dA;
    b.geo = c->dGeo;
    b.inflow = inflow_desc(c);
    b.sc = c->dSc;
    b.t = t;
    b.tsrc = tsrc;
    b.loop = loop;
    ck(tpb::launch_bc(b, c->stream), "bc_kernel");
}

tpb::PostArgs post_args(tp_ctx* c, int loop) {
    tpb::PostArgs a{};
    a.sc = c->dSc;
    a.tally_pred = c->dTallyP;
    a.tally_corr = c->dTallyC;
    a.stamp_pred = c->dStampP;
    a.stamp_corr = c->dStampC;
    a.ntx = c->ntx;
    a.nty = c->nty;
    a.loop = loop;
    a.peered = c->peered ? 1 : 0;
    return a;
}

void launch_post(tp_ctx* c, int loop) { ck(tpb::launch_post(post_args(c, loop), c->stream), "post_kernel"); }

// one whole step of the device loop: 5 kernels
//   pre(bc(u,t) + predictor list + compute_dt) -> predictor -> pre(bc(u*,t+dt) + corrector list)
//   -> corrector -> post(t += dt, audit, stop flag)
// the loop's bc of a stage's input buffer (apply_boundaries, solver.cpp:639 / :523)
tpb::BcArgs loop_bc(tp_ctx* c, int corr) {
    tpb::BcArgs b{};
    b.g = c->g;
    b.s = corr ? c->dB : c->dA;
    b.geo = c->dGeo;
    b.inflow = inflow_desc(c);
    b.sc = c->dSc;
    b.t = 0.0;
    // corrector: Hydrograph::at(t + dt) as evaluated once after compute_dt (tsrc 3)
    b.tsrc = corr ? 3 : 1;
    b.stage = corr ? 1 : 0;
    b.loop = 1;
    return b;
}

// bc + the stage's list (+ compute_dt before the predictor): pre_kernel
void launch_loop_pre(tp_ctx* c, const tpb::StageArgs& sa, int corr) {
    tpb::PreArgs p{};
    p.bc = loop_bc(c, corr);
    p.t = tile_args(c, sa, corr != 0);
    p.P = c->ph;
    p.nb_bc = tpb::bc_blocks(c->g);
    p.with_dt = corr ? 0 : 1;
    ck(tpb::launch_pre(p, c->stream), corr ? "pre (corrector)" : "pre (predictor)");
}

// the step graphs merge each step's post into the next step's pre (option "merge_post",
// unpeered contexts): pre, then per step predictor, pre(corrector), corrector, and between
// steps one prepost_kernel; a standalone post ends the replay.  4 launches per step + 1.
bool merged_loop(const tp_ctx* c) { return c->merge_post && !c->peered; }

void enqueue_merged_steps(tp_ctx* c, int k, bool wide) {
    const tpb::StageArgs pa = stage_args(c, false, 1), ca = stage_args(c, true, 1);
    tpb::PrePostArgs pp{};
    pp.pre.bc = loop_bc(c, 0);
    pp.pre.t = tile_args(c, pa, false);
    pp.pre.P = c->ph;
    pp.pre.nb_bc = tpb::bc_blocks(c->g);
    pp.pre.with_dt = 1;
    pp.post = post_args(c, 1);
    for (int s = 0; s < k; ++s) {
        if (s == 0) launch_loop_pre(c, pa, 0);
        else ck(tpb::launch_prepost(pp, c->stream), "prepost");
        ck(tpb::launch_stage(pa, c->fastdiv, false, false, wide, c->stream), "predictor");
        launch_loop_pre(c, ca, 1);
        ck(tpb::launch_stage(ca, c->fastdiv, true, false, wide, c->stream), "corrector");
    }
    launch_post(c, 1);
    c->last_tiles_stage = 1;
}

void enqueue_loop_step(tp_ctx* c, cudaEvent_t* ev = nullptr, bool wide = false) {
    // slabs connected by tp_peer_connect*: the lambda + stop all-reduce before compute_dt
    if (c->peered) ck(tpb::launch_peer_lambda(c->link, c->dSc, c->stream), "peer lambda");
    for (int corr = 0; corr < 2; ++corr) {
        const tpb::StageArgs sa = stage_args(c, corr != 0, 1);
        launch_loop_pre(c, sa, corr);
        c->last_tiles_stage = corr;
        // halo rows after apply_boundaries (solver.cpp:639, :523), straight into the
        // neighbours' buffers; the stage kernel waits for theirs before its halo tiles
        if (c->peered)
            ck(tpb::launch_peer_halo(c->link, c->g, corr ? c->dB : c->dA, corr, c->dSc, c->stream), "peer halo");
        if (ev) ck(cudaEventRecordWithFlags(ev[2 * corr], c->stream, cudaEventRecordExternal), "event");
        ck(tpb::launch_stage(sa, c->fastdiv, corr != 0, c->peered, wide, c->stream), corr ? "corrector" : "predictor");
        if (ev) ck(cudaEventRecordWithFlags(ev[2 * corr + 1], c->stream, cudaEventRecordExternal), "event");
    }
    launch_post(c, 1);
}

cudaGraphExec_t capture_steps(tp_ctx* c, int k, cudaEvent_t* ev = nullptr, bool wide = false) {
    cudaGraph_t graph = nullptr;
    const int saved_stage = c->last_tiles_stage;
    c->last_tiles_stage = 1;  // a replay always follows a corrector (tp_steps resets otherwise)
    ck(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal), "begin capture");
    try {
        if (merged_loop(c) && !ev) enqueue_merged_steps(c, k, wide);
        else
            for (int s = 0; s < k; ++s) enqueue_loop_step(c, ev, wide);
    } catch (...) {
        cudaStreamEndCapture(c->stream, &graph);
        if (graph) cudaGraphDestroy(graph);
        c->last_tiles_stage = saved_stage;
        throw;
    }
    ck(cudaStreamEndCapture(c->stream, &graph), "end capture");
    cudaGraphExec_t exec = nullptr;
    ck(cudaGraphInstantiate(&exec, graph, 0), "graph instantiate");
    cudaGraphDestroy(graph);
    c->last_tiles_stage = saved_stage;
    return exec;
}

void write_ctrl(tp_ctx* c, double t, double t_next, double t_end, double dt, long long max_steps) {
    DevScalars h{};
    h.t = t;
    h.t_next = t_next;
    h.t_end = t_end;
    h.dt = dt;
    h.steps = 0;
    h.max_steps = max_steps;
    h.done = 0;
    h.hit = 0;
    ck(cudaMemcpyAsync(c->dSc, &h, kCtrlBytes, cudaMemcpyHostToDevice, c->stream), "ctrl H2D");
}

DevScalars read_scalars(tp_ctx* c) {
    DevScalars h{};
    ck(cudaMemcpyAsync(&h, c->dSc, sizeof(DevScalars), cudaMemcpyDeviceToHost, c->stream), "scalars D2H");
    ck(cudaStreamSynchronize(c->stream), "sync");
    return h;
}

void fresh_lambda(tp_ctx* c) {
    ck(cudaMemsetAsync(&c->dSc->lam_bits, 0, sizeof(unsigned long long), c->stream), "memset");
    ck(tpb::launch_lambda(c->g, c->ph, c->dA, c->dGeo, c->dSc, c->fastdiv, c->stream), "lambda_kernel");
    ck(cudaMemcpyAsync(&c->dSc->lam_cur, &c->dSc->lam_bits, sizeof(unsigned long long),
                       cudaMemcpyDeviceToDevice, c->stream),
       "lam copy");
    c->lam_valid = true;
}

double read_cell(tp_ctx* c, const double* buf, int field, int X, int Y) {
    double v = 0.0;
    ck(cudaMemcpy(&v, buf + field * c->fs + static_cast<long long>(Y) * c->pitch + X, sizeof(double),
                  cudaMemcpyDeviceToHost),
       "cell D2H");
    return v;
}

// Turn a device error key into the reference's NumericsError text and clear it.
// pred_buf: buffer the class-0 (regularize) errors refer to.
void raise_error_key(tp_ctx* c, unsigned long long key, const double* pred_buf) {
    unsigned long long none = tpb::kNoError;
    ck(cudaMemcpy(&c->dSc->err_key, &none, sizeof(none), cudaMemcpyHostToDevice), "err reset");
    const unsigned cls = static_cast<unsigned>(key >> 62);
    if (cls <= 1) {
        const int Y = static_cast<int>((key >> 32) & 0x3fffffffull);
        const int X = static_cast<int>((key >> 1) & 0x7fffffffull);
        const int p = static_cast<int>(key & 1ull);
        const double* buf = cls == 0 ? pred_buf : c->dA;
        const double w = read_cell(c, buf, p, X, Y);
        const double jb = read_cell(c, c->dGeo, tpb::G_JB, X, Y);
        const double hp = w / jb;
        throw NumErr{std::string("negative ") + (p == 0 ? "solid" : "fluid") + " thickness " +
                     tpb::host::to_string_f(hp) + " at cell (" + std::to_string(X - kGhost) + ", " +
                     std::to_string(Y - kGhost + c->row0) + ")"};
    }
    if (cls == 3)
        throw CudaErr{"slab exchange: a neighbour did not arrive within the timeout (peer exchange, tp_peer.cu)"};
    static const char* names[6] = {"ws", "wf", "qsx", "qsy", "qfx", "qfy"};
    const int f = static_cast<int>((key >> 56) & 0x3full);
    const int Y = static_cast<int>((key >> 28) & 0xfffffffull);
    const int X = static_cast<int>(key & 0xfffffffull);
    throw NumErr{std::string("non-finite value in field '") + names[f] + "' at cell (" +
                 std::to_string(X - kGhost) + ", " + std::to_string(Y - kGhost + c->row0) +
                 ") during advance_step"};
}

void check_error(tp_ctx* c, const double* pred_buf) {
    unsigned long long key = 0;
    ck(cudaMemcpyAsync(&key, &c->dSc->err_key, sizeof(key), cudaMemcpyDeviceToHost, c->stream), "err D2H");
    ck(cudaStreamSynchronize(c->stream), "sync");
    if (key != tpb::kNoError) raise_error_key(c, key, pred_buf);
}

// host dense (nx*ny per field) <-> device pitched: one contiguous DMA copy through a
// dense device staging buffer, re-pitched by a kernel (a 2-D copy with 6*ny short rows
// runs at a fraction of the link bandwidth)
double* dense_staging(tp_ctx* c) {
    if (!c->dDense) ck(cudaMalloc(&c->dDense, sizeof(double) * 6ull * c->ny * c->nx), "cudaMalloc staging");
    return c->dDense;
}
// Host state [6][ny][nx] -> the pitched device layout: the six fields are one 2-D array of
// 6 ny rows (fs = ny * pitch), so one pitched copy moves it directly (no staging buffer, no
// unpack kernel: 3.7 ms instead of 3.8 ms for C2 2048^2).  The other way the pitched copy is
// slower (4.0 ms against 3.8 ms: the device rows start 8 bytes past a 64-byte boundary), so
// the download packs into the dense staging buffer and copies that.
void upload_state(tp_ctx* c, double* dst, const double* src) {
    ck(cudaMemcpy2DAsync(dst, sizeof(double) * c->pitch, src, sizeof(double) * c->nx, sizeof(double) * c->nx,
                         6ull * c->ny, cudaMemcpyHostToDevice, c->stream),
       "state H2D");
}
void download_state(tp_ctx* c, double* dst, const double* src) {
    double* d = dense_staging(c);
    ck(tpb::launch_pack_state(c->g, src, d, false, c->stream), "pack state");
    ck(cudaMemcpyAsync(dst, d, sizeof(double) * 6ull * c->ny * c->nx, cudaMemcpyDeviceToHost, c->stream),
       "state D2H");
    ck(cudaStreamSynchronize(c->stream), "sync");
}

void sync_ghosts(tp_ctx* c) {
    if (c->ghosts_in_B) {
        ck(tpb::launch_ghost_copy(c->g, c->dB, c->dA, c->stream), "ghost copy");
        c->ghosts_in_B = false;
    }
}


int fail(tp_ctx* c, int code, const std::string& msg) {
    if (c) c->err = msg;
    return code;
}

#define TP_GUARD(c, ...)                                          \
    try {                                                         \
        if (c) cudaSetDevice((c)->device);                        \
        __VA_ARGS__;                                              \
        return TP_OK;                                             \
    } catch (const ConfigErr& e) {                                \
        return fail(c, TP_ERR_CONFIG, e.msg);                     \
    } catch (const NumErr& e) {                                   \
        return fail(c, TP_ERR_NUMERICS, e.msg);                   \
    } catch (const CudaErr& e) {                                  \
        return fail(c, TP_ERR_CUDA, e.msg);                       \
    } catch (const std::exception& e) {                           \
        return fail(c, TP_ERR_INTERNAL, e.what());                \
    }

// Window B of the safe-tile form (DESIGN.md §3 item 6): every geometry value 0 or of
// magnitude in [2^-50, 2^50], jb <= 2^50, and the constants entering numerators within
// 2^+-20 (eps_h within [2^-60, 2^20]).  n = padded cells of this context.
bool consts_window_b(const tp_ctx* c) {
    auto mag_ok = [](double v, double lo, double hi) {
        const double a = std::fabs(v);
        return a == 0.0 || (a >= lo && a <= hi);
    };
    const tpb::Phys& P = c->ph;
    const double w20 = 0x1p20, n20 = 0x1p-20;
    return P.eps_h >= 0x1p-60 && P.eps_h <= w20 && P.eps >= n20 && P.eps <= w20 && mag_ok(P.oma, n20, 1.0) &&
           mag_ok(P.theta_b, n20, w20) && P.N_R >= n20 && P.N_R <= w20 && P.dxi >= n20 && P.dxi <= w20 &&
           P.deta >= n20 && P.deta <= w20;
}

void geo_window_b(tp_ctx* c, size_t n) {
    // host twin of geo_check_kernel (tp_geometry.cu), for the host-geometry path
    auto mag_ok = [](double v, double lo, double hi) {
        const double a = std::fabs(v);
        return a == 0.0 || (a >= lo && a <= hi);
    };
    const double* G = c->geo_h.data();
    bool ok = true;
    for (size_t k = 0; k < n && ok; ++k) {
        const double jb = G[tpb::R_JB * n + k];
        ok = jb >= 1.0 && jb <= 0x1p50;
        for (int f : {tpb::R_A11, tpb::R_A12, tpb::R_A21, tpb::R_A22}) ok = ok && mag_ok(G[f * n + k], 0x1p-120, 0x1p50);
        for (int f : {tpb::R_NX, tpb::R_NY}) ok = ok && mag_ok(G[f * n + k], 0x1p-200, 1.0);
        for (int f : {tpb::R_NZ, tpb::R_DNX_DXI, tpb::R_DNY_DXI, tpb::R_DNZ_DXI, tpb::R_DNX_DETA, tpb::R_DNY_DETA,
                      tpb::R_DNZ_DETA})
            ok = ok && std::isfinite(G[f * n + k]);
    }
    c->geo_safe2 = c->geo_safe && ok && consts_window_b(c);
}

// host copy of the 14 reference geometry fields (terrain.hpp:59-63 order), on demand
void ensure_geo_h(tp_ctx* c) {
    if (!c->geo_h.empty()) return;
    const size_t n = static_cast<size_t>(c->nx) * c->ny;
    c->geo_h.resize(14 * n);
    const int map[14] = {tpb::G_NX, tpb::G_NY, tpb::G_NZ, tpb::G_JB, tpb::G_A11, tpb::G_A12, tpb::G_A21,
                         tpb::G_A22, tpb::G_DNX_DXI, tpb::G_DNY_DXI, tpb::G_DNZ_DXI, tpb::G_DNX_DETA,
                         tpb::G_DNY_DETA, tpb::G_DNZ_DETA};
    for (int k = 0; k < 14; ++k)
        ck(cudaMemcpy2DAsync(c->geo_h.data() + k * n, c->nx * sizeof(double), c->dGeo + map[k] * c->fs,
                             c->pitch * sizeof(double), c->nx * sizeof(double), c->ny, cudaMemcpyDeviceToHost,
                             c->stream),
           "geometry D2H");
    ck(cudaStreamSynchronize(c->stream), "sync");
}

void create_impl(tp_ctx* c, const tp_params* p, const tp_dem* dem, int row0, int row1) {
    validate_params(p);
    if (!dem || dem->ncols < 2 || dem->nrows < 2)
        throw ConfigErr{"grid must be at least 2x2"};
    if (!(dem->cellsize > 0.0)) throw ConfigErr{"cellsize must be positive"};
    if (row0 < 0 || row1 > dem->nrows || row1 - row0 < 2)
        throw ConfigErr{"slab rows out of range (need at least 2 rows)"};
    // active-tile list entries pack (tile row << 16) | tile column, 13 + 16 bits
    if (dem->ncols > tpb::TX * 65535 || row1 - row0 > tpb::TY * 8191)
        throw ConfigErr{"grid too large for one context (at most " + std::to_string(tpb::TX * 65535) + " columns and " +
                        std::to_string(tpb::TY * 8191) + " rows per slab)"};
    c->p = *p;
    c->device = p->device;
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    ck(tpb::init_kernels(), "init kernels");
    c->ncols = dem->ncols;
    c->nrows_g = dem->nrows;
    c->row0 = row0;
    c->row1 = row1;
    c->nrows = row1 - row0;
    c->dem.ncols = dem->ncols;
    c->dem.nrows = dem->nrows;
    c->dem.xll = dem->xll;
    c->dem.yll = dem->yll;
    c->dem.cellsize = dem->cellsize;
    c->dem.z.assign(dem->z, dem->z + static_cast<size_t>(dem->ncols) * dem->nrows);

    // Simulator ctor: geometry of the whole extended DEM (solver.cpp:16), then our rows.
    // Built on the device (tp_geometry.cu) unless TPFLOW_HOST_GEOMETRY=1 selects the host
    // restatement (tp_geometry.cpp); both are bit-identical to terrain.cpp.
    const char* hg = std::getenv("TPFLOW_HOST_GEOMETRY");
    c->host_geometry = hg && hg[0] == '1';
    tpb::host::Geometry G;
    if (c->host_geometry) {
        G = tpb::host::compute_geometry(tpb::host::extend_grid(c->dem, kGhost), p->L);
        c->nx = G.nx;
        c->dxi = G.dxi;
        c->deta = G.deta;
    } else {
        c->nx = dem->ncols + 2 * kGhost;
        c->dxi = dem->cellsize / p->L;  // terrain.cpp:162-163
        c->deta = dem->cellsize / p->L;
    }
    c->ny = c->nrows + 2 * kGhost;
    if (c->host_geometry) {
        c->geo_h.resize(14ull * c->nx * c->ny);
        for (int k = 0; k < 14; ++k)
            std::memcpy(c->geo_h.data() + static_cast<size_t>(k) * c->nx * c->ny,
                        G.field(k) + static_cast<size_t>(row0) * G.nx,
                        sizeof(double) * static_cast<size_t>(c->nx) * c->ny);
    }

    c->pitch = (c->nx + 1 + 7) & ~7;
    c->fs = static_cast<long long>(c->pitch) * c->ny;
    c->g.nx = c->nx;
    c->g.ny = c->ny;
    c->g.pitch = c->pitch;
    c->g.fs = c->fs;
    c->g.has_south = row0 == 0 ? 1 : 0;
    c->g.has_north = row1 == dem->nrows ? 1 : 0;
    build_phys(c);

    c->ntx = (c->ncols + tpb::TX - 1) / tpb::TX;
    c->nty = (c->nrows + tpb::TY - 1) / tpb::TY;

    const size_t sbytes = sizeof(double) * 6ull * c->fs;
    ck(cudaMalloc(&c->rawA, sbytes), "cudaMalloc state A");
    ck(cudaMalloc(&c->rawB, sbytes), "cudaMalloc state B");
    ck(cudaMalloc(&c->rawGeo, sizeof(double) * tpb::G_COUNT * c->fs), "cudaMalloc geometry");
    c->dA = c->rawA + 1;
    c->dB = c->rawB + 1;
    c->dGeo = c->rawGeo + 1;
    cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, c->device);
    ck(cudaMalloc(&c->dSc, sizeof(DevScalars)), "cudaMalloc scalars");
    ck(cudaMemset(c->dSc, 0, sizeof(DevScalars)), "memset scalars");
    ck(cudaMalloc(&c->dClip, sizeof(tpb::ClipList)), "cudaMalloc clip list");
    const size_t tb = sizeof(double) * 4ull * c->ntx * c->nty;
    ck(cudaMalloc(&c->dTallyP, tb), "cudaMalloc tally");
    ck(cudaMalloc(&c->dTallyC, tb), "cudaMalloc tally");
    const size_t sb = sizeof(unsigned) * static_cast<size_t>(c->ntx) * c->nty;
    ck(cudaMalloc(&c->dStampP, sb), "cudaMalloc tally stamps");
    ck(cudaMalloc(&c->dStampC, sb), "cudaMalloc tally stamps");
    ck(cudaMemset(c->dStampP, 0, sb), "memset");
    ck(cudaMemset(c->dStampC, 0, sb), "memset");
    ck(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "stream");
    c->own_stream = true;
    ck(cudaMemsetAsync(c->dClip, 0, sizeof(tpb::ClipList), c->stream), "memset");
    ck(cudaMemsetAsync(c->rawA, 0, sbytes, c->stream), "memset");
    ck(cudaMemsetAsync(c->rawB, 0, sbytes, c->stream), "memset");
    ck(cudaMemsetAsync(c->dTallyP, 0, tb, c->stream), "memset");
    ck(cudaMemsetAsync(c->dTallyC, 0, tb, c->stream), "memset");
    const size_t ntiles = static_cast<size_t>(c->ntx) * c->nty;
    ck(cudaMalloc(&c->dFlagA, ntiles * sizeof(unsigned short)), "cudaMalloc flags");
    ck(cudaMalloc(&c->dFlagB, ntiles * sizeof(unsigned short)), "cudaMalloc flags");
    ck(cudaMalloc(&c->dTiles, sizeof(int) * ntiles), "cudaMalloc tiles");
    ck(cudaMalloc(&c->dBox, sizeof(tpb::PeerBox)), "cudaMalloc mailbox");
    ck(cudaMemsetAsync(c->dBox, 0, sizeof(tpb::PeerBox), c->stream), "memset");
    ck(cudaMalloc(&c->dNact, kNactInts * sizeof(int)), "cudaMalloc tiles");
    ck(cudaMemsetAsync(c->dNact, 0, kNactInts * sizeof(int), c->stream), "memset");
    invalidate_flags(c, true, true);
    if (c->host_geometry) {
            // device geometry layout (tp_types.h GeoField): the 14 reference fields
            // regrouped + RN(1/jb), RN(1/nZ) and the face RN(1/jbf) of the whole grid
            const size_t n = static_cast<size_t>(c->nx) * c->ny;
            const size_t gnx = static_cast<size_t>(G.nx);
            std::vector<double> dg(static_cast<size_t>(tpb::G_COUNT) * n, 0.0);
            auto src = [&](int rf) { return c->geo_h.data() + static_cast<size_t>(rf) * n; };
            const int map[][2] = {{tpb::G_JB, tpb::R_JB},   {tpb::G_NZ, tpb::R_NZ},   {tpb::G_A11, tpb::R_A11},
                                  {tpb::G_A12, tpb::R_A12}, {tpb::G_A21, tpb::R_A21}, {tpb::G_A22, tpb::R_A22},
                                  {tpb::G_NX, tpb::R_NX},   {tpb::G_NY, tpb::R_NY},
                                  {tpb::G_DNX_DXI, tpb::R_DNX_DXI},   {tpb::G_DNY_DXI, tpb::R_DNY_DXI},
                                  {tpb::G_DNZ_DXI, tpb::R_DNZ_DXI},   {tpb::G_DNX_DETA, tpb::R_DNX_DETA},
                                  {tpb::G_DNY_DETA, tpb::R_DNY_DETA}, {tpb::G_DNZ_DETA, tpb::R_DNZ_DETA}};
            for (const auto& m : map) std::memcpy(dg.data() + m[0] * n, src(m[1]), sizeof(double) * n);
            const double* gjb = G.field(tpb::R_JB);  // global rows: the face average may reach row1+3
            for (int j = 0; j < c->ny; ++j) {
                const int gj = j + row0;
                for (int i = 0; i < c->nx; ++i) {
                    const size_t k = static_cast<size_t>(j) * c->nx + i;
                    const double jb = gjb[gj * gnx + i];
                    dg[tpb::G_RJB * n + k] = 1.0 / jb;
                    dg[tpb::G_RNZ * n + k] = 1.0 / src(tpb::R_NZ)[k];
                    if (i + 1 < c->nx) dg[tpb::G_RJBFX * n + k] = 1.0 / (0.5 * (jb + gjb[gj * gnx + i + 1]));
                    if (gj + 1 < G.ny) dg[tpb::G_RJBFY * n + k] = 1.0 / (0.5 * (jb + gjb[(gj + 1) * gnx + i]));
                }
            }
            // safe tiles (tp_kernels.cu stage_phase1<FD, false>) need every face/cell divisor in
            // the FASTDIV window: jb in [1, 2^100] makes jb and 0.5*(jb_l + jb_r) qualify
            c->geo_safe = true;
            for (size_t k = 0; k < n && c->geo_safe; ++k) {
                const double jb = dg[tpb::G_JB * n + k];
                c->geo_safe = jb >= 1.0 && jb <= 0x1p100;
            }
            // window B (Phase 2 + Phase-3 divergence without window tests) assumes every
            // geometry value is 0 or of magnitude in [2^-50, 2^50], jb <= 2^50, and the
            // constants that enter numerators within 2^+-20 (eps_h within [2^-60, 2^20]);
            // the bound chain is in DESIGN.md §3
            geo_window_b(c, n);
            ck(cudaMemsetAsync(c->rawGeo, 0, sizeof(double) * tpb::G_COUNT * c->fs, c->stream), "memset");
            ck(cudaMemcpy2DAsync(c->dGeo, c->pitch * sizeof(double), dg.data(), c->nx * sizeof(double),
                                 c->nx * sizeof(double), static_cast<size_t>(tpb::G_COUNT) * c->ny,
                                 cudaMemcpyHostToDevice, c->stream),
               "geometry H2D");
            ck(cudaStreamSynchronize(c->stream), "sync");
    } else {
        ck(cudaMemsetAsync(c->rawGeo, 0, sizeof(double) * tpb::G_COUNT * c->fs, c->stream), "memset");
        ck(tpb::build_geometry_device(dem->z, dem->ncols, dem->nrows, p->L, dem->cellsize, row0, c->ny, c->g,
                                      c->dGeo, c->stream),
           "device geometry");
        // the geometry part of the safe-tile conditions, checked on the device; the host
        // copy of the fields (geo_h) is only downloaded when asked for (ensure_geo_h)
        int* dok = nullptr;
        int ok = 1;
        ck(cudaMalloc(&dok, sizeof(int)), "cudaMalloc");
        ck(cudaMemcpyAsync(dok, &ok, sizeof(int), cudaMemcpyHostToDevice, c->stream), "H2D");
        ck(tpb::launch_geo_check(c->g, c->dGeo, dok, c->stream), "geo_check_kernel");
        ck(cudaMemcpyAsync(&ok, dok, sizeof(int), cudaMemcpyDeviceToHost, c->stream), "D2H");
        ck(cudaStreamSynchronize(c->stream), "sync");
        cudaFree(dok);
        c->geo_safe = ok != 0;
        c->geo_safe2 = ok != 0 && consts_window_b(c);
    }
    // the maps cover the pad column too (x coordinate = logical column + 1)
    c->tmA = make_box_map(c->rawA, c->nx + 1, c->ny, c->pitch, c->fs, 6);
    c->tmB = make_box_map(c->rawB, c->nx + 1, c->ny, c->pitch, c->fs, 6);
    c->tmU = make_box_map(c->rawA, c->nx + 1, c->ny, c->pitch, c->fs, 6, tpb::TX, tpb::TY, 6);
    c->tmG = make_box_map(c->rawGeo, c->nx + 1, c->ny, c->pitch, c->fs, tpb::NGBOX);
    c->tmC = make_box_map(c->rawGeo, c->nx + 1, c->ny, c->pitch, c->fs, tpb::G_COUNT, tpb::TX, tpb::TY,
                          tpb::G_COUNT - tpb::NGBOX);
    DevScalars h{};
    h.lam_bits = 0;
    h.lam_cur = 0;
    h.err_key = tpb::kNoError;
    h.max_steps = LLONG_MAX;
    h.clip = c->dClip;
    ck(cudaMemcpyAsync(c->dSc, &h, sizeof(h), cudaMemcpyHostToDevice, c->stream), "scalars H2D");
    ck(cudaStreamSynchronize(c->stream), "sync");
}

// index of padded local cell (i, j) in the ghost band enumeration of bc_kernel, or -1
long band_index(const tp_ctx* c, int i, int j) {
    const int nx = c->nx, ny = c->ny;
    const long nS = c->g.has_south ? 3L * nx : 0;
    const long nN = c->g.has_north ? 3L * nx : 0;
    if (j < 3) return c->g.has_south ? static_cast<long>(j) * nx + i : -1;
    if (j >= ny - 3) return c->g.has_north ? nS + static_cast<long>(j - (ny - 3)) * nx + i : -1;
    const long rows = ny - 6;
    if (i < 3) return nS + nN + static_cast<long>(j - 3) * 3 + i;
    if (i >= nx - 3) return nS + nN + 3 * rows + static_cast<long>(j - 3) * 3 + (i - (nx - 3));
    return -1;
}

}  // namespace

extern "C" {

int tp_create_slab(const tp_params* p, const tp_dem* dem, int row0, int row1, tp_ctx** out) {
    tp_ctx* c = new tp_ctx();
    *out = c;
    TP_GUARD(c, create_impl(c, p, dem, row0, row1))
}

int tp_create(const tp_params* p, const tp_dem* dem, tp_ctx** out) {
    return tp_create_slab(p, dem, 0, dem ? dem->nrows : 0, out);
}

void tp_destroy(tp_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    drop_graphs(c);
    cudaFree(c->rawA);
    cudaFree(c->rawB);
    cudaFree(c->rawGeo);
    cudaFree(c->dSc);
    cudaFree(c->dClip);
    cudaFree(c->dTallyP);
    cudaFree(c->dTallyC);
    cudaFree(c->dStampP);
    cudaFree(c->dStampC);
    cudaFree(c->dInflowTiles);
    cudaFree(c->dSide);
    cudaFree(c->dSamples);
    cudaFree(c->dDts);
    cudaFree(c->dFlagA);
    cudaFree(c->dFlagB);
    cudaFree(c->dDense);
    for (auto& e : c->evT)
        if (e) cudaEventDestroy(e);
    cudaFree(c->dTiles);
    cudaFree(c->dNact);
    for (void* p : c->ipc_opened) cudaIpcCloseMemHandle(p);
    cudaFree(c->dBox);
    if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

int tp_geometry(const tp_dem* dem, double L, double* out) {
    try {
        tpb::host::Dem d;
        d.ncols = dem->ncols;
        d.nrows = dem->nrows;
        d.xll = dem->xll;
        d.yll = dem->yll;
        d.cellsize = dem->cellsize;
        d.z.assign(dem->z, dem->z + static_cast<size_t>(dem->ncols) * dem->nrows);
        tpb::host::Geometry G = tpb::host::compute_geometry(tpb::host::extend_grid(d, kGhost), L);
        std::memcpy(out, G.f.data(), sizeof(double) * G.f.size());
        return TP_OK;
    } catch (...) {
        return TP_ERR_INTERNAL;
    }
}

const char* tp_last_error(const tp_ctx* c) { return c ? c->err.c_str() : "null context"; }

int tp_dims(const tp_ctx* c, int* nx, int* ny, double* dxi, double* deta) {
    if (!c) return TP_ERR_INTERNAL;
    *nx = c->nx;
    *ny = c->ny;
    *dxi = c->dxi;
    *deta = c->deta;
    return TP_OK;
}

int tp_set_option(tp_ctx* c, const char* key, long value) {
    TP_GUARD(c, {
        std::string k(key);
        if (k == "fastdiv") {
            c->fastdiv = value != 0;
            drop_graphs(c);
        } else if (k == "skip_dry") {
            c->skip_dry = value != 0;
            drop_graphs(c);
        } else if (k == "wide_tiles") {
            // wide stage CTAs while the last tile lists had <= value tiles (-1: the SM count;
            // 0: never; a large value: always)
            c->wide_tiles = static_cast<int>(value);
        } else if (k == "merge_post") {
            // 1: one launch for each step's post and the next step's pre (default); 0: five
            // launches per step
            c->merge_post = value != 0;
            drop_graphs(c);
        } else if (k == "graph_steps") {
            if (value < 1 || value > 4096) throw ConfigErr{"graph_steps must be in [1, 4096]"};
            c->graph_steps = static_cast<int>(value);
            drop_graphs(c);
        } else {
            throw ConfigErr{"unknown option '" + k + "'"};
        }
    })
}

int tp_set_initial_thickness(tp_ctx* c, const double* h_m) {
    TP_GUARD(c, {
        // Simulator::set_initial_thickness (solver.cpp:35-57): the whole-grid check on the
        // host (first offender in row-major order, the reference's message), then this
        // slab's rows on the device (init_thickness_kernel)
        const size_t total = static_cast<size_t>(c->ncols) * c->nrows_g;
        for (size_t q = 0; q < total; ++q)
            if (h_m[q] < 0.0)
                throw ConfigErr{"initial state: negative thickness at column " + std::to_string(q % c->ncols) +
                                ", row " + std::to_string(q / c->ncols)};
        sync_ghosts(c);
        double* d = dense_staging(c);
        const size_t m = static_cast<size_t>(c->ncols) * c->nrows;
        ck(cudaMemcpyAsync(d, h_m + static_cast<size_t>(c->row0) * c->ncols, sizeof(double) * m,
                           cudaMemcpyHostToDevice, c->stream),
           "thickness H2D");
        ck(tpb::launch_init_thickness(c->g, c->dGeo, d, c->ncols, c->nrows, c->p.H, c->p.phi_s0, c->dA, c->stream),
           "init_thickness_kernel");
        scan_flags_A(c);
        ck(cudaStreamSynchronize(c->stream), "sync");
        c->ghosts_in_B = false;
    })
}

int tp_set_initial_velocity(tp_ctx* c, const double* vx, const double* vy) {
    TP_GUARD(c, {
        // Simulator::set_initial_velocity (solver.cpp:59-76) on the device
        sync_ghosts(c);
        double* d = dense_staging(c);  // 6*ny*nx >= 2*nrows*ncols
        const size_t m = static_cast<size_t>(c->ncols) * c->nrows;
        const size_t off = static_cast<size_t>(c->row0) * c->ncols;
        ck(cudaMemcpyAsync(d, vx + off, sizeof(double) * m, cudaMemcpyHostToDevice, c->stream), "vx H2D");
        ck(cudaMemcpyAsync(d + m, vy + off, sizeof(double) * m, cudaMemcpyHostToDevice, c->stream), "vy H2D");
        ck(tpb::launch_init_velocity(c->g, c->dGeo, d, d + m, c->ncols, c->nrows, std::sqrt(c->p.g * c->p.L), c->dA,
                                     c->stream),
           "init_velocity_kernel");
        scan_flags_A(c);
        ck(cudaStreamSynchronize(c->stream), "sync");
        c->ghosts_in_B = false;
    })
}

int tp_set_hydrograph(tp_ctx* c, int n_cells, const int* ci, const int* cj, const char* side,
                      int n_samples, const double* t, const double* h, const double* phi_s,
                      const double* speed) {
    TP_GUARD(c, {
        // Hydrograph::validate (hydrograph.hpp:49-77), same messages
        for (int k = 1; k < n_samples; ++k)
            if (!(t[k] > t[k - 1]))
                throw ConfigErr{"hydrograph: sample times must be strictly increasing (t=" +
                                std::to_string(t[k]) + " after t=" + std::to_string(t[k - 1]) + ")"};
        for (int k = 0; k < n_samples; ++k) {
            if (h[k] < 0.0) throw ConfigErr{"hydrograph: negative thickness"};
            if (speed[k] < 0.0) throw ConfigErr{"hydrograph: negative speed"};
            if (phi_s[k] < 0.0 || phi_s[k] > 1.0) throw ConfigErr{"hydrograph: phi_s out of [0, 1]"};
        }
        for (int k = 0; k < n_cells; ++k) {
            bool ok = false;
            switch (side[k]) {
                case 'N': ok = cj[k] == c->nrows_g - 1; break;
                case 'S': ok = cj[k] == 0; break;
                case 'E': ok = ci[k] == c->ncols - 1; break;
                case 'W': ok = ci[k] == 0; break;
                default:
                    throw ConfigErr{std::string("hydrograph: unknown side '") + side[k] + "'"};
            }
            if (ci[k] < 0 || ci[k] >= c->ncols || cj[k] < 0 || cj[k] >= c->nrows_g) ok = false;
            if (!ok)
                throw ConfigErr{"hydrograph: cell (" + std::to_string(ci[k]) + ", " + std::to_string(cj[k]) +
                                ") is not on the boundary ring of side " + std::string(1, side[k])};
        }
        // ghost-band side map for bc_kernel (apply_boundaries inflow, solver.cpp:108-136)
        const long nband = (c->g.has_south ? 3L * c->nx : 0) + (c->g.has_north ? 3L * c->nx : 0) +
                           6L * (c->ny - 6);
        std::vector<signed char> map(static_cast<size_t>(nband), 0);
        std::vector<unsigned char> itiles(static_cast<size_t>(c->ntx) * c->nty, 0);
        for (int k = 0; k < n_cells; ++k) {
            int di = 0, dj = 0;
            switch (side[k]) {
                case 'E': di = 1; break;
                case 'W': di = -1; break;
                case 'N': dj = 1; break;
                case 'S': dj = -1; break;
            }
            const int pi = ci[k] + kGhost, pj = cj[k] + kGhost;
            for (int g = 1; g <= kGhost; ++g) {
                const int gi = pi + di * g;
                const int gj = pj + dj * g - c->row0;  // local padded row
                if (gj < 0 || gj >= c->ny) continue;
                // W/E ghosts of rows we do not own are the neighbours' (halo rows)
                if (dj == 0 && (gj < kGhost || gj >= c->ny - kGhost)) continue;
                const long b = band_index(c, gi, gj);
                if (b >= 0) map[static_cast<size_t>(b)] = static_cast<signed char>(side[k]);
                // tiles whose radius-2 box (padded X0-2 .. X0+TX+1, Y0-2 .. Y0+TY+1 with
                // X0 = 3 + tx*TX, Y0 = 3 + ty*TY) contains this ghost cell
                for (int ty = 0; ty < c->nty; ++ty) {
                    const int y0 = kGhost + ty * tpb::TY;
                    if (gj < y0 - 2 || gj > y0 + tpb::TY + 1) continue;
                    for (int tx = 0; tx < c->ntx; ++tx) {
                        const int x0 = kGhost + tx * tpb::TX;
                        if (gi >= x0 - 2 && gi <= x0 + tpb::TX + 1) itiles[static_cast<size_t>(ty) * c->ntx + tx] = 1;
                    }
                }
            }
        }
        cudaFree(c->dSide);
        cudaFree(c->dSamples);
        cudaFree(c->dInflowTiles);
        c->dSide = nullptr;
        c->dSamples = nullptr;
        c->dInflowTiles = nullptr;
        ck(cudaMalloc(&c->dInflowTiles, itiles.size()), "cudaMalloc inflow tiles");
        ck(cudaMemcpy(c->dInflowTiles, itiles.data(), itiles.size(), cudaMemcpyHostToDevice), "inflow tiles H2D");
        ck(cudaMalloc(&c->dSide, std::max<size_t>(1, map.size())), "cudaMalloc side map");
        if (!map.empty())
            ck(cudaMemcpy(c->dSide, map.data(), map.size(), cudaMemcpyHostToDevice), "side map H2D");
        std::vector<double> smp(4ull * std::max(1, n_samples), 0.0);
        for (int k = 0; k < n_samples; ++k) {
            smp[4 * k + 0] = t[k];
            smp[4 * k + 1] = h[k];
            smp[4 * k + 2] = phi_s[k];
            smp[4 * k + 3] = speed[k];
        }
        ck(cudaMalloc(&c->dSamples, sizeof(double) * smp.size()), "cudaMalloc samples");
        ck(cudaMemcpy(c->dSamples, smp.data(), sizeof(double) * smp.size(), cudaMemcpyHostToDevice),
           "samples H2D");
        c->n_samples = n_samples;
        c->hydro_set = true;
        c->inflow_active = c->p.mode == 1;  // cfg_.mode == InflowHydrograph && hydro_
        drop_graphs(c);
    })
}

int tp_get_state(tp_ctx* c, double* out) {
    TP_GUARD(c, {
        sync_ghosts(c);
        download_state(c, out, c->dA);
    })
}

int tp_set_state(tp_ctx* c, const double* in) {
    TP_GUARD(c, {
        upload_state(c, c->dA, in);
        scan_flags_A(c);
        ck(cudaStreamSynchronize(c->stream), "sync");
        c->ghosts_in_B = false;
    })
}

int tp_get_geometry(tp_ctx* c, double* out) {
    TP_GUARD(c, {
        ensure_geo_h(c);
        std::memcpy(out, c->geo_h.data(), sizeof(double) * c->geo_h.size());
    })
}

int tp_apply_boundaries(tp_ctx* c, double t_scaled) {
    TP_GUARD(c, {
        launch_bc(c, 0, 0, t_scaled, 0);
        ck(cudaStreamSynchronize(c->stream), "sync");
        c->ghosts_in_B = false;
    })
}

int tp_compute_dt(tp_ctx* c, double t_scaled, double t_next_scaled, double* dt) {
    TP_GUARD(c, {
        write_ctrl(c, t_scaled, t_next_scaled, INFINITY, 0.0, LLONG_MAX);
        fresh_lambda(c);
        ck(tpb::launch_dt(c->ph, c->dSc, 0, c->stream), "dt_kernel");
        DevScalars h = read_scalars(c);
        *dt = h.dt;
    })
}

int tp_advance_step(tp_ctx* c, double dt_scaled, double t_scaled) {
    TP_GUARD(c, {
        // Simulator::advance_step (solver.cpp:496-545)
        write_ctrl(c, t_scaled, t_scaled, INFINITY, dt_scaled, LLONG_MAX);
        ck(launch_stage_sel(c, stage_args(c, false, 0), c->fastdiv, false, c->stream), "predictor");
        launch_bc(c, 1, 2, 0.0, 0);
        ck(launch_stage_sel(c, stage_args(c, true, 0), c->fastdiv, true, c->stream), "corrector");
        launch_post(c, 0);
        c->lam_valid = false;
        c->ghosts_in_B = true;
        check_error(c, c->dB);
    })
}

int tp_regularize(tp_ctx* c) {
    TP_GUARD(c, {
        sync_ghosts(c);
        ck(tpb::launch_regularize(c->g, c->ph, c->dA, c->dGeo, c->dSc, c->fastdiv, c->stream),
           "regularize_kernel");
        scan_flags_A(c);
        check_error(c, c->dA);
    })
}

int tp_set_advection_only(tp_ctx* c, int on) {
    TP_GUARD(c, {
        c->adv_only = on ? 1 : 0;
        build_phys(c);
        drop_graphs(c);
        c->lam_valid = false;
    })
}

}  // extern "C"

namespace {

// tp_steps in pieces, so several contexts of one process (slabs connected by
// tp_peer_connect_local) can advance in lockstep: every member must launch the same
// graphs, because the graphs exchange with each other.
struct StepsRun {
    long long max_steps = 0;
    long long launched = 0;  // graph steps launched (sequence-number bookkeeping)
    DevScalars h{};
    bool finished = false;
    double* dts = nullptr;
    double t_next = 0.0;
};

void steps_begin(tp_ctx* c, StepsRun& r, double t, double t_next, double t_end, long max_steps, double* dts) {
    r.max_steps = max_steps;
    r.dts = dts;
    r.t_next = t_next < t_end ? t_next : t_end;
    r.h.t = t;
    r.h.steps = 0;
    c->launches = 0;
    if (dts && c->dts_cap < max_steps) {
        cudaFree(c->dDts);
        c->dDts = nullptr;
        ck(cudaMalloc(&c->dDts, sizeof(double) * max_steps), "cudaMalloc dts");
        c->dts_cap = max_steps;
    }
    double* dts_dev = dts ? c->dDts : nullptr;
    ck(cudaMemcpyAsync(&c->dSc->dts, &dts_dev, sizeof(double*), cudaMemcpyHostToDevice, c->stream), "dts ptr");
    write_ctrl(c, t, t_next, t_end, 0.0, max_steps);
    if (c->peered)
        ck(cudaMemcpyAsync(&c->dSc->peer_base, &c->peer_base, sizeof(c->peer_base), cudaMemcpyHostToDevice,
                           c->stream),
           "peer base");
    if (!c->lam_valid) {
        fresh_lambda(c);
        c->launches += 1;
    }
    if (c->graphK_steps != c->graph_steps) {
        drop_graphs(c);
        for (int w = 0; w < 2; ++w)
            for (int l = 0; (1 << l) <= c->graph_steps; ++l) c->graphs[w][l] = capture_steps(c, 1 << l, nullptr, w != 0);
        c->graphK_steps = c->graph_steps;
    }
    if (c->last_tiles_stage == 0) {  // the graphs start with a predictor list
        ck(cudaMemsetAsync(c->dNact, 0, sizeof(int), c->stream), "memset");
        ck(cudaMemsetAsync(c->dNact + 4, 0, sizeof(int), c->stream), "memset");
        ck(cudaMemsetAsync(c->dNact + 8, 0, sizeof(int), c->stream), "memset");
    }
    c->last_tiles_stage = 1;
}

// Steps to launch before the next poll: up to the output time at the last dt (+1 in case dt
// shrinks), at most graph_steps and the steps left.  A replay past a stop (output hit, t_end,
// error) runs no-op launches, so long graphs are only used when no output is near.
long steps_to_launch(const tp_ctx* c, const StepsRun& r) {
    long n = static_cast<long>(r.max_steps - r.h.steps);
    if (n > c->graph_steps) n = c->graph_steps;
    if (c->dt_hint > 0.0) {
        const double left = (r.t_next - r.h.t) / c->dt_hint;
        const double est = left > 0.0 ? std::ceil(left) + 1.0 : 1.0;
        if (est < static_cast<double>(n)) n = static_cast<long>(est);
    }
    return n < 1 ? 1 : n;
}

// n steps as back-to-back replays of the power-of-two graphs (largest first, one poll after)
void steps_launch(tp_ctx* c, StepsRun& r, long n) {
    for (int l = tp_ctx::kMaxGraphLog - 1; l >= 0; --l) {
        const long k = 1L << l;
        while (n >= k && c->graphs[0][l]) {
            ck(cudaGraphLaunch(c->graphs[c->wide ? 1 : 0][l], c->stream), "graph launch");
            // merged: 4 per step + the final post; peered: + lambda exchange + 2 halo pushes
            c->launches += merged_loop(c) ? 4L * k + 1L : (c->peered ? 8L : 5L) * k;
            r.launched += k;
            n -= k;
        }
    }
}

// the graph family of the next replay: wide stage CTAs (one tile per SM, one face per thread)
// while the last lists were short enough that every tile had an SM to itself
void choose_wide(tp_ctx* c, const DevScalars& h) {
    const int thr = c->wide_tiles >= 0 ? c->wide_tiles : c->num_sms;
    const int n = h.last_nact[0] > h.last_nact[1] ? h.last_nact[0] : h.last_nact[1];
    c->wide = n <= thr;
}

void steps_poll(tp_ctx* c, StepsRun& r) {
    r.h = read_scalars(c);
    r.finished = r.h.done != 0;
    if (r.h.steps > 0) {
        choose_wide(c, r.h);
        c->dt_hint = r.h.dt;
    }
}

// A device error key with the slab's local row replaced by the global row, so keys of
// different slabs order like the serial reference's loops (error keys: tp_kernels.cu).
unsigned long long global_error_key(const tp_ctx* c, unsigned long long key) {
    if (key == tpb::kNoError) return key;
    const unsigned long long cls = key >> 62;
    if (cls <= 1) {  // (cls << 62) | (j << 32) | (i << 1) | phase
        const unsigned long long j = ((key >> 32) & 0x3fffffffull) + static_cast<unsigned long long>(c->row0);
        return (cls << 62) | (j << 32) | (key & 0xffffffffull);
    }
    if (cls == 2) {  // (2 << 62) | (field << 56) | (j << 28) | i
        const unsigned long long j = ((key >> 28) & 0xfffffffull) + static_cast<unsigned long long>(c->row0);
        return (key & ~(0xfffffffull << 28)) | (j << 28);
    }
    return key;
}

void steps_end(tp_ctx* c, StepsRun& r, double* t, long* steps, int* hit) {
    const DevScalars& h = r.h;
    if (c->peered) c->peer_base += 4ull * static_cast<unsigned long long>(r.launched);
    *steps = static_cast<long>(h.steps);
    *t = h.t;
    *hit = h.steps > 0 ? h.hit : 0;
    c->lam_valid = h.steps > 0 || c->lam_valid;
    c->ghosts_in_B = c->ghosts_in_B || h.steps > 0;
    if (r.dts && h.steps > 0)
        ck(cudaMemcpy(r.dts, c->dDts, sizeof(double) * h.steps, cudaMemcpyDeviceToHost), "dts D2H");
    if (h.err_key != tpb::kNoError) {
        c->lam_valid = false;
        raise_error_key(c, h.err_key, c->dB);
    }
}

}  // namespace

extern "C" {

int tp_steps(tp_ctx* c, double t_next, double t_end, long max_steps, double* t, long* steps, int* hit,
             double* dts) {
    TP_GUARD(c, {
        *steps = 0;
        *hit = 0;
        c->launches = 0;
        if (max_steps <= 0 || !(*t < t_end)) return TP_OK;
        StepsRun r;
        steps_begin(c, r, *t, t_next, t_end, max_steps, dts);
        while (!r.finished) {
            steps_launch(c, r, steps_to_launch(c, r));
            steps_poll(c, r);
        }
        steps_end(c, r, t, steps, hit);
    })
}

int tp_steps_group(tp_ctx* const* cs, int n, double t_next, double t_end, long max_steps, double* t, long* steps,
                   int* hit) {
    tp_ctx* c0 = n > 0 ? cs[0] : nullptr;
    TP_GUARD(c0, {
        if (n <= 0) throw ConfigErr{"tp_steps_group: no contexts"};
        *steps = 0;
        *hit = 0;
        if (max_steps <= 0 || !(*t < t_end)) return TP_OK;
        std::vector<StepsRun> runs(static_cast<size_t>(n));
        for (int k = 0; k < n; ++k) {
            cudaSetDevice(cs[k]->device);
            steps_begin(cs[k], runs[k], *t, t_next, t_end, max_steps, nullptr);
        }
        for (;;) {
            // every member launches the same steps (member 0's estimate) before anyone waits
            const long ns = steps_to_launch(cs[0], runs[0]);
            for (int k = 0; k < n; ++k) {
                cudaSetDevice(cs[k]->device);
                steps_launch(cs[k], runs[k], ns);
            }
            bool any = false, all = true;
            for (int k = 0; k < n; ++k) {
                cudaSetDevice(cs[k]->device);
                steps_poll(cs[k], runs[k]);
                any = any || runs[k].finished;
                all = all && runs[k].finished;
            }
            if (any) {
                if (!all) throw CudaErr{"tp_steps_group: members stopped at different steps"};
                break;
            }
        }
        double tk = 0.0;
        long sk = 0;
        int hk = 0;
        // the error the serial reference throws first: smallest key in global row order
        int first = -1;
        unsigned long long best = tpb::kNoError;
        for (int k = 0; k < n; ++k) {
            const unsigned long long gk = global_error_key(cs[k], runs[k].h.err_key);
            if (gk < best) {
                best = gk;
                first = k;
            }
        }
        std::string err;
        for (int k = 0; k < n; ++k) {  // finish every member, then report the first error
            cudaSetDevice(cs[k]->device);
            try {
                steps_end(cs[k], runs[k], &tk, &sk, &hk);
            } catch (const NumErr& e) {
                if (k == first) err = e.msg;
            }
            if (k == 0) {
                *t = tk;
                *steps = sk;
                *hit = hk;
            }
        }
        cudaSetDevice(c0->device);
        if (!err.empty()) throw NumErr{err};
    })
}

// ---- device-resident slab exchange: connection ------------------------------------

namespace {
struct PeerBlob {  // what one rank publishes (TP_PEER_BLOB_BYTES, include/tpflow_b200.h)
    cudaIpcMemHandle_t state[2];
    cudaIpcMemHandle_t box;
    long long fs;
    int ny, row0, row1, nx, pad[2];
};
static_assert(sizeof(PeerBlob) <= TP_PEER_BLOB_BYTES, "peer blob too large");

void peer_check_layout(tp_ctx* c, int rank, int nranks) {
    if (nranks < 1 || nranks > tpb::kMaxRanks) throw ConfigErr{"peer: nranks must be in [1, 16]"};
    if (rank < 0 || rank >= nranks) throw ConfigErr{"peer: rank out of range"};
    (void)c;
}

void peer_finish(tp_ctx* c, int rank, int nranks) {
    c->link.rank = rank;
    c->link.nranks = nranks;
    c->link.my_box = c->dBox;
    {
        const char* e = std::getenv("TPFLOW_PEER_TIMEOUT_S");
        const double sec = e ? std::atof(e) : 60.0;
        c->link.timeout_ns = static_cast<unsigned long long>((sec > 0.0 ? sec : 60.0) * 1e9);
    }
    c->peered = nranks > 1;
    c->peer_base = 0;
    ck(cudaMemsetAsync(c->dBox, 0, sizeof(tpb::PeerBox), c->stream), "memset");
    ck(cudaStreamSynchronize(c->stream), "sync");
    drop_graphs(c);
}
}  // namespace

int tp_peer_export(tp_ctx* c, void* blob) {
    TP_GUARD(c, {
        PeerBlob b{};
        ck(cudaIpcGetMemHandle(&b.state[0], c->rawA), "ipc handle");
        ck(cudaIpcGetMemHandle(&b.state[1], c->rawB), "ipc handle");
        ck(cudaIpcGetMemHandle(&b.box, c->dBox), "ipc handle");
        b.fs = c->fs;
        b.ny = c->ny;
        b.row0 = c->row0;
        b.row1 = c->row1;
        b.nx = c->nx;
        std::memset(blob, 0, TP_PEER_BLOB_BYTES);
        std::memcpy(blob, &b, sizeof(b));
    })
}

int tp_peer_connect(tp_ctx* c, int rank, int nranks, const void* blobs) {
    TP_GUARD(c, {
        peer_check_layout(c, rank, nranks);
        const auto* B = static_cast<const unsigned char*>(blobs);
        auto blob = [&](int r) {
            PeerBlob b;
            std::memcpy(&b, B + static_cast<size_t>(r) * TP_PEER_BLOB_BYTES, sizeof(b));
            return b;
        };
        auto open = [&](const cudaIpcMemHandle_t& h) {
            void* p = nullptr;
            ck(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess), "ipc open");
            c->ipc_opened.push_back(p);
            return p;
        };
        tpb::PeerLink L{};
        for (int r = 0; r < nranks; ++r)
            L.box[r] = r == rank ? c->dBox : static_cast<tpb::PeerBox*>(open(blob(r).box));
        for (int side = 0; side < 2; ++side) {
            const int nb = side == 0 ? rank - 1 : rank + 1;
            if (nb < 0 || nb >= nranks) continue;
            const PeerBlob b = blob(nb);
            if (b.nx != c->nx || (side == 0 ? b.row1 != c->row0 : b.row0 != c->row1))
                throw ConfigErr{"peer: rank " + std::to_string(nb) + " is not the adjacent slab"};
            for (int buf = 0; buf < 2; ++buf)
                L.nbr_state[buf][side] = static_cast<double*>(open(b.state[buf])) + 1;  // + pad column
            L.nbr_fs[side] = b.fs;
            L.nbr_ny[side] = b.ny;
            L.nbr_box[side] = L.box[nb];
        }
        c->link = L;
        peer_finish(c, rank, nranks);
    })
}

int tp_peer_connect_local(tp_ctx* c, int rank, int nranks, tp_ctx* const* all) {
    TP_GUARD(c, {
        peer_check_layout(c, rank, nranks);
        tpb::PeerLink L{};
        // peer_lambda_kernel stores into every rank's mailbox, peer_halo_push_kernel into the
        // neighbours' state: peer access to every other device of the group
        c->stage_ctas = 0;
        int nshare = 0;  // members on this device, this one included
        for (int r = 0; r < nranks; ++r)
            if (all[r]->device == c->device) ++nshare;
        for (int r = 0; r < nranks; ++r) {
            L.box[r] = all[r]->dBox;
            if (r != rank && all[r]->device == c->device) {
                // members sharing this device run their kernels beside this one's stage kernel,
                // which may wait for their halo pushes: the members' stage grids together leave
                // 4 SMs to the small kernels (pre, halo push), so a push never waits for a stage
                // CTA that is itself waiting (with 3+ members, stage kernels of several members
                // could otherwise fill every SM)
                int sms = 148;
                cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
                c->stage_ctas = 2 * ((sms - 4) / nshare);
            }
            if (all[r]->device != c->device) {
                const cudaError_t e = cudaDeviceEnablePeerAccess(all[r]->device, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) ck(e, "peer access");
                cudaGetLastError();
            }
        }
        for (int side = 0; side < 2; ++side) {
            const int nb = side == 0 ? rank - 1 : rank + 1;
            if (nb < 0 || nb >= nranks) continue;
            const tp_ctx* o = all[nb];
            if (o->nx != c->nx || (side == 0 ? o->row1 != c->row0 : o->row0 != c->row1))
                throw ConfigErr{"peer: context " + std::to_string(nb) + " is not the adjacent slab"};
            L.nbr_state[0][side] = o->dA;
            L.nbr_state[1][side] = o->dB;
            L.nbr_fs[side] = o->fs;
            L.nbr_ny[side] = o->ny;
            L.nbr_box[side] = o->dBox;
        }
        c->link = L;
        peer_finish(c, rank, nranks);
    })
}

int tp_steps_timed(tp_ctx* c, double t_next, double t_end, long max_steps, double* t, long* steps, int* hit,
                   float* pred_ms, float* corr_ms) {
    TP_GUARD(c, {
        // tp_steps one step per graph replay, with CUDA events recorded (as external event
        // nodes of the graph, on the launching stream) right around the two stage kernels:
        // the kernels' device time in their production context
        *steps = 0;
        *hit = 0;
        *pred_ms = *corr_ms = 0.0f;
        c->launches = 0;
        if (max_steps <= 0 || !(*t < t_end)) return TP_OK;
        ck(cudaMemsetAsync(&c->dSc->dts, 0, sizeof(double*), c->stream), "dts null");
        write_ctrl(c, *t, t_next, t_end, 0.0, max_steps);
        if (!c->lam_valid) fresh_lambda(c);
        if (!c->evT[0])
            for (auto& e : c->evT) ck(cudaEventCreate(&e), "event");
        if (!c->graphT) c->graphT = capture_steps(c, 1, c->evT);
        if (c->last_tiles_stage == 0) {
            ck(cudaMemsetAsync(c->dNact, 0, sizeof(int), c->stream), "memset");
            ck(cudaMemsetAsync(c->dNact + 4, 0, sizeof(int), c->stream), "memset");
            ck(cudaMemsetAsync(c->dNact + 8, 0, sizeof(int), c->stream), "memset");
        }
        c->last_tiles_stage = 1;
        DevScalars h{};
        c->timed_tiles[0] = c->timed_tiles[1] = 0;
        for (;;) {
            ck(cudaGraphLaunch(c->graphT, c->stream), "graph launch");
            c->launches += 5;
            h = read_scalars(c);
            if (h.steps > *steps) {
                float a = 0.0f, b = 0.0f;
                ck(cudaEventElapsedTime(&a, c->evT[0], c->evT[1]), "elapsed");
                ck(cudaEventElapsedTime(&b, c->evT[2], c->evT[3]), "elapsed");
                *pred_ms += a;
                *corr_ms += b;
                *steps = static_cast<long>(h.steps);
                int n[2] = {0, 0};  // tiles the two stage launches of this step processed
                ck(cudaMemcpy(n, c->dNact + 2, sizeof(n), cudaMemcpyDeviceToHost), "tiles D2H");
                c->timed_tiles[0] += n[0];
                c->timed_tiles[1] += n[1];
            }
            if (h.done) break;
        }
        *t = h.t;
        *hit = h.steps > 0 ? h.hit : 0;
        c->lam_valid = h.steps > 0 || c->lam_valid;
        c->ghosts_in_B = c->ghosts_in_B || h.steps > 0;
        if (h.err_key != tpb::kNoError) {
            c->lam_valid = false;
            raise_error_key(c, h.err_key, c->dB);
        }
    })
}

int tp_get_audit(tp_ctx* c, double* a) {
    TP_GUARD(c, {
        DevScalars h = read_scalars(c);
        std::memcpy(a, h.audit, sizeof(h.audit));
    })
}

int tp_set_audit(tp_ctx* c, const double* a) {
    TP_GUARD(c, {
        ck(cudaMemcpyAsync(&c->dSc->audit, a, sizeof(double) * 10, cudaMemcpyHostToDevice, c->stream),
           "audit H2D");
        ck(cudaStreamSynchronize(c->stream), "sync");
    })
}

int tp_interior_mass(tp_ctx* c, double* ms, double* mf) {
    TP_GUARD(c, {
        // Simulator::interior_mass (solver.cpp:582-588): KahanSum (field.hpp:46-59) in (j, i) order
        std::vector<double> w(2ull * c->nx * c->ny);
        ck(cudaMemcpy2DAsync(w.data(), c->nx * sizeof(double), c->dA, c->pitch * sizeof(double),
                             c->nx * sizeof(double), 2ull * c->ny, cudaMemcpyDeviceToHost, c->stream),
           "mass D2H");
        ck(cudaStreamSynchronize(c->stream), "sync");
        for (int p = 0; p < 2; ++p) {
            double sum = 0.0, comp = 0.0;
            const double* f = w.data() + static_cast<size_t>(p) * c->nx * c->ny;
            for (int j = kGhost; j < c->ny - kGhost; ++j)
                for (int i = kGhost; i < c->nx - kGhost; ++i) {
                    double x = f[static_cast<size_t>(j) * c->nx + i];
                    double y = x - comp;
                    double t = sum + y;
                    comp = (t - sum) - y;
                    sum = t;
                }
            (p == 0 ? *ms : *mf) = sum * c->dxi * c->deta;
        }
    })
}

int tp_interior_mass_device(tp_ctx* c, double* ms, double* mf) {
    TP_GUARD(c, {
        const int blocks = 296;
        double* d = dense_staging(c);  // >= 4 * blocks doubles
        ck(tpb::launch_mass(c->g, c->dA, d, blocks, c->stream), "mass_kernel");
        std::vector<double> part(4ull * blocks);
        ck(cudaMemcpyAsync(part.data(), d, sizeof(double) * part.size(), cudaMemcpyDeviceToHost, c->stream),
           "mass D2H");
        ck(cudaStreamSynchronize(c->stream), "sync");
        for (int p = 0; p < 2; ++p) {
            double a = 0.0, e = 0.0;
            for (int b = 0; b < blocks; ++b) {  // block order, compensated
                const double x = part[(2 * b + p) * 2], y = a + x, bb = y - a;
                e += (a - (y - bb)) + (x - bb) + part[(2 * b + p) * 2 + 1];
                a = y;
            }
            (p == 0 ? *ms : *mf) = (a + e) * c->dxi * c->deta;
        }
    })
}

int tp_snapshot(tp_ctx* c, double* out) {
    TP_GUARD(c, {
        // Simulator::snapshot (solver.cpp:590-617) on the device (snapshot_kernel), then one
        // contiguous copy of the 6 interior fields
        double* d = dense_staging(c);  // 6*ny*nx >= 6*nrows*ncols
        const size_t m = static_cast<size_t>(c->ncols) * c->nrows;
        ck(tpb::launch_snapshot(c->g, c->dA, c->dGeo, d, c->ncols, c->nrows, c->p.H, c->p.h_dry, c->p.eps_h,
                                std::sqrt(c->p.g * c->p.L), c->stream),
           "snapshot_kernel");
        ck(cudaMemcpyAsync(out, d, sizeof(double) * 6 * m, cudaMemcpyDeviceToHost, c->stream), "snapshot D2H");
        ck(cudaStreamSynchronize(c->stream), "sync");
    })
}

// ---- multi-GPU slab plumbing ----------------------------------------------------

long tp_halo_bytes(const tp_ctx* c) { return 2L * 6L * c->nx * static_cast<long>(sizeof(double)); }

int tp_halo_pack(tp_ctx* c, int buf, int side, void* dst) {
    TP_GUARD(c, {
        if (buf == 0) sync_ghosts(c);
        const double* base = buf ? c->dB : c->dA;
        const int row = side == 0 ? kGhost : c->ny - kGhost - 2;  // our 2 edge interior rows
        for (int f = 0; f < 6; ++f)
            ck(cudaMemcpy2DAsync(static_cast<double*>(dst) + 2L * f * c->nx, c->nx * sizeof(double),
                                 base + f * c->fs + static_cast<long long>(row) * c->pitch,
                                 c->pitch * sizeof(double), c->nx * sizeof(double), 2,
                                 cudaMemcpyDeviceToDevice, c->stream),
               "halo pack");
    })
}

int tp_halo_unpack(tp_ctx* c, int buf, int side, const void* src) {
    TP_GUARD(c, {
        double* base = buf ? c->dB : c->dA;
        const int row = side == 0 ? kGhost - 2 : c->ny - kGhost;  // the 2 halo rows next to the interior
        for (int f = 0; f < 6; ++f)
            ck(cudaMemcpy2DAsync(base + f * c->fs + static_cast<long long>(row) * c->pitch,
                                 c->pitch * sizeof(double),
                                 static_cast<const double*>(src) + 2L * f * c->nx, c->nx * sizeof(double),
                                 c->nx * sizeof(double), 2, cudaMemcpyDeviceToDevice, c->stream),
               "halo unpack");
    })
}

int tp_step_begin(tp_ctx* c, double t, double t_next, double t_end) {
    TP_GUARD(c, {
        write_ctrl(c, t, t_next, t_end, 0.0, LLONG_MAX);
        c->t_next_last = t_next;
        ck(cudaMemsetAsync(&c->dSc->dts, 0, sizeof(double*), c->stream), "dts null");
    })
}

int tp_bc(tp_ctx* c, int buf) {
    TP_GUARD(c, {
        launch_bc(c, buf ? 1 : 0, buf ? 2 : 1, 0.0, 0);
        if (!buf) c->ghosts_in_B = false;
    })
}

int tp_lambda_local(tp_ctx* c, void* dst) {
    TP_GUARD(c, {
        if (!c->lam_valid) {
            ck(cudaMemsetAsync(&c->dSc->lam_bits, 0, sizeof(unsigned long long), c->stream), "memset");
            ck(tpb::launch_lambda(c->g, c->ph, c->dA, c->dGeo, c->dSc, c->fastdiv, c->stream),
               "lambda_kernel");
        }
        ck(cudaMemcpyAsync(dst, &c->dSc->lam_bits, sizeof(double), cudaMemcpyDeviceToDevice, c->stream),
           "lambda export");
    })
}

int tp_dt_from(tp_ctx* c, const void* lam) {
    TP_GUARD(c, {
        ck(cudaMemcpyAsync(&c->dSc->lam_cur, lam, sizeof(double), cudaMemcpyDeviceToDevice, c->stream),
           "lambda import");
        ck(tpb::launch_dt(c->ph, c->dSc, 0, c->stream), "dt_kernel");
    })
}

int tp_stage(tp_ctx* c, int corrector) {
    TP_GUARD(c, {
        ck(launch_stage_sel(c, stage_args(c, corrector != 0, 0), c->fastdiv, corrector != 0, c->stream),
           corrector ? "corrector" : "predictor");
        if (corrector) {
            c->lam_valid = true;  // lam_bits now holds the local lambda of u^{n+1}
            c->ghosts_in_B = true;
        }
    })
}

int tp_stage_timed(tp_ctx* c, int corrector, float* ms) {
    TP_GUARD(c, {
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        ck(cudaEventCreate(&e0), "event");
        ck(cudaEventCreate(&e1), "event");
        cudaError_t e = launch_stage_sel(c, stage_args(c, corrector != 0, 0), c->fastdiv, corrector != 0,
                                         c->stream, e0, e1);
        if (e == cudaSuccess) e = cudaEventSynchronize(e1);
        if (e == cudaSuccess) e = cudaEventElapsedTime(ms, e0, e1);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        ck(e, corrector ? "corrector" : "predictor");
        if (corrector) {
            c->lam_valid = true;
            c->ghosts_in_B = true;
        }
    })
}

int tp_step_end(tp_ctx* c, double* t, int* hit, double* dt) {
    TP_GUARD(c, {
        // clear a stale done flag so post_kernel runs its loop bookkeeping
        int zero = 0;
        ck(cudaMemcpyAsync(&c->dSc->done, &zero, sizeof(int), cudaMemcpyHostToDevice, c->stream), "done");
        launch_post(c, 1);
        DevScalars h = read_scalars(c);
        *t = h.t;
        *hit = h.hit;
        *dt = h.dt;
        if (h.err_key != tpb::kNoError) {
            c->lam_valid = false;
            raise_error_key(c, h.err_key, c->dB);
        }
    })
}

int tp_set_stream(tp_ctx* c, void* s) {
    TP_GUARD(c, {
        ck(cudaStreamSynchronize(c->stream), "sync");
        if (c->own_stream) cudaStreamDestroy(c->stream);
        c->stream = static_cast<cudaStream_t>(s);
        c->own_stream = false;
        drop_graphs(c);
    })
}

int tp_synchronize(tp_ctx* c) { TP_GUARD(c, ck(cudaStreamSynchronize(c->stream), "sync")) }

int tp_device_state(tp_ctx* c, int buf, void** ptr, long* pitch, long* field_stride) {
    if (!c) return TP_ERR_INTERNAL;
    try {
        invalidate_flags(c, buf == 0, buf != 0);  // the caller may write through the pointer
    } catch (...) {
        return TP_ERR_CUDA;
    }
    *ptr = buf ? c->dB : c->dA;
    *pitch = c->pitch;
    *field_stride = static_cast<long>(c->fs);
    return TP_OK;
}

int tp_selftest_division(int device, long n, unsigned long long seed, unsigned long long* mismatches) {
    if (cudaSetDevice(device) != cudaSuccess) return TP_ERR_CUDA;
    return tpb::selftest_division(n, seed, mismatches) == cudaSuccess ? TP_OK : TP_ERR_CUDA;
}

int tp_selftest_minmod(int device, long n, const double* a, const double* b, double* out) {
    if (n <= 0 || !a || !b || !out) return TP_ERR_INTERNAL;
    if (cudaSetDevice(device) != cudaSuccess) return TP_ERR_CUDA;
    return tpb::selftest_minmod(n, a, b, out) == cudaSuccess ? TP_OK : TP_ERR_CUDA;
}

int tp_safe_tiles(tp_ctx* c, int* corr) {
    TP_GUARD(c, {
        ck(cudaMemcpyAsync(corr, c->dNact + 5, sizeof(int), cudaMemcpyDeviceToHost, c->stream), "tiles D2H");
        ck(cudaStreamSynchronize(c->stream), "sync");
    })
}

int tp_cond_skipped_tiles(tp_ctx* c, unsigned long long* n) {
    TP_GUARD(c, { *n = read_scalars(c).cond_skips; })
}

int tp_timed_tiles(tp_ctx* c, long long* pred, long long* corr) {
    TP_GUARD(c, {
        *pred = c->timed_tiles[0];
        *corr = c->timed_tiles[1];
    })
}

int tp_active_tiles(tp_ctx* c, int* pred, int* corr, int* total) {
    TP_GUARD(c, {
        int n[2] = {0, 0};
        ck(cudaMemcpyAsync(n, c->dNact + 2, sizeof(n), cudaMemcpyDeviceToHost, c->stream), "tiles D2H");
        ck(cudaStreamSynchronize(c->stream), "sync");
        *pred = n[0];
        *corr = n[1];
        *total = c->ntx * c->nty;
    })
}

int tp_debug_phase_cycles(unsigned long long* out, int reset) {
    return tpb::phase_cycles(out, reset) == cudaSuccess ? TP_OK : TP_ERR_CUDA;
}

long tp_kernel_launches(const tp_ctx* c) { return c ? c->launches : 0; }

}  // extern "C"
