// Plain data structures shared by the kernels (nvcc) and the host library (g++).
// No device code here: this header is included by tp_capi.cpp.
#pragma once

#include <cuda.h>

#include <cstdint>

namespace tpb {

struct Phys {
    // model constants (params.hpp:29-51, config.hpp:18-22), host-evaluated once
    double eps;        // ScalingConfig::epsilon()
    double alpha;      // alpha_rho
    double oma;        // 1.0 - alpha_rho
    double C_d, N_R, theta_b;
    double eps_chi;    // std::pow(eps, chi)          (physics.hpp:60, solver.cpp:470)
    double tan_d;      // params.tan_delta_b()        (params.hpp:38)
    double neg_eps_alpha;  // -eps * alpha_rho         (physics.hpp:147)
    double eps_NR;     // eps * N_R                   (physics.hpp:115)
    double h_dry, eps_h;
    double eps_h2;     // RN(eps_h * eps_h): max(h, eps_h)^2 of the desingularisation is this or h*h
    double dxi, deta, two_dxi, two_deta;
    double cell_area;  // dxi * deta                  (solver.cpp:140)
    double cfl;
    // RN(1/x) of the constant divisors (FASTDIV)
    double r_dxi, r_deta, r_two_dxi, r_two_deta, r_eps_NR, r_NR;
    // FASTDIV divisor window of the four grid constants (mkrcp_const's test, evaluated once)
    int ok_dxi, ok_deta, ok_two_dxi, ok_two_deta;
    int adv_only;      // Simulator::set_advection_only (solver.hpp:60-62)
    int cap_on;        // !(adv_only || tan_delta_b() == 0.0)  (solver.cpp:454)
};


// Host/API geometry order = TerrainGeometry declaration order (terrain.hpp:59-63).
enum RefGeoField {
    R_NX = 0, R_NY, R_NZ, R_JB, R_A11, R_A12, R_A21, R_A22,
    R_DNX_DXI, R_DNY_DXI, R_DNZ_DXI, R_DNX_DETA, R_DNY_DETA, R_DNZ_DETA, R_COUNT
};
// Device geometry layout: the reference's 14 fields regrouped so that the fields
// every stencil point needs form one contiguous TMA box (the first NGBOX), plus
// four host-derived reciprocals RN(1/x) of the geometric divisors (the shared
// reciprocals of the FASTDIV division, see tp_math.cuh).
enum GeoField {
    G_JB = 0, G_RJB, G_NZ, G_A11, G_A12, G_A21, G_A22,
    G_RJBFX,   // RN(1 / (0.5 * (jb(i,j) + jb(i+1,j))))  xi-face jbf (solver.cpp:242)
    G_RJBFY,   // RN(1 / (0.5 * (jb(i,j) + jb(i,j+1))))  eta-face jbf
    G_NX, G_NY, G_DNX_DXI, G_DNY_DXI, G_DNZ_DXI, G_DNX_DETA, G_DNY_DETA, G_DNZ_DETA,
    G_RNZ,     // RN(1 / nZ)
    G_COUNT
};
constexpr int NGBOX = 9;   // G_JB .. G_RJBFY staged per tile box by TMA
// State field order = MixtureState::fields() (state.hpp:29).
enum StateField { S_WS = 0, S_WF, S_QSX, S_QSY, S_QFX, S_QFY, S_COUNT };

constexpr unsigned long long kNoError = ~0ull;

// Clipped-mass audit events of regularize (solver.cpp:139-166): the reference adds
// -w * cell_area to audit.clipped cell by cell in (j, i) order, predictor then corrector.
// The stage kernels append (key, value) events here; post_kernel (and the standalone
// regularize's fold) sorts them by key and adds them in that order, so the audit is the
// reference's sum bit for bit.  key = (stage << 62) | (j << 32) | (i << 1) | phase.
// Past kClipCap events per fold the rest are added with atomics (order not reproduced).
constexpr int kClipCap = 8192;
struct ClipList {
    int n;                               // events appended since the last fold
    int overflow;                        // events added directly (cumulative, diagnostics)
    unsigned long long key[kClipCap];
    double val[kClipCap];
    int order[kClipCap];                 // fold scratch: event index by rank
};

// Device-resident step scalars: the time loop of Simulator::run
// (solver.cpp:637-649) lives here so the host never waits on dt.
struct DevScalars {
    double t;        // scaled time
    double t_next;   // target of this tp_steps call (min(next_out, t_end))
    double t_end;    // loop bound (solver.cpp:637)
    double dt;       // dt of the step in flight
    long long steps;
    long long max_steps;
    int done;        // stop flag: every loop kernel returns immediately when set
    int hit;         // exact_hit of the step in flight (solver.cpp:641)
    // Mode-II inflow ghosts of the [predictor, corrector] stage in flight are inside the
    // safe-tile window (inflow_window_ok): their tiles may take the safe forms.  Cleared by
    // every write_ctrl (the first predictor of a tp_steps call keeps the checked forms).
    int inflow_safe[2];
    unsigned long long lam_bits;  // atomicMax accumulator of lambda (bits of a double >= 0)
    unsigned long long lam_cur;   // lambda_max of the current state (compute_dt input)
    unsigned long long err_key;   // earliest error (see error keys in tp_kernels.cu)
    double audit[10];             // solid {initial, final, injected, outflow, clipped}, fluid {...}
    double* dts;                  // optional per-step dt record (device)
    unsigned long long peer_base; // sequence base of the slab exchange (tp_peer.cu)
    unsigned long long cond_skips;  // conditional tiles dropped by stage_kernel<PEER> (cumulative)
    ClipList* clip;               // regularize's clipped-mass events (see ClipList)
    int last_nact[2];             // tiles listed for the last predictor / corrector launch
    // ring-tally epoch: a stage stamps each ring tile's tally slot it writes with
    // 2 * epoch + 1 + stage; post folds the slots carrying this step's stamps, then advances it
    // (monotonic: write_ctrl never resets it, so a slot from an earlier call never matches)
    unsigned tally_epoch;
    // the step in flight as the corrector sees it at its start (device loop): the time and step
    // count after it and whether the loop stops after it for any reason but an error; read by
    // prepost_kernel's pre blocks, which must not read t / steps / hit (its post block rewrites them)
    double t_after;
    long long steps_after;
    int stop_after;
    // Hydrograph::at (sh, sphi, sspeed) at the [predictor, corrector] stage's bc time, evaluated
    // once by the kernel before that stage's bc (corrector end / compute_dt) and read by every
    // inflow ghost thread of the bc (BcArgs::tsrc 3) instead of each one scanning the samples
    double inflow_val[2][3];
};

struct GridDesc {
    int nx, ny;       // padded dims of this (slab of the) grid
    int pitch;        // row pitch in doubles
    long long fs;     // field stride in doubles
    int has_south, has_north;  // physical S/N boundaries (always 1 on a single device)
};

struct Inflow {
    int n_samples;
    const double* samples;  // [n][4] t, h, phi_s, speed (physical units)
    const signed char* ghost_side;  // per ghost-band index: 0 or 'E','W','N','S'
    double t_unit, H, v_unit;
    int active;
};

// Stage kernel tile: TX x TY interior cells, NT threads.  TX*TY*2 + TX + TY = 511
// faces <= 2 * NT, so the face work of a tile is exactly two rounds.
constexpr int TX = 16;
#ifndef TP_TY
#define TP_TY 15
#endif
constexpr int TY = TP_TY;
constexpr int NT = 256;
constexpr int W2 = TX + 4;
constexpr int H2 = TY + 4;
constexpr int BOX = W2 * H2;
constexpr int NFX = (TX + 1) * TY;
constexpr int NFY = TX * (TY + 1);

struct StageArgs {
    CUtensorMap tm_s;                // TMA descriptor of the stage input state (6 fields)
    CUtensorMap tm_g;                // TMA descriptor of the NGBOX box geometry fields
    CUtensorMap tm_c;                // TMA descriptor of the per-cell geometry fields (G_NX..G_RNZ), tile box
    CUtensorMap tm_u;                // corrector: TMA descriptor of u^n (6 fields), interior tile box
    GridDesc g;
    Phys ph;
    const double* __restrict__ s;    // stage input state (6 fields, ghosts filled)
    const double* __restrict__ u0;   // corrector: u^n (interior read at own cell only)
    double* out;                     // stage output state (interior written)
    const double* __restrict__ geo;  // 14 geometry fields
    DevScalars* sc;
    double* tally;                   // per-tile boundary mass tally [ntiles][4] (ring tiles)
    unsigned* tally_stamp;           // [ntiles]: 2 * epoch + 1 + stage of the slot's last write
    int ntx, nty;
    int loop;                        // 1 = obey sc->done (device-resident loop)
    int use_sc_dt;                   // read dt from sc (always 1 in practice)
    // active-tile list of this stage (TileArgs below); tiles not listed are bitwise no-ops
    const int* __restrict__ tiles;   // [ntiles] entries (tile row << 16) | tile column, count in *ntiles_active
    const int* ntiles_active;
    unsigned short* flag_out;        // per-tile TileFlag bits of `out` (nonzero bits per region)
    int* nact_stat;                  // [2] list length of the last predictor / corrector launch
    int* work;                       // dynamic tile scheduler counter of this stage (zeroed by tiles_kernel)
    int max_ctas;                    // grid cap (peer groups sharing one device leave SMs to the others)
    // Peer-joined slabs (stage_kernel<..., PEER = true>, tp_peer.cu): the listed tiles whose box
    // reads halo rows, and the conditional ones (kTileCond: bitwise no-ops unless the pushed rows
    // are nonzero in their columns), sit at the BACK of `tiles` (tiles[ntx*nty-1-k], k < *nback).
    // They are claimed after every other tile; the claiming thread waits for the neighbours'
    // halo rows of this stage first (halo_seq), so the NVLink transfer overlaps interior tiles.
    const int* nback;
    const unsigned long long* halo_seq[2];  // this slab's mailbox slots for the stage's buffer [side 0 = south]
    const unsigned int* halo_nz[2];         // [tile column] the pushed rows hold a bit other than +0.0
    int has_nbr[2];
    int nyi;                                // interior rows of this slab
    int peer_phase;                         // 1 + buffer: the stage's sequence-number phase (tp_peer.cu)
    unsigned long long timeout_ns;
    Inflow inflow;                          // corrector (device loop): the next predictor's inflow-window test
};

// Per-tile output flags: which regions of the tile's interior hold a value with a nonzero
// bit (the 2-cell bands and 2x2 corners are what a neighbour's radius-2 box reads).
// TF_UNSAFE2: some output value is neither +-0 nor of magnitude in [2^-100, 2^100), or a
// thickness is negative or -0 (the "safe tile" window, DESIGN.md §3 item 6).
enum TileFlag : unsigned {
    TF_ANY = 1u, TF_W = 2u, TF_E = 4u, TF_S = 8u, TF_N = 16u,
    TF_SW = 32u, TF_SE = 64u, TF_NW = 128u, TF_NE = 256u, TF_UNSAFE2 = 1024u,
    TF_ALL = 0xffffu
};
// list-entry bit: every state value the tile's box reads is +-0 or in the safe window
// (entries: tile column in bits 0-15, tile row in bits 16-28)
constexpr int kTileSafe = 1 << 30;
// list-entry bit (peer-joined slabs): a conditional tile (see StageArgs::nback)
constexpr int kTileCond = 1 << 29;
// A tile of a peer-joined slab that is a bitwise no-op except that its box reads halo rows
// is listed with kTileCond; stage_kernel<PEER> processes it only if the neighbour's pushed
// rows hold a bit other than +0.0 in its box columns (PeerBox::halo_nz, tp_peer.cu).
constexpr int kMaxTileCols = 2048;  // halo_nz entries per side (wider slabs list such tiles unconditionally)

// Dry-tile classification before a stage.  flag_in: per-tile flags of the stage's input
// buffer (the radius-2 box reads interior cells of the tile and the facing bands/corners
// of its 8 neighbours only); flag_out: flags of its output buffer.  A tile whose box
// and whose own output are all +0.0 bits is a bitwise no-op: it is left
// off the list (its ring tally slot keeps an old stamp, so post does not fold it).  Flags are conservative: all bits
// set = unknown.
struct TileArgs {
    const unsigned short* flag_in;
    const unsigned short* flag_out;
    int* tiles;
    int* ntiles_active;   // this stage's counter (zeroed by the other stage's tiles_kernel);
                          // [4] past it: this stage's safe-tile count
    int* ntiles_reset;    // the other stage's counter
    int* work;            // this stage's dynamic tile scheduler counter (zeroed here)
    int ntx, nty;
    int nxi, nyi;         // interior columns / rows of this context (a tile's box may reach the ghost band
                          // or the halo rows without being an edge tile: a last tile of one column / row)
    int skip;             // 0 = list every tile
    int ring_ineligible;  // 1 = ring tiles read ghosts not refreshed as copies (outside the device loop)
    const unsigned char* inflow_tiles;  // per tile: its box reads a Mode-II inflow ghost (never skip, never safe); may be null
    int south_ineligible, north_ineligible;  // slab edges next to halo rows: never skip
    int safe_ok;          // FASTDIV on, geometry and constants inside the safe-window bounds (tp_capi.cpp)
    int stage;            // 0 predictor, 1 corrector (DevScalars::inflow_safe index)
    int cond_halo;        // peer-joined slab: tiles whose box reads halo rows go to the back of `tiles`
                          // (StageArgs::nback), flagged kTileCond when otherwise a no-op
    int* nback;           // this stage's back-region count (zeroed by the other stage's tiles_kernel)
    int* nback_reset;     // the other stage's
    int loop;
    DevScalars* sc;
};

struct BcArgs {
    GridDesc g;
    double* s;
    const double* __restrict__ geo;
    Inflow inflow;
    DevScalars* sc;
    double t;       // used when tsrc == 0
    int tsrc;       // 0: t argument, 1: sc->t, 2: sc->t + sc->dt, 3: sc->inflow_val[stage]
    int stage;      // tsrc 3: 0 predictor, 1 corrector
    int loop;
};

// bc + tile list (+ dt before the predictor) of one device-loop stage in one launch
struct PreArgs {
    BcArgs bc;
    TileArgs t;
    Phys P;
    int nb_bc;    // blocks of the ghost band (bc_body); the tile blocks follow
    int with_dt;  // predictor: compute_dt's tail in block 0
};

struct PostArgs {
    DevScalars* sc;
    const double* tally_pred;
    const double* tally_corr;
    const unsigned* stamp_pred;   // DevScalars::tally_epoch stamps of the two tallies
    const unsigned* stamp_corr;
    int ntx, nty;
    int loop;
    int peered;   // slabs joined by tp_peer_connect*: a local error stops the loop through the
                  // next step's stop-flag exchange (peer_lambda_kernel), on every rank at once
};

// post of one step + pre of the next predictor in one launch (device loop, unpeered): the last
// block runs post_kernel's work and compute_dt, the others bc + the predictor's list
struct PrePostArgs {
    PreArgs pre;
    PostArgs post;
};


// ---- device-resident row-slab exchange (tp_peer.cu) ----------------------------
constexpr int kMaxRanks = 16;
// Per-context mailbox in device memory (exported by CUDA IPC across processes): the
// neighbours write halo-arrival sequence numbers, every rank writes its lambda slot.
struct PeerBox {
    unsigned long long halo_seq[2][2];          // [buf A/B][side 0 = from south, 1 = from north]
    // lambda / stop slots by step parity: a rank can run at most one step ahead of any
    // reader (its step-n+1 exchange waits for every rank's step-n+1 write, which each rank
    // makes only after reading its step-n slots), so two slots never collide
    unsigned long long lam_seq[2][kMaxRanks];   // [step & 1][rank] sequence of lam_val/stop_val
    unsigned long long lam_val[2][kMaxRanks];   // bits of the rank's local lambda (>= 0)
    unsigned long long stop_val[2][kMaxRanks];  // 1 if the rank stopped (error)
    unsigned int push_done[2][2];               // local: CTAs finished pushing [buf][side]
    unsigned int pad[4];
    // [buf][side][tile column]: 1 if the 2 pushed rows hold a bit other than +0.0 within the
    // columns tile tx's box reads (X0-2 .. X0+TX+1); written before halo_seq is released
    unsigned int halo_nz[2][2][kMaxTileCols];
};
// Where this slab's neighbours live (pointers valid in this process: own allocations,
// allocations of contexts in this process, or CUDA-IPC mappings of other processes').
struct PeerLink {
    double* nbr_state[2][2];     // [buf A/B][side 0 = rank-1 (south), 1 = rank+1 (north)]; null = none
    long long nbr_fs[2];
    int nbr_ny[2];
    PeerBox* nbr_box[2];
    PeerBox* box[kMaxRanks];     // every rank's mailbox (lambda all-reduce)
    PeerBox* my_box;
    int rank, nranks;
    unsigned long long timeout_ns;  // a wait without progress this long reports an error (TPFLOW_PEER_TIMEOUT_S, default 60)
};

}  // namespace tpb
