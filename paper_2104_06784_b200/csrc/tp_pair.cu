// stage_pair_kernel<FD, CORR>: the fused Heun stage with every face and every
// cell split across a lane PAIR — the even lane carries the solid phase
// (ws, qsx, qsy), the odd lane the fluid phase (wf, qfx, qfy).  Same tiles, same
// TMA staging and the same shared-memory carve-up as stage_kernel
// (tp_kernels.cu).  Each thread holds half a face's state and its dependent FP64
// chains are half as long; the hope was twice the resident warps, but the
// kernel's natural register demand stays ~124, so at this smem budget it runs
// 2 CTAs x 8 warps like stage_kernel and measures slower on fully wet tiles
// (profiles/).  Kept as option "kernel"=3 and tested.  The two lanes
// exchange only what couples the phases (h_s/h_f for h_total and the dry test,
// the two wave speeds for the KT coefficient `a`, the new thicknesses for lambda)
// with pair-masked shuffles; every value is computed with the reference's
// expression tree, so results are bit-identical to stage_kernel and to the
// reference (tests/test_gpu_parity.py runs both kernels).
#include <cuda_runtime.h>

#include "tp_math.cuh"
#include "tp_stage_common.cuh"
#include "tp_types.h"

namespace tpb {

constexpr int NTP = 512;  // threads per CTA of the pair kernel
constexpr int NPAIR = NTP / 2;
static_assert(NPAIR >= TX * TY, "Phase 3 maps one lane pair to each tile cell");

__device__ __forceinline__ double pshfl(unsigned pm, double v) { return __shfl_xor_sync(pm, v, 1); }

// One half (phase p) of the KT face flux of solver.cpp:239-316.  k = box index
// of the left/lower cell, d = 1 (xi) or W2 (eta).  o = {mass, x-momentum,
// y-momentum} fluxes of phase p.
template <bool FD, bool XI>
__device__ __forceinline__ void face_half(const int p, const unsigned pm, const double* __restrict__ S,
                                          const double* __restrict__ G, const int k, const Phys& P,
                                          double (&o)[3]) {
    constexpr int d = XI ? 1 : W2;
    const double* Sw = S + p * BOX;
    const double* Sx = S + (2 + 2 * p) * BOX;
    const double* Sy = S + (3 + 2 * p) * BOX;
    // solver.cpp:229-263: edges of the own phase's three fields
    const double Lw = edge_plus(Sw[k - d], Sw[k], Sw[k + d]);
    const double Rw = edge_minus(Sw[k], Sw[k + d], Sw[k + 2 * d]);
    const double Lx = edge_plus(Sx[k - d], Sx[k], Sx[k + d]);
    const double Rx = edge_minus(Sx[k], Sx[k + d], Sx[k + 2 * d]);
    const double Ly = edge_plus(Sy[k - d], Sy[k], Sy[k + d]);
    const double Ry = edge_minus(Sy[k], Sy[k + d], Sy[k + 2 * d]);
    const double Lqn = XI ? Lx : Ly, Lqt = XI ? Ly : Lx;
    const double Rqn = XI ? Rx : Ry, Rqt = XI ? Ry : Rx;
    // solver.cpp:242-245
    const double jbf = 0.5 * (G[G_JB * BOX + k] + G[G_JB * BOX + k + d]);
    const double cf = 0.5 * (G[G_NZ * BOX + k] + G[G_NZ * BOX + k + d]);
    const int gnn = XI ? G_A11 : G_A22, gnt = XI ? G_A12 : G_A21;
    const double ann = 0.5 * (G[gnn * BOX + k] + G[gnn * BOX + k + d]);
    const double ant = 0.5 * (G[gnt * BOX + k] + G[gnt * BOX + k + d]);
    const Rcp rj = mkrcp_const<FD>(jbf, G[(XI ? G_RJBFX : G_RJBFY) * BOX + k]);
    bool ok = rj.ok;
    double hL = dq<FD>(Lw, rj, ok), hR = dq<FD>(Rw, rj, ok);
    double jL = dq<FD>(Lqn, rj, ok), jR = dq<FD>(Rqn, rj, ok);
    if (!ok) {
        dfix<FD>(hL, Lw, rj);
        dfix<FD>(hR, Rw, rj);
        dfix<FD>(jL, Lqn, rj);
        dfix<FD>(jR, Rqn, rj);
    }
    // solver.cpp:265-275 (h_total = hL[0] + hL[1] in the reference's order)
    const double hLo = pshfl(pm, hL), hRo = pshfl(pm, hR);
    const double htL = p ? hLo + hL : hL + hLo;
    const double htR = p ? hRo + hR : hR + hRo;
    if (htL < P.h_dry && htR < P.h_dry) {  // same outcome on both lanes of the pair
        o[0] = o[1] = o[2] = 0.0;
        return;
    }
    // solver.cpp:277-285: even lane celL, odd lane celR, exchanged
    const double cel_own = sqrt(P.eps * cf * smax(p ? htR : htL, 0.0));
    const double cel_oth = pshfl(pm, cel_own);
    const double celL = p ? cel_oth : cel_own;
    const double celR = p ? cel_own : cel_oth;
    const double dL = smax(hL, 0.0), dR = smax(hR, 0.0);
    double fL, fR;
    if (FD) {
        bool okf = true;
        fL = desing_factor_g(dL, P.eps_h, okf);
        fR = desing_factor_g(dR, P.eps_h, okf);
        if (!okf) {
            fL = desing_factor<FD>(dL, P.eps_h);
            fR = desing_factor<FD>(dR, P.eps_h);
        }
    } else {
        fL = desing_factor<FD>(dL, P.eps_h);
        fR = desing_factor<FD>(dR, P.eps_h);
    }
    const double vnL = jL * fL, vnR = jR * fR;
    // a = max(max(0, m_solid), m_fluid) exactly as the reference's loop over p
    const double m_own = smax(fabs(vnL) + celL, fabs(vnR) + celR);
    const double m_oth = pshfl(pm, m_own);
    const double a = smax(smax(0.0, p ? m_oth : m_own), p ? m_own : m_oth);
    // solver.cpp:288-296
    double prL = 0.0, prR = 0.0;
    if (!P.adv_only) {
        if (p == 0) {
            prL = cf * P.oma * hL * 0.5;
            prR = cf * P.oma * hR * 0.5;
        } else {
            prL = cf * htL * 0.5;
            prR = cf * htR * 0.5;
        }
    }
    // physics::directional_flux (physics.hpp:84-95) + solver.cpp:298-315
    const double ejL = P.eps * jbf * htL;
    const double ejR = P.eps * jbf * htR;
    const double ha = 0.5 * a;
    const double flm = Lw * vnL, frm = Rw * vnR;
    const double fln = Lqn * vnL + ejL * ann * prL;
    const double frn = Rqn * vnR + ejR * ann * prR;
    const double flt = Lqt * vnL + ejL * ant * prL;
    const double frt = Rqt * vnR + ejR * ant * prR;
    o[0] = 0.5 * (flm + frm) - ha * (Rw - Lw);
    const double momn = 0.5 * (fln + frn) - ha * (Rqn - Lqn);
    const double momt = 0.5 * (flt + frt) - ha * (Rqt - Lqt);
    o[1] = XI ? momn : momt;
    o[2] = XI ? momt : momn;
}

// regularize (solver.cpp:139-166) of phase p + [check_finite (:482-494) of its
// three fields + lambda (:556-573) of the cell] + store, on a lane pair.
template <bool FD, bool CORR>
__device__ __forceinline__ void pair_epilogue(const int p, const unsigned pm, double (&un)[3], const Rcp& rj,
                                              double nZ, int X, int Y, const Phys& P, DevScalars* sc,
                                              double& lam_local, double* out, long long fs, long long o3) {
    bool okr = rj.ok;
    double hp = dq<FD>(un[0], rj, okr);
    if (!okr) dfix<FD>(hp, un[0], rj);
    if (hp < 0.0) {
        if (hp < -1e-12) {
            const unsigned long long key = (static_cast<unsigned long long>(CORR ? 1 : 0) << 62) |
                                           (static_cast<unsigned long long>(Y) << 32) |
                                           (static_cast<unsigned long long>(X) << 1) |
                                           static_cast<unsigned long long>(p);
            atomicMin(&sc->err_key, key);
        } else {
            atomicAdd(&sc->audit[5 * p + 4], -un[0] * P.cell_area);
            un[0] = 0.0;
            hp = 0.0;
        }
    }
    if (!(hp < 0.0) && hp < P.h_dry) {
        un[1] = 0.0;
        un[2] = 0.0;
    }
    if (CORR) {
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            if (!isfinite(un[q])) {
                const int f = q == 0 ? p : 1 + 2 * p + q;  // ws,wf,qsx,qsy,qfx,qfy
                const unsigned long long key = (2ull << 62) | (static_cast<unsigned long long>(f) << 56) |
                                               (static_cast<unsigned long long>(Y) << 28) |
                                               static_cast<unsigned long long>(X);
                atomicMin(&sc->err_key, key);
            }
        }
        // lambda of the new state: hp is exactly w_new / jb (0 after a clip)
        bool okl = rj.ok;
        double jx = dq<FD>(un[1], rj, okl), jy = dq<FD>(un[2], rj, okl);
        if (!okl) {
            dfix<FD>(jx, un[1], rj);
            dfix<FD>(jy, un[2], rj);
        }
        double f;
        if (FD) {
            bool okf = true;
            f = desing_factor_g(hp, P.eps_h, okf);
            if (!okf) f = desing_factor<FD>(hp, P.eps_h);
        } else {
            f = desing_factor<FD>(hp, P.eps_h);
        }
        const double ax = fabs(jx * f), ay = fabs(jy * f);
        const double ho = pshfl(pm, hp), axo = pshfl(pm, ax), ayo = pshfl(pm, ay);
        const double h = p ? ho + hp : hp + ho;
        if (!(h < P.h_dry)) {
            const double cel = sqrt(P.eps * nZ * h);
            const double lx = smax(p ? axo : ax, p ? ax : axo) + cel;
            const double ly = smax(p ? ayo : ay, p ? ay : ayo) + cel;
            lam_local = smax(lam_local, smax(lx, ly));
        }
    }
    out[p * fs + o3] = un[0];
    out[(2 + 2 * p) * fs + o3] = un[1];
    out[(3 + 2 * p) * fs + o3] = un[2];
}

template <bool FD, bool CORR>
__global__ void __launch_bounds__(NTP, 2) stage_pair_kernel(const __grid_constant__ StageArgs A) {
    extern __shared__ __align__(128) double sm[];
    __shared__ unsigned long long bar;
    double* S = sm + SM_S;
    const double* G = sm + SM_G;
    double* V = sm + SM_V;
    double* PJ = sm + SM_PJ;
    double* BR = sm + SM_BR;
    double* FX = sm + SM_FX;
    double* FY = sm + SM_FY;

    DevScalars* sc = A.sc;
    if (A.loop && *(volatile int*)&sc->done) return;

    const GridDesc& g = A.g;
    const Phys& P = A.ph;
    const int nx = g.nx, ny = g.ny, pitch = g.pitch;
    const double* __restrict__ geo = A.geo;
    const long long fs = g.fs;
    const int ntiles = A.ntx * A.nty;
    const double dt = sc->dt;
    const int tid = threadIdx.x;
    const int p = tid & 1;          // phase of this lane: 0 solid, 1 fluid
    const int pr = tid >> 1;        // pair index
    const unsigned pm = 3u << (tid & 30);  // the pair's lanes

    int tile = blockIdx.x;
    if (tid == 0) {
        mbar_init(&bar, 1);
        if (tile < ntiles) {
            const int bx0 = 1 + (tile % A.ntx) * TX, by0 = 1 + (tile / A.ntx) * TY;
            mbar_expect_tx(&bar, kTmaBytes);
            tma_load_3d(S, &A.tm_s, bx0 + 1, by0, 0, &bar);  // +1: leading pad column
            tma_load_3d(sm + SM_G, &A.tm_g, bx0 + 1, by0, 0, &bar);
        }
    }
    __syncthreads();
    double lam_local = 0.0;
    for (unsigned iter = 0; tile < ntiles; tile += gridDim.x, ++iter) {
        const int tix = tile % A.ntx, tiy = tile / A.ntx;
        const int X0 = 3 + tix * TX, Y0 = 3 + tiy * TY;
        // this pair's Phase-3 cell
        const int cx = pr % TX, cy = pr / TX;
        const int p3x = X0 + cx, p3y = Y0 + cy;
        const bool p3 = pr < TX * TY && p3x <= nx - 4 && p3y <= ny - 4;
        const long long o3 = static_cast<long long>(p3y) * pitch + p3x;
        const int bk = (cy + 2) * W2 + (cx + 2);
        if (iter == 0 && p3) {
            for (int f = G_NX + p; f <= G_RNZ; f += 2) prefetch_l2(geo + f * fs + o3);
            if (CORR) {
                prefetch_l2(A.u0 + p * fs + o3);
                prefetch_l2(A.u0 + (2 + 2 * p) * fs + o3);
                prefetch_l2(A.u0 + (3 + 2 * p) * fs + o3);
            }
        }
        auto issue_next = [&]() {
            const int nt = tile + gridDim.x;
            if (nt < ntiles) {
                const int bx0n = 1 + (nt % A.ntx) * TX, by0n = 1 + (nt / A.ntx) * TY;
                if (tid == 0) {
                    mbar_expect_tx(&bar, kTmaBytes);
                    tma_load_3d(S, &A.tm_s, bx0n + 1, by0n, 0, &bar);
                    tma_load_3d(sm + SM_G, &A.tm_g, bx0n + 1, by0n, 0, &bar);
                }
                const int qx = bx0n + 2 + cx, qy = by0n + 2 + cy;
                if (pr < TX * TY && qx <= nx - 4 && qy <= ny - 4) {
                    const long long oq = static_cast<long long>(qy) * pitch + qx;
                    for (int f = G_NX + p; f <= G_RNZ; f += 2) prefetch_l2(geo + f * fs + oq);
                    if (CORR) {
                        prefetch_l2(A.u0 + p * fs + oq);
                        prefetch_l2(A.u0 + (2 + 2 * p) * fs + oq);
                        prefetch_l2(A.u0 + (3 + 2 * p) * fs + oq);
                    }
                }
            }
        };
        mbar_wait(&bar, iter & 1u);

        // ---- dry-tile fast path (exact; see stage_kernel / DESIGN.md §3) ----------
        {
            unsigned long long acc = 0ull;
            for (int k = tid; k < 6 * BOX; k += NTP)
                acc |= static_cast<unsigned long long>(__double_as_longlong(S[k]));
            const double jb0 = p3 ? G[G_JB * BOX + bk] : 1.0;
            const double rjb0 = p3 ? G[G_RJB * BOX + bk] : 1.0;
            const double nz0 = p3 ? G[G_NZ * BOX + bk] : 1.0;
            if (!__syncthreads_or(acc != 0ull)) {
                issue_next();
                if (p3) {
                    if (!CORR) {
                        A.out[p * fs + o3] = 0.0;
                        A.out[(2 + 2 * p) * fs + o3] = 0.0;
                        A.out[(3 + 2 * p) * fs + o3] = 0.0;
                    } else {
                        double un[3] = {0.5 * (A.u0[p * fs + o3] + 0.0),
                                        0.5 * (A.u0[(2 + 2 * p) * fs + o3] + 0.0),
                                        0.5 * (A.u0[(3 + 2 * p) * fs + o3] + 0.0)};
                        const Rcp rj0 = mkrcp_const<FD>(jb0, rjb0);
                        pair_epilogue<FD, CORR>(p, pm, un, rj0, nz0, p3x, p3y, P, sc, lam_local, A.out, fs, o3);
                    }
                }
                if ((tix == 0 || tix == A.ntx - 1 || tiy == 0 || tiy == A.nty - 1) && tid < 4)
                    A.tally[4ll * tile + tid] = 0.0;
                continue;
            }
        }

        // ---- Phase 1: xi faces, eta faces, cell fields (one pair per item) --------
        constexpr int N1 = NFX + NFY + BOX;
        for (int it = pr; it < N1; it += NPAIR) {
            if (it < NFX) {
                const int fx = it % (TX + 1), ty = it / (TX + 1);
                double o[3];
                face_half<FD, true>(p, pm, S, G, (ty + 2) * W2 + fx + 1, P, o);
                FX[p * NFX + it] = o[0];
                FX[(2 + 2 * p) * NFX + it] = o[1];
                FX[(3 + 2 * p) * NFX + it] = o[2];
            } else if (it < NFX + NFY) {
                const int jt = it - NFX;
                const int tx = jt % TX, fy = jt / TX;
                double o[3];
                face_half<FD, false>(p, pm, S, G, (fy + 1) * W2 + tx + 2, P, o);
                FY[p * NFY + jt] = o[0];
                FY[(2 + 2 * p) * NFY + jt] = o[1];
                FY[(3 + 2 * p) * NFY + jt] = o[2];
            } else {
                if (P.adv_only) continue;
                const int k = it - NFX - NFY;
                // solver.cpp:172-184, phase p
                const double jb = G[G_JB * BOX + k];
                const Rcp rj = mkrcp_const<FD>(jb, G[G_RJB * BOX + k]);
                const double w = S[p * BOX + k], qx = S[(2 + 2 * p) * BOX + k], qy = S[(3 + 2 * p) * BOX + k];
                bool ok = rj.ok;
                double hp = dq<FD>(w, rj, ok), jx = dq<FD>(qx, rj, ok), jy = dq<FD>(qy, rj, ok);
                if (!ok) {
                    dfix<FD>(hp, w, rj);
                    dfix<FD>(jx, qx, rj);
                    dfix<FD>(jy, qy, rj);
                }
                double f;
                if (FD) {
                    bool okf = true;
                    f = desing_factor_g(hp, P.eps_h, okf);
                    if (!okf) f = desing_factor<FD>(hp, P.eps_h);
                } else {
                    f = desing_factor<FD>(hp, P.eps_h);
                }
                V[(2 * p) * BOX + k] = jx * f;
                V[(2 * p + 1) * BOX + k] = jy * f;
                const double ho = pshfl(pm, hp);
                if (p == 0) {
                    const double h = hp + ho;  // hs + hf
                    PJ[k] = jb * h * (G[G_NZ * BOX + k] * h * 0.5);  // solver.cpp:182
                }
            }
        }
        __syncthreads();

        // ---- Phase 2: viscous brackets on the tile's cross neighbours ------------
        const Rcp r2x = mkrcp_const<FD>(P.two_dxi, P.r_two_dxi);
        const Rcp r2y = mkrcp_const<FD>(P.two_deta, P.r_two_deta);
        if (!P.adv_only) {
            constexpr int NB1 = (TX + 2) * TY;
            constexpr int NB = NB1 + 2 * TX;
            for (int it = tid; it < NB; it += NTP) {
                int bx, by;
                if (it < NB1) {
                    bx = 1 + it % (TX + 2);
                    by = 2 + it / (TX + 2);
                } else {
                    const int r = it - NB1;
                    bx = 2 + r % TX;
                    by = (r < TX) ? 1 : TY + 2;
                }
                const int k = by * W2 + bx;
                const double jb = G[G_JB * BOX + k];
                const double a11 = G[G_A11 * BOX + k], a12 = G[G_A12 * BOX + k];
                const double a21 = G[G_A21 * BOX + k], a22 = G[G_A22 * BOX + k];
                const Rcp rj = mkrcp_const<FD>(jb, G[G_RJB * BOX + k]);
                const double* vxf = V + 2 * BOX;
                const double* vyf = V + 3 * BOX;
                const double n0 = S[0 * BOX + k] + S[1 * BOX + k];
                const double n1 = vxf[k + 1] - vxf[k - 1], n2 = vxf[k + W2] - vxf[k - W2];
                const double n3 = vyf[k + 1] - vyf[k - 1], n4 = vyf[k + W2] - vyf[k - W2];
                bool ok = rj.ok && r2x.ok && r2y.ok;
                double h = dq<FD>(n0, rj, ok);
                double gux = dq<FD>(n1, r2x, ok), guy = dq<FD>(n2, r2y, ok);
                double gwx = dq<FD>(n3, r2x, ok), gwy = dq<FD>(n4, r2y, ok);
                if (!ok) {
                    dfix<FD>(h, n0, rj);
                    dfix<FD>(gux, n1, r2x);
                    dfix<FD>(guy, n2, r2y);
                    dfix<FD>(gwx, n3, r2x);
                    dfix<FD>(gwy, n4, r2y);
                }
                const double jh = jb * h;
                BR[0 * BOX + k] = jh * (a11 * gux + a21 * guy);
                BR[1 * BOX + k] = jh * (a12 * gwx + a22 * gwy);
                BR[2 * BOX + k] = jh * ((a12 * gux + a22 * guy) + (a11 * gwx + a21 * gwy));
            }
        }
        // this lane's Phase-3 values out of the staged boxes (recycled below)
        double s3[3] = {0.0, 0.0, 0.0};
        double gjb = 1.0, grjb = 1.0, gnz = 1.0, ga11 = 0.0, ga12 = 0.0, ga21 = 0.0, ga22 = 0.0;
        if (p3) {
            s3[0] = S[p * BOX + bk];
            s3[1] = S[(2 + 2 * p) * BOX + bk];
            s3[2] = S[(3 + 2 * p) * BOX + bk];
            gjb = G[G_JB * BOX + bk];
            grjb = G[G_RJB * BOX + bk];
            gnz = G[G_NZ * BOX + bk];
            ga11 = G[G_A11 * BOX + bk];
            ga12 = G[G_A12 * BOX + bk];
            ga21 = G[G_A21 * BOX + bk];
            ga22 = G[G_A22 * BOX + bk];
        }
        __syncthreads();
        issue_next();

        // ---- Phase 3: residual + update + [cap] + [average] + regularize + [finite, lambda]
        if (p3) {
            const Rcp rdx = mkrcp_const<FD>(P.dxi, P.r_dxi);
            const Rcp rdy = mkrcp_const<FD>(P.deta, P.r_deta);
            const double jb = gjb;
            const Rcp rj = mkrcp_const<FD>(jb, grjb);
            const double nZ = gnz;
            const int f0 = p, f1 = 2 + 2 * p, f2 = 3 + 2 * p;
            const int fxo = cy * (TX + 1) + cx, fyo = cy * TX + cx;
            // flux divergence (solver.cpp:396-399) of the own three fields
            const double n0 = -(FX[f0 * NFX + fxo + 1] - FX[f0 * NFX + fxo]);
            const double n1 = -(FX[f1 * NFX + fxo + 1] - FX[f1 * NFX + fxo]);
            const double n2 = -(FX[f2 * NFX + fxo + 1] - FX[f2 * NFX + fxo]);
            const double m0 = -(FY[f0 * NFY + fyo + TX] - FY[f0 * NFY + fyo]);
            const double m1 = -(FY[f1 * NFY + fyo + TX] - FY[f1 * NFY + fyo]);
            const double m2 = -(FY[f2 * NFY + fyo + TX] - FY[f2 * NFY + fyo]);
            bool ok = rdx.ok && rdy.ok;
            double dx0 = dq<FD>(n0, rdx, ok), dx1 = dq<FD>(n1, rdx, ok), dx2 = dq<FD>(n2, rdx, ok);
            double dy0 = dq<FD>(m0, rdy, ok), dy1 = dq<FD>(m1, rdy, ok), dy2 = dq<FD>(m2, rdy, ok);
            if (!ok) {
                dfix<FD>(dx0, n0, rdx);
                dfix<FD>(dx1, n1, rdx);
                dfix<FD>(dx2, n2, rdx);
                dfix<FD>(dy0, m0, rdy);
                dfix<FD>(dy1, m1, rdy);
                dfix<FD>(dy2, m2, rdy);
            }
            double rhs[3] = {dx0 + dy0, dx1 + dy1, dx2 + dy2};

            double nX = 0.0, nY = 0.0, dXx = 0.0, dYx = 0.0, dZx = 0.0, dXy = 0.0, dYy = 0.0, dZy = 0.0;
            double rnzv = 1.0;
            if (!P.adv_only || P.cap_on) {
                nX = __ldg(geo + G_NX * fs + o3);
                nY = __ldg(geo + G_NY * fs + o3);
                dXx = __ldg(geo + G_DNX_DXI * fs + o3);
                dYx = __ldg(geo + G_DNY_DXI * fs + o3);
                dZx = __ldg(geo + G_DNZ_DXI * fs + o3);
                dXy = __ldg(geo + G_DNX_DETA * fs + o3);
                dYy = __ldg(geo + G_DNY_DETA * fs + o3);
                dZy = __ldg(geo + G_DNZ_DETA * fs + o3);
                rnzv = __ldg(geo + G_RNZ * fs + o3);
            }
            const Rcp rnz = mkrcp_const<FD>(nZ, rnzv);

            if (!P.adv_only) {
                // solver.cpp:406-445, the own phase's part
                const double vsx = V[0 * BOX + bk], vsy = V[1 * BOX + bk];
                const double vfx = V[2 * BOX + bk], vfy = V[3 * BOX + bk];
                const double vx = p ? vfx : vsx, vy = p ? vfy : vsy;
                const double gpx = PJ[bk + 1] - PJ[bk - 1], gpy = PJ[bk + W2] - PJ[bk - W2];
                const double nzv = -(nX * vx + nY * vy);
                bool ok2 = rj.ok && rnz.ok && r2x.ok && r2y.ok;
                double hp = dq<FD>(s3[0], rj, ok2);
                double vz = dq<FD>(nzv, rnz, ok2);
                double gPx = dq<FD>(gpx, r2x, ok2), gPy = dq<FD>(gpy, r2y, ok2);
                if (!ok2) {
                    dfix<FD>(hp, s3[0], rj);
                    dfix<FD>(vz, nzv, rnz);
                    dfix<FD>(gPx, gpx, r2x);
                    dfix<FD>(gPy, gpy, r2y);
                }
                const double ho = pshfl(pm, hp);
                const double hs = p ? ho : hp, hf = p ? hp : ho;
                const double h = hs + hf;
                double phi = 0.0, hsf_h = 0.0;
                if (!(h <= 0.0)) {
                    const Rcp rh = mkrcp<FD>(h);
                    const double hsf = hs * hf;
                    bool okh = rh.ok;
                    double q1 = dq<FD>(hp, rh, okh), q3 = dq<FD>(hsf, rh, okh);
                    if (!okh) {
                        dfix<FD>(q1, hp, rh);
                        dfix<FD>(q3, hsf, rh);
                    }
                    if (!(h < P.h_dry)) phi = q1;  // phi_p = h < h_dry ? 0 : h_p / h
                    hsf_h = q3;
                }
                // physics::curvature_accel (physics.hpp:47-52) and hydrostatic_terms (:56-69)
                const double kap = ((vx * dXx + vy * dYx) + vz * dZx) * vx + ((vx * dXy + vy * dYy) + vz * dZy) * vy;
                const double p_b = p ? smax(0.0, hf * (nZ - P.eps_chi * kap))
                                     : smax(0.0, hs * (nZ * P.oma - P.eps_chi * kap));
                const double snx = jb * p_b * nX, sny = jb * p_b * nY;
                const double Avx = ga11 * gPx + ga21 * gPy;
                const double Avy = ga12 * gPx + ga22 * gPy;
                double cx_ = 0.0, cy_ = 0.0;
                if (!(h <= 0.0)) {  // physics::drag_sources (physics.hpp:121-134)
                    const double common = jb * P.C_d * hsf_h;
                    cx_ = common * (vfx - vsx);
                    cy_ = common * (vfy - vsy);
                }
                if (p == 0) {
                    const double svx = (h <= 0.0) ? 0.0 : P.alpha * cx_;
                    const double svy = (h <= 0.0) ? 0.0 : P.alpha * cy_;
                    const double fsp = P.neg_eps_alpha * phi;
                    rhs[1] = rhs[1] + (snx + fsp * Avx + svx);
                    rhs[2] = rhs[2] + (sny + fsp * Avy + svy);
                } else {
                    const double svx = (h <= 0.0) ? 0.0 : -cx_;
                    const double svy = (h <= 0.0) ? 0.0 : -cy_;
                    const Rcp rNR = mkrcp_const<FD>(P.N_R, P.r_NR);
                    const Rcp reNR = mkrcp_const<FD>(P.eps_NR, P.r_eps_NR);
                    const double ephf = P.eps * phi;
                    const double cn = jb * hf * P.theta_b;
                    const double s1 = 2.0 * (BR[bk + 1] - BR[bk - 1]);
                    const double s2 = BR[2 * BOX + bk + W2] - BR[2 * BOX + bk - W2];
                    const double s3v = 2.0 * (BR[BOX + bk + W2] - BR[BOX + bk - W2]);
                    const double s4 = BR[2 * BOX + bk + 1] - BR[2 * BOX + bk - 1];
                    bool ok3 = rNR.ok && reNR.ok && r2x.ok && r2y.ok;
                    double coeff = dq<FD>(cn, reNR, ok3), visc = dq<FD>(ephf, rNR, ok3);
                    double v1 = dq<FD>(s1, r2x, ok3), v2 = dq<FD>(s2, r2y, ok3);
                    double v3 = dq<FD>(s3v, r2y, ok3), v4 = dq<FD>(s4, r2x, ok3);
                    if (!ok3) {
                        dfix<FD>(coeff, cn, reNR);
                        dfix<FD>(visc, ephf, rNR);
                        dfix<FD>(v1, s1, r2x);
                        dfix<FD>(v2, s2, r2y);
                        dfix<FD>(v3, s3v, r2y);
                        dfix<FD>(v4, s4, r2x);
                    }
                    const double sdx = -coeff * vfx, sdy = -coeff * vfy;
                    rhs[1] = rhs[1] + (snx + sdx + ephf * Avx + svx + visc * (v1 + v2));
                    rhs[2] = rhs[2] + (sny + sdy + ephf * Avy + svy + visc * (v3 + v4));
                }
            }

            // stage update of the own fields (solver.cpp:518 / :531)
            double un[3];
#pragma unroll
            for (int q = 0; q < 3; ++q) un[q] = s3[q] + dt * rhs[q];

            // Coulomb cap (solver.cpp:458-479): solid lane
            if (P.cap_on && p == 0) {
                const double qx = un[1], qy = un[2];
                if (!(qx == 0.0 && qy == 0.0)) {
                    bool okc = rj.ok;
                    double hs = dq<FD>(un[0], rj, okc);
                    double jx = dq<FD>(qx, rj, okc), jy = dq<FD>(qy, rj, okc);
                    if (!okc) {
                        dfix<FD>(hs, un[0], rj);
                        dfix<FD>(jx, qx, rj);
                        dfix<FD>(jy, qy, rj);
                    }
                    if (!(hs < P.h_dry)) {
                        double fsld;
                        if (FD) {
                            bool okf = true;
                            fsld = desing_factor_g(hs, P.eps_h, okf);
                            if (!okf) fsld = desing_factor<FD>(hs, P.eps_h);
                        } else {
                            fsld = desing_factor<FD>(hs, P.eps_h);
                        }
                        const double vsx = jx * fsld, vsy = jy * fsld;
                        const double vz = dv<FD>(-(nX * vsx + nY * vsy), rnz);
                        const double kap = ((vsx * dXx + vsy * dYx) + vz * dZx) * vsx + ((vsx * dXy + vsy * dYy) + vz * dZy) * vsy;
                        const double p_b_s = smax(0.0, hs * (nZ * P.oma - P.eps_chi * kap));
                        const double rate = jb * p_b_s * P.tan_d;
                        const double qnorm = sqrt(qx * qx + qy * qy);
                        const double num = dt * rate;
                        double frac;
                        if (FD) {
                            bool okq = true;
                            frac = ddiv_fast(num, qnorm, okq);
                            if (!okq) frac = num / qnorm;
                        } else {
                            frac = num / qnorm;
                        }
                        const double factor = smax(0.0, 1.0 - frac);
                        un[1] = qx * factor;
                        un[2] = qy * factor;
                    }
                }
            }
            if (CORR) {  // Heun average (solver.cpp:538-541)
                un[0] = 0.5 * (A.u0[f0 * fs + o3] + un[0]);
                un[1] = 0.5 * (A.u0[f1 * fs + o3] + un[1]);
                un[2] = 0.5 * (A.u0[f2 * fs + o3] + un[2]);
            }
            pair_epilogue<FD, CORR>(p, pm, un, rj, nZ, p3x, p3y, P, sc, lam_local, A.out, fs, o3);
        }

        // ---- boundary mass tally (solver.cpp:352-376), ring tiles
        const bool ring = tix == 0 || tix == A.ntx - 1 || tiy == 0 || tiy == A.nty - 1;
        if (ring && tid < 2) {
            const bool w_edge = X0 == 3;
            const bool e_edge = (nx - 4) >= X0 && (nx - 4) < X0 + TX;
            const bool s_edge = g.has_south && Y0 == 3;
            const bool n_edge = g.has_north && (ny - 4) >= Y0 && (ny - 4) < Y0 + TY;
            const int q = tid;
            const double wdt = dt * 0.5;
            double in = 0.0, outf = 0.0;
            auto add = [&](double outward) {
                if (outward >= 0.0) outf += outward;
                else in += -outward;
            };
            const int fxE = nx - 3 - X0;
            for (int ty = 0; ty < TY && Y0 + ty <= ny - 4; ++ty) {
                if (w_edge) add(-FX[q * NFX + ty * (TX + 1) + 0] * P.deta * wdt);
                if (e_edge) add(FX[q * NFX + ty * (TX + 1) + fxE] * P.deta * wdt);
            }
            const int fyN = ny - 3 - Y0;
            for (int tx = 0; tx < TX && X0 + tx <= nx - 4; ++tx) {
                if (s_edge) add(-FY[q * NFY + 0 * TX + tx] * P.dxi * wdt);
                if (n_edge) add(FY[q * NFY + fyN * TX + tx] * P.dxi * wdt);
            }
            double* t = A.tally + 4ll * tile;
            t[2 * q + 0] = in;
            t[2 * q + 1] = outf;
        }
        __syncthreads();
    }  // tile loop

    if (CORR) lam_block_max<NTP>(lam_local, sc);
}

static int g_sms_pair = 148;

template <bool FD, bool CORR>
static cudaError_t launch_pair_t(const StageArgs& a, cudaStream_t st) {
    const int ntiles = a.ntx * a.nty;
    dim3 grid(ntiles < 2 * g_sms_pair ? ntiles : 2 * g_sms_pair);
    stage_pair_kernel<FD, CORR><<<grid, NTP, sizeof(double) * SM_END, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_stage_pair(const StageArgs& a, bool fastdiv, bool corr, cudaStream_t st) {
    if (fastdiv) return corr ? launch_pair_t<true, true>(a, st) : launch_pair_t<true, false>(a, st);
    return corr ? launch_pair_t<false, true>(a, st) : launch_pair_t<false, false>(a, st);
}

cudaError_t init_pair_kernels() {
    const int smem = static_cast<int>(sizeof(double) * SM_END);
    cudaError_t e;
    int dev = 0;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
    if ((e = cudaDeviceGetAttribute(&g_sms_pair, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(stage_pair_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)) != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(stage_pair_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)) != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(stage_pair_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)) != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(stage_pair_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)) != cudaSuccess) return e;
    return cudaSuccess;
}

}  // namespace tpb
