// One Kurganov–Tadmor central face flux of the six-equation system.
// Restates Simulator::compute_face_fluxes' `face_flux` lambda
// (/root/reference/proj/src/solver.cpp:239-316) with physics::directional_flux
// (physics.hpp:84-95) and physics::desingularized_velocity (physics.hpp:33-37).
#pragma once

#include "tp_math.cuh"

namespace tpb {

// L[k], R[k]: reconstructed edge states of the 6 fields (ws,wf,qsx,qsy,qfx,qfy)
// on the left (cell i, +edge) and right (cell i+1, -edge) of the face.
// XI = true for a xi face (normal X: a_nn = a11, a_nt = a12), false for eta
// (normal Y: a_nn = a22, a_nt = a21).  out[6] in field order.
// rjbf = RN(1/jbf) precomputed on the host (geometry field G_RJBFX/G_RJBFY).
// CHK = false: the "safe tile" form without the FASTDIV window tests.
template <bool FD, bool XI, bool CHK = true>
__device__ __forceinline__ void face_flux(const double (&L)[6], const double (&R)[6], double jb_l,
                                          double jb_r, double nZ_l, double nZ_r, double ann_l,
                                          double ann_r, double ant_l, double ant_r, double rjbf,
                                          const Phys& P, double (&out)[6]) {
    // solver.cpp:242-245.  Safe tiles (CHK = false) keep a_nn, a_nt unhalved: the factor 1/2
    // is folded, with the pressure's 1/2, into one exact FMA per flux term (below)
    const double jbf = 0.5 * (jb_l + jb_r);
    const double cf = 0.5 * (nZ_l + nZ_r);
    const double ann = CHK ? 0.5 * (ann_l + ann_r) : ann_l + ann_r;
    const double ant = CHK ? 0.5 * (ant_l + ant_r) : ant_l + ant_r;
    const Rcp rj = mkrcp_const<FD, CHK>(jbf, rjbf);

    // solver.cpp:265-275
    bool ok = rj.ok;
    double hL0 = dq<FD, CHK>(L[0], rj, ok), hL1 = dq<FD, CHK>(L[1], rj, ok);
    double hR0 = dq<FD, CHK>(R[0], rj, ok), hR1 = dq<FD, CHK>(R[1], rj, ok);
    if (!ok) {
        dfix<FD>(hL0, L[0], rj);
        dfix<FD>(hL1, L[1], rj);
        dfix<FD>(hR0, R[0], rj);
        dfix<FD>(hR1, R[1], rj);
    }
    const double htL = hL0 + hL1;
    const double htR = hR0 + hR1;
    if (htL < P.h_dry && htR < P.h_dry) {
#pragma unroll
        for (int k = 0; k < 6; ++k) out[k] = 0.0;
        return;
    }

    // solver.cpp:277-285
    double celL, celR;
    if (CHK) {
        celL = sqrt(P.eps * cf * smax(htL, 0.0));
        celR = sqrt(P.eps * cf * smax(htR, 0.0));
    } else {  // safe tile: the argument is +-0 or >= 2^-274, so the branch-free sequence is IEEE sqrt
        // (and htL, htR are +0 or positive: max(h, 0.0) is h itself, see below)
        bool oks = true;
        celL = dsqrt_fast(P.eps * cf * htL, oks);
        celR = dsqrt_fast(P.eps * cf * htR, oks);
    }
    // normal / transverse momenta (solver.cpp:259-262)
    const double qnL0 = XI ? L[2] : L[3], qtL0 = XI ? L[3] : L[2];
    const double qnR0 = XI ? R[2] : R[3], qtR0 = XI ? R[3] : R[2];
    const double qnL1 = XI ? L[4] : L[5], qtL1 = XI ? L[5] : L[4];
    const double qnR1 = XI ? R[4] : R[5], qtR1 = XI ? R[5] : R[4];

    ok = rj.ok;
    double jL0 = dq<FD, CHK>(qnL0, rj, ok), jR0 = dq<FD, CHK>(qnR0, rj, ok);
    double jL1 = dq<FD, CHK>(qnL1, rj, ok), jR1 = dq<FD, CHK>(qnR1, rj, ok);
    if (!ok) {
        dfix<FD>(jL0, qnL0, rj);
        dfix<FD>(jR0, qnR0, rj);
        dfix<FD>(jL1, qnL1, rj);
        dfix<FD>(jR1, qnR1, rj);
    }
    // safe tile (CHK = false): every thickness of the box is +-0 or positive (TF_UNSAFE2), so
    // each minmod edge value uc + (+-0.5)*slope is +0 or positive (a nonzero slope has the sign
    // of both differences, so the exact sum is >= 0; a zero slope or uc = -0 gives +0), and so
    // are hL = edge / jbf and htL = hL0 + hL1: std::max(h, 0.0) returns h bit for bit
    const double dL0 = CHK ? smax(hL0, 0.0) : hL0, dR0 = CHK ? smax(hR0, 0.0) : hR0;
    const double dL1 = CHK ? smax(hL1, 0.0) : hL1, dR1 = CHK ? smax(hR1, 0.0) : hR1;
    double fL0, fR0, fL1, fR1;
    if (FD) {  // four desingularisation divisions, one shared slow-path branch
        bool okf = true;
        // safe tile: the d's are +0 or positive (above), so no signed-zero select is needed
        fL0 = desing_factor_g<CHK, !CHK>(dL0, P.eps_h, P.eps_h2, okf);
        fR0 = desing_factor_g<CHK, !CHK>(dR0, P.eps_h, P.eps_h2, okf);
        fL1 = desing_factor_g<CHK, !CHK>(dL1, P.eps_h, P.eps_h2, okf);
        fR1 = desing_factor_g<CHK, !CHK>(dR1, P.eps_h, P.eps_h2, okf);
        if (!okf) {
            fL0 = desing_factor<FD>(dL0, P.eps_h, P.eps_h2);
            fR0 = desing_factor<FD>(dR0, P.eps_h, P.eps_h2);
            fL1 = desing_factor<FD>(dL1, P.eps_h, P.eps_h2);
            fR1 = desing_factor<FD>(dR1, P.eps_h, P.eps_h2);
        }
    } else {
        fL0 = desing_factor<FD>(dL0, P.eps_h, P.eps_h2);
        fR0 = desing_factor<FD>(dR0, P.eps_h, P.eps_h2);
        fL1 = desing_factor<FD>(dL1, P.eps_h, P.eps_h2);
        fR1 = desing_factor<FD>(dR1, P.eps_h, P.eps_h2);
    }
    const double vnL0 = jL0 * fL0;
    const double vnR0 = jR0 * fR0;
    const double vnL1 = jL1 * fL1;
    const double vnR1 = jR1 * fR1;
    double a = 0.0;
    if (CHK) {
        a = smax(a, smax(fabs(vnL0) + celL, fabs(vnR0) + celR));
    } else {  // safe tile: |v| + cel is +0 or positive and never NaN, so max(0.0, x) is x bit for bit
        a = smax(fabs(vnL0) + celL, fabs(vnR0) + celR);
    }
    a = smax(a, smax(fabs(vnL1) + celL, fabs(vnR1) + celR));

    // solver.cpp:288-296
    double prL0, prR0, prL1, prR1;
    if (P.adv_only) {
        prL0 = prR0 = prL1 = prR1 = 0.0;
    } else if (CHK) {
        prL0 = cf * P.oma * hL0 * 0.5;
        prR0 = cf * P.oma * hR0 * 0.5;
        prL1 = cf * htL * 0.5;
        prR1 = cf * htR * 0.5;
    } else {  // safe tile: pressures without the exact factor 1/2 (folded below)
        prL0 = cf * P.oma * hL0;
        prR0 = cf * P.oma * hR0;
        prL1 = cf * htL;
        prR1 = cf * htR;
    }

    // physics::directional_flux (physics.hpp:84-95) + solver.cpp:298-315
    const double ejL = P.eps * jbf * htL;
    const double ejR = P.eps * jbf * htR;
    const double ha = 0.5 * a;
    // Safe tiles: every value is +-0 or of magnitude in [2^-800, 2^300] (DESIGN.md §3 item 6),
    // so scaling by 1/2 or 1/4 is exact and commutes with rounding:
    //   q*v + (ej*(ANN/2))*(X/2)   == fma(1/4, (ej*ANN)*X, q*v)
    //   (1/2)*(fl + fr) - ha*d     == fma(1/2, fl + fr, -(ha*d))
    // bit for bit (one rounding each side), two FP64 instructions fewer per term.
    auto pterm = [&](double qv, double ej, double anx, double pr) {
        return CHK ? qv + ej * anx * pr : __fma_rn(0.25, ej * anx * pr, qv);
    };
    auto kt = [&](double fl, double fr, double d) {
        return CHK ? 0.5 * (fl + fr) - ha * d : __fma_rn(0.5, fl + fr, -(ha * d));
    };
    // solid
    {
        const double flm = L[0] * vnL0, frm = R[0] * vnR0;
        const double fln = pterm(qnL0 * vnL0, ejL, ann, prL0);
        const double frn = pterm(qnR0 * vnR0, ejR, ann, prR0);
        const double flt = pterm(qtL0 * vnL0, ejL, ant, prL0);
        const double frt = pterm(qtR0 * vnR0, ejR, ant, prR0);
        const double mass = kt(flm, frm, R[0] - L[0]);
        const double momn = kt(fln, frn, qnR0 - qnL0);
        const double momt = kt(flt, frt, qtR0 - qtL0);
        out[0] = mass;
        out[2] = XI ? momn : momt;
        out[3] = XI ? momt : momn;
    }
    // fluid
    {
        const double flm = L[1] * vnL1, frm = R[1] * vnR1;
        const double fln = pterm(qnL1 * vnL1, ejL, ann, prL1);
        const double frn = pterm(qnR1 * vnR1, ejR, ann, prR1);
        const double flt = pterm(qtL1 * vnL1, ejL, ant, prL1);
        const double frt = pterm(qtR1 * vnR1, ejR, ant, prR1);
        const double mass = kt(flm, frm, R[1] - L[1]);
        const double momn = kt(fln, frn, qnR1 - qnL1);
        const double momt = kt(flt, frt, qtR1 - qtL1);
        out[1] = mass;
        out[4] = XI ? momn : momt;
        out[5] = XI ? momt : momn;
    }
}

}  // namespace tpb
