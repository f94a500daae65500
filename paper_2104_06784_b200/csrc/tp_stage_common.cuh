// Device helpers shared by the stage kernels: TMA + mbarrier PTX wrappers and the
// exact block-level maximum of the wave-speed bound.
#pragma once

#include <cuda.h>

#include "tp_math.cuh"
#include "tp_types.h"

namespace tpb {

// shared-memory carve-up of the stage kernel (doubles)
constexpr int SM_S = 0;                                   // [6][BOX] state box (TMA)
constexpr int SM_G = ((6 * BOX * 8 + 127) / 128) * 16;    // [NGBOX][BOX] geometry box (TMA), 128B aligned
constexpr int SM_V = SM_G + NGBOX * BOX;                  // [4][BOX] cell velocities
constexpr int SM_PJ = SM_V + 4 * BOX;                     // [BOX] jb*h*p_bar_f
constexpr int SM_BR = SM_PJ + BOX;                        // [3][BOX] viscous brackets
constexpr int SM_FX = SM_BR + 3 * BOX;                    // [6][NFX] xi face fluxes
constexpr int SM_FY = SM_FX + 6 * NFX;                    // [6][NFY] eta face fluxes
constexpr int SM_C = (((SM_FY + 6 * NFY) * 8 + 127) / 128) * 16;  // [NGCELL][TY][TX] per-cell geometry (TMA)
constexpr int NGCELL = G_COUNT - NGBOX;                   // nX, nY, 6 x dn, RN(1/nZ)
constexpr int SM_END = SM_C + NGCELL * TX * TY;
// corrector: the u^n tile (6 x TY x TX, TMA) lands in the velocity region, dead after Phase 2
constexpr int SM_U = ((SM_V * 8 + 127) / 128) * 16;
static_assert(SM_U + 6 * TX * TY <= SM_PJ + BOX, "u^n tile must fit the V/PJ region");
constexpr unsigned kTmaUBytes = 6 * TX * TY * 8;
constexpr unsigned kTmaCellBytes = NGCELL * TX * TY * 8;
static_assert((SM_C * 8) % 128 == 0, "cell-geometry TMA box must be 128-byte aligned");
constexpr unsigned kTmaBytes = (6 + NGBOX) * BOX * 8;

__device__ __forceinline__ double ldg(const double* p) { return __ldg(p); }

template <int NTHREADS = NT>
__device__ __forceinline__ void lam_block_max(double lam, DevScalars* sc) {
    // lam >= 0 (or NaN, which reduce_max ignores: std::max(m, NaN) == m)
    unsigned long long b = (lam == lam) ? static_cast<unsigned long long>(__double_as_longlong(lam)) : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long x = __shfl_xor_sync(0xffffffffu, b, o);
        b = x > b ? x : b;
    }
    __shared__ unsigned long long wmax[NTHREADS / 32];
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) wmax[w] = b;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long m = 0;
        for (int k = 0; k < NTHREADS / 32; ++k) m = wmax[k] > m ? wmax[k] : m;
        if (m) atomicMax(&sc->lam_bits, m);
    }
}

// One clipped-mass event of regularize (ClipList, tp_types.h); out of line (rare).
static __device__ __noinline__ void clip_record(DevScalars* sc, unsigned long long key, double val, int p) {
    ClipList* cl = sc->clip;
    const int k = atomicAdd(&cl->n, 1);
    if (k < kClipCap) {
        cl->key[k] = key;
        cl->val[k] = val;
    } else {
        atomicAdd(&sc->audit[5 * p + 4], val);
        atomicAdd(&cl->overflow, 1);
    }
}

// Fold the pending clip events into the audit in key order (= the reference's serial
// (stage, j, i) order per phase), by one whole block; resets the list.
template <int NTHREADS>
__device__ __forceinline__ void clip_fold_block(DevScalars* sc) {
    ClipList* cl = sc->clip;
    const int n = min(*(volatile int*)&cl->n, kClipCap);
    if (n == 0) return;  // uniform across the block
    for (int i = threadIdx.x; i < n; i += NTHREADS) {
        const unsigned long long ki = cl->key[i];
        int r = 0;
        for (int k = 0; k < n; ++k) {
            const unsigned long long kk = cl->key[k];
            r += (kk < ki || (kk == ki && k < i)) ? 1 : 0;
        }
        cl->order[r] = i;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int r = 0; r < n; ++r) {
            const int i = cl->order[r];
            const int p = static_cast<int>(cl->key[i] & 1ull);
            sc->audit[5 * p + 4] += cl->val[i];
        }
        cl->n = 0;
    }
    __syncthreads();
}

// ---------------------------------------------------------------------------
// TMA / mbarrier helpers (sm_90+ PTX, used here on sm_100a)
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* tm, int x, int y, int z,
                                            unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<unsigned long long>(tm)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
// TMA prefetch of a 3-D box into L2 (no shared-memory destination, no barrier)
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* tm, int x, int y, int z) {
    asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(
                     reinterpret_cast<unsigned long long>(tm)),
                 "r"(x), "r"(y), "r"(z)
                 : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}


}  // namespace tpb
