// System-scope acquire / release helpers of the device-resident slab exchange (tp_peer.cu
// and the PEER stage kernels): stores to a neighbour's buffers are made visible with
// __threadfence_system() + st.release.sys of a sequence number, read with ld.acquire.sys.
#pragma once

#include "tp_types.h"

namespace tpb {

// error class 3 of the device error keys (tp_kernels.cu): a neighbour did not arrive
constexpr unsigned long long kPeerTimeoutKey = (3ull << 62);

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// spin until *p >= seq; false on timeout (real exchanges take microseconds; the timeout only
// turns a lost rank into an error instead of a hang)
__device__ __forceinline__ bool wait_seq(const unsigned long long* p, unsigned long long seq,
                                         unsigned long long timeout_ns) {
    if (ld_acquire_sys(p) >= seq) return true;
    const unsigned long long t0 = gtime();
    for (;;) {
        __nanosleep(200);
        if (ld_acquire_sys(p) >= seq) return true;
        if (gtime() - t0 > timeout_ns) return false;
    }
}

// Sequence numbers of one step (steps = DevScalars::steps before the step's post).
// peer_base is advanced by the host after every tp_steps call by 4 * (graph steps launched),
// identically on every rank, so sequence numbers only grow (a step's numbers are at most
// base + 4 * (launched - 1) + 3 < the next call's first, base + 4 * launched + 1).
__device__ __forceinline__ unsigned long long seq_of(const DevScalars* sc, int phase) {
    return sc->peer_base + 4ull * static_cast<unsigned long long>(sc->steps) +
           static_cast<unsigned long long>(phase) + 1ull;
}

}  // namespace tpb
