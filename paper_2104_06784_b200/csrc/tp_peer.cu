// Device-resident row-slab exchange over peer memory (NVLink / CUDA IPC), SURVEY.md §8(e).
//
// One context per slab (one rank per GPU, or several contexts in one process).  Each
// step of the device loop exchanges, without the host:
//   * the wave-speed bound: every rank writes its local lambda (the bits of a double
//     >= 0, so the unsigned maximum is the floating maximum: exact, partition independent)
//     and its stop flag into every rank's mailbox, then each rank reduces its own mailbox
//     (peer_lambda_kernel, before compute_dt);
//   * the halo rows exactly where the reference refills ghosts (solver.cpp:639, :523):
//     after apply_boundaries each slab stores its 2 edge interior rows of all 6 fields,
//     at full padded width (W/E ghosts included, which keeps the reference's corner
//     semantics), straight into the neighbour's halo rows, then releases a sequence number
//     into the neighbour's mailbox (peer_halo_push_kernel); the neighbour's stage kernel
//     (stage_kernel<..., PEER>) acquires it before the first tile whose box reads those rows
//     (such tiles are listed last, so the transfer overlaps the interior tiles).
// Sequence numbers derive from the step counter, which every rank advances identically
// (dt is identical), so the graph of a step is the same on every rank.  Stores are
// made visible with __threadfence_system() + st.release.sys; waits use ld.acquire.sys.
// A wait that sees no progress for PeerLink::timeout_ns (60 s unless TPFLOW_PEER_TIMEOUT_S)
// sets the context's error key.
#include <cuda_runtime.h>

#include "tp_sync.cuh"
#include "tp_types.h"

namespace tpb {

// lambda + stop all-reduce of one step (one CTA of kMaxRanks threads).  Runs whatever
// the stop flag says, so every rank executes the same exchanges.
__global__ void peer_lambda_kernel(PeerLink L, DevScalars* sc) {
    __shared__ unsigned long long red[2][kMaxRanks];
    __shared__ int timed_out;
    const int k = threadIdx.x;
    const unsigned long long seq = seq_of(sc, 0);
    // exchange parity (PeerBox): peer_base / 4 + steps numbers the exchanges consecutively
    // across tp_steps calls (the host advances peer_base by 4 per graph step launched)
    const int slot = static_cast<int>(((sc->peer_base >> 2) + static_cast<unsigned long long>(sc->steps)) & 1ull);
    if (k == 0) timed_out = 0;
    __syncthreads();
    if (k < L.nranks) {
        PeerBox* b = L.box[k];
        b->lam_val[slot][L.rank] = sc->lam_cur;
        b->stop_val[slot][L.rank] = (sc->err_key != kNoError) ? 1ull : 0ull;
        __threadfence_system();
        st_release_sys(&b->lam_seq[slot][L.rank], seq);
    }
    __syncthreads();
    unsigned long long lam = 0ull, stop = 0ull;
    if (k < L.nranks) {
        if (wait_seq(&L.my_box->lam_seq[slot][k], seq, L.timeout_ns)) {
            lam = *(volatile unsigned long long*)&L.my_box->lam_val[slot][k];
            stop = *(volatile unsigned long long*)&L.my_box->stop_val[slot][k];
        } else {
            atomicExch(&timed_out, 1);
        }
    }
    red[0][k] = lam;
    red[1][k] = stop;
    __syncthreads();
    if (k == 0) {
        unsigned long long m = 0ull, st = 0ull;
        for (int r = 0; r < L.nranks; ++r) {
            m = red[0][r] > m ? red[0][r] : m;
            st |= red[1][r];
        }
        sc->lam_cur = m;
        if (st) sc->done = 1;
        if (timed_out) {
            atomicMin(&sc->err_key, kPeerTimeoutKey);
            sc->done = 1;
        }
    }
}

// Store this slab's 2 edge interior rows of buffer `buf` into each neighbour's halo rows,
// then release the sequence number into the neighbour's mailbox (last CTA per side).
//   to the south neighbour (rank-1): my rows 3,4   -> its rows ny-3, ny-2
//   to the north neighbour (rank+1): my rows ny-5, ny-4 -> its rows 1, 2
__global__ void peer_halo_push_kernel(PeerLink L, GridDesc g, const double* __restrict__ s, int buf,
                                      DevScalars* sc) {
    if (*(volatile int*)&sc->done) return;  // consistent on every rank (see peer_lambda_kernel)
    const int side = blockIdx.y;
    double* dst = L.nbr_state[buf][side];
    if (!dst) return;
    const long long n = 2ll * 6 * g.nx;  // 2 rows x 6 fields x padded width
    const int src_row = side == 0 ? 3 : g.ny - 5;
    const int dst_row = side == 0 ? L.nbr_ny[0] - 3 : 1;
    const long long dfs = L.nbr_fs[side];
    for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < n;
         e += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int i = static_cast<int>(e % g.nx);
        const long long r = e / g.nx;      // f * 2 + row
        const int f = static_cast<int>(r >> 1), dr = static_cast<int>(r & 1);
        dst[f * dfs + static_cast<long long>(dst_row + dr) * g.pitch + i] =
            s[f * g.fs + static_cast<long long>(src_row + dr) * g.pitch + i];
    }
    // per tile column of the receiver (same columns): does any pushed value inside the box
    // columns X0-2 .. X0+TX+1 have a bit other than +0.0 (its conditional tiles, stage_kernel<PEER>)
    const int ntx = (g.nx - 6 + TX - 1) / TX;
    unsigned int* nz = L.nbr_box[side]->halo_nz[buf][side == 0 ? 1 : 0];
    for (int tx = blockIdx.x * blockDim.x + threadIdx.x; tx < ntx && tx < kMaxTileCols;
         tx += gridDim.x * blockDim.x) {
        const int x0 = 3 + tx * TX - 2, x1 = min(3 + tx * TX + TX + 1, g.nx - 1);
        unsigned long long bits = 0ull;
        for (int f = 0; f < 6; ++f)
            for (int dr = 0; dr < 2; ++dr) {
                const double* row = s + f * g.fs + static_cast<long long>(src_row + dr) * g.pitch;
                for (int x = x0; x <= x1; ++x) bits |= static_cast<unsigned long long>(__double_as_longlong(row[x]));
            }
        nz[tx] = bits != 0ull ? 1u : 0u;
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned int* cnt = &L.my_box->push_done[buf][side];
        if (atomicAdd(cnt, 1u) == gridDim.x - 1) {  // the last CTA of this side
            *cnt = 0u;
            __threadfence_system();
            // the neighbour files data from its north (side 1) when we are its south
            st_release_sys(&L.nbr_box[side]->halo_seq[buf][side == 0 ? 1 : 0], seq_of(sc, 1 + buf));
        }
    }
}

cudaError_t launch_peer_lambda(const PeerLink& L, DevScalars* sc, cudaStream_t st) {
    peer_lambda_kernel<<<1, kMaxRanks, 0, st>>>(L, sc);
    return cudaGetLastError();
}
cudaError_t launch_peer_halo(const PeerLink& L, const GridDesc& g, const double* s, int buf, DevScalars* sc,
                             cudaStream_t st) {
    peer_halo_push_kernel<<<dim3(16, 2), 256, 0, st>>>(L, g, s, buf, sc);
    return cudaGetLastError();
}

}  // namespace tpb
