// FP64 pipe latency / throughput probe on sm_100a (development aid).
// lat: one warp, one dependent chain; thr: many warps x ILP chains.
#include <cstdio>
#include <cuda_runtime.h>
template <int OP, int ILP>
__global__ void k(double* out, int iters, long long* cyc) {
    double a[ILP];
    for (int i = 0; i < ILP; ++i) a[i] = 1.0 + threadIdx.x * 1e-9 + i * 1e-7;
    const double b = 0.999999, c = 1e-12;
    long long t0 = clock64();
    for (int n = 0; n < iters; ++n) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int i = 0; i < ILP; ++i) {
                if (OP == 0) a[i] = __fma_rn(a[i], b, c);
                if (OP == 1) a[i] = __dmul_rn(a[i], b);
                if (OP == 2) a[i] = __dadd_rn(a[i], c);
            }
    }
    long long t1 = clock64();
    double s = 0;
    for (int i = 0; i < ILP; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
// mixed: FP64 chain + independent integer work
__global__ void kmix(double* out, int iters, long long* cyc, int nint) {
    double a0 = 1.0 + threadIdx.x, a1 = 2.0 + threadIdx.x;
    unsigned x = threadIdx.x, y = threadIdx.x * 3;
    long long t0 = clock64();
    for (int n = 0; n < iters; ++n) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            a0 = __fma_rn(a0, 0.999999, 1e-12);
            a1 = __fma_rn(a1, 0.999999, 1e-12);
            for (int q = 0; q < 2; ++q) { x = x * 1664525u + y; y ^= x >> 3; }
        }
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + x + y;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int OP, int ILP>
void run(const char* name, int blocks, int threads) {
    double* o; long long* c; cudaMalloc(&o, 8 * blocks * threads); cudaMalloc(&c, 8);
    int it = 2000;
    k<OP, ILP><<<blocks, threads>>>(o, it, c);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<OP, ILP><<<blocks, threads>>>(o, it, c);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long cy; cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
    double ops = 8.0 * it * ILP;  // per thread
    double warps_per_smsp = (double)blocks * threads / 32 / (148 * 4);
    printf("%-5s ILP=%d blocks=%d thr=%d: %.2f cyc per dependent op (1 warp view), %.3f cyc/warp-instr/SMSP, %.1f Gop/s\n",
           name, ILP, blocks, threads, cy / (8.0 * it), cy / (ops * (blocks >= 148 ? warps_per_smsp : (double)threads / 32 / 4 > 1 ? (double)threads / 128 : 1)),
           ops * blocks * threads / (ms * 1e6));
    cudaFree(o); cudaFree(c);
}
int main() {
    run<0, 1>("dfma", 1, 32);
    run<1, 1>("dmul", 1, 32);
    run<2, 1>("dadd", 1, 32);
    run<0, 2>("dfma", 1, 32);
    run<0, 4>("dfma", 1, 32);
    run<0, 8>("dfma", 1, 32);
    run<0, 1>("dfma", 148, 128);
    run<0, 2>("dfma", 148, 128);
    run<0, 4>("dfma", 148, 128);
    run<0, 8>("dfma", 148, 128);
    run<0, 1>("dfma", 148, 256);
    run<0, 1>("dfma", 148, 512);
    run<0, 2>("dfma", 148, 512);
    run<0, 4>("dfma", 148, 512);
    run<0, 8>("dfma", 148, 1024);
    run<1, 4>("dmul", 148, 512);
    run<2, 4>("dadd", 148, 512);
    for (int nint = 0; nint < 1; ++nint) {
        double* o; long long* c; cudaMalloc(&o, 8 * 148 * 512); cudaMalloc(&c, 8);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        kmix<<<148, 512>>>(o, 2000, c, 0);
        cudaEventRecord(e0); kmix<<<148, 512>>>(o, 2000, c, 0); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        long long cy; cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
        printf("mix: 2 dfma + ~8 int per unit, 16 warps/SM: %.2f cyc per unit per warp, %.3f ms\n", cy / 16000.0, ms);
    }
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("clock %d kHz\n", clk);
    return 0;
}
