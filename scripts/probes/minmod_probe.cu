// Device check of the two minmod forms (tp_math.cuh) against a host reference.
#include <cstdio>
#include <cstring>
#include <cstdint>
#include <vector>
#include "../../paper_2104_06784_b200/csrc/tp_math.cuh"
using namespace tpb;
__global__ void k(const double* a, const double* b, double* o1, double* o2, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) { o1[i] = limited_slope(a[i], b[i]); o2[i] = limited_slope_fp(a[i], b[i]); }
}
static double ref(double a, double b) { if (a > 0.0 && b > 0.0) return b < a ? b : a; if (a < 0.0 && b < 0.0) return a < b ? b : a; return 0.0; }
static uint64_t s = 88172645463325252ull;
static uint64_t xr() { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; }
static double rd() {
    uint64_t k = xr(); int mode = k & 3; uint64_t b;
    double sp[] = {0.0, -0.0, 1.0, -1.0, 5e-324, -5e-324, 1e300, -1e300};
    if (mode == 0) return sp[xr() % 8];
    if (mode == 1) return (double)(int)(xr() % 7) - 3;
    b = xr(); if (((b >> 52) & 0x7ff) == 0x7ff) b ^= 1ull << 62; double d; memcpy(&d, &b, 8); return d;
}
int main() {
    const int n = 1 << 22;
    std::vector<double> a(n), b(n), o1(n), o2(n);
    for (int i = 0; i < n; ++i) { a[i] = rd(); b[i] = rd(); }
    double *da, *db, *d1, *d2;
    cudaMalloc(&da, n * 8); cudaMalloc(&db, n * 8); cudaMalloc(&d1, n * 8); cudaMalloc(&d2, n * 8);
    cudaMemcpy(da, a.data(), n * 8, cudaMemcpyHostToDevice); cudaMemcpy(db, b.data(), n * 8, cudaMemcpyHostToDevice);
    k<<<n / 256, 256>>>(da, db, d1, d2, n);
    cudaMemcpy(o1.data(), d1, n * 8, cudaMemcpyDeviceToHost); cudaMemcpy(o2.data(), d2, n * 8, cudaMemcpyDeviceToHost);
    long bad1 = 0, bad2 = 0;
    for (int i = 0; i < n; ++i) {
        double r = ref(a[i], b[i]);
        if (memcmp(&r, &o1[i], 8)) { if (bad1 < 5) printf("int: a=%a b=%a ref=%a got=%a\n", a[i], b[i], r, o1[i]); ++bad1; }
        if (memcmp(&r, &o2[i], 8)) { if (bad2 < 5) printf("fp:  a=%a b=%a ref=%a got=%a\n", a[i], b[i], r, o2[i]); ++bad2; }
    }
    printf("n=%d bad_int=%ld bad_fp=%ld\n", n, bad1, bad2);
    return 0;
}
