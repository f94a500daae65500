// Device check of smax/smin (std::max/std::min semantics) incl. signed zeros and NaN.
#include <cstdio>
#include <cstring>
#include <cstdint>
#include <cmath>
#include "../../paper_2104_06784_b200/csrc/tp_math.cuh"
using namespace tpb;
__global__ void k(const double* a, const double* b, double* o, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        o[6 * i + 0] = smax(a[i], b[i]);
        o[6 * i + 1] = smin(a[i], b[i]);
        o[6 * i + 2] = smax(a[i], 0.0);
        o[6 * i + 3] = smax(0.0, a[i]);
        o[6 * i + 4] = smin(a[i], 0.0);
        o[6 * i + 5] = smax(fabs(a[i]), fabs(b[i])) + 1.0;
    }
}
static double hmax(double a, double b) { return (a < b) ? b : a; }
static double hmin(double a, double b) { return (b < a) ? b : a; }
int main() {
    double vals[] = {0.0, -0.0, 1.0, -1.0, NAN, -NAN, INFINITY, -INFINITY, 5e-324, -5e-324, 2.5, -2.5};
    const int nv = sizeof(vals) / 8, n = nv * nv;
    double a[n], b[n], o[6 * n];
    for (int i = 0; i < nv; ++i) for (int j = 0; j < nv; ++j) { a[i * nv + j] = vals[i]; b[i * nv + j] = vals[j]; }
    double *da, *db, *dout;
    cudaMalloc(&da, n * 8); cudaMalloc(&db, n * 8); cudaMalloc(&dout, 6 * n * 8);
    cudaMemcpy(da, a, n * 8, cudaMemcpyHostToDevice); cudaMemcpy(db, b, n * 8, cudaMemcpyHostToDevice);
    k<<<1, 256>>>(da, db, dout, n);
    cudaMemcpy(o, dout, 6 * n * 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < n; ++i) {
        double r[6] = {hmax(a[i], b[i]), hmin(a[i], b[i]), hmax(a[i], 0.0), hmax(0.0, a[i]), hmin(a[i], 0.0), hmax(fabs(a[i]), fabs(b[i])) + 1.0};
        for (int q = 0; q < 6; ++q)
            if (memcmp(&r[q], &o[6 * i + q], 8)) { if (bad < 20) printf("op%d a=%a b=%a ref=%a got=%a\n", q, a[i], b[i], r[q], o[6 * i + q]); ++bad; }
    }
    printf("bad=%d of %d\n", bad, 6 * n);
    return 0;
}
