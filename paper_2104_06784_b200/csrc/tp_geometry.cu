// Terrain geometry on the device: extend_grid (terrain.cpp:113-145),
// the slope derivatives (:21-45), compute_geometry (:157-215) and basal_transform
// (:147-155), operation for operation with IEEE division/sqrt and no FMA contraction
// (--fmad=false), so every field is bit-identical to the reference's host geometry
// (tests/test_gpu_parity.py::test_device_geometry_bitwise).  Written straight into the
// device layout of tp_types.h (GeoField), with the four correctly rounded reciprocals.
#include <cuda_runtime.h>

#include "tp_types.h"

namespace tpb {

namespace {

// terrain.cpp:23-31
__device__ __forceinline__ double deriv(double m1, double p1, double spacing) { return (p1 - m1) / (2.0 * spacing); }
__device__ __forceinline__ double deriv_low(double f0, double f1, double f2, double spacing) {
    return (-3.0 * f0 + 4.0 * f1 - f2) / (2.0 * spacing);
}
__device__ __forceinline__ double deriv_high(double f0, double f1, double f2, double spacing) {
    return (3.0 * f0 - 4.0 * f1 + f2) / (2.0 * spacing);
}

struct Ext {  // the extended DEM (all global rows), dense NX x NY
    const double* z;
    int NX, NY;
};

// b(i, j) = z(i, j) / L on the extended grid (compute_geometry :170-173)
__device__ __forceinline__ double bval(const Ext& e, double L, int i, int j) {
    return e.z[static_cast<long long>(j) * e.NX + i] / L;
}

}  // namespace

// extend_grid part 1: the interior plus the west/east linear extrapolation of every
// interior row (terrain.cpp:125-137).  One thread per extended cell of the interior rows.
__global__ void geo_extend_we_kernel(const double* __restrict__ dem, int ncols, int nrows, double* __restrict__ z) {
    const int NX = ncols + 6;
    const long long n = static_cast<long long>(NX) * nrows;
    for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < n;
         k += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int jj = static_cast<int>(k / NX), i = static_cast<int>(k - static_cast<long long>(jj) * NX);
        const int j = jj + 3;
        const double* row = dem + static_cast<long long>(jj) * ncols;
        double v;
        if (i >= 3 && i < 3 + ncols) {
            v = row[i - 3];
        } else if (i < 3) {  // out.z(3-g, j) = out.z(3, j) + g*(out.z(3, j) - out.z(4, j))
            const int g = 3 - i;
            v = row[0] + g * (row[0] - row[1]);
        } else {             // out.z(e+g, j) = out.z(e, j) + g*(out.z(e, j) - out.z(e-1, j))
            const int g = i - (2 + ncols);
            v = row[ncols - 1] + g * (row[ncols - 1] - row[ncols - 2]);
        }
        z[static_cast<long long>(j) * NX + i] = v;
    }
}

// extend_grid part 2: the north/south extrapolation of every column, corners included
// (terrain.cpp:138-144), from the rows written by part 1.
__global__ void geo_extend_ns_kernel(int ncols, int nrows, double* __restrict__ z) {
    const int NX = ncols + 6;
    const int n = NX * 6;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const int i = k % NX, r = k / NX;  // r: 0..2 south ghosts (g = 3-r), 3..5 north (g = r-2)
        const int nr = 3 + nrows - 1;
        const double* z3 = z + 3ll * NX;
        const double* z4 = z + 4ll * NX;
        const double* zn = z + static_cast<long long>(nr) * NX;
        const double* zn1 = z + static_cast<long long>(nr - 1) * NX;
        if (r < 3) {
            const int g = 3 - r;
            z[static_cast<long long>(3 - g) * NX + i] = z3[i] + g * (z3[i] - z4[i]);
        } else {
            const int g = r - 2;
            z[static_cast<long long>(nr + g) * NX + i] = zn[i] + g * (zn[i] - zn1[i]);
        }
    }
}

// compute_geometry's first loop (terrain.cpp:175-202) on global extended rows [g0, g1):
// nX, nY, nZ, jb, a11, a12, a21, a22 into dense scratch rows (8 fields, row gj - g0).
__global__ void geo_pass1_kernel(Ext e, double L, double dxi, double deta, int g0, int g1,
                                 double* __restrict__ out) {
    const long long rows = g1 - g0;
    const long long n = rows * e.NX, fs = n;
    for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < n;
         k += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int jr = static_cast<int>(k / e.NX), i = static_cast<int>(k - static_cast<long long>(jr) * e.NX);
        const int j = g0 + jr;
        double bx, by;
        if (i == 0) bx = deriv_low(bval(e, L, 0, j), bval(e, L, 1, j), bval(e, L, 2, j), dxi);
        else if (i == e.NX - 1) bx = deriv_high(bval(e, L, e.NX - 1, j), bval(e, L, e.NX - 2, j), bval(e, L, e.NX - 3, j), dxi);
        else bx = deriv(bval(e, L, i - 1, j), bval(e, L, i + 1, j), dxi);
        if (j == 0) by = deriv_low(bval(e, L, i, 0), bval(e, L, i, 1), bval(e, L, i, 2), deta);
        else if (j == e.NY - 1) by = deriv_high(bval(e, L, i, e.NY - 1), bval(e, L, i, e.NY - 2), bval(e, L, i, e.NY - 3), deta);
        else by = deriv(bval(e, L, i, j - 1), bval(e, L, i, j + 1), deta);
        const double norm = sqrt(1.0 + (bx * bx + by * by));
        // basal_transform (terrain.cpp:147-155): columns (1,0,bx), (0,1,by), unit normal
        const double m02 = -bx / norm, m12 = -by / norm, m20 = bx, m21 = by, m22 = 1.0 / norm;
        const double det = norm;
        out[0 * fs + k] = -bx / norm;                         // nX
        out[1 * fs + k] = -by / norm;                         // nY
        out[2 * fs + k] = 1.0 / norm;                         // nZ
        out[3 * fs + k] = det;                                // jb
        out[4 * fs + k] = (1.0 * m22 - m12 * m21) / det;      // a11 = (m11 m22 - m12 m21) / det
        out[5 * fs + k] = (m02 * m21 - 0.0 * m22) / det;      // a12 = (m02 m21 - m01 m22) / det
        out[6 * fs + k] = (m12 * m20 - 0.0 * m22) / det;      // a21 = (m12 m20 - m10 m22) / det
        out[7 * fs + k] = (1.0 * m22 - m02 * m20) / det;      // a22 = (m00 m22 - m02 m20) / det
    }
}

// The device layout of the slab rows [row0, row0 + ny): the pass-1 fields, the normal
// derivatives (terrain.cpp:204-213, diff_x/diff_y of the stored normals) and the four
// reciprocals RN(1/jb), RN(1/nZ), RN(1/jbf) of the xi and eta faces.
__global__ void geo_pass2_kernel(const double* __restrict__ p1, int NX, int NY, int g0, int g1, int row0,
                                 int ny, double dxi, double deta, GridDesc g, double* __restrict__ geo) {
    const long long pfs = static_cast<long long>(g1 - g0) * NX;
    const long long n = static_cast<long long>(ny) * NX;
    for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < n;
         k += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int j = static_cast<int>(k / NX), i = static_cast<int>(k - static_cast<long long>(j) * NX);
        const int gj = row0 + j;
        auto at = [&](int f, int ii, int jj) { return p1[f * pfs + static_cast<long long>(jj - g0) * NX + ii]; };
        auto dx = [&](int f) {
            if (i == 0) return deriv_low(at(f, 0, gj), at(f, 1, gj), at(f, 2, gj), dxi);
            if (i == NX - 1) return deriv_high(at(f, NX - 1, gj), at(f, NX - 2, gj), at(f, NX - 3, gj), dxi);
            return deriv(at(f, i - 1, gj), at(f, i + 1, gj), dxi);
        };
        auto dy = [&](int f) {
            if (gj == 0) return deriv_low(at(f, i, 0), at(f, i, 1), at(f, i, 2), deta);
            if (gj == NY - 1) return deriv_high(at(f, i, NY - 1), at(f, i, NY - 2), at(f, i, NY - 3), deta);
            return deriv(at(f, i, gj - 1), at(f, i, gj + 1), deta);
        };
        const long long o = static_cast<long long>(j) * g.pitch + i;
        const double jb = at(3, i, gj), nZ = at(2, i, gj);
        geo[G_JB * g.fs + o] = jb;
        geo[G_RJB * g.fs + o] = 1.0 / jb;
        geo[G_NZ * g.fs + o] = nZ;
        geo[G_A11 * g.fs + o] = at(4, i, gj);
        geo[G_A12 * g.fs + o] = at(5, i, gj);
        geo[G_A21 * g.fs + o] = at(6, i, gj);
        geo[G_A22 * g.fs + o] = at(7, i, gj);
        geo[G_RJBFX * g.fs + o] = i + 1 < NX ? 1.0 / (0.5 * (jb + at(3, i + 1, gj))) : 0.0;
        geo[G_RJBFY * g.fs + o] = gj + 1 < NY ? 1.0 / (0.5 * (jb + at(3, i, gj + 1))) : 0.0;
        geo[G_NX * g.fs + o] = at(0, i, gj);
        geo[G_NY * g.fs + o] = at(1, i, gj);
        geo[G_DNX_DXI * g.fs + o] = dx(0);
        geo[G_DNY_DXI * g.fs + o] = dx(1);
        geo[G_DNZ_DXI * g.fs + o] = dx(2);
        geo[G_DNX_DETA * g.fs + o] = dy(0);
        geo[G_DNY_DETA * g.fs + o] = dy(1);
        geo[G_DNZ_DETA * g.fs + o] = dy(2);
        geo[G_RNZ * g.fs + o] = 1.0 / nZ;
    }
}

// Build the slab's device geometry from the DEM (host, dense ncols x nrows).
cudaError_t build_geometry_device(const double* dem_h, int ncols, int nrows, double L, double cellsize, int row0,
                                  int ny, const GridDesc& g, double* geo, cudaStream_t st) {
    const int NX = ncols + 6, NY = nrows + 6;
    const double dxi = cellsize / L, deta = cellsize / L;
    const int g0 = row0 - 2 < 0 ? 0 : row0 - 2;
    const int g1 = row0 + ny + 2 > NY ? NY : row0 + ny + 2;
    double *d_dem = nullptr, *d_z = nullptr, *d_p1 = nullptr;
    const size_t dem_b = sizeof(double) * static_cast<size_t>(ncols) * nrows;
    cudaError_t e = cudaMalloc(&d_dem, dem_b);
    if (e == cudaSuccess) e = cudaMalloc(&d_z, sizeof(double) * static_cast<size_t>(NX) * NY);
    if (e == cudaSuccess) e = cudaMalloc(&d_p1, sizeof(double) * 8ull * (g1 - g0) * NX);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d_dem, dem_h, dem_b, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) {
        geo_extend_we_kernel<<<1184, 256, 0, st>>>(d_dem, ncols, nrows, d_z);
        geo_extend_ns_kernel<<<64, 256, 0, st>>>(ncols, nrows, d_z);
        geo_pass1_kernel<<<1184, 256, 0, st>>>(Ext{d_z, NX, NY}, L, dxi, deta, g0, g1, d_p1);
        geo_pass2_kernel<<<1184, 256, 0, st>>>(d_p1, NX, NY, g0, g1, row0, ny, dxi, deta, g, geo);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(d_dem);  // null-safe
    cudaFree(d_z);
    cudaFree(d_p1);
    return e;
}

// ---- setup kernels on the device layout ------------------------------------------

// Simulator::set_initial_thickness (solver.cpp:35-57) on the slab's interior cells; h is
// the slab's rows of the thickness grid (dense ncols x nrows, metres).
__global__ void init_thickness_kernel(GridDesc g, const double* __restrict__ geo, const double* __restrict__ h,
                                      int ncols, int nrows, double H, double phi, double* s) {
    const long long n = static_cast<long long>(ncols) * nrows;
    for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < n;
         q += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int j = static_cast<int>(q / ncols), i = static_cast<int>(q - static_cast<long long>(j) * ncols);
        const long long k = static_cast<long long>(j + 3) * g.pitch + (i + 3);
        const double jb = geo[G_JB * g.fs + k];
        const double h_scaled = h[q] / H;
        s[0 * g.fs + k] = jb * h_scaled * phi;
        s[1 * g.fs + k] = jb * h_scaled * (1.0 - phi);
        s[2 * g.fs + k] = 0.0;
        s[3 * g.fs + k] = 0.0;
        s[4 * g.fs + k] = 0.0;
        s[5 * g.fs + k] = 0.0;
    }
}

// Simulator::set_initial_velocity (solver.cpp:59-76) on the slab's interior cells.
__global__ void init_velocity_kernel(GridDesc g, const double* __restrict__ geo, const double* __restrict__ vx,
                                     const double* __restrict__ vy, int ncols, int nrows, double vu, double* s) {
    const long long n = static_cast<long long>(ncols) * nrows;
    for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < n;
         q += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int j = static_cast<int>(q / ncols), i = static_cast<int>(q - static_cast<long long>(j) * ncols);
        const long long k = static_cast<long long>(j + 3) * g.pitch + (i + 3);
        const double jb = geo[G_JB * g.fs + k];
        const double hs = s[0 * g.fs + k] / jb;
        const double hf = s[1 * g.fs + k] / jb;
        const double ux = vx[q] / vu, uy = vy[q] / vu;
        s[2 * g.fs + k] = jb * hs * ux;
        s[3 * g.fs + k] = jb * hs * uy;
        s[4 * g.fs + k] = jb * hf * ux;
        s[5 * g.fs + k] = jb * hf * uy;
    }
}

// The geometry part of the safe-tile conditions (DESIGN.md §3 item 6): all 14 reference
// fields finite; jb in [1, 2^50] (so nZ = 1/jb >= 2^-50); the metric coefficients a_ij 0 or
// of magnitude in [2^-128, 2^50]; nX, nY 0 or of magnitude >= 2^-200.  (The normal
// derivatives only enter curvature terms, never a numerator.)  *ok starts at 1 and is
// cleared by any violation.
__global__ void geo_check_kernel(GridDesc g, const double* __restrict__ geo, int* ok) {
    const long long n = static_cast<long long>(g.ny) * g.nx;
    bool good = true;
    auto mag = [](double v, double lo, double hi) {
        const double a = fabs(v);
        return a == 0.0 || (a >= lo && a <= hi);  // NaN fails both
    };
    for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < n;
         q += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int j = static_cast<int>(q / g.nx), i = static_cast<int>(q - static_cast<long long>(j) * g.nx);
        const long long k = static_cast<long long>(j) * g.pitch + i;
        const double jb = geo[G_JB * g.fs + k];
        good = good && jb >= 1.0 && jb <= 0x1p50;
        good = good && mag(geo[G_A11 * g.fs + k], 0x1p-120, 0x1p50) && mag(geo[G_A12 * g.fs + k], 0x1p-120, 0x1p50) &&
               mag(geo[G_A21 * g.fs + k], 0x1p-120, 0x1p50) && mag(geo[G_A22 * g.fs + k], 0x1p-120, 0x1p50);
        good = good && mag(geo[G_NX * g.fs + k], 0x1p-200, 1.0) && mag(geo[G_NY * g.fs + k], 0x1p-200, 1.0);
        good = good && isfinite(geo[G_NZ * g.fs + k]) && isfinite(geo[G_DNX_DXI * g.fs + k]) &&
               isfinite(geo[G_DNY_DXI * g.fs + k]) && isfinite(geo[G_DNZ_DXI * g.fs + k]) &&
               isfinite(geo[G_DNX_DETA * g.fs + k]) && isfinite(geo[G_DNY_DETA * g.fs + k]) &&
               isfinite(geo[G_DNZ_DETA * g.fs + k]);
    }
    if (!__all_sync(0xffffffffu, good) && (threadIdx.x & 31) == 0) atomicAnd(ok, 0);
}

cudaError_t launch_init_thickness(const GridDesc& g, const double* geo, const double* h, int ncols, int nrows,
                                  double H, double phi, double* s, cudaStream_t st) {
    init_thickness_kernel<<<1184, 256, 0, st>>>(g, geo, h, ncols, nrows, H, phi, s);
    return cudaGetLastError();
}
cudaError_t launch_init_velocity(const GridDesc& g, const double* geo, const double* vx, const double* vy,
                                 int ncols, int nrows, double vu, double* s, cudaStream_t st) {
    init_velocity_kernel<<<1184, 256, 0, st>>>(g, geo, vx, vy, ncols, nrows, vu, s);
    return cudaGetLastError();
}
cudaError_t launch_geo_check(const GridDesc& g, const double* geo, int* ok, cudaStream_t st) {
    geo_check_kernel<<<592, 256, 0, st>>>(g, geo, ok);
    return cudaGetLastError();
}

}  // namespace tpb
