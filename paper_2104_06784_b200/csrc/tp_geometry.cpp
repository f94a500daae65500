// Terrain geometry on the host, restating /root/reference/proj/src/terrain.cpp
// (extend_grid :113-145, slopes :21-45, compute_geometry :157-215,
// basal_transform :147-155) operation for operation.  Built with
// -ffp-contract=off: the padded geometry fields are bit-identical to the
// reference's TerrainGeometry (checked by tests/test_geometry.py).
#include <cmath>
#include <cstdio>
#include <thread>

#include "tp_host.hpp"

namespace tpb {
namespace host {

namespace {

// terrain.cpp:23-31
inline double deriv(double m1, double p1, double spacing) { return (p1 - m1) / (2.0 * spacing); }
inline double deriv_low(double f0, double f1, double f2, double spacing) {
    return (-3.0 * f0 + 4.0 * f1 - f2) / (2.0 * spacing);
}
inline double deriv_high(double f0, double f1, double f2, double spacing) {
    return (3.0 * f0 - 4.0 * f1 + f2) / (2.0 * spacing);
}

// terrain.cpp:33-45 on a dense nx*ny field
inline double diff_x(const double* f, int nx, int i, int j, double d) {
    const double* r = f + static_cast<size_t>(j) * nx;
    if (i == 0) return deriv_low(r[0], r[1], r[2], d);
    if (i == nx - 1) return deriv_high(r[nx - 1], r[nx - 2], r[nx - 3], d);
    return deriv(r[i - 1], r[i + 1], d);
}
inline double diff_y(const double* f, int nx, int ny, int i, int j, double d) {
    auto at = [&](int jj) { return f[static_cast<size_t>(jj) * nx + i]; };
    if (j == 0) return deriv_low(at(0), at(1), at(2), d);
    if (j == ny - 1) return deriv_high(at(ny - 1), at(ny - 2), at(ny - 3), d);
    return deriv(at(j - 1), at(j + 1), d);
}

template <class F>
void parallel_rows(int ny, F&& fn) {
    unsigned hw = std::thread::hardware_concurrency();
    int nt = static_cast<int>(hw ? hw : 1);
    if (nt > 32) nt = 32;
    if (static_cast<long long>(ny) * 64 < 4096 || nt == 1) {
        fn(0, ny);
        return;
    }
    std::vector<std::thread> th;
    int chunk = (ny + nt - 1) / nt;
    for (int t = 0; t < nt; ++t) {
        int b = t * chunk, e = std::min(ny, b + chunk);
        if (b >= e) break;
        th.emplace_back([&, b, e] { fn(b, e); });
    }
    for (auto& x : th) x.join();
}

}  // namespace

Dem extend_grid(const Dem& grid, int ghost) {
    Dem out;
    out.ncols = grid.ncols + 2 * ghost;
    out.nrows = grid.nrows + 2 * ghost;
    out.cellsize = grid.cellsize;
    out.xll = grid.xll - ghost * grid.cellsize;
    out.yll = grid.yll - ghost * grid.cellsize;
    out.z.assign(static_cast<size_t>(out.ncols) * out.nrows, 0.0);
    const int W = out.ncols;
    auto Z = [&](int i, int j) -> double& { return out.z[static_cast<size_t>(j) * W + i]; };
    for (int j = 0; j < grid.nrows; ++j)
        for (int i = 0; i < grid.ncols; ++i)
            Z(i + ghost, j + ghost) = grid.z[static_cast<size_t>(j) * grid.ncols + i];
    // west/east over interior rows, then north/south over every column (corners)
    for (int j = ghost; j < ghost + grid.nrows; ++j) {
        for (int g = 1; g <= ghost; ++g) {
            Z(ghost - g, j) = Z(ghost, j) + g * (Z(ghost, j) - Z(ghost + 1, j));
            int e = ghost + grid.ncols - 1;
            Z(e + g, j) = Z(e, j) + g * (Z(e, j) - Z(e - 1, j));
        }
    }
    for (int i = 0; i < out.ncols; ++i) {
        for (int g = 1; g <= ghost; ++g) {
            Z(i, ghost - g) = Z(i, ghost) + g * (Z(i, ghost) - Z(i, ghost + 1));
            int n = ghost + grid.nrows - 1;
            Z(i, n + g) = Z(i, n) + g * (Z(i, n) - Z(i, n - 1));
        }
    }
    return out;
}

Geometry compute_geometry(const Dem& grid, double L) {
    Geometry geo;
    geo.nx = grid.ncols;
    geo.ny = grid.nrows;
    geo.dxi = grid.cellsize / L;
    geo.deta = grid.cellsize / L;
    const int nx = geo.nx, ny = geo.ny;
    const size_t n = static_cast<size_t>(nx) * ny;
    geo.f.assign(14 * n, 0.0);

    std::vector<double> b(n);
    for (size_t k = 0; k < n; ++k) b[k] = grid.z[k] / L;

    double* nX = geo.field(0);
    double* nY = geo.field(1);
    double* nZ = geo.field(2);
    double* jb = geo.field(3);
    double* a11 = geo.field(4);
    double* a12 = geo.field(5);
    double* a21 = geo.field(6);
    double* a22 = geo.field(7);
    const double dxi = geo.dxi, deta = geo.deta;
    parallel_rows(ny, [&](int j0, int j1) {
        for (int j = j0; j < j1; ++j) {
            for (int i = 0; i < nx; ++i) {
                const size_t k = static_cast<size_t>(j) * nx + i;
                double bx = diff_x(b.data(), nx, i, j, dxi);
                double by = diff_y(b.data(), nx, ny, i, j, deta);
                double norm = std::sqrt(1.0 + (bx * bx + by * by));
                nX[k] = -bx / norm;
                nY[k] = -by / norm;
                nZ[k] = 1.0 / norm;
                // basal_transform (terrain.cpp:147-155)
                double bn = std::sqrt(1.0 + (bx * bx + by * by));
                double m[3][3] = {{1.0, 0.0, -bx / bn}, {0.0, 1.0, -by / bn}, {bx, by, 1.0 / bn}};
                double det = norm;
                jb[k] = det;
                a11[k] = (m[1][1] * m[2][2] - m[1][2] * m[2][1]) / det;
                a12[k] = (m[0][2] * m[2][1] - m[0][1] * m[2][2]) / det;
                a21[k] = (m[1][2] * m[2][0] - m[1][0] * m[2][2]) / det;
                a22[k] = (m[0][0] * m[2][2] - m[0][2] * m[2][0]) / det;
            }
        }
    });
    // normal-derivative fields (terrain.cpp:204-213)
    parallel_rows(ny, [&](int j0, int j1) {
        for (int j = j0; j < j1; ++j) {
            for (int i = 0; i < nx; ++i) {
                const size_t k = static_cast<size_t>(j) * nx + i;
                geo.field(8)[k] = diff_x(nX, nx, i, j, dxi);
                geo.field(9)[k] = diff_x(nY, nx, i, j, dxi);
                geo.field(10)[k] = diff_x(nZ, nx, i, j, dxi);
                geo.field(11)[k] = diff_y(nX, nx, ny, i, j, deta);
                geo.field(12)[k] = diff_y(nY, nx, ny, i, j, deta);
                geo.field(13)[k] = diff_y(nZ, nx, ny, i, j, deta);
            }
        }
    });
    return geo;
}

std::string to_string_f(double v) {
    char buf[512];
    std::snprintf(buf, sizeof(buf), "%f", v);
    return buf;
}

}  // namespace host
}  // namespace tpb
