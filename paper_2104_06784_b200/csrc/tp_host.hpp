// Host-side (CPU) pieces of the framework that the reference computes on the
// host too: DEM extension + terrain geometry (built once, consumed by every
// kernel), and the snapshot conversion.  Compiled with -ffp-contract=off so the
// arithmetic is bit-identical to the reference build.
#pragma once

#include <string>
#include <vector>

namespace tpb {
namespace host {

constexpr int kGhost = 3;  // solver.hpp:14

// ElevationGrid (terrain.hpp:15-29) reduced to what the path needs.
struct Dem {
    int ncols = 0, nrows = 0;
    double xll = 0.0, yll = 0.0, cellsize = 0.0;
    std::vector<double> z;  // ncols*nrows, j-major, south row first
};

// extend_grid (terrain.cpp:113-145): ghost rings by linear extrapolation.
Dem extend_grid(const Dem& grid, int ghost);

// compute_geometry (terrain.cpp:157-215): 14 padded fields, TerrainGeometry
// declaration order, each nx*ny.  Rows are computed in parallel (pure per cell).
struct Geometry {
    int nx = 0, ny = 0;
    double dxi = 0.0, deta = 0.0;
    std::vector<double> f;  // 14 * nx * ny
    const double* field(int k) const { return f.data() + static_cast<size_t>(k) * nx * ny; }
    double* field(int k) { return f.data() + static_cast<size_t>(k) * nx * ny; }
};
Geometry compute_geometry(const Dem& ext, double L);

// std::to_string(double) == "%f"
std::string to_string_f(double v);

}  // namespace host
}  // namespace tpb
