// Synthetic inputs: the generators the reference declares but never defines
// (/root/reference/proj/include/tpflow/scenarios.hpp:12-33), same signatures.
#include <cmath>

#include "tpflow_b200.hpp"
#include "tpflow_b200_scenarios.hpp"

namespace tpflow_b200::scenarios {

namespace {

ElevationGrid make_grid(int ncols, int nrows, double cellsize) {
    ElevationGrid g;
    g.ncols = ncols;
    g.nrows = nrows;
    g.cellsize = cellsize;
    g.header_lines = {"ncols " + std::to_string(ncols), "nrows " + std::to_string(nrows), "xllcorner 0",
                      "yllcorner 0", "cellsize " + io::time_tag(cellsize), "NODATA_value -9999"};
    g.z = Field(ncols, nrows);
    return g;
}

double cx_m(int i, double cs) { return (i + 0.5) * cs; }

}  // namespace

ElevationGrid flat_dem(int ncols, int nrows, double cellsize, double z0) {
    ElevationGrid g = make_grid(ncols, nrows, cellsize);
    g.z.fill(z0);
    return g;
}

ElevationGrid incline_dem(int ncols, int nrows, double cellsize, double slope_deg) {
    ElevationGrid g = make_grid(ncols, nrows, cellsize);
    const double s = std::tan(slope_deg * M_PI / 180.0);
    for (int j = 0; j < nrows; ++j)
        for (int i = 0; i < ncols; ++i) g.z(i, j) = cx_m(i, cellsize) * s;  // descends in -X
    return g;
}

ElevationGrid bowl_dem(int ncols, int nrows, double cellsize, double depth) {
    ElevationGrid g = make_grid(ncols, nrows, cellsize);
    const double xc = 0.5 * ncols * cellsize, yc = 0.5 * nrows * cellsize;
    const double R = std::min(xc, yc);
    for (int j = 0; j < nrows; ++j)
        for (int i = 0; i < ncols; ++i) {
            const double dx = cx_m(i, cellsize) - xc, dy = cx_m(j, cellsize) - yc;
            g.z(i, j) = depth * ((dx * dx + dy * dy) / (R * R));
        }
    return g;
}

ElevationGrid channel_dem(int ncols, int nrows, double cellsize, double slope_deg, double wall_height) {
    ElevationGrid g = make_grid(ncols, nrows, cellsize);
    const double s = std::tan(slope_deg * M_PI / 180.0);
    const double half = 0.5 * nrows * cellsize;
    for (int j = 0; j < nrows; ++j)
        for (int i = 0; i < ncols; ++i) {
            const double w = (cx_m(j, cellsize) - half) / half;
            g.z(i, j) = cx_m(i, cellsize) * s + wall_height * w * w;
        }
    return g;
}

Field gaussian_release(int ncols, int nrows, double amplitude, double width, double cx, double cy, double base) {
    Field h(ncols, nrows);
    for (int j = 0; j < nrows; ++j)
        for (int i = 0; i < ncols; ++i) {
            const double r2 = (i - cx) * (i - cx) + (j - cy) * (j - cy);
            h(i, j) = amplitude * std::exp(-r2 / (width * width)) + base;
        }
    return h;
}

Hydrograph triangular_hydrograph(const ElevationGrid& dem, char side, int first_cell, int n_cells, double t0,
                                 double t1, double peak_h, double phi_s, double peak_speed) {
    Hydrograph hg;
    for (int k = first_cell; k < first_cell + n_cells; ++k) {
        Hydrograph::Cell c;
        c.side = side;
        if (side == 'E') { c.i = dem.ncols - 1; c.j = k; }
        else if (side == 'W') { c.i = 0; c.j = k; }
        else if (side == 'N') { c.i = k; c.j = dem.nrows - 1; }
        else { c.i = k; c.j = 0; }
        hg.cells.push_back(c);
    }
    hg.samples = {{t0, 0.0, phi_s, 0.0}, {0.5 * (t0 + t1), peak_h, phi_s, peak_speed}, {t1, 0.0, phi_s, 0.0}};
    return hg;
}

}  // namespace tpflow_b200::scenarios
