// Timing probe of the host snapshot writers (2048^2, 6 asc grids + contour CSV into /dev/shm/wt_out):
// g++ -std=gnu++20 -O2 -Ipaper_2104_06784_b200/host scripts/probes/writer_probe.cpp paper_2104_06784_b200/host/io.cpp -lpthread
#include <chrono>
#include <cstdio>
#include <string>
#include "tpflow_b200.hpp"
int main() {
    const int N = 2048;
    std::string text = "ncols " + std::to_string(N) + "\nnrows " + std::to_string(N) + "\nxllcorner 0\nyllcorner 0\ncellsize 5\nnodata_value -9999\n";
    std::string row; for (int i = 0; i < N; ++i) row += (i ? " 1" : "1"); row += "\n";
    for (int j = 0; j < N; ++j) text += row;
    auto dem = tpflow_b200::parse_dem_text(text, "t");
    tpflow_b200::SimSnapshot s; s.t = 10.0;
    tpflow_b200::Field* f[6] = {&s.h_total, &s.phi_s, &s.vX_s, &s.vY_s, &s.vX_f, &s.vY_f};
    for (int k = 0; k < 6; ++k) { *f[k] = tpflow_b200::Field(N, N); for (int j = 0; j < N; ++j) for (int i = 0; i < N; ++i) (*f[k])(i, j) = 0.001 * (i + j * 3 + k); }
    auto t0 = std::chrono::steady_clock::now();
    tpflow_b200::io::write_snapshot(s, dem, "/dev/shm/wt_out");
    auto t1 = std::chrono::steady_clock::now();
    tpflow_b200::io::write_contour_csv(s, dem, "/dev/shm/wt_out");
    auto t2 = std::chrono::steady_clock::now();
    std::printf("6 asc grids %.2f s, contour csv %.2f s\n", std::chrono::duration<double>(t1 - t0).count(), std::chrono::duration<double>(t2 - t1).count());
}
