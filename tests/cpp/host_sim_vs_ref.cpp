// TEST (GPU): tpflow_b200::Simulator / run_simulation (C++ host layer over the C ABI, sm_100a
// kernels) against the UNMODIFIED reference tpflow::Simulator in one process: same par_list,
// DEM, init and hydrograph files; RunReport, every snapshot file (bytes) and the final padded
// state (bits) must match.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "tpflow/io.hpp"
#include "tpflow/parallel.hpp"
#include "tpflow/solver.hpp"
#include "tpflow_b200.hpp"
#include "tpflow_b200_scenarios.hpp"

static int failures = 0;
#define EXPECT(c, msg)                                                                  \
    do {                                                                                \
        if (!(c)) {                                                                     \
            ++failures;                                                                 \
            std::fprintf(stderr, "FAIL %s:%d %s\n", __FILE__, __LINE__, std::string(msg).c_str()); \
        }                                                                               \
    } while (0)

static std::string slurp(const std::string& p) {
    std::ifstream f(p); std::stringstream s; s << f.rdbuf(); return s.str();
}

static void write_grid(const std::string& path, const tpflow_b200::ElevationGrid& g, const tpflow_b200::Field& f) {
    std::ofstream o(path);
    for (auto& l : g.header_lines) o << l << "\n";
    char b[64];
    for (int j = g.nrows - 1; j >= 0; --j) {
        for (int i = 0; i < g.ncols; ++i) { std::snprintf(b, sizeof b, "%.17g", f(i, j)); o << b << (i + 1 < g.ncols ? " " : ""); }
        o << "\n";
    }
}

static void run_case(const std::string& dir, const std::string& name, const std::string& par) {
    const std::string pfile = dir + "/" + name + ".par";
    { std::ofstream o(pfile); o << par; }
    if (std::system(("mkdir -p " + dir + "/out_ref_" + name + " " + dir + "/out_b200_" + name).c_str()) != 0) std::fprintf(stderr, "mkdir failed\n");
    // the reference: tpflow::run_simulation with the serial backend (goldens)
    tpflow::SimConfig cr = tpflow::io::parse_par_list(pfile);
    cr.out_dir = dir + "/out_ref_" + name;
    tpflow::Backend be(tpflow::BackendConfig::serial());
    tpflow::ElevationGrid demr = tpflow::load_dem(cr.dem_path);
    std::vector<std::string> files_r;
    tpflow::RunReport rr = tpflow::run_simulation(cr, be, [&](const tpflow::SimSnapshot& s) {
        for (auto& p : tpflow::io::write_snapshot(s, demr, cr.out_dir)) files_r.push_back(p);
        files_r.push_back(tpflow::io::write_contour_csv(s, demr, cr.out_dir));
    });
    // the drop-in: same call shape, B200 device
    tpflow_b200::SimConfig cb = tpflow_b200::io::parse_par_list(pfile);
    cb.out_dir = dir + "/out_b200_" + name;
    tpflow_b200::ElevationGrid demb = tpflow_b200::load_dem(cb.dem_path);
    std::vector<std::string> files_b;
    tpflow_b200::RunReport rb = tpflow_b200::run_simulation(cb, tpflow_b200::DeviceConfig{}, [&](const tpflow_b200::SimSnapshot& s) {
        for (auto& p : tpflow_b200::io::write_snapshot(s, demb, cb.out_dir)) files_b.push_back(p);
        files_b.push_back(tpflow_b200::io::write_contour_csv(s, demb, cb.out_dir));
    });
    EXPECT(rr.steps == rb.steps, name + ": steps " + std::to_string(rr.steps) + " vs " + std::to_string(rb.steps));
    EXPECT(rr.solid.initial == rb.solid.initial && rr.fluid.initial == rb.fluid.initial, name + ": initial mass");
    EXPECT(rr.solid.final_mass == rb.solid.final_mass && rr.fluid.final_mass == rb.fluid.final_mass, name + ": final mass");
    auto close = [](double a, double b) { return std::abs(a - b) <= 1e-12 * std::max(1.0, std::abs(a)); };
    EXPECT(close(rr.solid.injected, rb.solid.injected) && close(rr.solid.outflow, rb.solid.outflow) &&
           close(rr.fluid.injected, rb.fluid.injected) && close(rr.fluid.outflow, rb.fluid.outflow), name + ": audit");
    EXPECT(files_r.size() == files_b.size() && !files_r.empty(), name + ": output file count");
    for (std::size_t k = 0; k < files_r.size() && k < files_b.size(); ++k) {
        const std::string a = slurp(files_r[k]), b = slurp(files_b[k]);
        EXPECT(a == b && !a.empty(), name + ": output bytes differ: " + files_r[k]);
    }
    std::printf("%s: %ld steps, %zu output files compared, wall ref %.2fs b200 %.2fs\n", name.c_str(), rr.steps,
                files_r.size(), rr.wall_seconds, rb.wall_seconds);
}

int main(int argc, char** argv) {
    const std::string dir = argc > 1 ? argv[1] : "/tmp/tpb_host";
    if (std::system(("mkdir -p " + dir).c_str()) != 0) std::fprintf(stderr, "mkdir failed\n");
    // Mode-I: hill on an incline (input files written with %.17g so both read identical values)
    {
        auto dem = tpflow_b200::scenarios::incline_dem(72, 60, 5.0, 15.0);
        for (int j = 0; j < 60; ++j)
            for (int i = 0; i < 72; ++i)
                dem.z(i, j) += 20.0 * std::exp(-((i - 30.0) * (i - 30.0) + (j - 30.0) * (j - 30.0)) / 120.0);
        write_grid(dir + "/hill.asc", dem, dem.z);
        write_grid(dir + "/hill_h.asc", dem, tpflow_b200::scenarios::gaussian_release(72, 60, 4.0, 7.0, 50.0, 30.0));
        run_case(dir, "release",
                 "mode = release\ndem = " + dir + "/hill.asc\ninit = " + dir + "/hill_h.asc\nout_dir = x\n"
                 "t_end = 6\ndt_out = 1.5\ndelta_b = 16\nC_d = 6\nN_R = 268\ntheta_b = 5\nphi_s0 = 0.5\n");
    }
    // Mode-II: channel with a triangular hydrograph starting dry
    {
        auto dem = tpflow_b200::scenarios::channel_dem(90, 40, 5.0, 10.0, 25.0);
        write_grid(dir + "/chan.asc", dem, dem.z);
        std::ofstream q(dir + "/chan.hyd");
        for (int j = 15; j < 25; ++j) q << "cell 89 " << j << " E\n";
        q << "t h phi_s speed\n0 0 0.55 0\n10 2.0 0.55 3.0\n20 0 0.55 0\n";
        q.close();
        run_case(dir, "inflow",
                 "mode = inflow\ndem = " + dir + "/chan.asc\nhydrograph = " + dir + "/chan.hyd\nout_dir = x\n"
                 "t_end = 12\ndt_out = 0.5\ndelta_b = 16\nC_d = 6\nN_R = 268\ntheta_b = 5\nphi_s0 = 0.5\n");
    }
    std::printf("%s: %d failures\n", argv[0], failures);
    return failures ? 1 : 0;
}
