// tpflow_b200 — command-line entry points of SPEC.md's cli module (run / validate /
// bench), which the reference declares but does not ship
// (proj/CMakeLists.txt:16, no tools/).  Exit codes: 0 ok, 2 ConfigError, 3 IoError,
// 4 NumericsError, 5 device error, 6 validation failure (errors.hpp:8-21).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "tpflow_b200.hpp"
#include "tpflow_b200_scenarios.hpp"

using namespace tpflow_b200;

namespace {

int usage() {
    std::fprintf(stderr,
                 "usage: tpflow_b200 run <par_list> [--device N] [--no-output]\n"
                 "       tpflow_b200 validate [--suite all|conservation|quiescence|symmetry|inflow] [--device N]\n"
                 "       tpflow_b200 bench [--meshes 10000,50000,...] [--steps N] [--repeats R] [--device N]\n");
    return 2;
}

const char* opt(int argc, char** argv, const char* name, const char* def) {
    for (int k = 0; k + 1 < argc; ++k)
        if (std::strcmp(argv[k], name) == 0) return argv[k + 1];
    return def;
}

bool flag(int argc, char** argv, const char* name) {
    for (int k = 0; k < argc; ++k)
        if (std::strcmp(argv[k], name) == 0) return true;
    return false;
}

SimConfig mem_config(SimConfig::Mode mode, double t_end, double dt_out) {
    SimConfig c;
    c.mode = mode;
    c.t_end = t_end;
    c.dt_out = dt_out;
    c.dem_path = "<memory>";
    c.init_path = "<memory>";
    c.hydrograph_path = "<memory>";
    return c;
}

int cmd_run(int argc, char** argv) {
    if (argc < 1) return usage();
    const SimConfig cfg = io::parse_par_list(argv[0]);
    DeviceConfig dev;
    dev.device = std::atoi(opt(argc, argv, "--device", "0"));
    const bool write = !flag(argc, argv, "--no-output");
    const ElevationGrid dem = load_dem(cfg.dem_path);
    int n_out = 0;
    const RunReport r = run_simulation(cfg, dev, [&](const SimSnapshot& s) {
        if (!write) return;
        io::write_snapshot(s, dem, cfg.out_dir);
        io::write_contour_csv(s, dem, cfg.out_dir);
        ++n_out;
    });
    std::printf("steps %ld  wall %.3f s  snapshots %d\n", r.steps, r.wall_seconds, n_out);
    const MassAudit* a[2] = {&r.solid, &r.fluid};
    const char* names[2] = {"solid", "fluid"};
    for (int p = 0; p < 2; ++p)
        std::printf("%s: initial %.12e final %.12e injected %.6e outflow %.6e clipped %.3e drift %.3e (rel %.3e)\n",
                    names[p], a[p]->initial, a[p]->final_mass, a[p]->injected, a[p]->outflow, a[p]->clipped,
                    a[p]->drift(), a[p]->drift() / a[p]->reference());
    return 0;
}

struct Check {
    std::string name;
    double value, tol;
};

// SPEC.md acceptance criteria as device runs.
int cmd_validate(int argc, char** argv) {
    const std::string suite = opt(argc, argv, "--suite", "all");
    DeviceConfig dev;
    dev.device = std::atoi(opt(argc, argv, "--device", "0"));
    std::vector<Check> checks;
    auto want = [&](const char* s) { return suite == "all" || suite == s; };

    if (want("conservation")) {  // closed basin, 1000 steps: |drift| / initial < 1e-10
        ElevationGrid dem = scenarios::bowl_dem(96, 96, 5.0, 60.0);
        Simulator sim(mem_config(SimConfig::Mode::FiniteRelease, 1e9, 1e9), dem, dev);
        sim.set_initial_thickness(scenarios::gaussian_release(96, 96, 3.0, 8.0, 47.5, 47.5));
        double t = 0.0;
        const double m0 = sim.interior_mass_solid(), f0 = sim.interior_mass_fluid();
        sim.steps(t, 1e9, 1e9, 1000);
        checks.push_back({"conservation solid (1000 steps)", std::abs(sim.interior_mass_solid() - m0) / m0, 1e-10});
        checks.push_back({"conservation fluid (1000 steps)", std::abs(sim.interior_mass_fluid() - f0) / f0, 1e-10});
    }
    if (want("quiescence")) {  // uniform depth at rest on flat terrain stays at rest (1e-12)
        ElevationGrid dem = scenarios::flat_dem(64, 64, 5.0, 3.0);
        Simulator sim(mem_config(SimConfig::Mode::FiniteRelease, 1e9, 1e9), dem, dev);
        Field h(64, 64, 2.0);
        sim.set_initial_thickness(h);
        double t = 0.0;
        sim.steps(t, 1e9, 1e9, 1000);
        const SimSnapshot s = sim.snapshot(t, 1000);
        double vmax = 0.0;
        for (std::size_t k = 0; k < s.vX_s.size(); ++k)
            vmax = std::max({vmax, std::abs(s.vX_s[k]), std::abs(s.vY_s[k]), std::abs(s.vX_f[k]), std::abs(s.vY_f[k])});
        checks.push_back({"quiescence max |v| (1000 steps)", vmax, 1e-12});
    }
    if (want("symmetry")) {  // transpose symmetry, 100 steps (1e-12)
        const int n = 80;
        ElevationGrid dem = scenarios::bowl_dem(n, n, 5.0, 40.0);
        Simulator sim(mem_config(SimConfig::Mode::FiniteRelease, 1e9, 1e9), dem, dev);
        sim.set_initial_thickness(scenarios::gaussian_release(n, n, 4.0, 10.0, 30.0, 30.0));
        double t = 0.0;
        sim.steps(t, 1e9, 1e9, 100);
        const SimSnapshot s = sim.snapshot(t, 100);
        double d = 0.0, ref = 0.0;
        for (int j = 0; j < n; ++j)
            for (int i = 0; i < n; ++i) {
                d = std::max(d, std::abs(s.h_total(i, j) - s.h_total(j, i)));
                d = std::max(d, std::abs(s.vX_s(i, j) - s.vY_s(j, i)));
                ref = std::max(ref, std::abs(s.h_total(i, j)));
            }
        checks.push_back({"transpose symmetry (100 steps, rel)", d / std::max(ref, 1e-300), 1e-12});
    }
    if (want("inflow")) {  // Mode-II: final = initial + injected - outflow + clipped (1e-6 rel)
        ElevationGrid dem = scenarios::channel_dem(120, 48, 5.0, 10.0, 30.0);
        SimConfig cfg = mem_config(SimConfig::Mode::InflowHydrograph, 40.0, 0.5);
        Simulator sim(cfg, dem, dev);
        sim.set_hydrograph(scenarios::triangular_hydrograph(dem, 'E', 18, 12, 0.0, 30.0, 2.0, 0.55, 4.0));
        const RunReport r = sim.run(nullptr);
        checks.push_back({"Mode-II bookkeeping solid (rel)", std::abs(r.solid.drift()) / r.solid.reference(), 1e-6});
        checks.push_back({"Mode-II bookkeeping fluid (rel)", std::abs(r.fluid.drift()) / r.fluid.reference(), 1e-6});
    }
    int bad = 0;
    for (const auto& c : checks) {
        const bool ok = c.value <= c.tol;
        bad += !ok;
        std::printf("%-40s %.3e  (tol %.0e)  %s\n", c.name.c_str(), c.value, c.tol, ok ? "PASS" : "FAIL");
    }
    return bad ? 6 : 0;
}

// SPEC.md:428-440 mesh campaign (CFL-controlled device steps; mean of R repeats).
int cmd_bench(int argc, char** argv) {
    std::vector<long> meshes;
    std::stringstream ss(opt(argc, argv, "--meshes", "10000,50000,100000,250000,500000,1000000"));
    for (std::string tok; std::getline(ss, tok, ',');) meshes.push_back(std::atol(tok.c_str()));
    const long steps = std::atol(opt(argc, argv, "--steps", "1000"));
    const int repeats = std::atoi(opt(argc, argv, "--repeats", "3"));
    DeviceConfig dev;
    dev.device = std::atoi(opt(argc, argv, "--device", "0"));
    std::printf("mesh_count,backend,steps,mean_wall_seconds,cell_updates_per_s\n");
    for (long m : meshes) {
        const int n = std::max(8, static_cast<int>(std::lround(std::sqrt(static_cast<double>(m)))));
        ElevationGrid dem = scenarios::incline_dem(n, n, 5.0, 20.0);
        double total = 0.0;
        for (int r = 0; r < repeats; ++r) {
            Simulator sim(mem_config(SimConfig::Mode::FiniteRelease, 1e9, 1e9), dem, dev);
            sim.set_initial_thickness(scenarios::gaussian_release(n, n, 5.0, 0.1 * n, 0.5 * n, 0.5 * n));
            double t = 0.0;
            sim.steps(t, 1e9, 1e9, 5);  // warm-up
            const auto t0 = std::chrono::steady_clock::now();
            sim.steps(t, 1e9, 1e9, steps);
            total += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        }
        const double mean = total / repeats;
        std::printf("%ld,b200,%ld,%.6f,%.4e\n", static_cast<long>(n) * n, steps, mean,
                    static_cast<double>(n) * n * steps / mean);
    }
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) return usage();
    const std::string cmd = argv[1];
    try {
        if (cmd == "run") return cmd_run(argc - 2, argv + 2);
        if (cmd == "validate") return cmd_validate(argc - 2, argv + 2);
        if (cmd == "bench") return cmd_bench(argc - 2, argv + 2);
        return usage();
    } catch (const ConfigError& e) {
        std::fprintf(stderr, "config error: %s\n", e.what());
        return 2;
    } catch (const IoError& e) {
        std::fprintf(stderr, "io error: %s\n", e.what());
        return 3;
    } catch (const NumericsError& e) {
        std::fprintf(stderr, "numerics error: %s\n", e.what());
        return 4;
    } catch (const DeviceError& e) {
        std::fprintf(stderr, "device error: %s\n", e.what());
        return 5;
    }
}
