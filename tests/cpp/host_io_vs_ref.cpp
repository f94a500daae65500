// TEST (CPU): tpflow_b200's host I/O against the UNMODIFIED reference (tpflow::, oracle/_ref
// objects) in one process — parsed values, error messages and written file bytes must match.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

#include "tpflow/config.hpp"
#include "tpflow/errors.hpp"
#include "tpflow/io.hpp"
#include "tpflow/terrain.hpp"
#include "tpflow_b200.hpp"

static int failures = 0;
#define EXPECT(c, msg)                                                   \
    do {                                                                 \
        if (!(c)) {                                                      \
            ++failures;                                                  \
            std::fprintf(stderr, "FAIL %s:%d %s\n", __FILE__, __LINE__, (msg)); \
        }                                                                \
    } while (0)

template <class B, class A>
static std::string err_of(A fa) {
    try { fa(); } catch (const B& e) { return std::string("E:") + e.what(); }
    catch (const std::exception& e) { return std::string("X:") + e.what(); }
    return "ok";
}

static std::string slurp(const std::string& p) {
    std::ifstream f(p); std::stringstream s; s << f.rdbuf(); return s.str();
}

int main(int argc, char** argv) {
    const std::string dir = argc > 1 ? argv[1] : "/tmp";
    // ---- par_list: valid + every error class
    const std::vector<std::string> pars = {
        "mode = release\ndem = d.asc\ninit = h.asc\nout_dir = o\nt_end = 10\ndt_out = 1\n"
        "delta_b = 16\nC_d = 6.0\nN_R = 268\ntheta_b = 5.0\nphi_s0 = 0.5  # Table 1\ncfl=0.1\n",
        "mode = inflow\ndem = d.asc\nhydrograph = q.txt\nout_dir = o\nt_end = 60\ndt_out = 0.5\n"
        "delta_b = 20\nC_d = 4\nN_R = 100\ntheta_b = 3\nphi_s0 = 0.6\nalpha_rho=0.5\nchi=2\nL=2\nH=2\n",
        "mode = release\ndem = d.asc\nout_dir = o\nt_end = 10\ndt_out = 1\ndelta_b = 16\nC_d = 6\nN_R = 268\ntheta_b = 5\nphi_s0 = 0.5\n",
        "mode = release\nfoo = 1\n", "mode = release\nmode = inflow\n", "mode =\n", "just words\n",
        "dem = d.asc\n", "mode = sideways\ndem = d\ninit = i\nout_dir = o\nt_end = 1\ndt_out = 1\ndelta_b = 1\nC_d = 1\nN_R = 1\ntheta_b = 1\nphi_s0 = 0.5\n",
        "mode = release\ndem = d\ninit = i\nout_dir = o\nt_end = 1\ndt_out = 1\ndelta_b = 1\nC_d = 1\nN_R = 1\ntheta_b = 1\nphi_s0 = 0.5\ncfl = 0.2\n",
        "mode = release\ndem = d\ninit = i\nout_dir = o\nt_end = 1\ndt_out = 1\ndelta_b = 1x\nC_d = 1\nN_R = 1\ntheta_b = 1\nphi_s0 = 0.5\n",
        "mode = release\ndem = d\ninit = i\nout_dir = o\nt_end = -1\ndt_out = 1\ndelta_b = 1\nC_d = 1\nN_R = 1\ntheta_b = 1\nphi_s0 = 0.5\n",
        "mode = release\ndem = d\ninit = i\nout_dir = o\nt_end = 1\ndt_out = 1\ndelta_b = 95\nC_d = 1\nN_R = 1\ntheta_b = 1\nphi_s0 = 0.5\n",
    };
    for (const auto& t : pars) {
        std::string er, eb;
        tpflow::SimConfig cr; tpflow_b200::SimConfig cb;
        er = err_of<tpflow::ConfigError>([&] { cr = tpflow::io::parse_par_list_text(t, "p"); });
        eb = err_of<tpflow_b200::ConfigError>([&] { cb = tpflow_b200::io::parse_par_list_text(t, "p"); });
        EXPECT(er == eb, (er + " | " + eb).c_str());
        if (er == "ok" && eb == "ok") {
            EXPECT(cr.params.delta_b == cb.params.delta_b && cr.params.C_d == cb.params.C_d &&
                   cr.params.N_R == cb.params.N_R && cr.params.theta_b == cb.params.theta_b &&
                   cr.params.phi_s0 == cb.params.phi_s0 && cr.params.alpha_rho == cb.params.alpha_rho &&
                   cr.params.chi == cb.params.chi && cr.scaling.L == cb.scaling.L && cr.scaling.H == cb.scaling.H &&
                   cr.scaling.g == cb.scaling.g && cr.t_end == cb.t_end && cr.dt_out == cb.dt_out &&
                   cr.cfl == cb.cfl && cr.h_dry == cb.h_dry && cr.eps_h == cb.eps_h &&
                   (int)cr.mode == (int)cb.mode && cr.dem_path == cb.dem_path && cr.init_path == cb.init_path &&
                   cr.hydrograph_path == cb.hydrograph_path && cr.out_dir == cb.out_dir, "par_list values");
        }
    }
    // ---- DEM text: SPEC.md:54-57 examples + errors
    const std::vector<std::string> dems = {
        "ncols 2\nnrows 2\nxllcorner 0\nyllcorner 0\ncellsize 10\nNODATA_value -9999\n1 2\n3 4\n",
        "NCOLS 3\nNROWS 2\nXLLCORNER 5.5\nYLLCORNER -2\nCELLSIZE 2.5\nnodata_value -1\n1 2 3\n4 5 6\n",
        "ncols 2\nnrows 2\nxllcorner 0\nyllcorner 0\ncellsize 10\nNODATA_value -9999\n1 -9999\n3 4\n",
        "ncols 2\nnrows 2\nxllcorner 0\nyllcorner 0\ncellsize 10\nNODATA_value -9999\n1 2\n3\n",
        "ncols 2\nnrows 2\nxllcorner 0\nyllcorner 0\ncellsize 10\nNODATA_value -9999\n1 2\n3 4 5\n",
        "ncols 2\nnrows 2\n", "ncols 2\nrows 2\nxllcorner 0\nyllcorner 0\ncellsize 10\nNODATA_value -9999\n",
        "ncols 1\nnrows 2\nxllcorner 0\nyllcorner 0\ncellsize 10\nNODATA_value -9999\n1\n2\n",
        "ncols 2\nnrows 2\nxllcorner 0\nyllcorner 0\ncellsize 0\nNODATA_value -9999\n1 2\n3 4\n",
    };
    for (const auto& t : dems) {
        tpflow::ElevationGrid gr; tpflow_b200::ElevationGrid gb;
        const std::string er = err_of<tpflow::IoError>([&] { gr = tpflow::parse_dem_text(t, "d"); });
        const std::string eb = err_of<tpflow_b200::IoError>([&] { gb = tpflow_b200::parse_dem_text(t, "d"); });
        EXPECT(er == eb, (er + " | " + eb).c_str());
        if (er == "ok" && eb == "ok") {
            bool same = gr.ncols == gb.ncols && gr.nrows == gb.nrows && gr.xll == gb.xll && gr.yll == gb.yll &&
                        gr.cellsize == gb.cellsize && gr.nodata == gb.nodata && gr.header_lines == gb.header_lines;
            for (int j = 0; same && j < gr.nrows; ++j)
                for (int i = 0; i < gr.ncols; ++i) same = same && gr.z(i, j) == gb.z(i, j);
            EXPECT(same, "dem values");
        }
    }
    // ---- hydrograph text
    tpflow::ElevationGrid demr = tpflow::parse_dem_text(dems[1], "d");
    tpflow_b200::ElevationGrid demb = tpflow_b200::parse_dem_text(dems[1], "d");
    const std::vector<std::string> hyds = {
        "cell 2 0 E\ncell 2 1 E\nt h phi_s speed\n0 0.5 0.5 1.0\n60 1.0 0.5 2.0\n",
        "cell 0 1 N  # top\nt h phi_s speed\n0 0 0.5 0\n10 1 0.5 1\n5 2 0.5 1\n",
        "cell 1 1 E\nt h phi_s speed\n0 1 0.5 1\n", "cell 1 0 S\nt h phi_s speed\n0 -1 0.5 1\n",
        "cell 1 0 S\nt h phi_s speed\n0 1 1.5 1\n", "cell 1 0 Q\nt h phi_s speed\n0 1 0.5 1\n",
        "t h phi_s speed\n0 1 0.5 1\n", "cell 0 0 W\n", "cell 0 0 W\nt h x speed\n", "bogus\n",
        "cell 0 0 W\nt h phi_s speed\n0 1 0.5\n",
    };
    for (const auto& t : hyds) {
        tpflow::Hydrograph hr; tpflow_b200::Hydrograph hb;
        const std::string er = err_of<tpflow::ConfigError>([&] { hr = tpflow::io::parse_hydrograph_text(t, demr, "q"); });
        const std::string eb = err_of<tpflow_b200::ConfigError>([&] { hb = tpflow_b200::io::parse_hydrograph_text(t, demb, "q"); });
        EXPECT(er == eb, (er + " | " + eb).c_str());
        if (er == "ok") {
            bool same = hr.cells.size() == hb.cells.size() && hr.samples.size() == hb.samples.size();
            for (double tt : {-1.0, 0.0, 5.0, 30.0, 59.0, 60.0, 61.0}) {
                auto a = hr.at(tt); auto b = hb.at(tt);
                same = same && a.t == b.t && a.h == b.h && a.phi_s == b.phi_s && a.speed == b.speed;
            }
            EXPECT(same, "hydrograph values / at()");
        }
    }
    // ---- writers: identical bytes for identical snapshots
    tpflow::SimSnapshot sr; tpflow_b200::SimSnapshot sb;
    sr.t = sb.t = 181.82;
    tpflow::Field* fr[6] = {&sr.h_total, &sr.phi_s, &sr.vX_s, &sr.vY_s, &sr.vX_f, &sr.vY_f};
    tpflow_b200::Field* fb[6] = {&sb.h_total, &sb.phi_s, &sb.vX_s, &sb.vY_s, &sb.vX_f, &sb.vY_f};
    for (int k = 0; k < 6; ++k) {
        *fr[k] = tpflow::Field(3, 2); *fb[k] = tpflow_b200::Field(3, 2);
        for (int j = 0; j < 2; ++j)
            for (int i = 0; i < 3; ++i) (*fr[k])(i, j) = (*fb[k])(i, j) = 0.1234567 * (k + 1) * (i - j) + 1e-7 * k;
    }
    const std::string dr = dir + "/ref", db = dir + "/b200";
    if (std::system(("mkdir -p " + dr + " " + db).c_str()) != 0) std::fprintf(stderr, "mkdir failed\n");
    auto pr = tpflow::io::write_snapshot(sr, demr, dr);
    auto pb = tpflow_b200::io::write_snapshot(sb, demb, db);
    EXPECT(pr.size() == pb.size(), "snapshot file count");
    for (std::size_t k = 0; k < pr.size() && k < pb.size(); ++k)
        EXPECT(slurp(pr[k]) == slurp(pb[k]) && !slurp(pr[k]).empty(), ("snapshot bytes " + pr[k]).c_str());
    const std::string cr = tpflow::io::write_contour_csv(sr, demr, dr), cb = tpflow_b200::io::write_contour_csv(sb, demb, db);
    EXPECT(slurp(cr) == slurp(cb), "contour csv bytes");
    EXPECT(tpflow::io::time_tag(181.82) == tpflow_b200::io::time_tag(181.82), "time tag");
    {
        // a grid large enough for the multi-threaded writers (row blocks on every host thread)
        const int NC = 211, NR = 157;
        std::string text = "ncols " + std::to_string(NC) + "\nnrows " + std::to_string(NR) +
                           "\nxllcorner 100.5\nyllcorner -20\ncellsize 2.5\nnodata_value -9999\n";
        for (int j = 0; j < NR; ++j) {
            for (int i = 0; i < NC; ++i) text += std::to_string((i * 7 + j * 3) % 50) + (i + 1 < NC ? " " : "\n");
        }
        tpflow::ElevationGrid gr = tpflow::parse_dem_text(text, "big");
        tpflow_b200::ElevationGrid gb = tpflow_b200::parse_dem_text(text, "big");
        tpflow::SimSnapshot br; tpflow_b200::SimSnapshot bb;
        br.t = bb.t = 3600.0;
        tpflow::Field* gfr[6] = {&br.h_total, &br.phi_s, &br.vX_s, &br.vY_s, &br.vX_f, &br.vY_f};
        tpflow_b200::Field* gfb[6] = {&bb.h_total, &bb.phi_s, &bb.vX_s, &bb.vY_s, &bb.vX_f, &bb.vY_f};
        unsigned long long r = 2104;
        for (int k = 0; k < 6; ++k) {
            *gfr[k] = tpflow::Field(NC, NR); *gfb[k] = tpflow_b200::Field(NC, NR);
            for (int j = 0; j < NR; ++j)
                for (int i = 0; i < NC; ++i) {
                    r = r * 6364136223846793005ull + 1442695040888963407ull;
                    const double u = static_cast<double>(r >> 11) * (1.0 / 9007199254740992.0);
                    const double v = (i + j) % 17 == 0 ? -0.0 : (u - 0.4) * std::pow(10.0, (k + i) % 9 - 4);
                    (*gfr[k])(i, j) = (*gfb[k])(i, j) = v;
                }
        }
        const std::string dr2 = dir + "/ref_big", db2 = dir + "/b200_big";
        if (std::system(("mkdir -p " + dr2 + " " + db2).c_str()) != 0) std::fprintf(stderr, "mkdir failed\n");
        auto qr = tpflow::io::write_snapshot(br, gr, dr2);
        auto qb = tpflow_b200::io::write_snapshot(bb, gb, db2);
        for (std::size_t k = 0; k < qr.size() && k < qb.size(); ++k)
            EXPECT(slurp(qr[k]) == slurp(qb[k]) && !slurp(qr[k]).empty(), ("large snapshot bytes " + qr[k]).c_str());
        EXPECT(slurp(tpflow::io::write_contour_csv(br, gr, dr2)) == slurp(tpflow_b200::io::write_contour_csv(bb, gb, db2)),
               "large contour csv bytes");
    }
    std::printf("%s: %d failures\n", argv[0], failures);
    return failures ? 1 : 0;
}
