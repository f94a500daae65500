// tpflow_b200::Simulator — the reference's Simulator (solver.hpp:26-98) over the C ABI.
#include <chrono>
#include <climits>
#include <cmath>
#include <cstring>

#include "../../include/tpflow_b200.h"
#include "tpflow_b200.hpp"

namespace tpflow_b200 {

void Simulator::check(int rc) const {
    if (rc == TP_OK) return;
    const std::string msg = tp_last_error(ctx_);
    if (rc == TP_ERR_CONFIG) throw ConfigError(msg);
    if (rc == TP_ERR_IO) throw IoError(msg);
    if (rc == TP_ERR_NUMERICS) throw NumericsError(msg);
    throw DeviceError(msg);
}

// solver.cpp:13-33
Simulator::Simulator(SimConfig config, const ElevationGrid& dem, DeviceConfig device)
    : cfg_(std::move(config)), dem_(dem) {
    cfg_.validate();
    tp_params p{};
    p.delta_b = cfg_.params.delta_b;
    p.C_d = cfg_.params.C_d;
    p.N_R = cfg_.params.N_R;
    p.theta_b = cfg_.params.theta_b;
    p.phi_s0 = cfg_.params.phi_s0;
    p.alpha_rho = cfg_.params.alpha_rho;
    p.chi = cfg_.params.chi;
    p.L = cfg_.scaling.L;
    p.H = cfg_.scaling.H;
    p.g = cfg_.scaling.g;
    p.t_end = cfg_.t_end;
    p.dt_out = cfg_.dt_out;
    p.cfl = cfg_.cfl;
    p.h_dry = cfg_.h_dry;
    p.eps_h = cfg_.eps_h;
    p.mode = cfg_.mode == SimConfig::Mode::InflowHydrograph ? 1 : 0;
    p.device = device.device;
    tp_dem d{dem_.ncols, dem_.nrows, dem_.xll, dem_.yll, dem_.cellsize, dem_.z.data()};
    const int rc = tp_create(&p, &d, &ctx_);
    if (rc != TP_OK) {
        const std::string msg = ctx_ ? tp_last_error(ctx_) : "tp_create failed";
        tp_destroy(ctx_);
        ctx_ = nullptr;
        if (rc == TP_ERR_CONFIG) throw ConfigError(msg);
        throw DeviceError(msg);
    }
    check(tp_dims(ctx_, &nx_, &ny_, &dxi_, &deta_));
    check(tp_set_option(ctx_, "fastdiv", device.fastdiv ? 1 : 0));
    check(tp_set_option(ctx_, "graph_steps", device.graph_steps));
}

Simulator::~Simulator() { tp_destroy(ctx_); }

// solver.cpp:35-57
void Simulator::set_initial_thickness(const Field& h) {
    if (h.nx() != dem_.ncols || h.ny() != dem_.nrows)
        throw ConfigError("initial state: dimension mismatch with DEM (" + std::to_string(h.nx()) + "x" +
                          std::to_string(h.ny()) + " vs " + std::to_string(dem_.ncols) + "x" +
                          std::to_string(dem_.nrows) + ")");
    check(tp_set_initial_thickness(ctx_, h.data()));
}

// solver.cpp:59-76
void Simulator::set_initial_velocity(const Field& vx, const Field& vy) {
    if (vx.nx() != dem_.ncols || vx.ny() != dem_.nrows || !vx.same_shape(vy))
        throw ConfigError("initial velocity: dimension mismatch with DEM");
    check(tp_set_initial_velocity(ctx_, vx.data(), vy.data()));
}

// solver.cpp:78-81
void Simulator::set_hydrograph(Hydrograph hg) {
    hg.validate(dem_.ncols, dem_.nrows);
    std::vector<int> ci, cj;
    std::string side;
    for (const auto& c : hg.cells) {
        ci.push_back(c.i);
        cj.push_back(c.j);
        side.push_back(c.side);
    }
    std::vector<double> t, h, phi, sp;
    for (const auto& s : hg.samples) {
        t.push_back(s.t);
        h.push_back(s.h);
        phi.push_back(s.phi_s);
        sp.push_back(s.speed);
    }
    check(tp_set_hydrograph(ctx_, static_cast<int>(ci.size()), ci.data(), cj.data(), side.data(),
                            static_cast<int>(t.size()), t.data(), h.data(), phi.data(), sp.data()));
}

void Simulator::apply_boundaries(double t) { check(tp_apply_boundaries(ctx_, t)); }

void Simulator::apply_boundaries(MixtureState& s, double t) {
    set_state(s);
    apply_boundaries(t);
    s = state();
}

double Simulator::compute_dt(double t, double t_next) {
    double dt = 0.0;
    check(tp_compute_dt(ctx_, t, t_next, &dt));
    return dt;
}

void Simulator::advance_step(double dt, double t) { check(tp_advance_step(ctx_, dt, t)); }

void Simulator::regularize() { check(tp_regularize(ctx_)); }

void Simulator::set_advection_only(bool on) { check(tp_set_advection_only(ctx_, on ? 1 : 0)); }

long Simulator::steps(double& t, double t_next, double t_end, long max_steps, bool* hit) {
    long n = 0;
    int h = 0;
    check(tp_steps(ctx_, t_next, t_end, max_steps, &t, &n, &h, nullptr));
    if (hit) *hit = h != 0;
    return n;
}

MixtureState Simulator::state() const {
    MixtureState s(nx_, ny_);
    std::vector<double> buf(6ull * nx_ * ny_);
    check(tp_get_state(ctx_, buf.data()));
    auto f = s.fields();
    for (int k = 0; k < 6; ++k)
        std::memcpy(f[k]->data(), buf.data() + static_cast<std::size_t>(k) * nx_ * ny_,
                    sizeof(double) * nx_ * ny_);
    return s;
}

void Simulator::set_state(const MixtureState& s) {
    std::vector<double> buf(6ull * nx_ * ny_);
    auto f = s.fields();
    for (int k = 0; k < 6; ++k)
        std::memcpy(buf.data() + static_cast<std::size_t>(k) * nx_ * ny_, f[k]->data(),
                    sizeof(double) * nx_ * ny_);
    check(tp_set_state(ctx_, buf.data()));
}

std::vector<double> Simulator::geometry() const {
    std::vector<double> g(14ull * nx_ * ny_);
    check(tp_get_geometry(ctx_, g.data()));
    return g;
}

std::array<double, 10> Simulator::audit() const {
    std::array<double, 10> a{};
    check(tp_get_audit(ctx_, a.data()));
    return a;
}

void Simulator::set_audit(const std::array<double, 10>& a) { check(tp_set_audit(ctx_, a.data())); }

MassAudit Simulator::solid_audit() const {
    const auto a = audit();
    return MassAudit{a[0], a[1], a[2], a[3], a[4]};
}

MassAudit Simulator::fluid_audit() const {
    const auto a = audit();
    return MassAudit{a[5], a[6], a[7], a[8], a[9]};
}

double Simulator::interior_mass_solid() const {
    double ms = 0.0, mf = 0.0;
    check(tp_interior_mass(ctx_, &ms, &mf));
    return ms;
}

double Simulator::interior_mass_fluid() const {
    double ms = 0.0, mf = 0.0;
    check(tp_interior_mass(ctx_, &ms, &mf));
    return mf;
}

// solver.cpp:590-617 (computed on the host from the downloaded state by tp_snapshot)
SimSnapshot Simulator::snapshot(double t_scaled, long step_index) const {
    SimSnapshot snap;
    snap.t = t_scaled * cfg_.scaling.t_unit();
    snap.step_index = step_index;
    const int nc = dem_.ncols, nr = dem_.nrows;
    std::vector<double> buf(6ull * nc * nr);
    check(tp_snapshot(ctx_, buf.data()));
    Field* out[6] = {&snap.h_total, &snap.phi_s, &snap.vX_s, &snap.vY_s, &snap.vX_f, &snap.vY_f};
    for (int k = 0; k < 6; ++k) {
        *out[k] = Field(nc, nr);
        std::memcpy(out[k]->data(), buf.data() + static_cast<std::size_t>(k) * nc * nr, sizeof(double) * nc * nr);
    }
    return snap;
}

// solver.cpp:619-659; the loop body runs device-resident between output times
RunReport Simulator::run(const std::function<void(const SimSnapshot&)>& sink) {
    RunReport report;
    std::array<double, 10> a{};
    set_audit(a);
    regularize();
    a = audit();
    check(tp_interior_mass(ctx_, &a[0], &a[5]));
    set_audit(a);

    const double t_unit = cfg_.scaling.t_unit();
    const double t_end = cfg_.t_end / t_unit;
    const double dt_out = cfg_.dt_out / t_unit;
    double t = 0.0;
    long steps_done = 0;
    if (sink) sink(snapshot(t, steps_done));
    double next_out = dt_out;

    const auto t0 = std::chrono::steady_clock::now();
    while (t < t_end) {
        const double t_next = std::min(next_out, t_end);
        bool hit = false;
        steps_done += steps(t, t_next, t_end, LONG_MAX, &hit);
        if (hit) {
            if (sink) sink(snapshot(t, steps_done));
            if (t_next == next_out) next_out += dt_out;
        }
    }
    const auto t1 = std::chrono::steady_clock::now();

    report.steps = steps_done;
    report.wall_seconds = std::chrono::duration<double>(t1 - t0).count();
    a = audit();
    check(tp_interior_mass(ctx_, &a[1], &a[6]));
    set_audit(a);
    report.solid = MassAudit{a[0], a[1], a[2], a[3], a[4]};
    report.fluid = MassAudit{a[5], a[6], a[7], a[8], a[9]};
    return report;
}

// solver.cpp:661-677
RunReport run_simulation(const SimConfig& config, DeviceConfig device,
                         const std::function<void(const SimSnapshot&)>& sink) {
    const ElevationGrid dem = load_dem(config.dem_path);
    Simulator sim(config, dem, device);
    if (config.mode == SimConfig::Mode::FiniteRelease) {
        sim.set_initial_thickness(io::load_initial_thickness(config.init_path, dem));
        if (!config.init_vx_path.empty() || !config.init_vy_path.empty()) {
            if (config.init_vx_path.empty() || config.init_vy_path.empty())
                throw ConfigError("init_vx and init_vy must be given together");
            sim.set_initial_velocity(io::load_initial_thickness(config.init_vx_path, dem, true),
                                     io::load_initial_thickness(config.init_vy_path, dem, true));
        }
    } else {
        sim.set_hydrograph(io::load_hydrograph(config.hydrograph_path, dem));
    }
    return sim.run(sink);
}

}  // namespace tpflow_b200
