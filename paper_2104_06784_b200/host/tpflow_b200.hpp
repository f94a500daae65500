// tpflow_b200 — C++ host API of the B200 time-stepping core.
//
// The reference's public solver API (/root/reference/proj/include/tpflow/*.hpp:
// Field, ElevationGrid, ModelParams, ScalingConfig, SimConfig, Hydrograph,
// MixtureState, SimSnapshot, MassAudit, RunReport, Simulator, run_simulation and
// the io:: readers/writers) re-provided in namespace tpflow_b200 with the same
// names, argument meaning and exceptions, so host code written against
// `tpflow::` switches by changing the namespace.  Everything on the hot path runs
// in the sm_100a kernels behind the C ABI (include/tpflow_b200.h); this layer only
// parses inputs, marshals arrays and drives Simulator::run's loop
// (solver.cpp:619-659), whose inner steps are device-resident (tp_steps).
//
// Differences, all forced by device residency:
//   * Simulator takes a DeviceConfig instead of a `Backend&`;
//   * state() returns a downloaded copy (set_state uploads);
//   * the step pieces act on the device state (apply_boundaries(MixtureState&, t)
//     keeps the reference signature by uploading/downloading `s`).
#pragma once

#include <array>
#include <cstddef>
#include <functional>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

struct tp_ctx;

namespace tpflow_b200 {

inline constexpr int kGhost = 3;  // solver.hpp:14

// errors.hpp:8-21 (CLI exit codes 2/3/4)
struct ConfigError : std::runtime_error {
    explicit ConfigError(const std::string& m) : std::runtime_error(m) {}
};
struct IoError : std::runtime_error {
    explicit IoError(const std::string& m) : std::runtime_error(m) {}
};
struct NumericsError : std::runtime_error {
    explicit NumericsError(const std::string& m) : std::runtime_error(m) {}
};
struct DeviceError : std::runtime_error {  // CUDA failures (exit code 5)
    explicit DeviceError(const std::string& m) : std::runtime_error(m) {}
};

// field.hpp:11-43 — dense 2-D array, index (i east, j north), j-major.
class Field {
public:
    Field() = default;
    Field(int nx, int ny, double init = 0.0)
        : nx_(nx), ny_(ny), data_(static_cast<std::size_t>(nx) * ny, init) {}
    int nx() const { return nx_; }
    int ny() const { return ny_; }
    std::size_t size() const { return data_.size(); }
    double& operator()(int i, int j) { return data_[static_cast<std::size_t>(j) * nx_ + i]; }
    double operator()(int i, int j) const { return data_[static_cast<std::size_t>(j) * nx_ + i]; }
    double& operator[](std::size_t k) { return data_[k]; }
    double operator[](std::size_t k) const { return data_[k]; }
    double* data() { return data_.data(); }
    const double* data() const { return data_.data(); }
    void fill(double v) { data_.assign(data_.size(), v); }
    bool same_shape(const Field& o) const { return nx_ == o.nx_ && ny_ == o.ny_; }

private:
    int nx_ = 0, ny_ = 0;
    std::vector<double> data_;
};

// params.hpp:12-51
struct ScalingConfig {
    double L = 1.0, H = 1.0, g = 9.80665;
    double epsilon() const { return H / L; }
    double t_unit() const;
    double v_unit() const;
    void validate() const;
};

struct ModelParams {
    double delta_b = 16.0, C_d = 6.0, N_R = 268.0, theta_b = 5.0, phi_s0 = 0.5, alpha_rho = 0.4, chi = 1.0;
    double tan_delta_b() const;
    void validate() const;
};

// config.hpp:12-82
struct SimConfig {
    enum class Mode { FiniteRelease, InflowHydrograph };
    ModelParams params;
    ScalingConfig scaling;
    Mode mode = Mode::FiniteRelease;
    double t_end = 0.0, dt_out = 0.0, cfl = 0.1, h_dry = 1e-10, eps_h = 1e-6;
    std::string dem_path, init_path, init_vx_path, init_vy_path, hydrograph_path, out_dir = ".";
    void validate() const;
};

struct SimSnapshot {
    double t = 0.0;
    long step_index = 0;
    Field h_total, phi_s, vX_s, vY_s, vX_f, vY_f;
};

struct MassAudit {
    double initial = 0.0, final_mass = 0.0, injected = 0.0, outflow = 0.0, clipped = 0.0;
    double drift() const { return final_mass - (initial + injected - outflow + clipped); }
    double reference() const;
};

struct RunReport {
    long steps = 0;
    double wall_seconds = 0.0;
    MassAudit solid, fluid;
};

// hydrograph.hpp:12-77
struct Hydrograph {
    struct Cell {
        int i = 0, j = 0;
        char side = 'E';
    };
    struct Sample {
        double t = 0.0, h = 0.0, phi_s = 0.0, speed = 0.0;
    };
    std::vector<Cell> cells;
    std::vector<Sample> samples;
    Sample at(double t) const;
    void validate(int ncols, int nrows) const;
};

// terrain.hpp:15-29
struct ElevationGrid {
    int ncols = 0, nrows = 0;
    double xll = 0.0, yll = 0.0, cellsize = 0.0, nodata = -9999.0;
    std::vector<std::string> header_lines;
    Field z;
    bool congruent(const ElevationGrid& o) const {
        return ncols == o.ncols && nrows == o.nrows && xll == o.xll && yll == o.yll && cellsize == o.cellsize;
    }
};
ElevationGrid load_dem(const std::string& path);
ElevationGrid parse_dem_text(const std::string& text, const std::string& origin = "<memory>");

// state.hpp:13-30
struct MixtureState {
    int nx = 0, ny = 0;
    Field ws, wf, qsx, qsy, qfx, qfy;
    MixtureState() = default;
    MixtureState(int nx_, int ny_)
        : nx(nx_), ny(ny_), ws(nx_, ny_), wf(nx_, ny_), qsx(nx_, ny_), qsy(nx_, ny_), qfx(nx_, ny_), qfy(nx_, ny_) {}
    std::array<Field*, 6> fields() { return {&ws, &wf, &qsx, &qsy, &qfx, &qfy}; }
    std::array<const Field*, 6> fields() const { return {&ws, &wf, &qsx, &qsy, &qfx, &qfy}; }
    static constexpr const char* field_names[6] = {"ws", "wf", "qsx", "qsy", "qfx", "qfy"};
};

// io.hpp:15-40
namespace io {
SimConfig parse_par_list(const std::string& path);
SimConfig parse_par_list_text(const std::string& text, const std::string& origin = "<memory>");
Field load_initial_thickness(const std::string& path, const ElevationGrid& dem, bool allow_negative = false);
Hydrograph load_hydrograph(const std::string& path, const ElevationGrid& dem);
Hydrograph parse_hydrograph_text(const std::string& text, const ElevationGrid& dem,
                                 const std::string& origin = "<memory>");
std::string time_tag(double t_seconds);
std::vector<std::string> write_snapshot(const SimSnapshot& snap, const ElevationGrid& dem, const std::string& out_dir);
std::string write_contour_csv(const SimSnapshot& snap, const ElevationGrid& dem, const std::string& out_dir);
}  // namespace io

// replaces the reference's `Backend&` (parallel.hpp:40-84)
struct DeviceConfig {
    int device = 0;
    bool fastdiv = true;   // exact shared-reciprocal division
    int graph_steps = 16;  // device steps per CUDA graph replay
};

// solver.hpp:26-98
class Simulator {
public:
    Simulator(SimConfig config, const ElevationGrid& dem, DeviceConfig device = {});
    ~Simulator();
    Simulator(const Simulator&) = delete;
    Simulator& operator=(const Simulator&) = delete;

    void set_initial_thickness(const Field& h_meters);
    void set_initial_velocity(const Field& vx, const Field& vy);
    void set_hydrograph(Hydrograph hydrograph);

    RunReport run(const std::function<void(const SimSnapshot&)>& sink);

    // the step pieces (solver.hpp:41-47), scaled times, on the device state
    void apply_boundaries(double t_scaled);
    void apply_boundaries(MixtureState& s, double t_scaled);
    double compute_dt(double t_scaled, double t_next_scaled);
    void advance_step(double dt_scaled, double t_scaled);
    void regularize();
    SimSnapshot snapshot(double t_scaled, long step_index) const;
    // device-resident loop body (tp_steps): steps from t until the exact hit of t_next
    long steps(double& t_scaled, double t_next_scaled, double t_end_scaled, long max_steps, bool* hit = nullptr);

    MixtureState state() const;
    void set_state(const MixtureState& s);
    std::vector<double> geometry() const;  // 14 padded fields, terrain.hpp:59-63 order
    const SimConfig& config() const { return cfg_; }
    MassAudit solid_audit() const;
    MassAudit fluid_audit() const;
    double interior_mass_solid() const;
    double interior_mass_fluid() const;
    void set_advection_only(bool on);
    int nx() const { return nx_; }
    int ny() const { return ny_; }
    tp_ctx* handle() const { return ctx_; }

private:
    void check(int rc) const;
    std::array<double, 10> audit() const;
    void set_audit(const std::array<double, 10>& a);

    SimConfig cfg_;
    ElevationGrid dem_;
    tp_ctx* ctx_ = nullptr;
    int nx_ = 0, ny_ = 0;
    double dxi_ = 0.0, deta_ = 0.0;
};

// solver.hpp:101-102 / solver.cpp:661-677
RunReport run_simulation(const SimConfig& config, DeviceConfig device,
                         const std::function<void(const SimSnapshot&)>& sink);

}  // namespace tpflow_b200
