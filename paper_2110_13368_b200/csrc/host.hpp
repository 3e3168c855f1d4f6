// Host-side C++ mirror of the reference microenvironment API
// (/root/reference/proj/src/core/{mesh,solver,agents,backend,errors}.hpp).
//
// Callers keep the reference's types and entry-point shapes; the execution
// strategy argument (WorkerPool&, backend.hpp:34) becomes a DeviceBackend&
// that owns a device-resident copy of the field and runs the sm_100a
// kernels. Setup work that the reference also does on the host (Thomas
// coefficient precompute, Dirichlet map merging, agent grouping) stays here
// and reproduces the reference's bits exactly.
#pragma once

#include <array>
#include <cstdint>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace biodiff_b200 {

using index_t = std::int64_t;

// errors.hpp:9-24 — same three categories, same exit-code mapping.
struct config_error : std::runtime_error {
    explicit config_error(const std::string& w) : std::runtime_error(w) {}
};
struct io_error : std::runtime_error {
    explicit io_error(const std::string& w) : std::runtime_error(w) {}
};
struct state_error : std::runtime_error {
    explicit state_error(const std::string& w) : std::runtime_error(w) {}
};

// mesh.hpp:17-57
struct CartesianMesh {
    double x_min = 0, x_max = 0, y_min = 0, y_max = 0, z_min = 0, z_max = 0;
    double dx = 0, dy = 0, dz = 0;
    int nx = 0, ny = 0, nz = 0;

    static CartesianMesh from_bounds(double x_min, double x_max, double y_min, double y_max, double z_min,
                                     double z_max, double dx, double dy, double dz);
    index_t voxel_count() const { return static_cast<index_t>(nx) * ny * nz; }
    double voxel_volume() const { return dx * dy * dz; }
    index_t voxel_index(int i, int j, int k) const;
    std::array<int, 3> voxel_ijk(index_t n) const;
    index_t nearest_voxel(const std::array<double, 3>& p) const;
    bool contains(const std::array<double, 3>& p) const;
    bool is_boundary_voxel(int i, int j, int k) const
    {
        return i == 0 || i == nx - 1 || j == 0 || j == ny - 1 || k == 0 || k == nz - 1;
    }
    index_t boundary_voxel_count() const;
};

// mesh.hpp:62-90: values[n*S + s].
struct DensityField {
    std::vector<double> values;
    int substrates = 0;
    DensityField() = default;
    DensityField(index_t voxels, int S, double fill = 0.0)
        : values(static_cast<std::size_t>(voxels) * S, fill), substrates(S)
    {
    }
    index_t voxel_count() const { return substrates == 0 ? 0 : static_cast<index_t>(values.size()) / substrates; }
    double& at(index_t v, int s) { return values[static_cast<std::size_t>(v) * substrates + s]; }
    double at(index_t v, int s) const { return values[static_cast<std::size_t>(v) * substrates + s]; }
    bool all_finite() const; // mesh.cpp:95-99
};

// mesh.hpp:93-100 / mesh.cpp:101-136: PhysiCell's vector-of-vectors density
// (one std::vector per voxel) <-> the flat voxel-major layout the kernels
// use. Same checks and messages as the reference.
using NestedDensity = std::vector<std::vector<double>>;
DensityField translate_vector_to_array(const NestedDensity& nested);
NestedDensity translate_array_to_vector(const DensityField& field);

// mesh.hpp:103-110
struct SubstrateParams {
    std::string name;
    double diffusion_coefficient = 0.0;
    double decay_rate = 0.0;
    double initial_condition = 0.0;
};

// mesh.hpp:113-141
struct DirichletEntry {
    index_t voxel = 0;
    std::vector<std::uint8_t> mask;
    std::vector<double> values;
};

class DirichletMap {
public:
    void add(index_t voxel, std::vector<std::uint8_t> mask, std::vector<double> values, index_t voxel_count,
             int substrates);
    void add_single(index_t voxel, int substrate, double value, index_t voxel_count, int substrates);
    bool empty() const { return entries_.empty(); }
    std::size_t size() const { return entries_.size(); }
    const std::vector<DirichletEntry>& entries() const { return entries_; }
    void clear() { entries_.clear(); }

private:
    std::vector<DirichletEntry> entries_; // sorted by voxel, unique
};

// mesh.hpp:145-158
struct Microenvironment {
    CartesianMesh mesh;
    std::vector<SubstrateParams> substrates;
    DensityField field;
    DirichletMap dirichlet;
    int substrate_count() const { return static_cast<int>(substrates.size()); }
    static Microenvironment create(const CartesianMesh& mesh, std::vector<SubstrateParams> substrates);
};

// solver.hpp:12-33
enum class Axis { x = 0, y = 1, z = 2 };

struct SolverWorkspace {
    Axis axis = Axis::x;
    int n = 0;
    int substrates = 0;
    double dt = 0.0;
    int dims = 0;
    std::vector<double> off_diag;
    std::vector<double> denom_inv;
    std::vector<double> c_back;
};

SolverWorkspace precompute_thomas_coefficients(const CartesianMesh& mesh, const std::vector<double>& diffusion,
                                               const std::vector<double>& decay, double dt, Axis axis, int dims);

struct SolverWorkspaces {
    std::optional<SolverWorkspace> x, y, z;
    int dims = 0;
    double dt = 0.0;
    static SolverWorkspaces build(const CartesianMesh& mesh, const std::vector<SubstrateParams>& substrates,
                                  double dt);
};

// agents.hpp:14-24
struct CellAgent {
    std::int64_t id = 0;
    std::array<double, 3> position{};
    double volume = 0.0;
    std::vector<double> secretion_rates;
    std::vector<double> uptake_rates;
    std::vector<double> saturation_densities;
    index_t voxel = 0;
};

// agents.hpp:30-65
class AgentPopulation {
public:
    AgentPopulation() = default;
    AgentPopulation(std::vector<CellAgent> agents, const CartesianMesh& mesh, int substrates);
    std::size_t size() const { return agents_.size(); }
    bool empty() const { return agents_.empty(); }
    const std::vector<CellAgent>& agents() const { return agents_; }
    const std::vector<std::pair<index_t, std::vector<std::size_t>>>& grouping() const { return groups_; }
    void set_position(std::int64_t id, const std::array<double, 3>& position);
    void rebuild_voxel_grouping(const CartesianMesh& mesh);

private:
    void validate(const CartesianMesh& mesh, int substrates) const;
    std::vector<CellAgent> agents_;
    std::vector<std::pair<index_t, std::vector<std::size_t>>> groups_;
};

class DeviceSession; // device state + kernels (device.cuh)

// The execution strategy that replaces WorkerPool (backend.hpp:34-66). It
// owns the device-resident field for one Microenvironment; the host copy
// (env.field) is refreshed only by download(). Results are bitwise equal to
// the reference's serial backend.
class DeviceBackend {
public:
    explicit DeviceBackend(int device = 0);
    ~DeviceBackend();
    DeviceBackend(const DeviceBackend&) = delete;
    DeviceBackend& operator=(const DeviceBackend&) = delete;

    // Uploads mesh, field, Dirichlet map and workspaces (and agents, if given).
    void attach(const Microenvironment& env, const SolverWorkspaces& ws, const AgentPopulation* agents = nullptr);
    void upload(const DensityField& field);
    void download(DensityField& field);
    // The nested (vector-of-vectors) layout straight to / from HBM: packed on
    // the host with translate_vector_to_array's checks, one copy each way.
    void upload(const NestedDensity& nested);
    void download(NestedDensity& nested);
    void attach_agents(const AgentPopulation& agents);
    const AgentPopulation* attached_agents() const { return agents_from_; }
    DeviceSession& session()
    {
        if (!session_) throw state_error("device backend not attached");
        return *session_;
    }

private:
    int device_;
    const AgentPopulation* agents_from_ = nullptr;
    std::unique_ptr<DeviceSession> session_;
};

// solver.hpp:72-73 / agents.hpp:72-73 with the device backend. The field
// argument stays device-resident; call backend.download(env.field) to read it.
void diffuse_decay_step(Microenvironment& env, const SolverWorkspaces& workspaces, DeviceBackend& backend);
void cell_sources_sinks_step(DensityField& field, const AgentPopulation& agents, const CartesianMesh& mesh,
                             double dt, DeviceBackend& backend);

std::string format_double(double v);

// text.cpp:16-76 (the reference's token rules: std::from_chars over the
// trimmed token, the whole token must parse; std::invalid_argument
// "invalid number '<token>' for <what>").
std::string format_int(std::int64_t v);
std::string trim(const std::string& s);
std::vector<std::string> split_csv_line(const std::string& line);
double parse_double(const std::string& token, const std::string& what);
std::int64_t parse_int(const std::string& token, const std::string& what);

// config.cpp:416-477 / 479-491: agent CSV ingest and export. Header
// "id,x,y,z,volume" + ",S_<name>,U_<name>,target_<name>" per substrate;
// errors are config_error("agent file <path> line <n>: ...") / io_error.
AgentPopulation load_agents(const std::string& path, const CartesianMesh& mesh,
                            const std::vector<std::string>& substrate_names);
void save_agents(const std::vector<CellAgent>& agents, const std::vector<std::string>& substrate_names,
                 const std::string& path);

} // namespace biodiff_b200
