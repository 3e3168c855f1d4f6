// Host-side setup of the reference microenvironment API (see host.hpp).
// Every numeric routine here must reproduce the reference's bits: it is the
// source of the coefficients the device kernels consume.
#include "host.hpp"

#include <algorithm>
#include <charconv>
#include <cmath>
#include <fstream>
#include <unordered_set>

namespace biodiff_b200 {

std::string format_double(double v)
{
    char buf[64];
    auto r = std::to_chars(buf, buf + sizeof(buf), v);
    return std::string(buf, r.ptr);
}

// mesh.cpp:12-44: counts rounded from the extent, upper bounds snapped.
CartesianMesh CartesianMesh::from_bounds(double x_min, double x_max, double y_min, double y_max, double z_min,
                                         double z_max, double dx, double dy, double dz)
{
    if (!(dx > 0.0) || !(dy > 0.0) || !(dz > 0.0))
        throw config_error("mesh spacing must be positive (dx=" + format_double(dx) + " dy=" + format_double(dy) +
                           " dz=" + format_double(dz) + ")");
    auto count = [](double lo, double hi, double h, const char* axis) {
        const int n = static_cast<int>(std::llround((hi - lo) / h));
        if (n < 1) throw config_error(std::string("domain extent along ") + axis + " is smaller than one voxel");
        return n;
    };
    CartesianMesh m;
    m.dx = dx;
    m.dy = dy;
    m.dz = dz;
    m.nx = count(x_min, x_max, dx, "x");
    m.ny = count(y_min, y_max, dy, "y");
    m.nz = count(z_min, z_max, dz, "z");
    m.x_min = x_min;
    m.y_min = y_min;
    m.z_min = z_min;
    m.x_max = x_min + m.nx * dx;
    m.y_max = y_min + m.ny * dy;
    m.z_max = z_min + m.nz * dz;
    return m;
}

index_t CartesianMesh::voxel_index(int i, int j, int k) const
{
    if (i < 0 || i >= nx || j < 0 || j >= ny || k < 0 || k >= nz)
        throw std::out_of_range("voxel index (" + std::to_string(i) + "," + std::to_string(j) + "," +
                                std::to_string(k) + ") outside mesh");
    return static_cast<index_t>(i) + static_cast<index_t>(j) * nx + static_cast<index_t>(k) * nx * ny;
}

std::array<int, 3> CartesianMesh::voxel_ijk(index_t n) const
{
    if (n < 0 || n >= voxel_count()) throw std::out_of_range("flat voxel index outside mesh");
    const index_t plane = static_cast<index_t>(nx) * ny;
    const index_t rem = n % plane;
    return {static_cast<int>(rem % nx), static_cast<int>(rem / nx), static_cast<int>(n / plane)};
}

bool CartesianMesh::contains(const std::array<double, 3>& p) const
{
    return p[0] >= x_min && p[0] <= x_max && p[1] >= y_min && p[1] <= y_max && p[2] >= z_min && p[2] <= z_max;
}

// mesh.cpp:72-88: containing voxel, upper boundary clamps to the last one.
index_t CartesianMesh::nearest_voxel(const std::array<double, 3>& p) const
{
    if (!contains(p))
        throw std::domain_error("position (" + format_double(p[0]) + "," + format_double(p[1]) + "," +
                                format_double(p[2]) + ") outside the simulation domain");
    auto cell = [](double v, double lo, double h, int n) {
        return std::clamp(static_cast<int>(std::floor((v - lo) / h)), 0, n - 1);
    };
    return voxel_index(cell(p[0], x_min, dx, nx), cell(p[1], y_min, dy, ny), cell(p[2], z_min, dz, nz));
}

index_t CartesianMesh::boundary_voxel_count() const
{
    const index_t inner = static_cast<index_t>(std::max(nx - 2, 0)) * std::max(ny - 2, 0) * std::max(nz - 2, 0);
    return voxel_count() - inner;
}

// mesh.cpp:138-159: sorted unique entries; re-adding a voxel merges masks.
void DirichletMap::add(index_t voxel, std::vector<std::uint8_t> mask, std::vector<double> values,
                       index_t voxel_count, int substrates)
{
    if (voxel < 0 || voxel >= voxel_count)
        throw std::out_of_range("Dirichlet voxel " + std::to_string(voxel) + " outside mesh");
    if (mask.size() != static_cast<std::size_t>(substrates) || values.size() != static_cast<std::size_t>(substrates))
        throw std::invalid_argument("Dirichlet mask/value length must equal the substrate count");
    auto it = std::lower_bound(entries_.begin(), entries_.end(), voxel,
                               [](const DirichletEntry& e, index_t v) { return e.voxel < v; });
    if (it != entries_.end() && it->voxel == voxel) {
        for (int s = 0; s < substrates; ++s)
            if (mask[s]) {
                it->mask[s] = 1;
                it->values[s] = values[s];
            }
        return;
    }
    entries_.insert(it, DirichletEntry{voxel, std::move(mask), std::move(values)});
}

void DirichletMap::add_single(index_t voxel, int substrate, double value, index_t voxel_count, int substrates)
{
    if (substrate < 0 || substrate >= substrates) throw std::invalid_argument("Dirichlet substrate index out of range");
    std::vector<std::uint8_t> mask(substrates, 0);
    std::vector<double> values(substrates, 0.0);
    mask[substrate] = 1;
    values[substrate] = value;
    add(voxel, std::move(mask), std::move(values), voxel_count, substrates);
}

// mesh.cpp:173-195 (without the nested-vector staging: same values).
Microenvironment Microenvironment::create(const CartesianMesh& mesh, std::vector<SubstrateParams> substrates)
{
    if (substrates.empty()) throw config_error("a microenvironment needs at least one substrate");
    for (const auto& s : substrates) {
        if (s.diffusion_coefficient < 0.0)
            throw config_error("substrate '" + s.name + "' has negative diffusion coefficient");
        if (s.decay_rate < 0.0) throw config_error("substrate '" + s.name + "' has negative decay rate");
    }
    Microenvironment env;
    env.mesh = mesh;
    env.substrates = std::move(substrates);
    const int S = env.substrate_count();
    env.field = DensityField(mesh.voxel_count(), S);
    for (std::size_t v = 0; v < static_cast<std::size_t>(mesh.voxel_count()); ++v)
        for (int s = 0; s < S; ++s) env.field.values[v * S + s] = env.substrates[s].initial_condition;
    return env;
}

// solver.cpp:47-97. The expressions are written in the reference's
// evaluation order so the host (compiled without FMA contraction, see
// Makefile) produces identical bits.
SolverWorkspace precompute_thomas_coefficients(const CartesianMesh& mesh, const std::vector<double>& diffusion,
                                               const std::vector<double>& decay_rate, double dt, Axis axis,
                                               int dims)
{
    if (!(dt > 0.0)) throw std::invalid_argument("solver step size must be positive, got " + format_double(dt));
    if (dims < 1 || dims > 3) throw std::invalid_argument("decay split count must be 1, 2, or 3");
    if (diffusion.empty()) throw std::invalid_argument("no substrates to precompute coefficients for");
    if (diffusion.size() != decay_rate.size()) throw std::invalid_argument("diffusion/decay length mismatch");

    const int n = axis == Axis::x ? mesh.nx : axis == Axis::y ? mesh.ny : mesh.nz;
    const double h = axis == Axis::x ? mesh.dx : axis == Axis::y ? mesh.dy : mesh.dz;
    const int S = static_cast<int>(diffusion.size());

    SolverWorkspace ws;
    ws.axis = axis;
    ws.n = n;
    ws.substrates = S;
    ws.dt = dt;
    ws.dims = dims;
    ws.off_diag.assign(S, 0.0);
    ws.denom_inv.assign(static_cast<std::size_t>(n) * S, 0.0);
    ws.c_back.assign(static_cast<std::size_t>(n) * S, 0.0);
    for (int s = 0; s < S; ++s) {
        const double q = dt * diffusion[s] / (h * h);
        const double decay = 1.0 + dt * decay_rate[s] / dims;
        ws.off_diag[s] = q;
        auto diag = [&](int i) {
            if (n == 1) return decay;
            return (i == 0 || i == n - 1) ? decay + q : decay + 2.0 * q;
        };
        double denom = diag(0);
        ws.denom_inv[s] = 1.0 / denom;
        ws.c_back[s] = (n > 1) ? q * ws.denom_inv[s] : 0.0;
        for (int i = 1; i < n; ++i) {
            denom = diag(i) - q * ws.c_back[static_cast<std::size_t>(i - 1) * S + s];
            const double dinv = 1.0 / denom;
            ws.denom_inv[static_cast<std::size_t>(i) * S + s] = dinv;
            if (i < n - 1) ws.c_back[static_cast<std::size_t>(i) * S + s] = q * dinv;
        }
    }
    return ws;
}

// solver.cpp:277-287: x always; y, z only when the mesh extends along them.
SolverWorkspaces SolverWorkspaces::build(const CartesianMesh& mesh, const std::vector<SubstrateParams>& substrates,
                                         double dt)
{
    std::vector<double> D, L;
    for (const auto& s : substrates) {
        D.push_back(s.diffusion_coefficient);
        L.push_back(s.decay_rate);
    }
    SolverWorkspaces w;
    w.dt = dt;
    w.dims = 1 + (mesh.ny > 1 ? 1 : 0) + (mesh.nz > 1 ? 1 : 0);
    w.x = precompute_thomas_coefficients(mesh, D, L, dt, Axis::x, w.dims);
    if (mesh.ny > 1) w.y = precompute_thomas_coefficients(mesh, D, L, dt, Axis::y, w.dims);
    if (mesh.nz > 1) w.z = precompute_thomas_coefficients(mesh, D, L, dt, Axis::z, w.dims);
    return w;
}

// agents.cpp:12-18
AgentPopulation::AgentPopulation(std::vector<CellAgent> agents, const CartesianMesh& mesh, int substrates)
    : agents_(std::move(agents))
{
    validate(mesh, substrates);
    rebuild_voxel_grouping(mesh);
}

// agents.cpp:20-43: same checks, same exception types, same order.
void AgentPopulation::validate(const CartesianMesh& mesh, int substrates) const
{
    std::unordered_set<std::int64_t> ids;
    ids.reserve(agents_.size());
    const auto S = static_cast<std::size_t>(substrates);
    for (const auto& a : agents_) {
        if (!ids.insert(a.id).second) throw std::invalid_argument("duplicate agent id " + std::to_string(a.id));
        if (!(a.volume > 0.0))
            throw std::invalid_argument("agent " + std::to_string(a.id) + " has non-positive volume");
        if (a.secretion_rates.size() != S || a.uptake_rates.size() != S || a.saturation_densities.size() != S)
            throw std::invalid_argument("agent " + std::to_string(a.id) +
                                        " rate vectors do not match the substrate count");
        for (std::size_t s = 0; s < S; ++s)
            if (a.secretion_rates[s] < 0.0 || a.uptake_rates[s] < 0.0 || a.saturation_densities[s] < 0.0)
                throw std::invalid_argument("agent " + std::to_string(a.id) +
                                            " has a negative rate or saturation density");
        if (!mesh.contains(a.position))
            throw std::domain_error("agent " + std::to_string(a.id) + " position outside the domain");
    }
}

void AgentPopulation::set_position(std::int64_t id, const std::array<double, 3>& position)
{
    for (auto& a : agents_)
        if (a.id == id) {
            a.position = position;
            return;
        }
    throw std::invalid_argument("no agent with id " + std::to_string(id));
}

// agents.cpp:56-73: cache voxels, stable order by (voxel, id), cut groups.
void AgentPopulation::rebuild_voxel_grouping(const CartesianMesh& mesh)
{
    for (auto& a : agents_) a.voxel = mesh.nearest_voxel(a.position);
    std::vector<std::size_t> order(agents_.size());
    for (std::size_t i = 0; i < order.size(); ++i) order[i] = i;
    std::sort(order.begin(), order.end(), [&](std::size_t l, std::size_t r) {
        if (agents_[l].voxel != agents_[r].voxel) return agents_[l].voxel < agents_[r].voxel;
        return agents_[l].id < agents_[r].id;
    });
    groups_.clear();
    for (std::size_t i : order) {
        if (groups_.empty() || groups_.back().first != agents_[i].voxel) groups_.push_back({agents_[i].voxel, {}});
        groups_.back().second.push_back(i);
    }
}

// ---- mesh.cpp:95-136: nested <-> flat --------------------------------------

bool DensityField::all_finite() const
{
    return std::all_of(values.begin(), values.end(), [](double v) { return std::isfinite(v); });
}

DensityField translate_vector_to_array(const NestedDensity& nested)
{
    DensityField field;
    if (nested.empty()) return field;
    const std::size_t substrates = nested.front().size();
    field.substrates = static_cast<int>(substrates);
    field.values.reserve(nested.size() * substrates);
    for (std::size_t v = 0; v < nested.size(); ++v) {
        if (nested[v].size() != substrates)
            throw std::invalid_argument("ragged nested density: voxel " + format_int(static_cast<std::int64_t>(v)) +
                                        " holds " + format_int(static_cast<std::int64_t>(nested[v].size())) +
                                        " substrates, expected " + format_int(static_cast<std::int64_t>(substrates)));
        field.values.insert(field.values.end(), nested[v].begin(), nested[v].end());
    }
    return field;
}

NestedDensity translate_array_to_vector(const DensityField& field)
{
    if (field.substrates <= 0) {
        if (!field.values.empty()) throw std::invalid_argument("density field with values but no substrate count");
        return {};
    }
    if (field.values.size() % field.substrates != 0)
        throw std::invalid_argument("density array length is not a multiple of the substrate count");
    const index_t voxels = field.voxel_count();
    NestedDensity nested(static_cast<std::size_t>(voxels));
    for (index_t v = 0; v < voxels; ++v) {
        auto begin = field.values.begin() + v * field.substrates;
        nested[v].assign(begin, begin + field.substrates);
    }
    return nested;
}

// ---- text.cpp:16-76 --------------------------------------------------------

std::string format_int(std::int64_t v)
{
    char buf[32];
    auto r = std::to_chars(buf, buf + sizeof(buf), v);
    return std::string(buf, r.ptr);
}

std::string trim(const std::string& s)
{
    const char* ws = " \t\r\n";
    const auto b = s.find_first_not_of(ws);
    if (b == std::string::npos) return {};
    const auto e = s.find_last_not_of(ws);
    return s.substr(b, e - b + 1);
}

std::vector<std::string> split_csv_line(const std::string& line)
{
    std::vector<std::string> fields;
    std::size_t start = 0;
    while (true) {
        const std::size_t comma = line.find(',', start);
        if (comma == std::string::npos) {
            fields.emplace_back(line.substr(start));
            break;
        }
        fields.emplace_back(line.substr(start, comma - start));
        start = comma + 1;
    }
    return fields;
}

namespace {

[[noreturn]] void bad_token(const std::string& token, const std::string& what)
{
    throw std::invalid_argument("invalid number '" + token + "' for " + what);
}

} // namespace

double parse_double(const std::string& token, const std::string& what)
{
    const std::string t = trim(token);
    double value = 0.0;
    const auto r = std::from_chars(t.data(), t.data() + t.size(), value);
    if (r.ec != std::errc{} || r.ptr != t.data() + t.size() || t.empty()) bad_token(token, what);
    return value;
}

std::int64_t parse_int(const std::string& token, const std::string& what)
{
    const std::string t = trim(token);
    std::int64_t value = 0;
    const auto r = std::from_chars(t.data(), t.data() + t.size(), value);
    if (r.ec != std::errc{} || r.ptr != t.data() + t.size() || t.empty()) bad_token(token, what);
    return value;
}

// ---- config.cpp:407-491: agent CSV -----------------------------------------

namespace {

[[noreturn]] void agent_fail(const std::string& path, std::size_t line, const std::string& msg)
{
    throw config_error("agent file " + path + " line " + format_int(static_cast<std::int64_t>(line)) + ": " + msg);
}

std::string agent_header(const std::vector<std::string>& names)
{
    std::string h = "id,x,y,z,volume";
    for (const auto& n : names) h += ",S_" + n + ",U_" + n + ",target_" + n;
    return h;
}

} // namespace

AgentPopulation load_agents(const std::string& path, const CartesianMesh& mesh,
                            const std::vector<std::string>& substrate_names)
{
    std::ifstream in(path, std::ios::binary);
    if (!in) throw config_error("agent file not found: " + path);
    const std::string expected = agent_header(substrate_names);
    std::string line;
    std::size_t line_no = 0;
    if (!std::getline(in, line)) throw config_error("agent file " + path + " is empty");
    ++line_no;
    if (trim(line) != expected) agent_fail(path, line_no, "header must be '" + expected + "'");
    const std::size_t S = substrate_names.size();
    std::vector<CellAgent> agents;
    while (std::getline(in, line)) {
        ++line_no;
        const std::string stripped = trim(line);
        if (stripped.empty()) continue;
        const auto f = split_csv_line(stripped);
        if (f.size() != 5 + 3 * S)
            agent_fail(path, line_no,
                       "expected " + format_int(static_cast<std::int64_t>(5 + 3 * S)) + " fields, got " +
                           format_int(static_cast<std::int64_t>(f.size())));
        try {
            CellAgent a;
            a.id = parse_int(f[0], "id");
            a.position = {parse_double(f[1], "x"), parse_double(f[2], "y"), parse_double(f[3], "z")};
            a.volume = parse_double(f[4], "volume");
            a.secretion_rates.resize(S);
            a.uptake_rates.resize(S);
            a.saturation_densities.resize(S);
            for (std::size_t s = 0; s < S; ++s) {
                a.secretion_rates[s] = parse_double(f[5 + 3 * s], "secretion rate");
                a.uptake_rates[s] = parse_double(f[6 + 3 * s], "uptake rate");
                a.saturation_densities[s] = parse_double(f[7 + 3 * s], "target density");
            }
            agents.push_back(std::move(a));
        } catch (const std::invalid_argument& e) {
            agent_fail(path, line_no, e.what());
        }
    }
    try {
        return AgentPopulation(std::move(agents), mesh, static_cast<int>(S));
    } catch (const std::exception& e) {
        throw config_error("agent file " + path + ": " + e.what());
    }
}

void save_agents(const std::vector<CellAgent>& agents, const std::vector<std::string>& substrate_names,
                 const std::string& path)
{
    std::ofstream out(path, std::ios::binary);
    if (!out) throw io_error("cannot open " + path + " for writing");
    out << agent_header(substrate_names) << "\n";
    for (const auto& a : agents) {
        out << format_int(a.id) << ',' << format_double(a.position[0]) << ',' << format_double(a.position[1]) << ','
            << format_double(a.position[2]) << ',' << format_double(a.volume);
        for (std::size_t s = 0; s < substrate_names.size(); ++s)
            out << ',' << format_double(a.secretion_rates[s]) << ',' << format_double(a.uptake_rates[s]) << ','
                << format_double(a.saturation_densities[s]);
        out << "\n";
    }
    if (!out) throw io_error("failed writing " + path);
}

} // namespace biodiff_b200
