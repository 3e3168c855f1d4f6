// extern "C" boundary (include/biodiff_b200.h) over the host mirror and the
// device session. Exceptions are mapped to status codes exactly as the
// reference maps its exception types to exit codes (errors.hpp:9-24,
// SPEC.md:499): config_error -> 1, io_error -> 4, everything else -> 2.
#include "../../include/biodiff_b200.h"

#include "config.hpp"
#include "device.hpp"
#include "engine.hpp"
#include "host.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <optional>
#include <memory>
#include <new>
#include <string>
#include <type_traits>

using namespace biodiff_b200;

struct biodiff_session {
    std::unique_ptr<DeviceSession> dev;
    CartesianMesh mesh; // the GLOBAL mesh (for a z-slab, dev->mesh() is the slab)
    int S = 0;          // substrates of the GLOBAL problem (parameter arrays are [S])
    int s0 = 0, s1 = 0; // substrate shard [s0, s1) held by this session (all: 0, S)
    bool slab = false;
    int z0 = 0, z1 = 0; // slab planes [z0, z1)
    int replicas = 1;   // ensemble size (stacked replica-major)
    bool sharded() const { return s1 - s0 != S; }
};

namespace {

thread_local std::string g_last_error;

template <class F>
int guarded(F&& f)
{
    try {
        f();
        return BIODIFF_OK;
    } catch (const config_error& e) {
        g_last_error = e.what();
        return BIODIFF_ERR_CONFIG;
    } catch (const io_error& e) {
        g_last_error = e.what();
        return BIODIFF_ERR_IO;
    } catch (const std::bad_alloc&) {
        g_last_error = "out of host memory";
        return BIODIFF_ERR_STATE;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return BIODIFF_ERR_STATE;
    } catch (...) {
        g_last_error = "unknown error";
        return BIODIFF_ERR_STATE;
    }
}

CartesianMesh to_mesh(const biodiff_mesh* m)
{
    if (!m) throw std::invalid_argument("null mesh");
    CartesianMesh c;
    c.x_min = m->x_min;
    c.x_max = m->x_max;
    c.y_min = m->y_min;
    c.y_max = m->y_max;
    c.z_min = m->z_min;
    c.z_max = m->z_max;
    c.dx = m->dx;
    c.dy = m->dy;
    c.dz = m->dz;
    c.nx = m->nx;
    c.ny = m->ny;
    c.nz = m->nz;
    if (c.nx < 1 || c.ny < 1 || c.nz < 1) throw config_error("mesh voxel counts must be positive");
    if (!(c.dx > 0.0) || !(c.dy > 0.0) || !(c.dz > 0.0)) throw config_error("mesh spacing must be positive");
    return c;
}

void from_mesh(const CartesianMesh& c, biodiff_mesh* m)
{
    m->x_min = c.x_min;
    m->x_max = c.x_max;
    m->y_min = c.y_min;
    m->y_max = c.y_max;
    m->z_min = c.z_min;
    m->z_max = c.z_max;
    m->dx = c.dx;
    m->dy = c.dy;
    m->dz = c.dz;
    m->nx = c.nx;
    m->ny = c.ny;
    m->nz = c.nz;
}

DeviceSession& dev(biodiff_session* s)
{
    if (!s || !s->dev) throw std::invalid_argument("null session");
    return *s->dev;
}

Axis to_axis(int32_t a)
{
    if (a < 0 || a > 2) throw std::invalid_argument("axis must be 0 (x), 1 (y) or 2 (z)");
    return static_cast<Axis>(a);
}

void need(const void* p, const char* what)
{
    if (!p) throw std::invalid_argument(std::string("null pointer: ") + what);
}

// A substrate shard keeps columns [s0, s1) of every per-substrate array.
template <class T>
std::vector<T> columns(const T* a, std::int64_t rows, int S, int s0, int s1)
{
    std::vector<T> out(static_cast<std::size_t>(rows) * (s1 - s0));
    for (std::int64_t r = 0; r < rows; ++r)
        std::copy(a + r * S + s0, a + r * S + s1, out.begin() + r * (s1 - s0));
    return out;
}

// The shard's view of a validated population (same agents and ids, rates of
// substrates [s0, s1) only). Substrates are independent in the reaction
// update (agents.cpp:103-108), so the shard's result columns are bitwise
// those of the unsharded step.
AgentPopulation shard_population(const biodiff_session* s, const AgentPopulation& pop)
{
    if (!s->sharded()) return pop;
    std::vector<CellAgent> v = pop.agents();
    for (CellAgent& c : v) {
        auto cut = [&](std::vector<double>& x) { x = std::vector<double>(x.begin() + s->s0, x.begin() + s->s1); };
        cut(c.secretion_rates);
        cut(c.uptake_rates);
        cut(c.saturation_densities);
    }
    return AgentPopulation(std::move(v), s->mesh, s->s1 - s->s0);
}

// Uploads SolverWorkspaces built on the GLOBAL mesh. For a z-slab the z
// workspace is sliced to the slab's rows (the global factorisation, so the
// zero-inflow slab solve is the reference recurrence minus the inflow terms)
// and the slab's unit-inflow responses are computed:
//   phi_m : forward value at row m for d_in = 1 (zero RHS), Phi = its back substitution
//   psi_m : back-substituted value at row m for x_in = 1 (zero RHS)
void upload_workspaces(biodiff_session* s, const SolverWorkspaces& ws)
{
    DeviceSession& d = *s->dev;
    if (!s->slab) {
        d.set_workspaces(ws);
        return;
    }
    if (!ws.x) throw state_error("solver workspaces not built");
    const int S = s->s1 - s->s0; // the workspaces hold the shard's substrates
    auto put = [&](const std::optional<SolverWorkspace>& w) {
        if (w) d.set_workspace(w->axis, w->n, w->dims, w->dt, w->off_diag.data(), w->denom_inv.data(), w->c_back.data());
    };
    put(ws.x);
    put(ws.y);
    if (!ws.z) return;
    const SolverWorkspace& z = *ws.z;
    const int n = s->z1 - s->z0;
    std::vector<double> dinv(z.denom_inv.begin() + static_cast<std::ptrdiff_t>(s->z0) * S,
                             z.denom_inv.begin() + static_cast<std::ptrdiff_t>(s->z1) * S);
    std::vector<double> cb(z.c_back.begin() + static_cast<std::ptrdiff_t>(s->z0) * S,
                           z.c_back.begin() + static_cast<std::ptrdiff_t>(s->z1) * S);
    d.set_workspace(Axis::z, n, z.dims, z.dt, z.off_diag.data(), dinv.data(), cb.data());
    std::vector<double> phi(static_cast<std::size_t>(n) * S), Phi(phi.size()), psi(phi.size()), phi_last(S);
    for (int sub = 0; sub < S; ++sub) {
        const double q = z.off_diag[sub];
        auto at = [&](int m) { return static_cast<std::size_t>(m) * S + sub; };
        double f = 1.0;
        for (int m = 0; m < n; ++m) {
            f = (0.0 + q * f) * dinv[at(m)];
            phi[at(m)] = f;
        }
        Phi[at(n - 1)] = phi[at(n - 1)];
        for (int m = n - 2; m >= 0; --m) Phi[at(m)] = phi[at(m)] + cb[at(m)] * Phi[at(m + 1)];
        double g = cb[at(n - 1)] * 1.0; // zero on the last slab (global last row has c_back = 0)
        psi[at(n - 1)] = g;
        for (int m = n - 2; m >= 0; --m) {
            g = cb[at(m)] * g;
            psi[at(m)] = g;
        }
        phi_last[sub] = phi[at(n - 1)];
    }
    d.set_slab_spikes(Phi.data(), psi.data(), phi_last.data());
}

} // namespace

extern "C" {

const char* biodiff_last_error(void) { return g_last_error.c_str(); }

int32_t biodiff_version(void) { return 10000; }

int32_t biodiff_build_flags(void)
{
#ifdef BIODIFF_EXPERIMENTAL
    return 1;
#else
    return 0;
#endif
}

int biodiff_mesh_from_bounds(double x_min, double x_max, double y_min, double y_max, double z_min, double z_max,
                             double dx, double dy, double dz, biodiff_mesh* out)
{
    return guarded([&] {
        need(out, "out");
        from_mesh(CartesianMesh::from_bounds(x_min, x_max, y_min, y_max, z_min, z_max, dx, dy, dz), out);
    });
}

int biodiff_nearest_voxel(const biodiff_mesh* mesh, const double position[3], int64_t* voxel)
{
    return guarded([&] {
        need(position, "position");
        need(voxel, "voxel");
        *voxel = to_mesh(mesh).nearest_voxel({position[0], position[1], position[2]});
    });
}

int biodiff_parse_agents_csv(const biodiff_mesh* mesh, const char* path, const char* const* names, int32_t substrates,
                             int64_t* n, int64_t* ids, double* xyz, double* volume, double* secretion, double* uptake,
                             double* saturation)
{
    return guarded([&] {
        need(path, "path");
        need(names, "names");
        need(n, "n");
        std::vector<std::string> v;
        for (int s = 0; s < substrates; ++s) {
            need(names[s], "substrate name");
            v.emplace_back(names[s]);
        }
        const AgentPopulation pop = load_agents(path, to_mesh(mesh), v);
        const auto& all = pop.agents();
        *n = static_cast<int64_t>(all.size());
        if (!ids || !xyz || !volume || !secretion || !uptake || !saturation) return;
        const int S = substrates;
        for (std::size_t a = 0; a < all.size(); ++a) {
            ids[a] = all[a].id;
            for (int c = 0; c < 3; ++c) xyz[3 * a + c] = all[a].position[c];
            volume[a] = all[a].volume;
            for (int s = 0; s < S; ++s) {
                secretion[a * S + s] = all[a].secretion_rates[s];
                uptake[a * S + s] = all[a].uptake_rates[s];
                saturation[a * S + s] = all[a].saturation_densities[s];
            }
        }
    });
}

int biodiff_write_agents_csv(const char* path, const char* const* names, int32_t substrates, int64_t n,
                             const int64_t* ids, const double* xyz, const double* volume, const double* secretion,
                             const double* uptake, const double* saturation)
{
    return guarded([&] {
        need(path, "path");
        need(names, "names");
        if (n < 0) throw std::invalid_argument("negative agent count");
        if (n > 0) {
            need(ids, "ids");
            need(xyz, "xyz");
            need(volume, "volume");
            need(secretion, "secretion");
            need(uptake, "uptake");
            need(saturation, "saturation");
        }
        std::vector<std::string> v;
        for (int s = 0; s < substrates; ++s) {
            need(names[s], "substrate name");
            v.emplace_back(names[s]);
        }
        const int S = substrates;
        std::vector<CellAgent> agents(static_cast<std::size_t>(n));
        for (int64_t a = 0; a < n; ++a) {
            CellAgent& c = agents[a];
            c.id = ids[a];
            c.position = {xyz[3 * a], xyz[3 * a + 1], xyz[3 * a + 2]};
            c.volume = volume[a];
            c.secretion_rates.assign(secretion + a * S, secretion + (a + 1) * S);
            c.uptake_rates.assign(uptake + a * S, uptake + (a + 1) * S);
            c.saturation_densities.assign(saturation + a * S, saturation + (a + 1) * S);
        }
        save_agents(agents, v, path);
    });
}

int biodiff_precompute_thomas(const biodiff_mesh* mesh, int32_t substrates, const double* diffusion,
                              const double* decay, double dt, int32_t axis, int32_t dims, double* off_diag,
                              double* denom_inv, double* c_back)
{
    return guarded([&] {
        need(diffusion, "diffusion");
        need(decay, "decay");
        need(off_diag, "off_diag");
        need(denom_inv, "denom_inv");
        need(c_back, "c_back");
        if (substrates < 1) throw std::invalid_argument("no substrates to precompute coefficients for");
        const SolverWorkspace w = precompute_thomas_coefficients(
            to_mesh(mesh), std::vector<double>(diffusion, diffusion + substrates),
            std::vector<double>(decay, decay + substrates), dt, to_axis(axis), dims);
        std::memcpy(off_diag, w.off_diag.data(), sizeof(double) * w.off_diag.size());
        std::memcpy(denom_inv, w.denom_inv.data(), sizeof(double) * w.denom_inv.size());
        std::memcpy(c_back, w.c_back.data(), sizeof(double) * w.c_back.size());
    });
}

int biodiff_device_count(int32_t* count)
{
    return guarded([&] {
        need(count, "count");
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess) n = 0;
        int usable = 0;
        for (int d = 0; d < n; ++d) {
            cudaDeviceProp p;
            if (cudaGetDeviceProperties(&p, d) == cudaSuccess && p.major == 10) ++usable;
        }
        *count = usable;
    });
}

int biodiff_session_create(const biodiff_mesh* mesh, int32_t substrates, int32_t device, biodiff_session** out)
{
    return guarded([&] {
        need(out, "out");
        *out = nullptr;
        auto s = std::make_unique<biodiff_session>();
        s->mesh = to_mesh(mesh);
        s->S = substrates;
        s->s1 = substrates;
        s->dev = std::make_unique<DeviceSession>(s->mesh, substrates, device);
        *out = s.release();
    });
}

int biodiff_session_destroy(biodiff_session* session)
{
    return guarded([&] { delete session; });
}

int biodiff_set_substrates(biodiff_session* session, const double* diffusion, const double* decay, double dt)
{
    return guarded([&] {
        need(diffusion, "diffusion");
        need(decay, "decay");
        dev(session);
        // Every substrate of the global problem is validated; a shard builds
        // the workspaces of its own (the coefficients are per-substrate, so
        // the bits equal the unsharded build's columns, solver.cpp:72-95).
        std::vector<SubstrateParams> params;
        for (int s = 0; s < session->S; ++s) {
            if (diffusion[s] < 0.0) throw config_error("substrate has negative diffusion coefficient");
            if (decay[s] < 0.0) throw config_error("substrate has negative decay rate");
            if (s >= session->s0 && s < session->s1)
                params.push_back({"s" + std::to_string(s), diffusion[s], decay[s], 0.0});
        }
        upload_workspaces(session, SolverWorkspaces::build(session->mesh, params, dt));
    });
}

int biodiff_set_workspace(biodiff_session* session, int32_t axis, int32_t n, int32_t dims, double dt,
                          const double* off_diag, const double* denom_inv, const double* c_back)
{
    return guarded([&] {
        need(off_diag, "off_diag");
        need(denom_inv, "denom_inv");
        need(c_back, "c_back");
        dev(session).set_workspace(to_axis(axis), n, dims, dt, off_diag, denom_inv, c_back);
    });
}

int biodiff_set_dirichlet(biodiff_session* session, int64_t count, const int64_t* voxel, const uint8_t* mask,
                          const double* values)
{
    return guarded([&] {
        if (count < 0) throw std::invalid_argument("negative Dirichlet entry count");
        if (count > 0) {
            need(voxel, "voxel");
            need(mask, "mask");
            need(values, "values");
        }
        DeviceSession& d = dev(session);
        const int S = session->S;
        DirichletMap map;
        for (int64_t e = 0; e < count; ++e)
            map.add(voxel[e], std::vector<std::uint8_t>(mask + e * S, mask + (e + 1) * S),
                    std::vector<double>(values + e * S, values + (e + 1) * S),
                    session->mesh.voxel_count() * session->replicas, S);
        if (session->sharded()) { // the merged entries' columns [s0, s1); entries that clamp none of them go
            const int s0 = session->s0, s1 = session->s1;
            DirichletMap cut;
            for (const auto& e : map.entries()) {
                std::vector<std::uint8_t> m(e.mask.begin() + s0, e.mask.begin() + s1);
                if (std::none_of(m.begin(), m.end(), [](std::uint8_t b) { return b != 0; })) continue;
                cut.add(e.voxel, std::move(m), std::vector<double>(e.values.begin() + s0, e.values.begin() + s1),
                        session->mesh.voxel_count(), s1 - s0);
            }
            map = std::move(cut);
        }
        const int SL = session->s1 - session->s0;
        if (!session->slab) {
            d.set_dirichlet(map);
        } else { // keep the slab's entries, in local voxel indices
            const std::int64_t plane = static_cast<std::int64_t>(session->mesh.nx) * session->mesh.ny;
            const std::int64_t lo = session->z0 * plane, hi = session->z1 * plane;
            DirichletMap local;
            for (const auto& e : map.entries())
                if (e.voxel >= lo && e.voxel < hi)
                    local.add(e.voxel - lo, e.mask, e.values, hi - lo, SL);
            d.set_dirichlet(local);
        }
    });
}

namespace {

std::vector<std::string> substrate_names(const biodiff_session* session, const char* const* names)
{
    need(names, "names");
    std::vector<std::string> v;
    for (int s = 0; s < session->S; ++s) {
        need(names[s], "substrate name");
        v.emplace_back(names[s]);
    }
    return v;
}

// `pop` holds all S substrates; a shard installs its columns.
void install_agents(biodiff_session* session, const AgentPopulation& full)
{
    DeviceSession& d = dev(session);
    if (session->replicas > 1) throw state_error("ensembles take agents through biodiff_ensemble_set_agents");
    const AgentPopulation pop = shard_population(session, full);
    if (!session->slab) {
        d.set_agents(pop);
    } else {
        const std::int64_t plane = static_cast<std::int64_t>(session->mesh.nx) * session->mesh.ny;
        d.set_agents_range(pop, session->mesh, session->z0 * plane, session->z1 * plane);
    }
}

} // namespace

int biodiff_set_agents(biodiff_session* session, int64_t n, const int64_t* ids, const double* positions,
                       const double* volume, const double* secretion, const double* uptake,
                       const double* saturation)
{
    return guarded([&] {
        if (n < 0) throw std::invalid_argument("negative agent count");
        if (n > 0) {
            need(ids, "ids");
            need(positions, "positions");
            need(volume, "volume");
            need(secretion, "secretion");
            need(uptake, "uptake");
            need(saturation, "saturation");
        }
        dev(session);
        const int S = session->S;
        std::vector<CellAgent> agents(static_cast<std::size_t>(n));
        for (int64_t a = 0; a < n; ++a) {
            CellAgent& c = agents[a];
            c.id = ids[a];
            c.position = {positions[3 * a], positions[3 * a + 1], positions[3 * a + 2]};
            c.volume = volume[a];
            c.secretion_rates.assign(secretion + a * S, secretion + (a + 1) * S);
            c.uptake_rates.assign(uptake + a * S, uptake + (a + 1) * S);
            c.saturation_densities.assign(saturation + a * S, saturation + (a + 1) * S);
        }
        install_agents(session, AgentPopulation(std::move(agents), session->mesh, S)); // host validation
    });
}

int biodiff_agent_grouping(biodiff_session* session, int64_t* groups, int64_t* group_voxel, int64_t* group_offsets,
                           int64_t* order)
{
    return guarded([&] {
        need(groups, "groups");
        DeviceSession& d = dev(session);
        if (!group_voxel || !group_offsets || !order) {
            *groups = d.download_grouping(nullptr, nullptr, nullptr);
            return;
        }
        *groups = d.download_grouping(group_voxel, group_offsets, order);
    });
}

int biodiff_agent_count(biodiff_session* session, int64_t* n)
{
    return guarded([&] {
        need(n, "n");
        *n = dev(session).agent_count();
    });
}

int biodiff_set_agent_positions(biodiff_session* session, const double* xyz, int64_t n)
{
    return guarded([&] {
        if (n > 0) need(xyz, "xyz");
        dev(session).set_agent_positions(xyz, n);
    });
}

int biodiff_set_agent_position(biodiff_session* session, int64_t id, const double* xyz)
{
    return guarded([&] {
        need(xyz, "xyz");
        dev(session).set_agent_position(id, xyz);
    });
}

int biodiff_agent_positions_device(biodiff_session* session, double** xyz)
{
    return guarded([&] {
        need(xyz, "xyz");
        *xyz = dev(session).agent_positions_device();
    });
}

int biodiff_rebuild_voxel_grouping(biodiff_session* session)
{
    return guarded([&] { dev(session).rebuild_voxel_grouping(); });
}

int biodiff_sample_agent_densities(biodiff_session* session, double* out, int64_t count)
{
    return guarded([&] {
        need(out, "out");
        dev(session).sample_agent_densities(out, count);
    });
}

int biodiff_download_agents(biodiff_session* session, int64_t* ids, double* xyz, double* volume, double* secretion,
                            double* uptake, double* saturation)
{
    return guarded([&] { dev(session).download_agents(ids, xyz, volume, secretion, uptake, saturation); });
}


int biodiff_load_agents_csv(biodiff_session* session, const char* path, const char* const* names)
{
    return guarded([&] {
        need(path, "path");
        const auto v = substrate_names(session, names);
        install_agents(session, load_agents(path, session->mesh, v));
    });
}

int biodiff_save_agents_csv(biodiff_session* session, const char* path, const char* const* names)
{
    return guarded([&] {
        need(path, "path");
        const auto v = substrate_names(session, names);
        DeviceSession& d = dev(session);
        if (session->sharded())
            throw state_error("a substrate shard holds only its substrates' rates: save agents from an unsharded "
                              "session");
        const std::int64_t n = d.agent_count();
        const int S = session->S;
        std::vector<std::int64_t> ids(n);
        std::vector<double> xyz(3 * n), vol(n), sec(n * S), upt(n * S), sat(n * S);
        d.download_agents(ids.data(), xyz.data(), vol.data(), sec.data(), upt.data(), sat.data());
        std::vector<CellAgent> agents(n);
        for (std::int64_t a = 0; a < n; ++a) {
            CellAgent& c = agents[a];
            c.id = ids[a];
            c.position = {xyz[3 * a], xyz[3 * a + 1], xyz[3 * a + 2]};
            c.volume = vol[a];
            c.secretion_rates.assign(sec.begin() + a * S, sec.begin() + (a + 1) * S);
            c.uptake_rates.assign(upt.begin() + a * S, upt.begin() + (a + 1) * S);
            c.saturation_densities.assign(sat.begin() + a * S, sat.begin() + (a + 1) * S);
        }
        save_agents(agents, v, path);
    });
}

namespace {

void to_c_clock(const SimulationClock& c, biodiff_clock* o)
{
    o->dt_diff = c.dt_diff;
    o->dt_mech = c.dt_mech;
    o->dt_cell = c.dt_cell;
    o->t_max = c.t_max;
    o->per_mech = c.per_mech;
    o->per_cell = c.per_cell;
    o->total_steps = c.total_steps;
    o->diffusion_steps = c.diffusion_steps;
    o->mechanics_steps = c.mechanics_steps;
    o->cell_steps = c.cell_steps;
    o->t_now = c.t_now();
    o->pending = c.pending;
}

} // namespace

int biodiff_clock_make(double dt_diff, double dt_mech, double dt_cell, double t_max, biodiff_clock* clock)
{
    return guarded([&] {
        need(clock, "clock");
        to_c_clock(SimulationClock::make(dt_diff, dt_mech, dt_cell, t_max), clock);
    });
}

int biodiff_run_simulation(biodiff_session* session, biodiff_clock* clock, int32_t with_sources,
                           double snapshot_interval, biodiff_hook mechanics, biodiff_hook cell, biodiff_hook snapshot,
                           void* user, biodiff_run_metrics* metrics)
{
    return guarded([&] {
        need(clock, "clock");
        SimulationClock c = SimulationClock::make(clock->dt_diff, clock->dt_mech, clock->dt_cell, clock->t_max);
        if (clock->diffusion_steps < 0 || clock->mechanics_steps < 0 || clock->cell_steps < 0)
            throw std::invalid_argument("negative clock counters");
        c.diffusion_steps = clock->diffusion_steps;
        c.mechanics_steps = clock->mechanics_steps;
        c.cell_steps = clock->cell_steps;
        if (clock->pending & ~std::int64_t{7}) throw std::invalid_argument("unknown pending bits in the clock");
        c.pending = clock->pending;
        auto wrap = [&](biodiff_hook h, const char* which) -> std::function<void(const SimulationClock&)> {
            if (!h) return {};
            return [h, user, which](const SimulationClock& k) {
                biodiff_clock v;
                to_c_clock(k, &v);
                if (h(user, &v) != 0) throw state_error(std::string(which) + " hook aborted the run");
            };
        };
        EngineHooks hooks;
        hooks.mechanics = wrap(mechanics, "mechanics");
        hooks.cell = wrap(cell, "cell");
        hooks.snapshot = wrap(snapshot, "snapshot");
        hooks.snapshot_interval = snapshot_interval;
        RunMetrics m;
        try {
            m = run_simulation(dev(session), c, with_sources != 0, hooks);
        } catch (...) {
            to_c_clock(c, clock); // counters as far as the run got
            throw;
        }
        to_c_clock(c, clock);
        if (metrics) {
            metrics->wall_seconds = m.wall_seconds;
            metrics->diffusion_seconds = m.diffusion_seconds;
            metrics->hook_seconds = m.hook_seconds;
            metrics->snapshot_seconds = m.snapshot_seconds;
            metrics->diffusion_steps = m.diffusion_steps;
            metrics->mechanics_steps = m.mechanics_steps;
            metrics->cell_steps = m.cell_steps;
            metrics->snapshots = m.snapshots;
        }
    });
}

int biodiff_translate_vector_to_array(const double* const* voxels, const int64_t* counts, int64_t nvox, double* out,
                                      int32_t* substrates)
{
    return guarded([&] {
        need(substrates, "substrates");
        if (nvox < 0) throw std::invalid_argument("negative voxel count");
        if (nvox > 0) {
            need(voxels, "voxels");
            need(counts, "counts");
        }
        NestedDensity nested(static_cast<std::size_t>(nvox));
        for (int64_t v = 0; v < nvox; ++v) {
            if (counts[v] < 0) throw std::invalid_argument("negative substrate count");
            if (counts[v] > 0) need(voxels[v], "voxel values");
            nested[v].assign(voxels[v], voxels[v] + counts[v]);
        }
        const DensityField f = translate_vector_to_array(nested);
        *substrates = f.substrates;
        if (out) std::copy(f.values.begin(), f.values.end(), out);
    });
}

int biodiff_upload_field_nested(biodiff_session* session, const double* const* voxels, const int64_t* counts,
                                int64_t nvox)
{
    return guarded([&] {
        DeviceSession& d = dev(session);
        if (nvox != d.value_count() / d.substrates()) throw state_error("density field size does not match the mesh");
        need(voxels, "voxels");
        need(counts, "counts");
        const int S = d.substrates();
        std::vector<double> flat(static_cast<std::size_t>(d.value_count()));
        for (int64_t v = 0; v < nvox; ++v) {
            if (counts[v] != S)  // translate_vector_to_array's ragged check (mesh.cpp:110-114)
                throw std::invalid_argument("ragged nested density: voxel " + format_int(v) + " holds " +
                                            format_int(counts[v]) + " substrates, expected " + format_int(S));
            need(voxels[v], "voxel values");
            std::copy(voxels[v], voxels[v] + S, flat.begin() + v * S);
        }
        d.upload(flat.data(), static_cast<std::int64_t>(flat.size()));
        d.synchronize();
    });
}

int biodiff_download_field_nested(biodiff_session* session, double* const* voxels, int64_t nvox)
{
    return guarded([&] {
        DeviceSession& d = dev(session);
        if (nvox != d.value_count() / d.substrates()) throw state_error("density field size does not match the mesh");
        need(voxels, "voxels");
        const int S = d.substrates();
        std::vector<double> flat(static_cast<std::size_t>(d.value_count()));
        d.download(flat.data(), static_cast<std::int64_t>(flat.size()));
        for (int64_t v = 0; v < nvox; ++v) {
            need(voxels[v], "voxel values");
            std::copy(flat.begin() + v * S, flat.begin() + (v + 1) * S, voxels[v]);
        }
    });
}

int biodiff_field_all_finite(biodiff_session* session, int32_t* finite)
{
    return guarded([&] {
        need(finite, "finite");
        *finite = dev(session).all_finite() ? 1 : 0;
    });
}

int biodiff_upload_field(biodiff_session* session, const double* values, int64_t count)
{
    return guarded([&] {
        need(values, "values");
        dev(session).upload(values, count);
    });
}

int biodiff_fill_field(biodiff_session* session, const double* initial)
{
    return guarded([&] {
        need(initial, "initial");
        dev(session).fill(initial + session->s0);
    });
}

int biodiff_upload_field_global(biodiff_session* session, const double* values, int64_t count)
{
    return guarded([&] {
        need(values, "values");
        DeviceSession& d = dev(session);
        if (session->replicas > 1) throw state_error("ensembles upload their stacked field with biodiff_upload_field");
        if (count != session->mesh.voxel_count() * session->S)
            throw state_error("global field size does not match the global mesh and substrates");
        const std::int64_t plane = static_cast<std::int64_t>(session->mesh.nx) * session->mesh.ny;
        const std::int64_t v0 = session->slab ? session->z0 * plane : 0;
        const double* src = values + v0 * session->S;
        if (!session->sharded()) {
            d.upload(src, d.value_count());
            return;
        }
        const std::int64_t nvox = d.value_count() / d.substrates();
        const std::vector<double> packed = columns(src, nvox, session->S, session->s0, session->s1);
        d.upload(packed.data(), static_cast<std::int64_t>(packed.size()));
        d.synchronize();
    });
}

int biodiff_download_field_global(biodiff_session* session, double* values, int64_t count)
{
    return guarded([&] {
        need(values, "values");
        DeviceSession& d = dev(session);
        if (session->replicas > 1) throw state_error("ensembles download their stacked field with biodiff_download_field");
        if (count != session->mesh.voxel_count() * session->S)
            throw state_error("global field size does not match the global mesh and substrates");
        const std::int64_t plane = static_cast<std::int64_t>(session->mesh.nx) * session->mesh.ny;
        const std::int64_t v0 = session->slab ? session->z0 * plane : 0;
        double* dst = values + v0 * session->S;
        if (!session->sharded()) {
            d.download(dst, d.value_count());
            return;
        }
        const int SL = d.substrates();
        std::vector<double> packed(static_cast<std::size_t>(d.value_count()));
        d.download(packed.data(), d.value_count());
        const std::int64_t nvox = d.value_count() / SL;
        for (std::int64_t v = 0; v < nvox; ++v)
            std::copy(packed.begin() + v * SL, packed.begin() + (v + 1) * SL, dst + v * session->S + session->s0);
    });
}

int biodiff_download_field(biodiff_session* session, double* values, int64_t count)
{
    return guarded([&] {
        need(values, "values");
        dev(session).download(values, count);
    });
}

int biodiff_download_field_range(biodiff_session* session, int64_t offset, int64_t count, double* values)
{
    return guarded([&] {
        need(values, "values");
        dev(session).download_range(values, offset, count);
    });
}

int biodiff_diffusion_sweep(biodiff_session* session, int32_t axis)
{
    return guarded([&] { dev(session).sweep(to_axis(axis)); });
}

int biodiff_apply_dirichlet(biodiff_session* session)
{
    return guarded([&] { dev(session).apply_dirichlet(); });
}

int biodiff_diffuse_decay_step(biodiff_session* session)
{
    return guarded([&] { dev(session).diffuse_decay_step(); });
}

int biodiff_cell_sources_sinks_step(biodiff_session* session, double dt)
{
    return guarded([&] { dev(session).sources(dt); });
}

int biodiff_advance(biodiff_session* session, int64_t steps, double dt, int32_t with_sources)
{
    return guarded([&] { dev(session).advance(steps, dt, with_sources != 0); });
}

int biodiff_prepare_advance(biodiff_session* session, int64_t steps, double dt, int32_t with_sources)
{
    return guarded([&] { dev(session).prepare_advance(steps, dt, with_sources != 0); });
}

int biodiff_synchronize(biodiff_session* session)
{
    return guarded([&] { dev(session).synchronize(); });
}

int biodiff_session_stream(biodiff_session* session, void** stream)
{
    return guarded([&] {
        need(stream, "stream");
        *stream = dev(session).stream();
    });
}

int biodiff_set_kernel_timing(biodiff_session* session, int32_t enabled)
{
    return guarded([&] { dev(session).set_kernel_timing(enabled != 0); });
}

int biodiff_kernel_times(biodiff_session* session, int32_t* n, int64_t* launches, double* milliseconds)
{
    return guarded([&] {
        need(n, "n");
        *n = kNumKernelClasses;
        if (launches && milliseconds) dev(session).kernel_times(launches, milliseconds);
    });
}

int biodiff_event_record(biodiff_session* session, int32_t slot)
{
    return guarded([&] { dev(session).event_record(slot); });
}

int biodiff_event_elapsed(biodiff_session* session, int32_t begin, int32_t end, double* milliseconds)
{
    return guarded([&] {
        need(milliseconds, "milliseconds");
        *milliseconds = dev(session).event_elapsed(begin, end);
    });
}

int biodiff_launch_count(biodiff_session* session, int64_t* launches)
{
    return guarded([&] {
        need(launches, "launches");
        *launches = dev(session).launch_count();
    });
}

int biodiff_cross_check(biodiff_session* session, const double* other, int64_t count, double abs_tol,
                        double rel_tol, double* max_abs, double* max_rel, int64_t* worst_index, int32_t* pass)
{
    return guarded([&] {
        need(other, "other");
        need(max_abs, "max_abs");
        need(max_rel, "max_rel");
        need(worst_index, "worst_index");
        need(pass, "pass");
        bool p = false;
        std::int64_t w = -1;
        dev(session).cross_check(other, count, abs_tol, rel_tol, max_abs, max_rel, &w, &p);
        *worst_index = w;
        *pass = p ? 1 : 0;
    });
}

// ---- ensembles ---------------------------------------------------------------

int biodiff_ensemble_create(const biodiff_mesh* mesh, int32_t substrates, int32_t replicas, int32_t device,
                            biodiff_session** out)
{
    return guarded([&] {
        need(out, "out");
        *out = nullptr;
        auto s = std::make_unique<biodiff_session>();
        s->mesh = to_mesh(mesh);
        s->S = substrates;
        s->s1 = substrates;
        s->replicas = replicas;
        s->dev = std::make_unique<DeviceSession>(s->mesh, substrates, device, replicas);
        *out = s.release();
    });
}

// Per-replica SolverWorkspaces::build (solver.cpp:277-287), uploaded as
// replicas consecutive coefficient sets per axis.
int biodiff_ensemble_set_substrates(biodiff_session* session, const double* diffusion, const double* decay, double dt)
{
    return guarded([&] {
        need(diffusion, "diffusion");
        need(decay, "decay");
        DeviceSession& d = dev(session);
        const int S = d.substrates(), R = d.replicas();
        std::vector<SolverWorkspaces> all;
        for (int r = 0; r < R; ++r) {
            std::vector<SubstrateParams> params;
            for (int s = 0; s < S; ++s) {
                const double D = diffusion[r * S + s], L = decay[r * S + s];
                if (D < 0.0) throw config_error("substrate has negative diffusion coefficient");
                if (L < 0.0) throw config_error("substrate has negative decay rate");
                params.push_back({"s" + std::to_string(s), D, L, 0.0});
            }
            all.push_back(SolverWorkspaces::build(session->mesh, params, dt));
        }
        auto upload = [&](auto member) {
            if (!(all[0].*member)) return;
            const SolverWorkspace& w0 = *(all[0].*member);
            std::vector<double> q, dinv, cb;
            for (const auto& ws : all) {
                const SolverWorkspace& w = *(ws.*member);
                q.insert(q.end(), w.off_diag.begin(), w.off_diag.end());
                dinv.insert(dinv.end(), w.denom_inv.begin(), w.denom_inv.end());
                cb.insert(cb.end(), w.c_back.begin(), w.c_back.end());
            }
            d.set_workspace(w0.axis, w0.n, w0.dims, w0.dt, q.data(), dinv.data(), cb.data());
        };
        upload(&SolverWorkspaces::x);
        upload(&SolverWorkspaces::y);
        upload(&SolverWorkspaces::z);
    });
}

// Agents of all replicas: replica[n] in [0, replicas); ids must be unique
// within a replica. Each replica's population is validated and grouped as
// AgentPopulation does (agents.cpp:12-73).
int biodiff_ensemble_set_agents(biodiff_session* session, int64_t n, const int32_t* replica, const int64_t* ids,
                                const double* positions, const double* volume, const double* secretion,
                                const double* uptake, const double* saturation)
{
    return guarded([&] {
        DeviceSession& d = dev(session);
        const int S = d.substrates(), R = d.replicas();
        if (n < 0) throw std::invalid_argument("negative agent count");
        if (n > 0) {
            need(replica, "replica");
            need(ids, "ids");
            need(positions, "positions");
            need(volume, "volume");
            need(secretion, "secretion");
            need(uptake, "uptake");
            need(saturation, "saturation");
        }
        std::vector<std::vector<CellAgent>> per(R);
        for (int64_t a = 0; a < n; ++a) {
            if (replica[a] < 0 || replica[a] >= R) throw std::invalid_argument("agent replica out of range");
            CellAgent c;
            c.id = ids[a];
            c.position = {positions[3 * a], positions[3 * a + 1], positions[3 * a + 2]};
            c.volume = volume[a];
            c.secretion_rates.assign(secretion + a * S, secretion + (a + 1) * S);
            c.uptake_rates.assign(uptake + a * S, uptake + (a + 1) * S);
            c.saturation_densities.assign(saturation + a * S, saturation + (a + 1) * S);
            per[replica[a]].push_back(std::move(c));
        }
        std::vector<AgentPopulation> pops;
        pops.reserve(R);
        for (int r = 0; r < R; ++r) pops.emplace_back(std::move(per[r]), session->mesh, S);
        std::vector<const AgentPopulation*> ptrs;
        for (const auto& p : pops) ptrs.push_back(&p);
        d.set_agents_multi(ptrs);
    });
}

// ---- z-slab decomposition -------------------------------------------------

int biodiff_zslab_create(const biodiff_mesh* global_mesh, int32_t substrates, int32_t z0, int32_t z1, int32_t device,
                         biodiff_session** out)
{
    return guarded([&] {
        need(out, "out");
        *out = nullptr;
        auto s = std::make_unique<biodiff_session>();
        s->mesh = to_mesh(global_mesh);
        if (z0 < 0 || z1 > s->mesh.nz || z0 >= z1) throw config_error("z-slab planes must satisfy 0 <= z0 < z1 <= nz");
        s->S = substrates;
        s->s1 = substrates;
        s->slab = true;
        s->z0 = z0;
        s->z1 = z1;
        CartesianMesh local = s->mesh;
        local.nz = z1 - z0;
        local.z_min = s->mesh.z_min + z0 * s->mesh.dz;
        local.z_max = s->mesh.z_min + z1 * s->mesh.dz;
        s->dev = std::make_unique<DeviceSession>(local, substrates, device);
        s->dev->configure_slab(s->mesh.nz, z0);
        *out = s.release();
    });
}

int biodiff_shard_create(const biodiff_mesh* global_mesh, int32_t substrates, int32_t s0, int32_t s1, int32_t z0,
                         int32_t z1, int32_t device, biodiff_session** out)
{
    return guarded([&] {
        need(out, "out");
        *out = nullptr;
        auto s = std::make_unique<biodiff_session>();
        s->mesh = to_mesh(global_mesh);
        if (substrates < 1) throw config_error("a shard needs at least one substrate");
        if (s0 < 0 || s1 > substrates || s0 >= s1)
            throw config_error("substrate shard must satisfy 0 <= s0 < s1 <= substrates");
        if (z0 < 0 || z1 > s->mesh.nz || z0 >= z1) throw config_error("z-slab planes must satisfy 0 <= z0 < z1 <= nz");
        s->S = substrates;
        s->s0 = s0;
        s->s1 = s1;
        CartesianMesh local = s->mesh;
        s->slab = !(z0 == 0 && z1 == s->mesh.nz);
        if (s->slab) {
            s->z0 = z0;
            s->z1 = z1;
            local.nz = z1 - z0;
            local.z_min = s->mesh.z_min + z0 * s->mesh.dz;
            local.z_max = s->mesh.z_min + z1 * s->mesh.dz;
        }
        s->dev = std::make_unique<DeviceSession>(local, s1 - s0, device);
        if (s->slab) s->dev->configure_slab(s->mesh.nz, z0);
        *out = s.release();
    });
}

int biodiff_shard_info(biodiff_session* session, int32_t* s0, int32_t* s1, int32_t* substrates)
{
    return guarded([&] {
        need(s0, "s0");
        need(s1, "s1");
        need(substrates, "substrates");
        dev(session);
        *s0 = session->s0;
        *s1 = session->s1;
        *substrates = session->S;
    });
}

int biodiff_zslab_info(biodiff_session* session, int32_t* z0, int32_t* z1, int32_t* nz_global)
{
    return guarded([&] {
        need(z0, "z0");
        need(z1, "z1");
        need(nz_global, "nz_global");
        dev(session);
        *z0 = session->slab ? session->z0 : 0;
        *z1 = session->slab ? session->z1 : session->mesh.nz;
        *nz_global = session->mesh.nz;
    });
}

int biodiff_nccl_unique_id(uint8_t* out)
{
    return guarded([&] {
        need(out, "out");
        nccl_unique_id(out);
    });
}

int biodiff_zslab_connect_nccl(biodiff_session* session, const uint8_t* unique_id, int32_t nranks, int32_t rank)
{
    return guarded([&] {
        need(unique_id, "unique_id");
        if (!session || !session->slab) throw state_error("not a z-slab session");
        dev(session).connect_nccl(unique_id, nranks, rank);
    });
}

int biodiff_zslab_connect_host(biodiff_session* session, int32_t nranks, int32_t rank, biodiff_plane_exchange fn,
                               void* user)
{
    return guarded([&] {
        if (!session || !session->slab) throw state_error("not a z-slab session");
        static_assert(std::is_same_v<DeviceSession::HostExchange, biodiff_plane_exchange>, "callback ABI");
        dev(session).connect_host_transport(nranks, rank, fn, user);
    });
}

int biodiff_zslab_link_local(biodiff_session** sessions, int32_t count)
{
    return guarded([&] {
        need(sessions, "sessions");
        std::vector<DeviceSession*> v;
        for (int32_t p = 0; p < count; ++p) v.push_back(&dev(sessions[p]));
        DeviceSession::link_local(v);
    });
}

int biodiff_zslab_group_advance(biodiff_session** sessions, int32_t count, int64_t steps, double dt,
                                int32_t with_sources)
{
    return guarded([&] {
        need(sessions, "sessions");
        if (steps < 0) throw std::invalid_argument("step count must be non-negative");
        std::vector<DeviceSession*> v;
        for (int32_t p = 0; p < count; ++p) v.push_back(&dev(sessions[p]));
        DeviceSession::group_advance(v, steps, dt, with_sources != 0);
    });
}

} // extern "C"

// ---- XML configuration (config.hpp; the reference's config.hpp:75-116) ----

namespace {

SimConfig config_from(const char* xml, const char* path)
{
    if (path) return parse_config(path);
    need(xml, "xml");
    return parse_config_text(xml);
}

} // namespace

int biodiff_config_canonical(const char* xml, const char* path, char* out, int64_t capacity, int64_t* needed)
{
    return guarded([&] {
        need(needed, "needed");
        const std::string text = serialize_config(config_from(xml, path));
        *needed = static_cast<int64_t>(text.size()) + 1;
        if (out && capacity >= *needed) std::memcpy(out, text.c_str(), text.size() + 1);
    });
}

int biodiff_config_save(const char* xml, const char* path, const char* out_path)
{
    return guarded([&] {
        need(out_path, "out_path");
        save_config(config_from(xml, path), out_path);
    });
}

int biodiff_config_build(const char* xml, const char* path, int64_t* voxels, int32_t* substrates,
                         int64_t* dirichlet_count, int64_t* agent_count, double* field, int64_t* dir_voxel,
                         uint8_t* dir_mask, double* dir_values, int64_t* ids, double* positions, double* volume,
                         double* secretion, double* uptake, double* saturation)
{
    return guarded([&] {
        need(voxels, "voxels");
        need(substrates, "substrates");
        need(dirichlet_count, "dirichlet_count");
        need(agent_count, "agent_count");
        const SimConfig cfg = config_from(xml, path);
        const Microenvironment env = build_microenvironment(cfg);
        const AgentPopulation agents = build_agents(cfg, env.mesh);
        const int S = env.substrate_count();
        *voxels = env.mesh.voxel_count();
        *substrates = S;
        *dirichlet_count = static_cast<int64_t>(env.dirichlet.size());
        *agent_count = static_cast<int64_t>(agents.size());
        if (!field) return; // sizes only
        std::memcpy(field, env.field.values.data(), sizeof(double) * env.field.values.size());
        int64_t e = 0;
        for (const auto& d : env.dirichlet.entries()) {
            dir_voxel[e] = d.voxel;
            std::copy(d.mask.begin(), d.mask.end(), dir_mask + e * S);
            std::copy(d.values.begin(), d.values.end(), dir_values + e * S);
            ++e;
        }
        int64_t a = 0;
        for (const auto& c : agents.agents()) {
            ids[a] = c.id;
            std::copy(c.position.begin(), c.position.end(), positions + 3 * a);
            volume[a] = c.volume;
            std::copy(c.secretion_rates.begin(), c.secretion_rates.end(), secretion + a * S);
            std::copy(c.uptake_rates.begin(), c.uptake_rates.end(), uptake + a * S);
            std::copy(c.saturation_densities.begin(), c.saturation_densities.end(), saturation + a * S);
            ++a;
        }
    });
}

int biodiff_session_from_config(const char* xml, const char* path, int32_t device, biodiff_session** out,
                                biodiff_clock* clock)
{
    return guarded([&] {
        need(out, "out");
        *out = nullptr;
        const SimConfig cfg = config_from(xml, path);
        const Microenvironment env = build_microenvironment(cfg);
        const AgentPopulation agents = build_agents(cfg, env.mesh);
        auto s = std::make_unique<biodiff_session>();
        s->mesh = env.mesh;
        s->S = env.substrate_count();
        s->s1 = s->S;
        s->dev = std::make_unique<DeviceSession>(s->mesh, s->S, device);
        upload_workspaces(s.get(), SolverWorkspaces::build(env.mesh, env.substrates, cfg.dt_diff));
        s->dev->set_dirichlet(env.dirichlet);
        if (!agents.empty()) install_agents(s.get(), agents);
        s->dev->upload(env.field.values.data(), static_cast<std::int64_t>(env.field.values.size()));
        if (clock) to_c_clock(SimulationClock::make(cfg.dt_diff, cfg.dt_mech, cfg.dt_cell, cfg.max_time), clock);
        *out = s.release();
    });
}
