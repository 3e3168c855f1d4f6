// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// An extern "C" driver over the UNMODIFIED reference sources, compiled where
// they lie under /root/reference/proj/src/core by oracle/Makefile into
// oracle/_ref/libbiodiff_ref.so. It builds reference objects programmatically
// (mirroring build_microenvironment config.cpp:494-527 and build_agents
// config.cpp:529-566, since config.cpp needs the absent Boost) and drives the
// reference's own entry points:
//   SolverWorkspaces::build        solver.cpp:277-287
//   diffusion_sweep                solver.cpp:248-265
//   apply_dirichlet_conditions     solver.cpp:267-275
//   diffuse_decay_step             solver.cpp:289-299
//   cell_sources_sinks_step        agents.cpp:75-112
//   AgentPopulation (grouping)     agents.cpp:12-73
//   run_convergence_test           validation.cpp:65-110
//   run_dirichlet_mutant_check     validation.cpp:274-287
// The step loop [diffuse_decay_step; cell_sources_sinks_step] is SPEC.md:297
// (the engine itself is absent from the snapshot).
//
// Only tests/ and bench.py (reference arm / cpu_baseline) load this library.
#include "core/agents.hpp"
#include "core/backend.hpp"
#include "core/errors.hpp"
#include "core/mesh.hpp"
#include "core/solver.hpp"
#include "core/text.hpp"
#include "core/validation.hpp"

#include <fstream>
#include <sstream>

#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

using namespace biodiff;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f)
{
    try {
        f();
        return 0;
    } catch (const config_error& e) {
        g_err = e.what();
        return 1;
    } catch (const io_error& e) {
        g_err = e.what();
        return 4;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

struct RefCtx {
    Microenvironment env;
    std::optional<SolverWorkspaces> ws;
    AgentPopulation agents;
    std::unique_ptr<WorkerPool> pool;
};

} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// load_agents (config.cpp:416-477) restated over the reference's own pieces
// (text.cpp trim / split_csv_line / parse_int / parse_double / format_int and
// the AgentPopulation ctor, agents.cpp:12-43): config.cpp itself needs the
// absent Boost. Stores the population in the context.
int ref_load_agents(void* h, const char* path, const char* const* names, int S)
{
    return guarded([&] {
        auto* c = static_cast<RefCtx*>(h);
        auto fail = [](const std::string& m) -> void { throw config_error(m); };
        auto agent_fail = [&](std::size_t line, const std::string& msg) {
            fail(std::string("agent file ") + path + " line " + format_int(static_cast<std::int64_t>(line)) + ": " +
                 msg);
        };
        std::ifstream in(path, std::ios::binary);
        if (!in) fail(std::string("agent file not found: ") + path);
        std::string expected = "id,x,y,z,volume";
        for (int s = 0; s < S; ++s)
            expected += std::string(",S_") + names[s] + ",U_" + names[s] + ",target_" + names[s];
        std::string line;
        std::size_t line_no = 0;
        if (!std::getline(in, line)) fail(std::string("agent file ") + path + " is empty");
        ++line_no;
        if (trim(line) != expected) agent_fail(line_no, "header must be '" + expected + "'");
        std::vector<CellAgent> agents;
        while (std::getline(in, line)) {
            ++line_no;
            const std::string stripped = trim(line);
            if (stripped.empty()) continue;
            const auto fields = split_csv_line(stripped);
            if (fields.size() != 5 + 3 * static_cast<std::size_t>(S))
                agent_fail(line_no, "expected " + format_int(5 + 3 * S) + " fields, got " +
                                        format_int(static_cast<std::int64_t>(fields.size())));
            try {
                CellAgent a;
                a.id = parse_int(fields[0], "id");
                a.position = {parse_double(fields[1], "x"), parse_double(fields[2], "y"), parse_double(fields[3], "z")};
                a.volume = parse_double(fields[4], "volume");
                a.secretion_rates.resize(S);
                a.uptake_rates.resize(S);
                a.saturation_densities.resize(S);
                for (int s = 0; s < S; ++s) {
                    a.secretion_rates[s] = parse_double(fields[5 + 3 * s], "secretion rate");
                    a.uptake_rates[s] = parse_double(fields[6 + 3 * s], "uptake rate");
                    a.saturation_densities[s] = parse_double(fields[7 + 3 * s], "target density");
                }
                agents.push_back(std::move(a));
            } catch (const std::invalid_argument& e) {
                agent_fail(line_no, e.what());
            }
        }
        try {
            c->agents = AgentPopulation(std::move(agents), c->env.mesh, S);
        } catch (const std::exception& e) {
            fail(std::string("agent file ") + path + ": " + e.what());
        }
    });
}

int64_t ref_agent_count(void* h) { return static_cast<int64_t>(static_cast<RefCtx*>(h)->agents.size()); }

int ref_get_agents(void* h, int64_t* ids, double* pos, double* vol, double* sec, double* upt, double* sat)
{
    return guarded([&] {
        const auto& all = static_cast<RefCtx*>(h)->agents.agents();
        for (std::size_t a = 0; a < all.size(); ++a) {
            const std::size_t S = all[a].secretion_rates.size();
            ids[a] = all[a].id;
            for (int k = 0; k < 3; ++k) pos[3 * a + k] = all[a].position[k];
            vol[a] = all[a].volume;
            for (std::size_t s = 0; s < S; ++s) {
                sec[a * S + s] = all[a].secretion_rates[s];
                upt[a * S + s] = all[a].uptake_rates[s];
                sat[a * S + s] = all[a].saturation_densities[s];
            }
        }
    });
}

// translate_vector_to_array (mesh.cpp:101-119) of the reference on a nested
// density given as per-voxel pointers; out may be null (count only).
int ref_translate_vector_to_array(const double* const* voxels, const int64_t* counts, int64_t nvox, double* out,
                                  int* substrates)
{
    return guarded([&] {
        NestedDensity nested(static_cast<std::size_t>(nvox));
        for (int64_t v = 0; v < nvox; ++v) nested[v].assign(voxels[v], voxels[v] + counts[v]);
        const DensityField f = translate_vector_to_array(nested);
        *substrates = f.substrates;
        if (out) std::copy(f.values.begin(), f.values.end(), out);
    });
}

// translate_array_to_vector (mesh.cpp:121-136) round trip: flat -> nested -> flat.
int ref_translate_round_trip(const double* flat, int64_t count, int S, double* out)
{
    return guarded([&] {
        DensityField f;
        f.substrates = S;
        f.values.assign(flat, flat + count);
        const NestedDensity nested = translate_array_to_vector(f);
        int64_t k = 0;
        for (const auto& v : nested)
            for (double x : v) out[k++] = x;
    });
}

// cross_check (validation.cpp:112-137) of the reference on two flat fields.
int ref_cross_check(const double* a, const double* b, int64_t count, int S, double abs_tol, double rel_tol,
                    double* max_abs, double* max_rel, int64_t* worst, int* pass)
{
    return guarded([&] {
        DensityField fa, fb;
        fa.substrates = fb.substrates = S;
        fa.values.assign(a, a + count);
        fb.values.assign(b, b + count);
        const CrossCheckReport r = cross_check(fa, fb, abs_tol, rel_tol);
        *max_abs = r.max_abs;
        *max_rel = r.max_rel;
        *worst = r.worst_value_index;
        *pass = r.pass ? 1 : 0;
    });
}

// format_int (text.cpp:16-21).
int ref_format_int(int64_t v, char* out, int cap)
{
    const std::string s = format_int(v);
    if (static_cast<int>(s.size()) + 1 > cap) return 1;
    std::memcpy(out, s.c_str(), s.size() + 1);
    return 0;
}

// Builds a Microenvironment. When `staged` is nonzero the reference's own
// Microenvironment::create (nested-vector staging, mesh.cpp:173-195) is used;
// otherwise the public fields are filled directly (SURVEY.md §7 hard part 8),
// which yields the identical field without the 3x staging memory.
int ref_create(const double* bounds, const double* spacing, int S, const double* D, const double* lambda,
               const double* ic, int workers, int staged, void** out)
{
    return guarded([&] {
        auto ctx = std::make_unique<RefCtx>();
        const CartesianMesh mesh = CartesianMesh::from_bounds(bounds[0], bounds[1], bounds[2], bounds[3], bounds[4],
                                                              bounds[5], spacing[0], spacing[1], spacing[2]);
        std::vector<SubstrateParams> params;
        for (int s = 0; s < S; ++s) params.push_back({"s" + std::to_string(s), D[s], lambda[s], ic[s]});
        if (staged) {
            ctx->env = Microenvironment::create(mesh, std::move(params));
        } else {
            ctx->env.mesh = mesh;
            ctx->env.substrates = std::move(params);
            ctx->env.field.substrates = S;
            ctx->env.field.values.resize(static_cast<std::size_t>(mesh.voxel_count()) * S);
            for (std::size_t v = 0; v < static_cast<std::size_t>(mesh.voxel_count()); ++v)
                for (int s = 0; s < S; ++s) ctx->env.field.values[v * S + s] = ic[s];
        }
        ctx->pool = std::make_unique<WorkerPool>(workers <= 0 ? BackendKind::serial()
                                                              : BackendKind::make_parallel(workers));
        *out = ctx.release();
    });
}

void ref_destroy(void* h) { delete static_cast<RefCtx*>(h); }

int ref_mesh_dims(void* h, int* n)
{
    auto* c = static_cast<RefCtx*>(h);
    n[0] = c->env.mesh.nx;
    n[1] = c->env.mesh.ny;
    n[2] = c->env.mesh.nz;
    return 0;
}

int ref_set_field(void* h, const double* v, int64_t count)
{
    return guarded([&] {
        auto* c = static_cast<RefCtx*>(h);
        if (static_cast<std::size_t>(count) != c->env.field.values.size())
            throw std::invalid_argument("field size mismatch");
        std::memcpy(c->env.field.values.data(), v, sizeof(double) * count);
    });
}

int ref_get_field(void* h, double* v, int64_t count)
{
    return guarded([&] {
        auto* c = static_cast<RefCtx*>(h);
        if (static_cast<std::size_t>(count) != c->env.field.values.size())
            throw std::invalid_argument("field size mismatch");
        std::memcpy(v, c->env.field.values.data(), sizeof(double) * count);
    });
}

// values[offset, offset + count) of the field: lets the tests hash a C4-sized
// (34 GB) field in pieces instead of holding a second copy of it.
int ref_get_field_range(void* h, int64_t offset, int64_t count, double* v)
{
    return guarded([&] {
        auto* c = static_cast<RefCtx*>(h);
        if (offset < 0 || count < 0 || static_cast<std::size_t>(offset + count) > c->env.field.values.size())
            throw std::invalid_argument("field range out of bounds");
        std::memcpy(v, c->env.field.values.data() + offset, sizeof(double) * count);
    });
}

// DirichletMap::add (mesh.cpp:138-159), one call per entry in caller order.
int ref_add_dirichlet(void* h, int64_t count, const int64_t* voxel, const uint8_t* mask, const double* values)
{
    return guarded([&] {
        auto* c = static_cast<RefCtx*>(h);
        const int S = c->env.substrate_count();
        for (int64_t e = 0; e < count; ++e)
            c->env.dirichlet.add(voxel[e], std::vector<std::uint8_t>(mask + e * S, mask + (e + 1) * S),
                                 std::vector<double>(values + e * S, values + (e + 1) * S),
                                 c->env.mesh.voxel_count(), S);
    });
}

// Reads back the canonical (sorted, merged) Dirichlet entries.
int64_t ref_dirichlet_size(void* h) { return static_cast<int64_t>(static_cast<RefCtx*>(h)->env.dirichlet.size()); }

int ref_get_dirichlet(void* h, int64_t* voxel, uint8_t* mask, double* values)
{
    auto* c = static_cast<RefCtx*>(h);
    const int S = c->env.substrate_count();
    int64_t e = 0;
    for (const auto& d : c->env.dirichlet.entries()) {
        voxel[e] = d.voxel;
        for (int s = 0; s < S; ++s) {
            mask[e * S + s] = d.mask[s];
            values[e * S + s] = d.values[s];
        }
        ++e;
    }
    return 0;
}

// Boundary clamp exactly as build_microenvironment (config.cpp:506-525).
int ref_add_boundary_dirichlet(void* h, const uint8_t* mask, const double* values)
{
    return guarded([&] {
        auto* c = static_cast<RefCtx*>(h);
        const auto& mesh = c->env.mesh;
        const int S = c->env.substrate_count();
        std::vector<std::uint8_t> m(mask, mask + S);
        std::vector<double> v(values, values + S);
        for (int k = 0; k < mesh.nz; ++k)
            for (int j = 0; j < mesh.ny; ++j)
                for (int i = 0; i < mesh.nx; ++i)
                    if (mesh.is_boundary_voxel(i, j, k))
                        c->env.dirichlet.add(mesh.voxel_index(i, j, k), m, v, mesh.voxel_count(), S);
    });
}

// AgentPopulation ctor (agents.cpp:12-18): validate + grouping.
int ref_set_agents(void* h, int64_t n, const int64_t* ids, const double* pos, const double* volume,
                   const double* secretion, const double* uptake, const double* saturation)
{
    return guarded([&] {
        auto* c = static_cast<RefCtx*>(h);
        const int S = c->env.substrate_count();
        std::vector<CellAgent> agents;
        agents.reserve(static_cast<std::size_t>(n));
        for (int64_t a = 0; a < n; ++a) {
            CellAgent ag;
            ag.id = ids[a];
            ag.position = {pos[3 * a], pos[3 * a + 1], pos[3 * a + 2]};
            ag.volume = volume[a];
            ag.secretion_rates.assign(secretion + a * S, secretion + (a + 1) * S);
            ag.uptake_rates.assign(uptake + a * S, uptake + (a + 1) * S);
            ag.saturation_densities.assign(saturation + a * S, saturation + (a + 1) * S);
            agents.push_back(std::move(ag));
        }
        c->agents = AgentPopulation(std::move(agents), c->env.mesh, S);
    });
}

int64_t ref_group_count(void* h) { return static_cast<int64_t>(static_cast<RefCtx*>(h)->agents.grouping().size()); }

int ref_get_grouping(void* h, int64_t* group_voxel, int64_t* group_offsets, int64_t* order)
{
    auto* c = static_cast<RefCtx*>(h);
    int64_t g = 0, m = 0;
    for (const auto& [voxel, idxs] : c->agents.grouping()) {
        group_voxel[g] = voxel;
        group_offsets[g] = m;
        for (std::size_t i : idxs) order[m++] = static_cast<int64_t>(i);
        ++g;
    }
    group_offsets[g] = m;
    return 0;
}

int ref_build_workspaces(void* h, double dt)
{
    return guarded([&] {
        auto* c = static_cast<RefCtx*>(h);
        c->ws = SolverWorkspaces::build(c->env.mesh, c->env.substrates, dt);
    });
}

// Copies one axis workspace; returns 3 if the axis is inactive.
int ref_get_workspace(void* h, int axis, double* off_diag, double* denom_inv, double* c_back, int* dims)
{
    auto* c = static_cast<RefCtx*>(h);
    if (!c->ws) return 2;
    const std::optional<SolverWorkspace>& w = axis == 0 ? c->ws->x : axis == 1 ? c->ws->y : c->ws->z;
    if (!w) return 3;
    std::memcpy(off_diag, w->off_diag.data(), sizeof(double) * w->off_diag.size());
    std::memcpy(denom_inv, w->denom_inv.data(), sizeof(double) * w->denom_inv.size());
    std::memcpy(c_back, w->c_back.data(), sizeof(double) * w->c_back.size());
    *dims = w->dims;
    return 0;
}

int ref_sweep(void* h, int axis)
{
    return guarded([&] {
        auto* c = static_cast<RefCtx*>(h);
        if (!c->ws) throw state_error("workspaces not built");
        const std::optional<SolverWorkspace>& w = axis == 0 ? c->ws->x : axis == 1 ? c->ws->y : c->ws->z;
        if (!w) throw state_error("axis not active");
        diffusion_sweep(c->env.field, c->env.mesh, *w, *c->pool);
    });
}

int ref_apply_dirichlet(void* h)
{
    return guarded([&] {
        auto* c = static_cast<RefCtx*>(h);
        apply_dirichlet_conditions(c->env.field, c->env.dirichlet);
    });
}

int ref_diffuse_decay_step(void* h)
{
    return guarded([&] {
        auto* c = static_cast<RefCtx*>(h);
        if (!c->ws) throw state_error("workspaces not built");
        diffuse_decay_step(c->env, *c->ws, *c->pool);
    });
}

int ref_sources_step(void* h, double dt)
{
    return guarded([&] {
        auto* c = static_cast<RefCtx*>(h);
        cell_sources_sinks_step(c->env.field, c->agents, c->env.mesh, dt, *c->pool);
    });
}

// The SPEC.md:297 inner loop: steps x [diffuse_decay_step; cell_sources_sinks_step].
// *seconds receives the steady_clock time of the loop alone.
int ref_run(void* h, int64_t steps, double dt, int with_sources, double* seconds)
{
    return guarded([&] {
        auto* c = static_cast<RefCtx*>(h);
        if (!c->ws) c->ws = SolverWorkspaces::build(c->env.mesh, c->env.substrates, dt);
        const auto t0 = std::chrono::steady_clock::now();
        for (int64_t s = 0; s < steps; ++s) {
            diffuse_decay_step(c->env, *c->ws, *c->pool);
            if (with_sources) cell_sources_sinks_step(c->env.field, c->agents, c->env.mesh, dt, *c->pool);
        }
        const auto t1 = std::chrono::steady_clock::now();
        if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    });
}

// Method 1 (validation.cpp:65-110). kind 0 temporal, 1 spatial.
int ref_convergence(int kind, int levels, double* order, double* steps, double* errors, int* pass)
{
    return guarded([&] {
        const ConvergenceReport r =
            run_convergence_test(kind == 0 ? RefineKind::temporal : RefineKind::spatial, levels);
        *order = r.fitted_order;
        for (std::size_t i = 0; i < r.points.size(); ++i) {
            steps[i] = r.points[i].step;
            errors[i] = r.points[i].linf_error;
        }
        *pass = r.pass ? 1 : 0;
    });
}

// text.cpp:9-14 format_double (shortest round trip, std::to_chars).
int ref_format_double(double v, char* out, int cap)
{
    const std::string s = format_double(v);
    if (static_cast<int>(s.size()) + 1 > cap) return 2;
    std::memcpy(out, s.c_str(), s.size() + 1);
    return 0;
}

// validation.cpp:155-200 write_snapshot_pgm / write_snapshot_table of the
// current field into `out` (NUL-terminated); returns the byte count needed.
int64_t ref_snapshot(void* h, int table, int substrate, int z_slice, char* out, int64_t cap)
{
    auto* c = static_cast<RefCtx*>(h);
    std::ostringstream os;
    try {
        if (table)
            write_snapshot_table(c->env.field, c->env.mesh, substrate, z_slice, os);
        else
            write_snapshot_pgm(c->env.field, c->env.mesh, substrate, z_slice, os);
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
    const std::string s = os.str();
    if (out && static_cast<int64_t>(s.size()) + 1 <= cap) std::memcpy(out, s.c_str(), s.size() + 1);
    return static_cast<int64_t>(s.size()) + 1;
}

// Method 3 mutant (validation.cpp:274-287): flags = {clean, crosscheck, table}.
int ref_mutant_check(int* flags)
{
    return guarded([&] {
        const MutantCheckReport r = run_dirichlet_mutant_check();
        flags[0] = r.clean_reproducible;
        flags[1] = r.crosscheck_detected;
        flags[2] = r.table_detected;
    });
}

} // extern "C"
