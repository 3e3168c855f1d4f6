// INTEGRATION.md §1, compiled: the reference's OWN types (headers under
// /root/reference/proj/src, objects from oracle/_ref built by oracle/Makefile)
// bound to libbiodiff_b200.so through include/biodiff_b200.h, the way a
// maintainer would swap the reference's WorkerPool for the B200 session.
//
//   bind_to_b200()        — INTEGRATION.md §1 (reference types -> C ABI)
//   main                  — runs N steps on the GPU through the binding and
//                           the reference's own loop (diffuse_decay_step,
//                           solver.cpp:289-299; cell_sources_sinks_step,
//                           agents.cpp:75-112) on a WorkerPool, and compares
//                           the final fields bit for bit.
//
// build: oracle/Makefile target `binding` (needs /root/reference here; the
// binary, oracle/_ref/reference_binding, travels to the GPU box);
// run: tests/test_reference_binding_gpu.py.
// The reference's config.cpp (build_microenvironment) needs the absent Boost,
// so the Microenvironment is assembled from the reference's public types the
// same way build_microenvironment does (config.cpp:494-566): boundary
// Dirichlet shell + interior entries, agents validated by AgentPopulation.
#include "core/agents.hpp"  // reference
#include "core/backend.hpp" // reference
#include "core/mesh.hpp"    // reference
#include "core/solver.hpp"  // reference

#include "biodiff_b200.h" // this repo

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

using namespace biodiff;

namespace {

void ok(int status, const char* what)
{
    if (status != BIODIFF_OK) throw std::runtime_error(std::string(what) + ": " + biodiff_last_error());
}

// ---- the reference's Microenvironment, SolverWorkspaces
// and AgentPopulation handed to the B200 session through the C ABI.
biodiff_session* bind_to_b200(const Microenvironment& env, const SolverWorkspaces& ws, const AgentPopulation& agents,
                              int device)
{
    const int S = env.substrate_count();
    const CartesianMesh& g = env.mesh;
    biodiff_mesh m{g.x_min, g.x_max, g.y_min, g.y_max, g.z_min, g.z_max, g.dx, g.dy, g.dz, g.nx, g.ny, g.nz};
    biodiff_session* s = nullptr;
    ok(biodiff_session_create(&m, S, device, &s), "biodiff_session_create");

    // SolverWorkspace bits, axis by axis (solver.hpp:24-33)
    for (const auto* w : {&ws.x, &ws.y, &ws.z})
        if (*w)
            ok(biodiff_set_workspace(s, static_cast<int32_t>((*w)->axis), (*w)->n, (*w)->dims, (*w)->dt,
                                     (*w)->off_diag.data(), (*w)->denom_inv.data(), (*w)->c_back.data()),
               "biodiff_set_workspace");

    // DirichletMap entries (mesh.hpp:113-141)
    std::vector<int64_t> vox;
    std::vector<uint8_t> mask;
    std::vector<double> val;
    for (const auto& e : env.dirichlet.entries()) {
        vox.push_back(e.voxel);
        mask.insert(mask.end(), e.mask.begin(), e.mask.end());
        val.insert(val.end(), e.values.begin(), e.values.end());
    }
    ok(biodiff_set_dirichlet(s, static_cast<int64_t>(vox.size()), vox.data(), mask.data(), val.data()),
       "biodiff_set_dirichlet");

    // Agents (agents.hpp:14-24); the library re-validates and re-groups them
    // exactly as AgentPopulation does (agents.cpp:20-73).
    std::vector<int64_t> ids;
    std::vector<double> pos, vol, sec, upt, sat;
    for (const auto& a : agents.agents()) {
        ids.push_back(a.id);
        pos.insert(pos.end(), a.position.begin(), a.position.end());
        vol.push_back(a.volume);
        sec.insert(sec.end(), a.secretion_rates.begin(), a.secretion_rates.end());
        upt.insert(upt.end(), a.uptake_rates.begin(), a.uptake_rates.end());
        sat.insert(sat.end(), a.saturation_densities.begin(), a.saturation_densities.end());
    }
    ok(biodiff_set_agents(s, static_cast<int64_t>(ids.size()), ids.data(), pos.data(), vol.data(), sec.data(),
                          upt.data(), sat.data()),
       "biodiff_set_agents");

    ok(biodiff_upload_field(s, env.field.values.data(), static_cast<int64_t>(env.field.values.size())),
       "biodiff_upload_field");
    return s;
}

// Deterministic generator (no <random> distribution differences across libstdc++).
struct Lcg {
    uint64_t x;
    double next() // [0, 1)
    {
        x = x * 6364136223846793005ull + 1442695040888963407ull;
        return static_cast<double>(x >> 11) * (1.0 / 9007199254740992.0);
    }
};

} // namespace

int main(int argc, char** argv)
{
    try {
        const int steps = argc > 1 ? std::atoi(argv[1]) : 200;
        const int workers = argc > 2 ? std::atoi(argv[2]) : 8;
        // 60 x 44 x 36 voxels of 20 um, 3 substrates (build_microenvironment's
        // shape of case: oxygen-like with a boundary shell, two others free).
        const double dx = 20.0, dt = 0.01;
        const CartesianMesh mesh = CartesianMesh::from_bounds(-600, 600, -440, 440, -360, 360, dx, dx, dx);
        std::vector<SubstrateParams> subs = {{"oxygen", 1.0e5, 0.1, 38.0},
                                             {"signal", 3.0e3, 0.02, 0.0},
                                             {"drug", 8.0e2, 0.005, 1.5}};
        Microenvironment env = Microenvironment::create(mesh, subs);
        const int S = env.substrate_count();
        const index_t nvox = mesh.voxel_count();
        // Dirichlet: substrate 0 on every boundary voxel (config.cpp:506-525),
        // plus interior entries clamping substrates 1 and 2.
        for (int k = 0; k < mesh.nz; ++k)
            for (int j = 0; j < mesh.ny; ++j)
                for (int i = 0; i < mesh.nx; ++i) {
                    if (!(i == 0 || j == 0 || k == 0 || i == mesh.nx - 1 || j == mesh.ny - 1 || k == mesh.nz - 1))
                        continue;
                    const index_t v = i + static_cast<index_t>(mesh.nx) * (j + static_cast<index_t>(mesh.ny) * k);
                    env.dirichlet.add_single(v, 0, 38.0, nvox, S);
                }
        Lcg rng{20261017};
        for (int e = 0; e < 12; ++e) {
            const int i = 3 + static_cast<int>(rng.next() * (mesh.nx - 6));
            const int j = 3 + static_cast<int>(rng.next() * (mesh.ny - 6));
            const int k = 3 + static_cast<int>(rng.next() * (mesh.nz - 6));
            const index_t v = i + static_cast<index_t>(mesh.nx) * (j + static_cast<index_t>(mesh.ny) * k);
            env.dirichlet.add(v, {0, 1, static_cast<uint8_t>(e % 2)}, {0.0, 5.0 + e, 0.25 * e}, nvox, S);
        }
        // 1500 agents in a ball (ids shuffled, several per voxel in the core).
        std::vector<CellAgent> cells;
        for (int a = 0; a < 1500; ++a) {
            CellAgent c;
            c.id = 100000 - 37 * a;
            const double r = 260.0 * std::cbrt(rng.next());
            const double u = 2.0 * rng.next() - 1.0, ph = 6.283185307179586 * rng.next();
            const double st = std::sqrt(1.0 - u * u);
            c.position = {r * st * std::cos(ph), r * st * std::sin(ph), r * u};
            c.volume = 2494.0 * (0.5 + rng.next());
            c.secretion_rates = {0.0, 10.0 * rng.next(), a % 7 == 0 ? 2.0 : 0.0};
            c.uptake_rates = {10.0 * rng.next(), 0.1 * rng.next(), 0.5 * rng.next()};
            c.saturation_densities = {0.0, 1.0 + rng.next(), 3.0};
            cells.push_back(std::move(c));
        }
        const AgentPopulation agents(std::move(cells), mesh, S);
        const SolverWorkspaces ws = SolverWorkspaces::build(mesh, env.substrates, dt);

        // GPU, through the binding
        biodiff_session* s = bind_to_b200(env, ws, agents, 0);
        ok(biodiff_advance(s, steps, dt, 1), "biodiff_advance");
        std::vector<double> gpu(env.field.values.size());
        ok(biodiff_download_field(s, gpu.data(), static_cast<int64_t>(gpu.size())), "biodiff_download_field");
        ok(biodiff_session_destroy(s), "biodiff_session_destroy");

        // The reference's own loop on its WorkerPool
        WorkerPool pool(workers <= 1 ? BackendKind::serial() : BackendKind::make_parallel(workers));
        for (int n = 0; n < steps; ++n) {
            diffuse_decay_step(env, ws, pool);
            cell_sources_sinks_step(env.field, agents, env.mesh, dt, pool);
        }
        std::size_t diff = 0;
        for (std::size_t q = 0; q < gpu.size(); ++q)
            if (std::memcmp(&gpu[q], &env.field.values[q], sizeof(double)) != 0) ++diff;
        std::printf("reference_binding: %d steps, %zu values (%dx%dx%d x %d), %zu differ from the reference\n", steps,
                    gpu.size(), mesh.nx, mesh.ny, mesh.nz, S, diff);
        return diff == 0 ? 0 : 1;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "reference_binding: %s\n", e.what());
        return 2;
    }
}
