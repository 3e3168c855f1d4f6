// Drives the C++ host mirror (paper_2110_13368_b200/csrc/host.hpp) exactly
// as a reference caller would: Microenvironment::create, boundary Dirichlet
// (config.cpp:506-525), AgentPopulation, SolverWorkspaces::build, then the
// entry points with a DeviceBackend in place of WorkerPool.
//
//   host_api_driver cpu <out.bin>   host-only set-up artefacts (coefficients, grouping)
//   host_api_driver gpu <out.bin>   the final field after `steps` device steps
#include "host.hpp"

#include <cstdio>
#include <cstring>
#include <fstream>
#include <random>
#include <string>

using namespace biodiff_b200;

int main(int argc, char** argv)
{
    if (argc < 3) {
        std::fprintf(stderr, "usage: %s cpu|gpu out.bin\n", argv[0]);
        return 1;
    }
    const std::string mode = argv[1];
    try {
        const CartesianMesh mesh = CartesianMesh::from_bounds(-200, 200, -180, 180, -160, 160, 20, 20, 20);
        Microenvironment env = Microenvironment::create(
            mesh, {SubstrateParams{"oxygen", 1e5, 0.1, 38.0}, SubstrateParams{"factor", 1e3, 0.016, 0.0}});
        const int S = env.substrate_count();
        for (int k = 0; k < mesh.nz; ++k)
            for (int j = 0; j < mesh.ny; ++j)
                for (int i = 0; i < mesh.nx; ++i)
                    if (mesh.is_boundary_voxel(i, j, k))
                        env.dirichlet.add(mesh.voxel_index(i, j, k), {1, 0}, {38.0, 0.0}, mesh.voxel_count(), S);
        env.dirichlet.add_single(mesh.voxel_index(7, 5, 4), 1, 2.5, mesh.voxel_count(), S);
        std::mt19937_64 rng(42); // build_agents placement (config.cpp:543-562)
        std::uniform_real_distribution<double> ux(mesh.x_min, mesh.x_max), uy(mesh.y_min, mesh.y_max),
            uz(mesh.z_min, mesh.z_max);
        std::vector<CellAgent> cells;
        for (int a = 0; a < 150; ++a) {
            CellAgent c;
            c.id = 1000 - a;
            c.position = {ux(rng), uy(rng), uz(rng)};
            if (a % 10 == 0) c.position = {1.0, 2.0, 3.0}; // collisions in one voxel
            c.volume = 2494.0;
            c.secretion_rates = {0.0, 1.0};
            c.uptake_rates = {10.0, 0.1};
            c.saturation_densities = {0.0, 1.0};
            cells.push_back(c);
        }
        const AgentPopulation agents(cells, mesh, S);
        const double dt = 0.01;
        const SolverWorkspaces ws = SolverWorkspaces::build(mesh, env.substrates, dt);
        std::ofstream out(argv[2], std::ios::binary);
        auto put = [&](const void* p, std::size_t n) { out.write(static_cast<const char*>(p), n); };
        if (mode == "cpu") {
            for (const auto* w : {&ws.x, &ws.y, &ws.z}) {
                put((*w)->off_diag.data(), sizeof(double) * (*w)->off_diag.size());
                put((*w)->denom_inv.data(), sizeof(double) * (*w)->denom_inv.size());
                put((*w)->c_back.data(), sizeof(double) * (*w)->c_back.size());
            }
            for (const auto& [voxel, idxs] : agents.grouping()) {
                const std::int64_t v = voxel, n = static_cast<std::int64_t>(idxs.size());
                put(&v, 8);
                put(&n, 8);
                for (std::size_t i : idxs) {
                    const std::int64_t ii = static_cast<std::int64_t>(i);
                    put(&ii, 8);
                }
            }
            std::printf("ok cpu %d %d %d dirichlet=%zu groups=%zu\n", mesh.nx, mesh.ny, mesh.nz, env.dirichlet.size(),
                        agents.grouping().size());
            return 0;
        }
        DeviceBackend gpu(0);
        gpu.attach(env, ws, &agents);
        // The field once more through PhysiCell's vector-of-vectors layout
        // (mesh.cpp:101-136) — same values, so the run must not change.
        gpu.upload(translate_array_to_vector(env.field));
        const int steps = 25;
        for (int s = 0; s < steps; ++s) {
            diffuse_decay_step(env, ws, gpu);                             // solver.hpp:72
            cell_sources_sinks_step(env.field, agents, env.mesh, dt, gpu); // agents.hpp:72
        }
        NestedDensity nested;
        gpu.download(nested);
        env.field = translate_vector_to_array(nested);
        if (!env.field.all_finite()) throw state_error("non-finite density after the run");
        put(env.field.values.data(), sizeof(double) * env.field.values.size());
        std::printf("ok gpu %zu values\n", env.field.values.size());
        return 0;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 2;
    }
}
