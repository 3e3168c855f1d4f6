// ref_config_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// extern "C" access to the reference's own XML config layer
// (/root/reference/proj/src/core/config.cpp, compiled where it lies against
// the Boost.PropertyTree shim in oracle/boost_shim/ — Boost itself is absent):
//   parse_config / parse_config_text   config.cpp:295-323 (+ parse_tree 128-233, validate 248-288)
//   serialize_config                   config.cpp:325-398
//   build_microenvironment             config.cpp:494-527
//   build_agents                       config.cpp:529-566
// and a run of the reference's step loop from a config, the
// oracle of the product's config ingest (paper_2110_13368_b200/csrc/config.cpp).
#include "core/agents.hpp"
#include "core/backend.hpp"
#include "core/config.hpp"
#include "core/errors.hpp"
#include "core/solver.hpp"

#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

using namespace biodiff;

namespace {

thread_local std::string g_cfg_err;

template <class F>
int cfg_guarded(F&& f)
{
    try {
        f();
        return 0;
    } catch (const config_error& e) {
        g_cfg_err = e.what();
        return 1;
    } catch (const io_error& e) {
        g_cfg_err = e.what();
        return 4;
    } catch (const state_error& e) {
        g_cfg_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_cfg_err = e.what();
        return 3;
    }
}

SimConfig parse_either(const char* xml, const char* path)
{
    return path ? parse_config(path) : parse_config_text(xml);
}

int copy_out(const std::string& s, char* out, int64_t cap, int64_t* needed)
{
    *needed = static_cast<int64_t>(s.size()) + 1;
    if (out && cap >= *needed) std::memcpy(out, s.c_str(), s.size() + 1);
    return 0;
}

} // namespace

extern "C" {

const char* ref_config_last_error() { return g_cfg_err.c_str(); }

// serialize_config(parse_config_text(xml)) (or parse_config(path) when path is set).
int ref_config_canonical(const char* xml, const char* path, char* out, int64_t cap, int64_t* needed)
{
    return cfg_guarded([&] { copy_out(serialize_config(parse_either(xml, path)), out, cap, needed); });
}

// build_microenvironment + build_agents: sizes, then (second call) contents.
int ref_config_build(const char* xml, const char* path, int64_t* nvox, int* S, int64_t* ndir, int64_t* nagents,
                     double* field, int64_t* dir_voxel, uint8_t* dir_mask, double* dir_values, int64_t* ids,
                     double* pos, double* vol, double* sec, double* upt, double* sat)
{
    return cfg_guarded([&] {
        const SimConfig cfg = parse_either(xml, path);
        const Microenvironment env = build_microenvironment(cfg);
        const AgentPopulation agents = build_agents(cfg, env.mesh);
        *nvox = env.mesh.voxel_count();
        *S = env.substrate_count();
        *ndir = static_cast<int64_t>(env.dirichlet.size());
        *nagents = static_cast<int64_t>(agents.size());
        if (!field) return;
        std::memcpy(field, env.field.values.data(), sizeof(double) * env.field.values.size());
        int64_t e = 0;
        for (const auto& d : env.dirichlet.entries()) {
            dir_voxel[e] = d.voxel;
            for (int s = 0; s < *S; ++s) {
                dir_mask[e * *S + s] = d.mask[s];
                dir_values[e * *S + s] = d.values[s];
            }
            ++e;
        }
        int64_t a = 0;
        for (const auto& c : agents.agents()) {
            ids[a] = c.id;
            for (int k = 0; k < 3; ++k) pos[3 * a + k] = c.position[k];
            vol[a] = c.volume;
            for (int s = 0; s < *S; ++s) {
                sec[a * *S + s] = c.secretion_rates[s];
                upt[a * *S + s] = c.uptake_rates[s];
                sat[a * *S + s] = c.saturation_densities[s];
            }
            ++a;
        }
    });
}

// The reference's own loop from a config: `steps` x [diffuse_decay_step;
// cell_sources_sinks_step] at dt_diff on `workers` threads (0: serial).
int ref_config_run(const char* xml, const char* path, int64_t steps, int workers, double* field, int64_t count)
{
    return cfg_guarded([&] {
        const SimConfig cfg = parse_either(xml, path);
        Microenvironment env = build_microenvironment(cfg);
        const AgentPopulation agents = build_agents(cfg, env.mesh);
        const SolverWorkspaces ws = SolverWorkspaces::build(env.mesh, env.substrates, cfg.dt_diff);
        WorkerPool pool(workers <= 0 ? BackendKind::serial() : BackendKind::make_parallel(workers));
        for (int64_t n = 0; n < steps; ++n) {
            diffuse_decay_step(env, ws, pool);
            cell_sources_sinks_step(env.field, agents, env.mesh, cfg.dt_diff, pool);
        }
        if (static_cast<int64_t>(env.field.values.size()) != count) throw std::invalid_argument("field size mismatch");
        std::memcpy(field, env.field.values.data(), sizeof(double) * count);
    });
}

} // extern "C"
