// XML simulation configuration (the reference's
// config.hpp:13-116 schema). A caller that drives the reference from an XML
// file (`<simulation>` with domain, overall, parallel, microenvironment,
// agents, save) gets the same configuration, microenvironment (boundary
// Dirichlet shell) and agent population here, and a ready device session
// through biodiff_session_from_config (include/biodiff_b200.h).
//
// Own implementation (Boost is absent from this image): a small XML reader
// (elements, text, CDATA, comments, processing instructions, the five
// predefined entities and character references; attributes are detected and
// rejected, as the schema has none) and a table-driven strict schema. Parity
// with the reference's own parser — compiled in oracle/ against a Boost shim —
// is tested on the canonical serialization, the built microenvironment and
// agents, and the error category (config_error) of malformed inputs
// (tests/test_config.py).
#pragma once

#include "host.hpp"

#include <cstdint>
#include <optional>
#include <string>
#include <vector>

namespace biodiff_b200 {

// config.hpp:15-23
struct SubstrateConfig {
    std::string name;
    double diffusion_coefficient = 0.0;
    double decay_rate = 0.0;
    double initial_condition = 0.0;
    std::optional<double> dirichlet_boundary_value; // clamp on every boundary voxel
};

// config.hpp:29-39: `count` identical agents, placed uniformly at random
// (std::mt19937_64(seed), x then y then z) or all at the domain center.
struct InlineAgentsConfig {
    std::int64_t count = 0;
    std::string placement = "random";
    std::uint64_t seed = 0;
    double volume = 2494.0;
    std::vector<double> secretion_rates;
    std::vector<double> uptake_rates;
    std::vector<double> saturation_densities;
};

// config.hpp:43-73 (same fields and defaults).
struct SimConfig {
    double x_min = -1000.0, x_max = 1000.0;
    double y_min = -1000.0, y_max = 1000.0;
    double z_min = -1000.0, z_max = 1000.0;
    double dx = 20.0, dy = 20.0, dz = 20.0;
    double max_time = 60.0;
    double dt_diff = 0.01;
    double dt_mech = 0.1;
    double dt_cell = 6.0;
    bool parallel_backend = false;
    int num_threads = 1;
    std::vector<SubstrateConfig> substrates;
    std::optional<std::string> agent_file;
    std::optional<InlineAgentsConfig> inline_agents;
    double snapshot_interval = 60.0;
    std::string output_folder = "output";

    void validate() const; // throws config_error naming the field
    CartesianMesh mesh() const;
    int substrate_count() const { return static_cast<int>(substrates.size()); }
};

SimConfig parse_config(const std::string& path);          // file (+ agent file must exist)
SimConfig parse_config_text(const std::string& xml_text); // in-memory document
std::string serialize_config(const SimConfig& config);   // canonical form; parses back to the same config
void save_config(const SimConfig& config, const std::string& path);

// The microenvironment of a config: mesh, substrates at their initial
// conditions, and every boundary voxel clamped for the substrates that give
// dirichlet_boundary_value (config.cpp:494-527 semantics).
Microenvironment build_microenvironment(const SimConfig& config);
// The agent source of a config: the agent file, the inline block, or none.
AgentPopulation build_agents(const SimConfig& config, const CartesianMesh& mesh);

} // namespace biodiff_b200
