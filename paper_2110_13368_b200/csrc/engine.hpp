// Engine loop: SimulationClock, RunMetrics, run_simulation
// over a DeviceSession. See engine.cpp.
#pragma once

#include "host.hpp"

#include <cstdint>
#include <functional>
#include <string>
#include <vector>

namespace biodiff_b200 {

class DeviceSession;

// SPEC.md:275-281.
struct SimulationClock {
    double dt_diff = 0.01, dt_mech = 0.1, dt_cell = 6.0, t_max = 60.0;
    std::int64_t per_mech = 10, per_cell = 60, total_steps = 6000;
    std::int64_t diffusion_steps = 0, mechanics_steps = 0, cell_steps = 0;
    // Boundary work not yet completed (a hook that threw is re-run first on
    // resume): the counters are bumped when a boundary is reached, the bits
    // are cleared when the matching hook returns.
    enum : std::int64_t { kPendingSnapshot = 1, kPendingMechanics = 2, kPendingCell = 4 };
    std::int64_t pending = 0;
    double t_now() const { return static_cast<double>(diffusion_steps) * dt_diff; }
    // Validated clock (config_error on non-integral ratios, config.cpp:237-244).
    static SimulationClock make(double dt_diff, double dt_mech, double dt_cell, double t_max);
};

// SPEC.md:283-291 (device time of the step replays; host time of hooks and
// snapshots; wall time of the whole run).
struct RunMetrics {
    double wall_seconds = 0.0, diffusion_seconds = 0.0, hook_seconds = 0.0, snapshot_seconds = 0.0;
    std::int64_t diffusion_steps = 0, mechanics_steps = 0, cell_steps = 0, snapshots = 0;
    std::vector<std::string> as_lines() const; // key=value lines
};

struct EngineHooks {
    std::function<void(const SimulationClock&)> mechanics; // every mechanics step (default no-op)
    std::function<void(const SimulationClock&)> cell;      // every per_cell mechanics steps
    std::function<void(const SimulationClock&)> snapshot;  // every snapshot_interval simulated minutes
    double snapshot_interval = 0.0;                        // 0 = no snapshots
};

RunMetrics run_simulation(DeviceSession& session, SimulationClock& clock, bool with_sources, const EngineHooks& hooks);

} // namespace biodiff_b200
