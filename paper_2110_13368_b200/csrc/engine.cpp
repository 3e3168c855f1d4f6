// The engine loop around the hot path (SPEC.md:271-336 `sim-engine`; the
// reference's core/engine.cpp is absent from the snapshot,
// proj/src/CMakeLists.txt:11), native C++ over a DeviceSession.
//
// Three-tier clock dt_diff <= dt_mech <= dt_cell with integral ratios
// (config.cpp:237-244; default 10 diffusion steps per mechanics step, 60
// mechanics steps per cell step); time is counted in integer diffusion steps
// (t_now = steps * dt_diff). Each mechanics interval is ONE
// device call — DeviceSession::advance(per_mech), a CUDA-graph replay — so the
// field stays in HBM for the whole run and the orchestration thread only wakes
// up for the hooks (no-ops by default) and for snapshots.
#include "engine.hpp"

#include "device.hpp"

#include <chrono>
#include <cmath>

namespace biodiff_b200 {

namespace {

// Positive integral a / b (config.cpp:237-244) or config_error.
std::int64_t integral_ratio(double a, double b, const char* what)
{
    if (!(a > 0.0 && b > 0.0)) throw config_error(std::string(what) + ": step sizes must be positive");
    const double r = a / b;
    const double n = std::round(r);
    if (n < 1.0 || std::fabs(r - n) > 1e-9 * std::max(1.0, r))
        throw config_error(std::string(what) + ": ratio " + format_double(r) + " is not a positive integer");
    return static_cast<std::int64_t>(n);
}

double seconds_since(std::chrono::steady_clock::time_point t0)
{
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

} // namespace

SimulationClock SimulationClock::make(double dt_diff, double dt_mech, double dt_cell, double t_max)
{
    SimulationClock c;
    c.dt_diff = dt_diff;
    c.dt_mech = dt_mech;
    c.dt_cell = dt_cell;
    c.t_max = t_max;
    c.per_mech = integral_ratio(dt_mech, dt_diff, "dt_mech / dt_diff");
    c.per_cell = integral_ratio(dt_cell, dt_mech, "dt_cell / dt_mech");
    if (!(t_max >= 0.0)) throw config_error("max_time must be non-negative");
    // Stop when t_now >= t_max (SPEC.md run_simulation post): the step count
    // whose time first reaches t_max; an integral ratio within 1e-9 counts as exact.
    const double x = t_max / dt_diff;
    const double r = std::round(x);
    c.total_steps = static_cast<std::int64_t>(std::fabs(x - r) <= 1e-9 * std::max(1.0, x) ? r : std::ceil(x));
    return c;
}

std::vector<std::string> RunMetrics::as_lines() const
{
    auto d = [](const char* k, double v) { return std::string(k) + "=" + format_double(v); };
    auto i = [](const char* k, std::int64_t v) { return std::string(k) + "=" + format_int(v); };
    return {d("wall_seconds", wall_seconds),       d("diffusion_seconds", diffusion_seconds),
            d("hook_seconds", hook_seconds),       d("snapshot_seconds", snapshot_seconds),
            i("diffusion_steps", diffusion_steps), i("mechanics_steps", mechanics_steps),
            i("cell_steps", cell_steps),           i("snapshots", snapshots)};
}

// SPEC.md run_simulation: for each mechanics step {per_mech x [diffuse_decay_step;
// cell_sources_sinks_step]}; every per_cell mechanics steps the cell hook;
// snapshots every `snapshot_interval` simulated minutes; stop at t_max.
RunMetrics run_simulation(DeviceSession& session, SimulationClock& clock, bool with_sources, const EngineHooks& hooks)
{
    RunMetrics m;
    const auto t0 = std::chrono::steady_clock::now();
    std::int64_t snap_every = 0;
    if (hooks.snapshot_interval > 0.0) {
        snap_every = static_cast<std::int64_t>(std::llround(hooks.snapshot_interval / clock.dt_diff));
        if (snap_every < 1) throw config_error("snapshot interval shorter than one diffusion step");
    }
    // Resume: the next snapshot is the first multiple of snap_every after the
    // clock's position (a snapshot AT the position is pending or done).
    std::int64_t next_snap = snap_every ? (clock.diffusion_steps / snap_every + 1) * snap_every : 0;

    // Device time is accumulated per segment of uninterrupted device calls: an
    // event pair around each segment, read (one host sync) only when a hook is
    // about to run or at the end — null hooks never make the host wait.
    bool open = false;
    auto open_segment = [&] {
        if (!open) {
            session.event_record(14);
            open = true;
        }
    };
    auto close_segment = [&] {
        if (open) {
            session.event_record(15);
            m.diffusion_seconds += session.event_elapsed(14, 15) / 1e3;
            open = false;
        }
    };
    // Drains the pending boundary work in the reference order: snapshot,
    // mechanics, cell. A hook that throws leaves its bit (and the later ones) set.
    auto drain = [&] {
        if (clock.pending & SimulationClock::kPendingSnapshot) {
            if (hooks.snapshot) {
                close_segment();
                const auto ts = std::chrono::steady_clock::now();
                hooks.snapshot(clock);
                m.snapshot_seconds += seconds_since(ts);
            }
            ++m.snapshots;
            clock.pending &= ~SimulationClock::kPendingSnapshot;
        }
        if (clock.pending & SimulationClock::kPendingMechanics) {
            if (hooks.mechanics) {
                close_segment();
                const auto th = std::chrono::steady_clock::now();
                hooks.mechanics(clock);
                m.hook_seconds += seconds_since(th);
            }
            clock.pending &= ~SimulationClock::kPendingMechanics;
        }
        if (clock.pending & SimulationClock::kPendingCell) {
            if (hooks.cell) {
                close_segment();
                const auto th = std::chrono::steady_clock::now();
                hooks.cell(clock);
                m.hook_seconds += seconds_since(th);
            }
            clock.pending &= ~SimulationClock::kPendingCell;
        }
    };
    try {
        drain(); // work left over from an aborted run
        while (clock.diffusion_steps < clock.total_steps) {
            std::int64_t n = std::min(clock.per_mech - clock.diffusion_steps % clock.per_mech,
                                      clock.total_steps - clock.diffusion_steps);
            if (snap_every) n = std::min(n, next_snap - clock.diffusion_steps);
            open_segment();
            session.advance(n, clock.dt_diff, with_sources);
            clock.diffusion_steps += n;
            if (snap_every && clock.diffusion_steps == next_snap) {
                clock.pending |= SimulationClock::kPendingSnapshot;
                next_snap += snap_every;
            }
            if (clock.diffusion_steps % clock.per_mech == 0) {
                ++clock.mechanics_steps;
                clock.pending |= SimulationClock::kPendingMechanics;
                if (clock.mechanics_steps % clock.per_cell == 0) {
                    ++clock.cell_steps;
                    clock.pending |= SimulationClock::kPendingCell;
                }
            }
            drain();
        }
        close_segment();
    } catch (...) {
        open = false; // the open segment's time is dropped with the aborted run
        throw;
    }
    session.synchronize();
    m.wall_seconds = seconds_since(t0);
    m.diffusion_steps = clock.diffusion_steps;
    m.mechanics_steps = clock.mechanics_steps;
    m.cell_steps = clock.cell_steps;
    return m;
}

} // namespace biodiff_b200
