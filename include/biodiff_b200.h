/*
 * biodiff_b200.h — C ABI of the B200-native LOD diffusion step.
 *
 * This is the "extern-C API" the reference's build declares but whose
 * sources are absent from the snapshot (libbiodiff SHARED from capi/capi.cpp
 * and include/biodiff/biodiff.h, /root/reference/proj/src/CMakeLists.txt:17-23).
 * Every entry point below names the reference C++ interface it stands in for.
 *
 * Conventions:
 *   - Every function returns an int status; no exception crosses the ABI.
 *       BIODIFF_OK          0
 *       BIODIFF_ERR_CONFIG  1  config_error            (errors.hpp:9-12)
 *       BIODIFF_ERR_STATE   2  state_error, std::invalid_argument, std::domain_error,
 *                              std::out_of_range, CUDA failures (errors.hpp:19-22)
 *       BIODIFF_ERR_IO      4  io_error                (errors.hpp:14-17)
 *     biodiff_last_error() returns the message of the calling thread's last failure.
 *   - Host arrays are caller-owned and copied (or read) during the call; the
 *     session owns all device memory. Plain pointers and sizes only.
 *   - Field layout is the reference's (mesh.hpp:59-61):
 *       values[(i + j*nx + k*nx*ny)*S + s], FP64.
 *   - One host thread drives a session at a time (backend.hpp:44-45).
 *   - The CUDA path is the only compute path: there is no CPU fallback. A
 *     session cannot be created without a visible sm_100 device.
 */
#ifndef BIODIFF_B200_H
#define BIODIFF_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BIODIFF_OK 0
#define BIODIFF_ERR_CONFIG 1
#define BIODIFF_ERR_STATE 2
#define BIODIFF_ERR_IO 4

#define BIODIFF_AXIS_X 0
#define BIODIFF_AXIS_Y 1
#define BIODIFF_AXIS_Z 2

/* CartesianMesh (mesh.hpp:17-57). */
typedef struct biodiff_mesh {
    double x_min, x_max, y_min, y_max, z_min, z_max;
    double dx, dy, dz;
    int32_t nx, ny, nz;
} biodiff_mesh;

typedef struct biodiff_session biodiff_session;

/* ---- library / host-side helpers (no device work) ---------------------- */

/* Message of this thread's last failed call ("" if none). */
const char* biodiff_last_error(void);

/* ABI version: major*10000 + minor*100 + patch. */
int32_t biodiff_version(void);

/* Build flags: bit 0 = EXPERIMENTAL=1 build (measured-and-rejected kernel
   variants compiled in for A/B runs). */
int32_t biodiff_build_flags(void);

/* CartesianMesh::from_bounds (mesh.hpp:28-31, mesh.cpp:12-44). */
int biodiff_mesh_from_bounds(double x_min, double x_max, double y_min, double y_max, double z_min, double z_max,
                             double dx, double dy, double dz, biodiff_mesh* out);

/* CartesianMesh::nearest_voxel (mesh.hpp:42-45, mesh.cpp:72-88). */
int biodiff_nearest_voxel(const biodiff_mesh* mesh, const double position[3], int64_t* voxel);

/* precompute_thomas_coefficients (solver.hpp:35-40, solver.cpp:47-97) for
 * one axis: off_diag[S], denom_inv[n*S], c_back[n*S] with n the axis length.
 * D, lambda: per-substrate diffusion coefficient and decay rate. */
int biodiff_precompute_thomas(const biodiff_mesh* mesh, int32_t substrates, const double* diffusion,
                              const double* decay, double dt, int32_t axis, int32_t dims, double* off_diag,
                              double* denom_inv, double* c_back);

/* Number of usable sm_100 devices (0 when none). */
int biodiff_device_count(int32_t* count);

/* ---- sessions: device-resident Microenvironment + WorkerPool stand-in --- */

/* Creates a session bound to `device`, with a device-resident DensityField of
 * mesh.voxel_count()*substrates values (zero-filled). The session is the
 * execution-strategy plugin that replaces WorkerPool& (backend.hpp:34-66,
 * select_backend SPEC.md:303-311). */
int biodiff_session_create(const biodiff_mesh* mesh, int32_t substrates, int32_t device, biodiff_session** out);
int biodiff_session_destroy(biodiff_session* session);

/* SolverWorkspaces::build (solver.hpp:66-67, solver.cpp:277-287): builds the
 * x/y/z workspaces on the host exactly as the reference does and uploads
 * their bits. D, lambda: per-substrate arrays of length S. */
int biodiff_set_substrates(biodiff_session* session, const double* diffusion, const double* decay, double dt);

/* Upload of one prebuilt SolverWorkspace (solver.hpp:24-33): off_diag[S],
 * denom_inv[n*S], c_back[n*S]. `dims` and `dt` must agree across axes. */
int biodiff_set_workspace(biodiff_session* session, int32_t axis, int32_t n, int32_t dims, double dt,
                          const double* off_diag, const double* denom_inv, const double* c_back);

/* Replaces the DirichletMap (mesh.hpp:124-141) with `count` entries:
 * voxel[count], mask[count*S] (nonzero = clamped), values[count*S]. Entries
 * may come in any order; duplicates merge as DirichletMap::add does
 * (mesh.cpp:138-159: later adds win per masked substrate). */
int biodiff_set_dirichlet(biodiff_session* session, int64_t count, const int64_t* voxel, const uint8_t* mask,
                          const double* values);

/* Replaces the AgentPopulation (agents.hpp:30-65): validates as the
 * reference ctor does (agents.cpp:20-43) on the host, then builds the
 * (voxel, id) grouping ON THE DEVICE (agents.cpp:56-73 as a radix-sort
 * pipeline, csrc/agents.cu). positions[3n], volume[n],
 * secretion/uptake/saturation[n*S]. The device keeps the agents in this
 * input order ("agent index" below). */
int biodiff_set_agents(biodiff_session* session, int64_t n, const int64_t* ids, const double* positions,
                       const double* volume, const double* secretion, const double* uptake,
                       const double* saturation);

/* Group count of the current agent grouping and a copy of it:
 * group_voxel[G], group_offsets[G+1], order[n] (agent indices in the
 * caller's order) — AgentPopulation::grouping() (agents.hpp:43-47). With
 * only `groups` non-null, returns the count alone. */
int biodiff_agent_grouping(biodiff_session* session, int64_t* groups, int64_t* group_voxel,
                           int64_t* group_offsets, int64_t* order);

/* Moving agents (agents.hpp:49-56). Positions change on the device; the
 * grouping is stale until biodiff_rebuild_voxel_grouping (the reference's
 * contract: "the caller is expected to rebuild the voxel grouping before
 * the next reaction step").
 *   set_agent_positions : all n positions, xyz[3n] host, agent-index order;
 *                         synchronous (the buffer may be reused on return).
 *                         A page-locked, device-mapped buffer (cudaHostAlloc,
 *                         torch pin_memory), 16-byte aligned, is read by a
 *                         zero-copy kernel, any other buffer by a DMA copy
 *   set_agent_position  : AgentPopulation::set_position(id, p) (agents.cpp:45-54);
 *                         status 2 "no agent with id" if absent
 *   agent_positions_device: the device xyz[3n] buffer (stream-ordered with
 *                         the session stream) for movers running on the GPU
 *   rebuild_voxel_grouping: agents.cpp:56-73 on the device; status 2 with
 *                         mesh.cpp:74-76's message if a position left the
 *                         domain (the previous grouping is kept, as in the
 *                         reference)
 *   sample_agent_densities: what every agent senses — the density values of
 *                         its cached voxel (field.values[agent.voxel*S + s],
 *                         mesh.hpp:62-90, agents.hpp:22) — into host
 *                         out[n*S] in agent-index order; agents outside this
 *                         session's voxels (other z-slabs) read NaN. A
 *                         page-locked, device-mapped `out` is written by the
 *                         gather kernel directly; synchronous either way. */
int biodiff_agent_count(biodiff_session* session, int64_t* n);
int biodiff_set_agent_positions(biodiff_session* session, const double* xyz, int64_t n);
int biodiff_set_agent_position(biodiff_session* session, int64_t id, const double* xyz);
int biodiff_agent_positions_device(biodiff_session* session, double** xyz);
int biodiff_rebuild_voxel_grouping(biodiff_session* session);
int biodiff_sample_agent_densities(biodiff_session* session, double* out, int64_t count);

/* The device's agents in agent-index order (null outputs are skipped):
 * ids[n], xyz[3n], volume[n], secretion/uptake/saturation[n*S]. */
int biodiff_download_agents(biodiff_session* session, int64_t* ids, double* xyz, double* volume,
                            double* secretion, double* uptake, double* saturation);

/* Agent CSV files (config.cpp:416-491): load_agents + set_agents, and
 * save_agents of the device's current agents. Header
 * "id,x,y,z,volume" then ",S_<name>,U_<name>,target_<name>" per substrate;
 * names[S] are the substrate names. Errors: status 1 (config_error
 * "agent file <path> line <n>: ...") or 4 (io_error). */
int biodiff_load_agents_csv(biodiff_session* session, const char* path, const char* const* names);

/* Host-only agent file I/O (no device needed): parse + validate an agent
 * file on `mesh` (call with null arrays to get *n, then with arrays of that
 * size), and write agents in the reference's format (format_double = the
 * shortest round-trip std::to_chars, text.cpp:9-14). */
int biodiff_parse_agents_csv(const biodiff_mesh* mesh, const char* path, const char* const* names, int32_t substrates,
                             int64_t* n, int64_t* ids, double* xyz, double* volume, double* secretion, double* uptake,
                             double* saturation);
int biodiff_write_agents_csv(const char* path, const char* const* names, int32_t substrates, int64_t n,
                             const int64_t* ids, const double* xyz, const double* volume, const double* secretion,
                             const double* uptake, const double* saturation);
int biodiff_save_agents_csv(biodiff_session* session, const char* path, const char* const* names);

/* ---- engine loop (the reference's engine.cpp is absent) ----
 * Three-tier clock dt_diff <= dt_mech <= dt_cell with integral ratios
 * (config.cpp:237-244), integer step counting (t_now = steps * dt_diff),
 * one CUDA-graph advance per mechanics interval, hooks on the calling thread
 * between device calls. A hook returning non-zero aborts the run (status 2). */
typedef struct biodiff_clock {
    double dt_diff, dt_mech, dt_cell, t_max;
    int64_t per_mech, per_cell, total_steps;           /* derived by biodiff_clock_make */
    int64_t diffusion_steps, mechanics_steps, cell_steps; /* counters (in/out of a run) */
    double t_now;                                      /* diffusion_steps * dt_diff */
    int64_t pending; /* boundary hooks not yet completed (1 snapshot, 2 mechanics, 4 cell): counters are
                        bumped when a boundary is reached; a hook that aborts the run keeps its bit and
                        is re-run first when the run resumes */
} biodiff_clock;

typedef struct biodiff_run_metrics {
    double wall_seconds, diffusion_seconds, hook_seconds, snapshot_seconds;
    int64_t diffusion_steps, mechanics_steps, cell_steps, snapshots;
} biodiff_run_metrics;

typedef int (*biodiff_hook)(void* user, const biodiff_clock* clock);

/* Validated clock with zero counters; status 1 (config_error) on
 * non-integral ratios or negative t_max. */
int biodiff_clock_make(double dt_diff, double dt_mech, double dt_cell, double t_max, biodiff_clock* clock);

/* run_simulation (SPEC.md run_simulation): continues from clock's counters
 * to total_steps; snapshot hook every snapshot_interval simulated minutes
 * (0 = none); null hooks are no-ops. */
int biodiff_run_simulation(biodiff_session* session, biodiff_clock* clock, int32_t with_sources,
                           double snapshot_interval, biodiff_hook mechanics, biodiff_hook cell, biodiff_hook snapshot,
                           void* user, biodiff_run_metrics* metrics);

/* PhysiCell's vector-of-vectors density (mesh.hpp:93-100, mesh.cpp:101-136):
 *   translate_vector_to_array : host only; voxels[v] points at counts[v]
 *       values; writes the flat voxel-major array to out (if non-null) and
 *       the substrate count; status 2 "ragged nested density: voxel ..." as
 *       the reference when counts differ.
 *   upload_field_nested / download_field_nested: the session field from /
 *       to per-voxel host buffers (one pack + one copy each way).
 *   field_all_finite : DensityField::all_finite (mesh.cpp:95-99) on the device. */
int biodiff_translate_vector_to_array(const double* const* voxels, const int64_t* counts, int64_t nvox, double* out,
                                      int32_t* substrates);
int biodiff_upload_field_nested(biodiff_session* session, const double* const* voxels, const int64_t* counts,
                                int64_t nvox);
int biodiff_download_field_nested(biodiff_session* session, double* const* voxels, int64_t nvox);
int biodiff_field_all_finite(biodiff_session* session, int32_t* finite);

/* Fills every voxel with the per-substrate values initial[S] on the device —
 * the initial condition of Microenvironment::create (mesh.cpp:173-195)
 * without staging a host copy of the field. */
int biodiff_fill_field(biodiff_session* session, const double* initial);

/* Host <-> device copies of the DensityField values (a1 layout). */
int biodiff_upload_field(biodiff_session* session, const double* values, int64_t count);
int biodiff_download_field(biodiff_session* session, double* values, int64_t count);
/* values[offset, offset + count) of the session's device field (the flat
 * array download_field returns), e.g. to read back a 34 GB field in pieces.
 * Status 2 when the range leaves the field. */
int biodiff_download_field_range(biodiff_session* session, int64_t offset, int64_t count, double* values);

/* diffusion_sweep (solver.hpp:51-52, solver.cpp:248-265) along one axis. */
int biodiff_diffusion_sweep(biodiff_session* session, int32_t axis);

/* apply_dirichlet_conditions (solver.hpp:55, solver.cpp:267-275). */
int biodiff_apply_dirichlet(biodiff_session* session);

/* diffuse_decay_step (solver.hpp:72-73, solver.cpp:289-299): x, y, z sweeps
 * (active axes) with the Dirichlet clamp fused into the last sweep. */
int biodiff_diffuse_decay_step(biodiff_session* session);

/* cell_sources_sinks_step (agents.hpp:72-73, agents.cpp:75-112). */
int biodiff_cell_sources_sinks_step(biodiff_session* session, double dt);

/* The engine's inner loop: steps x [diffuse_decay_step;
 * cell_sources_sinks_step(dt)]; sources are skipped when with_sources == 0.
 * dt must equal the workspace dt. Runs asynchronously on the session stream
 * (captured once into a CUDA graph per (steps-chunk, with_sources)). */
int biodiff_advance(biodiff_session* session, int64_t steps, double dt, int32_t with_sources);

/* Captures and instantiates the CUDA graphs biodiff_advance(steps, dt,
 * with_sources) replays, without running any step (a timed advance then
 * excludes the one-time capture). Same argument checks as biodiff_advance. */
int biodiff_prepare_advance(biodiff_session* session, int64_t steps, double dt, int32_t with_sources);

/* Blocks until all queued work of the session is done. */
int biodiff_synchronize(biodiff_session* session);

/* The session's CUDA stream (a cudaStream_t), for callers that want to
 * order their own work or events against it. */
int biodiff_session_stream(biodiff_session* session, void** stream);

/* Kernel-level timing: when enabled, every kernel launch on the session is
 * bracketed by CUDA events on the session stream; biodiff_kernel_times
 * returns, per kernel class, the number of launches and the summed device
 * milliseconds since the last reset. Classes: 0 sweep_x, 1 sweep_y,
 * 2 sweep_z, 3 dirichlet, 4 sources, 5 aux (set-up kernels: per-dt source factors,
 * cross_check), 6 sweep_xy (the fused x+y sweep of 3-D steps). Returns the
 * number of classes in *n. */
int biodiff_set_kernel_timing(biodiff_session* session, int32_t enabled);
int biodiff_kernel_times(biodiff_session* session, int32_t* n, int64_t* launches, double* milliseconds);

/* Records CUDA event `slot` (0..15) on the session stream / returns the
 * device milliseconds between two recorded slots (synchronizes on `end`). */
int biodiff_event_record(biodiff_session* session, int32_t slot);
int biodiff_event_elapsed(biodiff_session* session, int32_t begin, int32_t end, double* milliseconds);

/* Number of kernel launches issued by the session since creation. */
int biodiff_launch_count(biodiff_session* session, int64_t* launches);

/* Device-side cross_check (validation.hpp:61-65, validation.cpp:112-137)
 * of the session field against a host field: max_abs, max_rel, worst value
 * index, pass (|a-b| <= abs_tol + rel_tol*max(|a|,|b|) everywhere). */
int biodiff_cross_check(biodiff_session* session, const double* other, int64_t count, double abs_tol,
                        double rel_tol, double* max_abs, double* max_rel, int64_t* worst_index, int32_t* pass);

/* ---- ensembles (C5: independent replicas; new) -------------
 * `replicas` independent microenvironments on the same mesh in one session,
 * stacked replica-major: values[(r*voxels + v)*S + s]. Each replica has its
 * own diffusion/decay (D[r*S + s], lambda[r*S + s]) and agents; Dirichlet
 * entries use stacked voxel indices r*voxels + v. One kernel launch per sweep
 * covers every replica. upload/download/fill act on the whole stack. */
int biodiff_ensemble_create(const biodiff_mesh* mesh, int32_t substrates, int32_t replicas, int32_t device,
                            biodiff_session** out);
int biodiff_ensemble_set_substrates(biodiff_session* session, const double* diffusion, const double* decay,
                                    double dt);
int biodiff_ensemble_set_agents(biodiff_session* session, int64_t n, const int32_t* replica, const int64_t* ids,
                                const double* positions, const double* volume, const double* secretion,
                                const double* uptake, const double* saturation);

/* ---- z-slab decomposition across GPUs (new — the reference
 * has no domain decomposition) ------------------------------
 * A z-slab session owns global planes [z0, z1) of `global_mesh` (its field
 * holds nx*ny*(z1-z0)*S values). set_substrates / set_dirichlet / set_agents
 * take the GLOBAL inputs (global voxel indices, all agents) and keep the
 * slab's share. The z sweep is a partitioned solve: zero-inflow slab solves
 * plus two nearest-neighbour plane exchanges and an inflow correction (see
 * paper_2110_13368_b200/csrc/slab.cu). The interface recurrences are exact,
 * so any slab thickness >= 1 plane is accepted; results match the single
 * domain to rounding (the correction re-associates: not bit-identical). */
int biodiff_zslab_create(const biodiff_mesh* global_mesh, int32_t substrates, int32_t z0, int32_t z1, int32_t device,
                         biodiff_session** out);
int biodiff_zslab_info(biodiff_session* session, int32_t* z0, int32_t* z1, int32_t* nz_global);

/* ---- substrate shards (new) -------------------------------
 * Substrates are independent in every part of the step (coefficients per
 * substrate solver.cpp:72-95, Dirichlet masks per substrate solver.cpp:273,
 * the reaction update per substrate agents.cpp:103-108), so a session may
 * hold substrates [s0, s1) of an S-substrate problem and run with no
 * communication; its results are bit-identical to those columns of the
 * unsharded run. A shard may also be a z-slab (planes [z0, z1); pass 0, nz
 * for the whole mesh): S/k substrate shards x P z-slabs.
 * Like z-slabs, a shard takes the GLOBAL inputs — set_substrates(D[S],
 * lambda[S]), set_dirichlet(mask/values [count*S]), set_agents(rates
 * [n*S]), load_agents_csv(names[S]), fill_field(initial[S]) — and keeps
 * its share. Field buffers of upload_field / download_field / nested /
 * sample_agent_densities / download_agents are in the shard's own layout
 * (values[v*(s1-s0) + s - s0] over its voxels); upload_field_global /
 * download_field_global move the shard's part of a GLOBAL a1-layout field
 * (values[v*S + s], every voxel of the global mesh; only the shard's
 * columns and planes are read / written). save_agents_csv needs every
 * substrate and is refused on a shard (status 2). */
int biodiff_shard_create(const biodiff_mesh* global_mesh, int32_t substrates, int32_t s0, int32_t s1, int32_t z0,
                         int32_t z1, int32_t device, biodiff_session** out);
int biodiff_shard_info(biodiff_session* session, int32_t* s0, int32_t* s1, int32_t* substrates);
int biodiff_upload_field_global(biodiff_session* session, const double* values, int64_t count);
int biodiff_download_field_global(biodiff_session* session, double* values, int64_t count);

/* One slab per process: NCCL communicator over all slabs (rank = slab index,
 * ordered by z). biodiff_nccl_unique_id fills 128 bytes on rank 0, to be
 * broadcast by the caller. biodiff_advance then runs the exchanges on the
 * session stream. */
int biodiff_nccl_unique_id(uint8_t* out);
int biodiff_zslab_connect_nccl(biodiff_session* session, const uint8_t* unique_id, int32_t nranks, int32_t rank);

/* The same one-slab-per-process step with the planes moved by the CALLER:
 * fn(user, send, send_peer, recv, recv_peer, count) must send `count`
 * doubles from host `send` (when non-null) to rank send_peer and receive
 * `count` doubles from recv_peer into host `recv` (when non-null); return 0
 * on success. Called on the advancing thread, in the NCCL path's order and
 * pieces (e.g. over a gloo process group; also how a non-NCCL caller plugs
 * its own transport in). */
typedef int (*biodiff_plane_exchange)(void* user, const double* send, int32_t send_peer, double* recv,
                                      int32_t recv_peer, int64_t count);
int biodiff_zslab_connect_host(biodiff_session* session, int32_t nranks, int32_t rank, biodiff_plane_exchange fn,
                               void* user);

/* Several slabs in one process (one or more GPUs): link them in z order and
 * advance them together (device/peer copies move the planes). */
int biodiff_zslab_link_local(biodiff_session** sessions, int32_t count);
int biodiff_zslab_group_advance(biodiff_session** sessions, int32_t count, int64_t steps, double dt,
                                int32_t with_sources);

/* ---- XML configuration (the reference's config.hpp:75-116 schema) ---------
 * `xml` is an in-memory document, or `path` (when non-null) a file:
 * <simulation> with <domain>, <overall>, <parallel>, <microenvironment>
 * (<substrate>*), <agents> (file | inline count/placement/seed/volume/rates),
 * <save>; unknown elements, attributes, repeats and invalid values are
 * status 1 (config_error) naming the element. */

/* serialize_config(parse_config(...)) (config.cpp:325-398 canonical form);
 * `needed` = bytes including the terminator; `out` filled when large enough. */
int biodiff_config_canonical(const char* xml, const char* path, char* out, int64_t capacity, int64_t* needed);
/* save_config (config.cpp:400-406). */
int biodiff_config_save(const char* xml, const char* path, const char* out_path);
/* build_microenvironment + build_agents (config.cpp:494-566): sizes (field ==
 * NULL), then field[voxels*substrates], Dirichlet entries (voxel, mask[S],
 * values[S]) and agents (ids, positions[3n], volume, secretion/uptake/
 * saturation[n*S]). */
int biodiff_config_build(const char* xml, const char* path, int64_t* voxels, int32_t* substrates,
                         int64_t* dirichlet_count, int64_t* agent_count, double* field, int64_t* dir_voxel,
                         uint8_t* dir_mask, double* dir_values, int64_t* ids, double* positions, double* volume,
                         double* secretion, double* uptake, double* saturation);
/* A ready session for a config: mesh, SolverWorkspaces::build at dt_diff,
 * the boundary Dirichlet shell, the agents, the initial field; `clock`
 * (optional) = biodiff_clock_make(dt_diff, dt_mech, dt_cell, max_time). */
int biodiff_session_from_config(const char* xml, const char* path, int32_t device, biodiff_session** out,
                                biodiff_clock* clock);

#ifdef __cplusplus
}
#endif

#endif /* BIODIFF_B200_H */
