// DeviceSession: the device-resident state of one Microenvironment and the
// launch logic of the sm_100a kernels (kernels.cu). Plain C++ interface so
// host.cpp / capi.cpp need no CUDA headers.
#pragma once

#include "host.hpp"

#include <cstdint>
#include <map>
#include <unordered_map>
#include <string>
#include <vector>

namespace biodiff_b200 {

namespace kernels {
struct Clamp;
struct Coef;
} // namespace kernels
using kernels_Clamp = kernels::Clamp;
using kernels_Coef = kernels::Coef;

enum KernelClass {
    kSweepX = 0,
    kSweepY = 1,
    kSweepZ = 2,
    kDirichlet = 3,
    kSources = 4,
    kAux = 5,
    kSweepXY = 6, // fused x+y sweeps through L2 (plane clusters xyc.cuh, or xy2.cuh)
    kSweepXYZ = 7, // ensembles: x, y and z of a replica by one cluster (xyc.cuh)
    kResident = 8, // L2-resident grids: every step of an advance() in one cooperative launch (resident.cuh)
    kNumKernelClasses = 9
};

// Device-side copy of one SolverWorkspace (solver.hpp:24-33).
struct DeviceWorkspace {
    bool active = false;
    int n = 0;
    int dims = 0;
    double dt = 0.0;
    double* q = nullptr;      // [S]
    double* dinv = nullptr;   // [n*S]
    double* cb = nullptr;     // [n*S]
    double* dconst = nullptr; // [S] settled denom_inv (rows settle..n-2)
    double* cconst = nullptr; // [S] settled c_back
    double* dinvT = nullptr;  // [R][S][n] denom_inv, substrate-major (ring2 unsettled rows)
    double* cbT = nullptr;    // [R][S][n] c_back
    int settle = 0;           // first row of the bit-constant region (n = none); max over replicas
    int* settle_r = nullptr;  // [R] per-replica settle rows (ensembles), or nullptr
};

// Which kernel implementation a sweep uses (chosen per axis at set-up; the
// env var BIODIFF_SWEEP_PATH=smem|global forces one for A/B measurements).
// smem_ring2  : ring of chunk slots, register-chunk bodies, compile-time slot
//               count, x moved by one swizzled TMA box per chunk (default, ring2.cuh)
// smem_ring   : ring of chunk slots + backward recompute (r01 kernels)
// smem_bulk   : whole line resident in shared memory, persistent CTAs
// smem_plain  : whole line resident, plain loads (rows not 16-byte aligned)
// global      : one thread per chain straight from global memory
enum class SweepPath { smem_ring2, smem_ring, smem_bulk, smem_plain, global };

inline bool is_ring(SweepPath p) { return p == SweepPath::smem_ring2 || p == SweepPath::smem_ring; }

// Host-side analysis of a workspace's coefficient columns: the first row
// from which denom_inv and c_back are bit-constant up to row n-2 (max over
// substrates), and those constants.
int settle_row(int n, int S, const double* dinv, const double* cb, std::vector<double>& dconst,
               std::vector<double>& cconst);

// NCCL unique id (NCCL_UNIQUE_ID_BYTES = 128 bytes) for connect_nccl.
void nccl_unique_id(unsigned char* out);

class DeviceSession {
public:
    // `replicas` > 1: an ensemble of independent microenvironments on the same
    // mesh, stacked replica-major in one field (values[(r*nvox + v)*S + s]),
    // each with its own coefficient set (C5).
    DeviceSession(const CartesianMesh& mesh, int substrates, int device, int replicas = 1);
    ~DeviceSession();
    DeviceSession(const DeviceSession&) = delete;
    DeviceSession& operator=(const DeviceSession&) = delete;

    const CartesianMesh& mesh() const { return mesh_; }
    int substrates() const { return S_; }
    int replicas() const { return replicas_; }
    std::int64_t value_count() const { return mesh_.voxel_count() * S_ * replicas_; }
    void set_agents_multi(const std::vector<const AgentPopulation*>& pops);

    void set_workspace(Axis axis, int n, int dims, double dt, const double* q, const double* dinv, const double* cb);
    void set_workspaces(const SolverWorkspaces& ws);
    void set_dirichlet(const DirichletMap& map);
    void set_agents(const AgentPopulation& agents);
    const AgentPopulation& agents() const { return agents_; }

    // ---- on-device agent grouping (agents.cu) ------------
    // Agents live on the device in input order (set_agents order; ensembles:
    // replica-major). Moving them and regrouping needs no host round trip.
    std::int64_t agent_count() const { return n_agents_; }
    void set_agent_positions(const double* xyz, std::int64_t n);   // host xyz[3n], input order
    void set_agent_position(std::int64_t id, const double* xyz);   // AgentPopulation::set_position
    double* agent_positions_device() const { return in_pos_; }     // device xyz[3n] (caller-side movers)
    void rebuild_voxel_grouping();                                  // agents.cpp:56-73 on the device
    // Group CSR in (voxel, id) order: returns G; voxel[G], offsets[G+1], order[grouped agents].
    std::int64_t download_grouping(std::int64_t* group_voxel, std::int64_t* group_offsets, std::int64_t* order);
    void download_agents(std::int64_t* ids, double* pos, double* vol, double* sec, double* upt, double* sat);
    // Densities at each agent's voxel (after the last rebuild), host out[N*S] in input order.
    void sample_agent_densities(double* out, std::int64_t count);

    void upload(const double* values, std::int64_t count);
    void fill(const double* initial); // [S] per-substrate initial condition
    void download(double* values, std::int64_t count);
    void download_range(double* values, std::int64_t offset, std::int64_t count); // values[offset, +count)
    // advance() runs as one cooperative launch of the resident kernel (L2-resident grids).
    bool resident_path() const;
    bool small_path() const; // advance() runs as one launch of one thread-block cluster (field in its smem)

    void sweep(Axis axis);                 // diffusion_sweep, no clamp
    void apply_dirichlet();                // apply_dirichlet_conditions
    void diffuse_decay_step();             // x, y, z (+ fused clamp) + residual clamp
    void sources(double dt);               // cell_sources_sinks_step
    void advance(std::int64_t steps, double dt, bool with_sources);
    void prepare_advance(std::int64_t steps, double dt, bool with_sources); // capture graphs, run nothing
    void synchronize();
    void* stream() const { return stream_; }
    void event_record(int slot);
    double event_elapsed(int begin, int end);

    void set_kernel_timing(bool on);
    void kernel_times(std::int64_t* launches, double* ms);
    std::int64_t launch_count() const { return launches_; }
    SweepPath path(Axis axis) const { return path_[static_cast<int>(axis)]; }

    bool all_finite(); // DensityField::all_finite on the device field
    void cross_check(const double* other, std::int64_t count, double abs_tol, double rel_tol, double* max_abs,
                     double* max_rel, std::int64_t* worst, bool* pass);

    // ---- z-slab decomposition --------------------------
    // This session holds global planes [z0, z0 + mesh().nz) of a mesh with
    // nz_global planes. Must be called before any set_* call.
    void configure_slab(int nz_global, int z0);
    bool is_slab() const { return slab_; }
    int slab_z0() const { return z0_; }
    int slab_nz_global() const { return nzg_; }
    // Global-mesh boundary test for a local voxel (z faces are global).
    bool is_boundary_local(int i, int j, int k_local) const;
    std::int64_t boundary_count_local() const;
    // Responses to a unit inflow at the slab top (Phi, back-substituted) and
    // bottom (psi), [n*S], and the forward response at the last row [S].
    void set_slab_spikes(const double* Phi, const double* psi, const double* phi_last);
    // Neighbour transports: NCCL (one slab per rank), a host callback (one
    // slab per rank; the planes cross the host — e.g. a gloo process group —
    // through pinned buffers), or in-process.
    void connect_nccl(const unsigned char* unique_id, int nranks, int rank);
    // fn(user, send, send_peer, recv, recv_peer, count) moves `count` doubles:
    // `send` (host, or null) to rank send_peer and from recv_peer into `recv`
    // (host, or null); non-zero return = failure.
    using HostExchange = int (*)(void* user, const double* send, std::int32_t send_peer, double* recv,
                                 std::int32_t recv_peer, std::int64_t count);
    void connect_host_transport(int nranks, int rank, HostExchange fn, void* user);
    static void link_local(const std::vector<DeviceSession*>& slabs);
    static void group_advance(const std::vector<DeviceSession*>& slabs, std::int64_t steps, double dt,
                              bool with_sources);
    void set_agents_range(const AgentPopulation& agents, const CartesianMesh& global_mesh, std::int64_t vox_lo,
                          std::int64_t vox_hi);

private:
    // ---- resident multi-step kernel (resident.cuh) -------------------------
    int resident_mode_ = -1;       // BIODIFF_RESIDENT: 0 off, 1 forced where supported, -1 auto
    unsigned* res_cnt_ = nullptr;  // dataflow counters: [nz] planes | [tpr] ranges | [ny] rows
    int* res_tile_cnt_ = nullptr;  // per-z-tile list scratch (counts / fill cursor)
    int* res_dir_off_ = nullptr;   // [tiles+1] residual Dirichlet entries per z tile
    int* res_dir_idx_ = nullptr;
    int* res_grp_off_ = nullptr;   // [tiles+1] agent groups per z tile
    int* res_grp_idx_ = nullptr;
    int* res_grp_tile_ = nullptr;  // z tile of each group entry (the sources phase's row waits)
    void* res_grp_desc_ = nullptr; // kernels::ResSrc per group entry (voxel, agent range)
    std::int64_t res_grp_cap_ = 0; // capacity of res_grp_idx_ (items)
    bool res_dir_valid_ = false;   // lists match the current Dirichlet split / grouping
    bool res_grp_valid_ = false;
    int resident_tpr() const { return (mesh_.nx * S_ + 31) / 32; }
    int resident_smem_per_warp() const;
    int resident_coef_doubles() const;
    void build_resident_list(const std::int64_t* vox, const std::int64_t* lo, const std::int64_t* hi,
                             std::int64_t cap, int* off, int* idx, int* tile);
    void launch_resident(std::int64_t steps, double dt, bool with_sources);
    // ---- one-cluster kernel (small.cuh): fields that fit a cluster's smem
    int small_mode_ = -1; // BIODIFF_SMALL: 0 off, 1 forced where it fits, -1 auto
    bool small_config(int& cl, int& planes, int& pitch, int& smem_bytes, bool& grid) const;
    void launch_small(std::int64_t steps, double dt, bool with_sources);

    bool slab_ = false;
    int nzg_ = 0;
    int z0_ = 0;
    double* slab_phi_ = nullptr;       // [n_local*S] Phi (response to D_{p-1})
    double* slab_psi_ = nullptr;       // [n_local*S] Psi (response to X_{p+1})
    double* slab_philast_ = nullptr;   // [S] forward response at the last row
    double* plane_bottom_ = nullptr;   // exported zero-inflow forward value of the last row
    double* plane_top_ = nullptr;      // exported zero-inflow unclamped x_hat of row 0
    double* plane_din_ = nullptr;      // D_{p-1} received (0 on slab 0)
    double* plane_dout_ = nullptr;     // D_p, sent to slab p+1
    double* plane_xin_ = nullptr;      // X_{p+1} received (0 on the last slab)
    double* plane_xtop_ = nullptr;     // X_p, sent to slab p-1
    void* nccl_comm_ = nullptr;
    HostExchange host_xchg_ = nullptr; // host-callback transport
    void* host_xchg_user_ = nullptr;
    double* host_send_ = nullptr;      // pinned staging planes of the host transport
    double* host_recv_ = nullptr;
    bool remote_ = false;              // one slab per rank (NCCL or host transport)
    int nccl_rank_ = 0, nccl_ranks_ = 1;
    DeviceSession* prev_slab_ = nullptr; // in-process transport
    DeviceSession* next_slab_ = nullptr;
    bool has_prev() const { return remote_ ? nccl_rank_ > 0 : prev_slab_ != nullptr; }
    bool has_next() const { return remote_ ? nccl_rank_ < nccl_ranks_ - 1 : next_slab_ != nullptr; }
    void slab_phase_xy();   // x, y sweeps + the interface pre-pass (dhat, xhat0)
    void slab_phase_fwdfix(std::int64_t off, std::int64_t count);
    void slab_phase_topfix(std::int64_t off, std::int64_t count);
    void slab_phase_z();    // z sweep with the D_{p-1} / X_{p+1} inflows (+ shell clamp)
    void slab_phase_finish(bool with_sources, double dt);
    void slab_step_nccl(bool with_sources, double dt);
    void nccl_exchange(double* send, int send_peer, double* recv, int recv_peer, std::int64_t count);
    std::vector<std::pair<std::int64_t, std::int64_t>> plane_pieces() const; // chain pipelining
    const double* z_in_lo_ = nullptr; // inflow planes for the next z launch (slab_phase_z)
    const double* z_in_hi_ = nullptr;
    std::int64_t plane_count() const { return static_cast<std::int64_t>(mesh_.nx) * mesh_.ny * S_; }
    bool agent_filter_ = false; // z-slab: groups keep global voxels in [filter_lo_, filter_hi_), made local
    std::int64_t filter_lo_ = 0, filter_hi_ = 0;
    bool agent_mesh_set_ = false; // z-slab: agents are located on the global mesh
    CartesianMesh agent_mesh_;
    void release_slab();

    void check_ready(Axis axis) const;
    void launch_sweep(Axis axis, bool clamp);
    void launch_ring2(int ax, bool do_clamp, const kernels_Clamp& cl, const kernels_Coef& coef);
    void launch_xy_sweeps(); // x then y, no clamp (3-D steps): fused through L2 when enabled
    bool xy_fusable() const;
    void launch_xy2();
    void launch_residual_dirichlet(bool all_entries);
    void launch_sources(double dt);
    void step_body(bool with_sources, double dt);
    void advance_body(std::int64_t n, double dt, bool with_sources);
    void check_advance(std::int64_t steps, double dt) const;
    bool uses_graphs() const;
    static constexpr std::int64_t kGraphSteps = 50; // steps per captured graph
    std::pair<void*, int>& graph_for(std::int64_t n, double dt, bool with_sources);
    void begin_kernel(int cls);
    void end_kernel(int cls);
    void invalidate_graphs();
    void choose_paths();

    CartesianMesh mesh_;
    int S_ = 0;
    int device_ = 0;
    int replicas_ = 1;
    void* stream_ = nullptr; // cudaStream_t
    double* rho_ = nullptr;
    DeviceWorkspace ws_[3];
    int dims_ = 0;
    double dt_ = 0.0;
    SweepPath path_[3] = {SweepPath::global, SweepPath::global, SweepPath::global};
    int sm_count_ = 148;
    bool ring_persist_x_ = true;   // persistent ring kernels per axis (BIODIFF_RING_PERSIST)
    bool ring_persist_yz_ = false;
    bool xy_fused_ = false;          // BIODIFF_XY_FUSED=1 (lagged tickets) / 2 (plane clusters)
    int xy_mode_ = 0;
    void launch_xy_cluster(bool three);
    bool xy_cluster_pays() const;
    bool xyz_cluster_pays() const;
    int long_line_hint(int nch) const;
    void launch_k(const void* fn, unsigned grid, unsigned block, void** args, std::size_t smem, const char* what);
    bool pdl_ = false; // programmatic dependent launch of the step kernels
    int l2_hints_ = 0;               // ring2 L2 cache hints, BIODIFF_L2_HINTS bitmask (1 loads, 2 stores)
    int l2_keep_from8_ = 4; // L2 hint bit 2: reloaded chunks k >= keep_from8/8 of them keep their first load
    // Ensembles: replica batches that stay resident in L2 across several
    // steps (advance). rbn_ = 0: kernels cover every replica.
    int rb0_ = 0, rbn_ = 0;
    int batch_replicas_ = 0;          // replicas per L2 batch (0 = no batching)
    int batch_steps_ = 10;            // steps per batch visit
    std::vector<std::int64_t> dir_res_rep_off_; // residual Dirichlet entries per replica (host, R+1)
    int batch_nr() const { return rbn_ ? rbn_ : replicas_; }
    void step_body_batches(bool with_sources, double dt, std::int64_t steps);
    unsigned* xy_ctr_ = nullptr;     // ticket + per-plane x-done counters of the fused kernel
    unsigned* xyc_ctr_ = nullptr;    // plane counter of the plane-cluster kernel
    int xy_lag_ = 0;                 // chosen lag (planes) of the last fused launch
    int sweep_smem_bytes(int axis, bool bulk) const;
    int ring_slots(int axis) const;
    int ring_smem_bytes(int axis) const;
    int ring2_smem_bytes(int axis) const;
    int smem_align_slack_ = 1024; // extra dynamic smem to 1024-align the ring2 slots (0 when the base is aligned)
    bool ring2_ok(int axis) const;

    // Dirichlet: every entry (for apply_dirichlet), plus the split used by
    // the fused step: a per-substrate "whole boundary shell" rule evaluated in
    // the last sweep's epilogue and the residual entries it does not cover.
    std::int64_t dir_all_count_ = 0;
    std::int64_t* dir_all_voxel_ = nullptr;
    std::uint8_t* dir_all_mask_ = nullptr;
    double* dir_all_values_ = nullptr;
    std::int64_t dir_res_count_ = 0;
    std::int64_t* dir_res_voxel_ = nullptr;
    std::uint8_t* dir_res_mask_ = nullptr;
    double* dir_res_values_ = nullptr;
    std::uint64_t shell_mask_ = 0;
    double* shell_values_ = nullptr; // [S]

    // Agents: input-order arrays (in_*), the id-rank order, sort scratch,
    // and the group CSR + per-agent parameters in group order.
    AgentPopulation agents_;
    std::int64_t groups_ = 0;          // host copy of the last rebuild's group count
    std::int64_t grouped_agents_ = 0;  // agents inside the mesh (slab) after the last rebuild
    std::int64_t n_agents_ = 0;        // agent capacity (all agents handed to set_agents)
    std::int64_t* in_ids_ = nullptr;
    double* in_pos_ = nullptr;
    int* in_rep_ = nullptr;
    double* in_vol_ = nullptr;
    double* in_sec_ = nullptr;
    double* in_upt_ = nullptr;
    double* in_sat_ = nullptr;
    std::int64_t* id_order_ = nullptr;
    std::int64_t* keys_a_ = nullptr;
    std::int64_t* keys_b_ = nullptr;
    std::int64_t* vals_b_ = nullptr;   // agent indices in (voxel, id) order
    std::int64_t* keys_c_ = nullptr;   // the next rebuild's sort output (swapped in when it succeeds)
    std::int64_t* vals_c_ = nullptr;
    std::int64_t* agent_rank_ = nullptr; // agent -> position in (voxel, id) order (the density gather)
    // The CUB regrouping pipeline captured once per sort-output buffer.
    struct RegroupGraph {
        void* exec = nullptr;
        std::int64_t n = -1;
        int end_bit = -1;
        std::int64_t* keys = nullptr;
        int kernels = 0;
    };
    RegroupGraph regroup_graphs_[2];
    int sort_parity_ = 0; // which of the two sort-output pairs keys_c_ / vals_c_ is (its graph slot)
    void destroy_regroup_graphs();
    void mark_factors(bool computed);
    int* flags_ = nullptr;
    std::int64_t* scan_ = nullptr;
    std::int64_t* agent_counts_ = nullptr; // [0] groups, [1] grouped agents (device)
    std::int64_t* rep_groups_ = nullptr;   // [R+1] first group of each replica (device)
    void* host_pin_ = nullptr;             // 64 pinned host bytes: the regrouping's read-backs
    bool zc_positions_ = true;             // mapped caller buffers: positions read / densities written by kernels
    std::vector<std::int64_t> rep_agents_; // agents per replica (host)
    unsigned long long* agent_bad_ = nullptr;
    void* cub_tmp_ = nullptr;
    std::size_t cub_bytes_ = 0;
    std::unordered_map<std::int64_t, std::int64_t> id_index_;
    void release_agents();
    std::int64_t* group_voxel_ = nullptr;
    std::int64_t* group_offsets_ = nullptr;
    double* agent_volume_ = nullptr;
    double* agent_secretion_ = nullptr;
    double* agent_uptake_ = nullptr;
    double* agent_saturation_ = nullptr;
    double* agent_add_ = nullptr;     // [N*S] (f*sec)*target for factors_dt_
    double* agent_den_ = nullptr;     // [N*S] 1 + f*(sec+upt)
    double* agent_sample_ = nullptr;  // [N*S] sample_agent_densities scratch
    std::uint64_t factors_dt_bits_ = 0;
    bool factors_valid_ = false;
    void ensure_source_factors(double dt);

    // Launch accounting / timing.
    std::int64_t launches_ = 0;
    bool timing_ = false;
    std::vector<std::pair<int, std::pair<void*, void*>>> pending_events_;
    std::vector<void*> event_pool_;
    std::int64_t class_launches_[kNumKernelClasses] = {};
    double class_ms_[kNumKernelClasses] = {};
    int kernels_per_step_ = 0;

    // Graph cache for advance(): key (steps in graph, with_sources, dt bits).
    struct GraphKey {
        std::int64_t steps;
        bool sources;
        std::uint64_t dt_bits;
        bool operator<(const GraphKey& o) const
        {
            if (steps != o.steps) return steps < o.steps;
            if (sources != o.sources) return sources < o.sources;
            return dt_bits < o.dt_bits;
        }
    };
    std::map<GraphKey, std::pair<void*, int>> graphs_; // cudaGraphExec_t, kernels per replay
    void* slots_[16] = {};                              // cudaEvent_t for event_record()
    alignas(64) unsigned char res_tmap_[2][128] = {}; // resident kernel's y / z tensor maps
    bool res_tmap_ok_ = false;
    alignas(64) unsigned char tmap_[3][128] = {};       // CUtensorMap per axis (x: swizzled 4-D view for ring2)
    bool tmap_ok_[3] = {false, false, false};
    void build_tensor_maps();
};

} // namespace biodiff_b200
