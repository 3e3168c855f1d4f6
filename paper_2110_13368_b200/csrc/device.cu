// DeviceSession: device memory, kernel selection and launch, CUDA-graph
// capture of the step loop, and the DeviceBackend glue of host.hpp.
#include "device.hpp"
#include "kernels.cuh"
#include "ring.cuh"
#include "ring2.cuh"
#ifdef BIODIFF_EXPERIMENTAL
#include "xy2.cuh" // lagged-ticket x+y (measured slower; EXPERIMENTAL=1 builds only)
#endif
#include "xyc.cuh"
#include "resident.cuh"
#include "small.cuh"

#include <cstdio>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>

namespace biodiff_b200 {

namespace {

void ck(cudaError_t e, const char* what)
{
    if (e != cudaSuccess) throw state_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

template <class T>
void dfree(T*& p)
{
    if (p) cudaFree(p);
    p = nullptr;
}

template <class T>
T* dalloc_copy(const T* host, std::size_t count, cudaStream_t st)
{
    T* d = nullptr;
    if (count == 0) return nullptr;
    ck(cudaMalloc(&d, sizeof(T) * count), "cudaMalloc");
    ck(cudaMemcpyAsync(d, host, sizeof(T) * count, cudaMemcpyHostToDevice, st), "cudaMemcpyAsync H2D");
    return d;
}

const char* env_or(const char* name, const char* dflt)
{
    const char* v = std::getenv(name);
    return v ? v : dflt;
}

__global__ void smem_base_probe(unsigned* out)
{
    extern __shared__ __align__(1024) unsigned char smem[];
    if (threadIdx.x == 0) *out = ptx::smem_addr(smem);
}

} // namespace

int settle_row(int n, int S, const double* dinv, const double* cb, std::vector<double>& dconst,
               std::vector<double>& cconst)
{
    dconst.assign(S, 0.0);
    cconst.assign(S, 0.0);
    if (n < 3) return n;
    int settle = 0;
    for (int s = 0; s < S; ++s) {
        const double dv = dinv[static_cast<std::size_t>(n - 2) * S + s];
        const double cv = cb[static_cast<std::size_t>(n - 2) * S + s];
        dconst[s] = dv;
        cconst[s] = cv;
        int m = n - 2;
        while (m > 0 && std::memcmp(&dinv[static_cast<std::size_t>(m - 1) * S + s], &dv, 8) == 0 &&
               std::memcmp(&cb[static_cast<std::size_t>(m - 1) * S + s], &cv, 8) == 0)
            --m;
        settle = std::max(settle, m);
    }
    // Row 0 is special (fwd_first) and never uses the shortcut.
    return std::max(settle, 1);
}

void DeviceSession::build_tensor_maps()
{
    for (auto& ok : tmap_ok_) ok = false;
    res_tmap_ok_ = false;
    const long long rowlen = static_cast<long long>(mesh_.nx) * S_;
    if (rowlen % 2 != 0) return; // strides must be multiples of 16 bytes
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) return;
    using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    auto encode = reinterpret_cast<Encode>(fn);
    // 4-D view (row element, j, k, replica); replicas = 1 outside ensembles.
    const cuuint64_t dims[4] = {static_cast<cuuint64_t>(rowlen), static_cast<cuuint64_t>(mesh_.ny),
                                static_cast<cuuint64_t>(mesh_.nz), static_cast<cuuint64_t>(replicas_)};
    const cuuint64_t strides[3] = {static_cast<cuuint64_t>(rowlen) * 8, static_cast<cuuint64_t>(rowlen) * mesh_.ny * 8,
                                   static_cast<cuuint64_t>(rowlen) * mesh_.ny * mesh_.nz * 8};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    // x (ring2): 4-D view (16 doubles, j, plane, 16-double piece of the line),
    // box (16, L, 1, 2S) = one 32-position chunk of L lines, 128-byte swizzle.
    if ((S_ == 1 || S_ == 2 || S_ == 4) && rowlen % 16 == 0) {
        const cuuint64_t xd[4] = {16, static_cast<cuuint64_t>(mesh_.ny),
                                  static_cast<cuuint64_t>(mesh_.nz) * static_cast<cuuint64_t>(replicas_),
                                  static_cast<cuuint64_t>(rowlen / 16)};
        const cuuint64_t xs[3] = {static_cast<cuuint64_t>(rowlen) * 8, static_cast<cuuint64_t>(rowlen) * mesh_.ny * 8,
                                  128};
        const cuuint32_t xb[4] = {16, static_cast<cuuint32_t>(kernels::kLanes / S_), 1,
                                  static_cast<cuuint32_t>(2 * S_)};
        CUresult r = encode(reinterpret_cast<CUtensorMap*>(tmap_[0]), CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, rho_, xd, xs,
                            xb, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        tmap_ok_[0] = (r == CUDA_SUCCESS);
    }
    // resident kernel (L2-resident grids): y / z boxes of 32 columns x ceil(n/4) positions
    res_tmap_ok_ = false;
    if (replicas_ == 1 && mesh_.ny <= 1024 && mesh_.nz <= 1024) {
        const cuuint32_t py = static_cast<cuuint32_t>((mesh_.ny + 3) / 4), pz = static_cast<cuuint32_t>((mesh_.nz + 3) / 4);
        const cuuint32_t by[4] = {static_cast<cuuint32_t>(kernels::kLanes), py, 1, 1};
        const cuuint32_t bz[4] = {static_cast<cuuint32_t>(kernels::kLanes), 1, pz, 1};
        res_tmap_ok_ = py <= 256 && pz <= 256 &&
                       encode(reinterpret_cast<CUtensorMap*>(res_tmap_[0]), CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, rho_,
                              dims, strides, by, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS &&
                       encode(reinterpret_cast<CUtensorMap*>(res_tmap_[1]), CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, rho_,
                              dims, strides, bz, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS &&
                       std::getenv("BIODIFF_RES_NO_TMA") == nullptr;
    }
    for (int ax = 1; ax <= 2; ++ax) {
        const cuuint32_t box[4] = {static_cast<cuuint32_t>(kernels::kLanes),
                                   static_cast<cuuint32_t>(ax == 1 ? kernels::kChunk : 1),
                                   static_cast<cuuint32_t>(ax == 2 ? kernels::kChunk : 1), 1};
        CUresult r = encode(reinterpret_cast<CUtensorMap*>(tmap_[ax]), CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, rho_,
                            dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        tmap_ok_[ax] = (r == CUDA_SUCCESS);
    }
}

DeviceSession::DeviceSession(const CartesianMesh& mesh, int substrates, int device, int replicas)
    : mesh_(mesh), S_(substrates), device_(device), replicas_(replicas)
{
    if (substrates < 1) throw config_error("a session needs at least one substrate");
    if (replicas < 1) throw config_error("an ensemble needs at least one replica");
    if (mesh.nx < 1 || mesh.ny < 1 || mesh.nz < 1) throw config_error("mesh has an empty axis");
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
        throw state_error("no CUDA device visible: the B200 path has no CPU fallback");
    if (device < 0 || device >= count) throw config_error("device index out of range");
    ck(cudaSetDevice(device), "cudaSetDevice");
    cudaDeviceProp prop;
    ck(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
    if (prop.major != 10)
        throw state_error(std::string("device ") + prop.name + " is not sm_100 (Blackwell B200); this build targets sm_100a only");
    sm_count_ = prop.multiProcessorCount;
    // Persistent ring CTAs measured faster for x (C3: 234 -> 223 us) and
    // slower for y/z (211 -> 229 us): default "x". "1"/"all", "0"/"none".
    const std::string persist = env_or("BIODIFF_RING_PERSIST", "x");
    ring_persist_x_ = persist != "0" && persist != "none";
    ring_persist_yz_ = persist == "1" || persist == "all";
    // x+y fusion: BIODIFF_XY_FUSED = 0 off, 1 lagged tickets (xy2.cuh), 2
    // plane clusters (xyc.cuh); default "auto" = plane clusters where they
    // pay (xy_cluster_pays(): enough items per plane, the planes of all
    // clusters fit in L2), else off.
    {
        const std::string m = env_or("BIODIFF_XY_FUSED", "auto");
        xy_mode_ = m == "auto" ? -1 : std::atoi(m.c_str());
        xy_fused_ = xy_mode_ != 0;
#ifndef BIODIFF_EXPERIMENTAL
        if (xy_mode_ == 1)
            throw config_error("BIODIFF_XY_FUSED=1 (lagged-ticket x+y, xy2.cuh) needs a build with EXPERIMENTAL=1");
#endif
    }
    l2_hints_ = std::atoi(env_or("BIODIFF_L2_HINTS", "2")); // stores evict_first: C3 0.635 -> 0.629 ms; load hints slower
    l2_keep_from8_ = std::atoi(env_or("BIODIFF_L2_KEEP_FROM8", "4"));
    // Programmatic dependent launch of the step kernels: opt-in. Measured in
    // graph replay: C1 28.2 -> 30.3 us, C2 49.3 -> 53.2 us per step, C3 no
    // change (the kernels' griddepcontrol.wait is a no-op without it).
    pdl_ = std::atoi(env_or("BIODIFF_PDL", "0")) != 0;
    zc_positions_ = std::atoi(env_or("BIODIFF_ZC_POSITIONS", "1")) != 0;
    if (replicas_ > 1) { // L2 replica batches (step_body_batches)
        const double replica_mb = static_cast<double>(mesh.voxel_count()) * substrates * 8.0 / 1e6;
        const double budget = std::atof(env_or("BIODIFF_L2_BATCH_MB", "0")); // opt-in: measured slower (C5 latency-bound)
        const int nb = budget > 0.0 ? std::max(1, static_cast<int>(budget / replica_mb)) : 0;
        batch_replicas_ = (nb > 0 && nb < replicas_) ? nb : 0;
        batch_steps_ = std::max(1, std::atoi(env_or("BIODIFF_BATCH_STEPS", "10")));
    }
    nzg_ = mesh.nz;
    cudaStream_t st;
    ck(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "cudaStreamCreate");
    stream_ = st;
    ck(cudaMalloc(&rho_, sizeof(double) * value_count()), "cudaMalloc field");
    ck(cudaMemsetAsync(rho_, 0, sizeof(double) * value_count(), st), "cudaMemset field");
    ck(cudaMalloc(&shell_values_, sizeof(double) * S_), "cudaMalloc shell");
    ck(cudaMemsetAsync(shell_values_, 0, sizeof(double) * S_, st), "cudaMemset shell");
    {   // Is the dynamic shared-memory base 1024-byte aligned (no slack needed for the swizzled slots)?
        unsigned* probe = nullptr;
        unsigned base = 1;
        ck(cudaMalloc(&probe, sizeof(unsigned)), "cudaMalloc");
        smem_base_probe<<<1, 32, 4096, st>>>(probe);
        ck(cudaMemcpyAsync(&base, probe, sizeof(unsigned), cudaMemcpyDeviceToHost, st), "probe");
        ck(cudaStreamSynchronize(st), "sync");
        cudaFree(probe);
        smem_align_slack_ = (base % 1024 == 0) ? 0 : 1024;
    }
    build_tensor_maps();
    choose_paths();
    // Ticket + per-plane counters of the fused x+y kernel (allocated here:
    // launches may be captured into graphs).
    ck(cudaMalloc(&xy_ctr_, sizeof(unsigned) * (1 + static_cast<std::size_t>(mesh.nz) * replicas_)), "cudaMalloc");
    ck(cudaMalloc(&xyc_ctr_, sizeof(unsigned)), "cudaMalloc");
    small_mode_ = std::atoi(env_or("BIODIFF_SMALL", "-1")); // -1 auto, 0 off, 1 forced where it fits
    {
        // auto: off when another kernel family is forced for an A/B run
        const std::string m = env_or("BIODIFF_RESIDENT", "auto");
        resident_mode_ = m == "auto" ? -1 : std::atoi(m.c_str());
        for (const char* k : {"BIODIFF_SWEEP_PATH", "BIODIFF_XY_FUSED", "BIODIFF_XYZ_CLUSTER", "BIODIFF_L2_BATCH_MB",
                              "BIODIFF_RING_SLOTS", "BIODIFF_NO_GRAPH"})
            if (resident_mode_ == -1 && std::getenv(k) && std::string(std::getenv(k)) != "auto") resident_mode_ = 0;
    }
    {
        const std::size_t tiles = static_cast<std::size_t>(resident_tpr()) * mesh.ny;
        ck(cudaMalloc(&res_cnt_, sizeof(unsigned) * kernels::kCntPad *
                                     (static_cast<std::size_t>(mesh.nz) + resident_tpr() + 2 * mesh.ny)),
           "cudaMalloc");
        ck(cudaMalloc(&res_tile_cnt_, sizeof(int) * tiles), "cudaMalloc");
        ck(cudaMalloc(&res_dir_off_, sizeof(int) * (tiles + 1)), "cudaMalloc");
        ck(cudaMalloc(&res_grp_off_, sizeof(int) * (tiles + 1)), "cudaMalloc");
    }
}

DeviceSession::~DeviceSession()
{
    cudaSetDevice(device_);
    if (stream_) cudaStreamSynchronize(static_cast<cudaStream_t>(stream_));
    invalidate_graphs();
    for (auto& w : ws_) {
        dfree(w.q);
        dfree(w.dinv);
        dfree(w.cb);
        dfree(w.dconst);
        dfree(w.cconst);
        dfree(w.dinvT);
        dfree(w.cbT);
        dfree(w.settle_r);
    }
    dfree(rho_);
    dfree(dir_all_voxel_);
    dfree(dir_all_mask_);
    dfree(dir_all_values_);
    dfree(dir_res_voxel_);
    dfree(dir_res_mask_);
    dfree(dir_res_values_);
    dfree(shell_values_);
    dfree(xy_ctr_);
    dfree(xyc_ctr_);
    if (host_pin_) cudaFreeHost(host_pin_);
    dfree(res_cnt_);
    dfree(res_tile_cnt_);
    dfree(res_dir_off_);
    dfree(res_dir_idx_);
    dfree(res_grp_off_);
    dfree(res_grp_idx_);
    dfree(res_grp_tile_);
    dfree(res_grp_desc_);
    release_agents();
    release_slab();
    for (auto& pe : pending_events_) {
        cudaEventDestroy(static_cast<cudaEvent_t>(pe.second.first));
        cudaEventDestroy(static_cast<cudaEvent_t>(pe.second.second));
    }
    for (void* e : event_pool_) cudaEventDestroy(static_cast<cudaEvent_t>(e));
    for (void* e : slots_)
        if (e) cudaEventDestroy(static_cast<cudaEvent_t>(e));
    if (stream_) cudaStreamDestroy(static_cast<cudaStream_t>(stream_));
}

void DeviceSession::choose_paths()
{
    // Per axis: the async persistent tile kernel (x: bulk copies, y/z: TMA)
    // when the line fits in shared memory and the rows are 16-byte aligned,
    // else the plain whole-line tile, else the global two-pass kernel.
    // BIODIFF_SWEEP_PATH=global|smem_plain forces a path (A/B measurements).
    const std::string force = env_or("BIODIFF_SWEEP_PATH", "auto");
    const int rowlen = mesh_.nx * S_;
    const bool aligned = (rowlen % 2) == 0;
    constexpr int kMaxSmem = 227 * 1024;
    for (int ax = 0; ax < 3; ++ax) {
        const bool fits_lanes = !(ax == 0 && S_ > kernels::kLanes);
        const bool async_ok = fits_lanes && aligned && (ax == 0 || tmap_ok_[ax]);
        const int bulk_bytes = sweep_smem_bytes(ax, true);
        const int plain_bytes = sweep_smem_bytes(ax, false);
        SweepPath p = SweepPath::global;
        if (ring2_ok(ax) && ring2_smem_bytes(ax) <= kMaxSmem && (force == "auto" || force == "ring2"))
            p = SweepPath::smem_ring2;
        else if (async_ok && ring_smem_bytes(ax) <= kMaxSmem && (force == "auto" || force == "ring" || force == "ring2"))
            p = SweepPath::smem_ring;
        else if (async_ok && bulk_bytes <= kMaxSmem && force != "smem_plain" && force != "global")
            p = SweepPath::smem_bulk;
        else if (fits_lanes && plain_bytes <= kMaxSmem && force != "global")
            p = SweepPath::smem_plain;
        path_[ax] = p;
        const int n = ax == 0 ? mesh_.nx : ax == 1 ? mesh_.ny : mesh_.nz;
        if (replicas_ > 1 && n > 1 && !is_ring(p))
            throw config_error("ensembles need the ring sweep kernels (rows with an even number of doubles, lines "
                               "that fit a shared-memory ring)");
    }
}

// Ring kernels: NS chunk slots (BIODIFF_RING_SLOTS, default 4) + mbarriers +
// one checkpoint per chunk and lane.
int DeviceSession::ring_slots(int axis) const
{
    const int n = axis == 0 ? mesh_.nx : axis == 1 ? mesh_.ny : mesh_.nz;
    const int nch = (n + kernels::kChunk - 1) / kernels::kChunk;
    // x: 2 slots (C3, after the bank-conflict-free lane map: 2 slots 208 us,
    // 3 slots 218, 4 slots 218 — occupancy is register-bound at 8 CTAs/SM
    // either way); y / z: 3 (2 and 4 measured slower).
    const char* e = std::getenv("BIODIFF_RING_SLOTS");
    if (axis == 0 && std::getenv("BIODIFF_X_SLOTS")) e = std::getenv("BIODIFF_X_SLOTS");
    const int want = e ? std::max(2, std::atoi(e)) : (axis == 0 ? 2 : 3);
    // Short y / z lines (<= 2 chunks): two slot sets, alternate tiles (ring2
    // solve_short2) so the next tile loads while this one computes (C5
    // 64-point lines: y 1253 -> 1197 us, z 1294 -> 1246; x measured slower).
    if (!e && axis != 0 && nch <= 2 && std::getenv("BIODIFF_NO_SHORT") == nullptr) return 2 * nch;
#ifdef BIODIFF_EXPERIMENTAL
    return std::min(nch, want);
#else
    return std::min(nch, std::min(want, 3)); // 4 slots: EXPERIMENTAL=1 builds (measured slower)
#endif
}

int DeviceSession::ring_smem_bytes(int axis) const
{
    const int n = axis == 0 ? mesh_.nx : axis == 1 ? mesh_.ny : mesh_.nz;
    const int nch = (n + kernels::kChunk - 1) / kernels::kChunk;
    const int ns = ring_slots(axis);
    int slot;
    if (axis == 0) {
        const int L = std::max(1, kernels::kLanes / S_);
        slot = L * (kernels::kChunk * S_ + ((S_ + 1) / 2) * 2);
    } else {
        slot = kernels::kChunk * kernels::kLanes;
    }
    return kernels::bar_bytes(ns) + (ns * slot + nch * kernels::kLanes) * 8;
}

// ring2 (ring2.cuh): x needs the swizzled 4-D map (S in {1, 2, 4}, rows a
// multiple of 16 doubles); y / z the plain TMA maps.
bool DeviceSession::ring2_ok(int axis) const
{
    if (!tmap_ok_[axis]) return false;
    const int ns = ring_slots(axis);
    return ns >= 1 && ns <= 4;
}

int DeviceSession::ring2_smem_bytes(int axis) const
{
    const int n = axis == 0 ? mesh_.nx : axis == 1 ? mesh_.ny : mesh_.nz;
    const int nch = (n + kernels::kChunk - 1) / kernels::kChunk;
    return kernels::ring2_smem_bytes(ring_slots(axis), nch) - 1024 + smem_align_slack_;
}

// Dynamic shared memory of the tile kernels (bulk: chunk slots + mbarriers;
// plain: whole lines).
int DeviceSession::sweep_smem_bytes(int axis, bool bulk) const
{
    const int n = axis == 0 ? mesh_.nx : axis == 1 ? mesh_.ny : mesh_.nz;
    const int nch = (n + kernels::kChunk - 1) / kernels::kChunk;
    const int pad = ((S_ + 1) / 2) * 2;
    if (axis == 0) {
        const int L = std::max(1, kernels::kLanes / S_);
        if (bulk) return kernels::bar_bytes(nch) + nch * L * (kernels::kChunk * S_ + pad) * 8;
        return L * (((n * S_ + 15) / 16) * 16 + pad) * 8;
    }
    if (bulk) return kernels::bar_bytes(nch) + nch * kernels::kChunk * kernels::kLanes * 8;
    return kernels::kLanes * n * 8;
}

void DeviceSession::invalidate_graphs()
{
    for (auto& g : graphs_) cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(g.second.first));
    graphs_.clear();
    destroy_regroup_graphs(); // they carry dt and the mesh (source factors in the gather)
}

void DeviceSession::set_workspace(Axis axis, int n, int dims, double dt, const double* q, const double* dinv,
                                  const double* cb)
{
    ck(cudaSetDevice(device_), "cudaSetDevice");
    const int ax = static_cast<int>(axis);
    const int expect = ax == 0 ? mesh_.nx : ax == 1 ? mesh_.ny : mesh_.nz;
    if (n != expect) throw state_error("workspace line length " + std::to_string(n) + " does not match the mesh axis");
    if (dims < 1 || dims > 3) throw std::invalid_argument("decay split count must be 1, 2, or 3");
    if (!(dt > 0.0)) throw std::invalid_argument("solver step size must be positive");
    auto st = static_cast<cudaStream_t>(stream_);
    ck(cudaStreamSynchronize(st), "sync");
    DeviceWorkspace& w = ws_[ax];
    dfree(w.q);
    dfree(w.dinv);
    dfree(w.cb);
    dfree(w.dconst);
    dfree(w.cconst);
    dfree(w.dinvT);
    dfree(w.cbT);
    dfree(w.settle_r);
    // Ensembles: replicas_ consecutive coefficient sets (q[R*S], dinv/cb[R*n*S]);
    // the settle row is the max over replicas (warp-uniform in the kernels);
    // ring2 / cluster tiles hold one replica each and use the replica's own
    // settle row (settle_r) instead.
    const std::size_t set = static_cast<std::size_t>(n) * S_;
    w.q = dalloc_copy(q, static_cast<std::size_t>(S_) * replicas_, st);
    w.dinv = dalloc_copy(dinv, set * replicas_, st);
    w.cb = dalloc_copy(cb, set * replicas_, st);
    std::vector<double> dc, cc;
    w.settle = 0;
    std::vector<int> sr(static_cast<std::size_t>(replicas_));
    for (int r = 0; r < replicas_; ++r) {
        std::vector<double> dcr, ccr;
        sr[r] = settle_row(n, S_, dinv + r * set, cb + r * set, dcr, ccr);
        w.settle = std::max(w.settle, sr[r]);
        dc.insert(dc.end(), dcr.begin(), dcr.end());
        cc.insert(cc.end(), ccr.begin(), ccr.end());
    }
    if (std::getenv("BIODIFF_NO_SETTLE")) {
        w.settle = n;
        for (int& v : sr) v = n;
    }
    if (replicas_ > 1 && !std::getenv("BIODIFF_SETTLE_MAX")) w.settle_r = dalloc_copy(sr.data(), sr.size(), st);
    w.dconst = dalloc_copy(dc.data(), dc.size(), st);
    w.cconst = dalloc_copy(cc.data(), cc.size(), st);
    {   // Substrate-major copies (same bits) for ring2's unsettled rows.
        std::vector<double> dT(set * replicas_), cT(set * replicas_);
        for (int r = 0; r < replicas_; ++r)
            for (int m = 0; m < n; ++m)
                for (int sb = 0; sb < S_; ++sb) {
                    const std::size_t from = r * set + static_cast<std::size_t>(m) * S_ + sb;
                    const std::size_t to = (static_cast<std::size_t>(r) * S_ + sb) * n + m;
                    dT[to] = dinv[from];
                    cT[to] = cb[from];
                }
        w.dinvT = dalloc_copy(dT.data(), dT.size(), st);
        w.cbT = dalloc_copy(cT.data(), cT.size(), st);
        ck(cudaStreamSynchronize(st), "sync");
    }
    ck(cudaStreamSynchronize(st), "sync"); // host staging vectors go out of scope
    w.n = n;
    w.dims = dims;
    w.dt = dt;
    w.active = true;
    dims_ = dims;
    dt_ = dt;
    invalidate_graphs();
}

void DeviceSession::set_workspaces(const SolverWorkspaces& ws)
{
    if (!ws.x) throw state_error("solver workspaces not built");
    for (int ax = 0; ax < 3; ++ax) ws_[ax].active = false;
    auto put = [&](const std::optional<SolverWorkspace>& w) {
        if (!w) return;
        if (w->substrates != S_) throw state_error("workspace substrate count does not match the field");
        set_workspace(w->axis, w->n, w->dims, w->dt, w->off_diag.data(), w->denom_inv.data(), w->c_back.data());
    };
    put(ws.x);
    put(ws.y);
    put(ws.z);
}

// Splits the map into the per-substrate boundary-shell rule (evaluated in
// the last sweep's epilogue) and residual entries. Writes of distinct
// (voxel, substrate) pairs commute, so the split is bitwise equivalent to
// applying every entry after the sweeps (solver.cpp:298).
void DeviceSession::set_dirichlet(const DirichletMap& map)
{
    ck(cudaSetDevice(device_), "cudaSetDevice");
    auto st = static_cast<cudaStream_t>(stream_);
    ck(cudaStreamSynchronize(st), "sync");
    const int S = S_;
    const auto& entries = map.entries();
    const std::int64_t count = static_cast<std::int64_t>(entries.size());
    std::vector<std::int64_t> vox(count);
    std::vector<std::uint8_t> mask(count * S);
    std::vector<double> vals(count * S);
    for (std::int64_t e = 0; e < count; ++e) {
        const auto& d = entries[e];
        if (d.voxel < 0 || d.voxel >= mesh_.voxel_count() * replicas_)
            throw std::out_of_range("Dirichlet voxel outside mesh");
        vox[e] = d.voxel;
        for (int s = 0; s < S; ++s) {
            mask[e * S + s] = d.mask[s] ? 1 : 0;
            vals[e * S + s] = d.values[s];
        }
    }
    // Shell analysis.
    const std::int64_t nboundary = boundary_count_local() * replicas_;
    std::uint64_t shell = 0;
    std::vector<double> shell_vals(S, 0.0);
    if (S <= 64 && nboundary > 0) {
        for (int s = 0; s < S; ++s) {
            std::int64_t hits = 0;
            bool first = true, same = true;
            double v0 = 0.0;
            for (std::int64_t e = 0; e < count && same; ++e) {
                if (!mask[e * S + s]) continue;
                const auto ijk = mesh_.voxel_ijk(vox[e] % mesh_.voxel_count());
                if (!is_boundary_local(ijk[0], ijk[1], ijk[2])) continue;
                const double v = vals[e * S + s];
                if (first) {
                    v0 = v;
                    first = false;
                } else if (std::memcmp(&v, &v0, sizeof(double)) != 0) {
                    same = false;
                }
                ++hits;
            }
            if (same && hits == nboundary) {
                shell |= (1ull << s);
                shell_vals[s] = v0;
            }
        }
    }
    std::vector<std::int64_t> rvox;
    std::vector<std::uint8_t> rmask;
    std::vector<double> rvals;
    for (std::int64_t e = 0; e < count; ++e) {
        const auto ijk = mesh_.voxel_ijk(vox[e] % mesh_.voxel_count());
        const bool boundary = is_boundary_local(ijk[0], ijk[1], ijk[2]);
        bool any = false;
        for (int s = 0; s < S; ++s) {
            const bool covered = boundary && ((shell >> s) & 1ull);
            if (mask[e * S + s] && !covered) any = true;
        }
        if (!any) continue;
        rvox.push_back(vox[e]);
        for (int s = 0; s < S; ++s) {
            const bool covered = boundary && ((shell >> s) & 1ull);
            rmask.push_back(mask[e * S + s] && !covered ? 1 : 0);
            rvals.push_back(vals[e * S + s]);
        }
    }
    dfree(dir_all_voxel_);
    dfree(dir_all_mask_);
    dfree(dir_all_values_);
    dfree(dir_res_voxel_);
    dfree(dir_res_mask_);
    dfree(dir_res_values_);
    dir_all_count_ = count;
    dir_all_voxel_ = dalloc_copy(vox.data(), vox.size(), st);
    dir_all_mask_ = dalloc_copy(mask.data(), mask.size(), st);
    dir_all_values_ = dalloc_copy(vals.data(), vals.size(), st);
    dir_res_count_ = static_cast<std::int64_t>(rvox.size());
    dir_res_voxel_ = dalloc_copy(rvox.data(), rvox.size(), st);
    dir_res_mask_ = dalloc_copy(rmask.data(), rmask.size(), st);
    dir_res_values_ = dalloc_copy(rvals.data(), rvals.size(), st);
    // Residual entries are in voxel order, hence replica-major: per-replica
    // offsets for the L2 replica batches.
    dir_res_rep_off_.assign(static_cast<std::size_t>(replicas_) + 1, 0);
    for (int r = 0; r <= replicas_; ++r)
        dir_res_rep_off_[r] = std::lower_bound(rvox.begin(), rvox.end(), static_cast<std::int64_t>(r) * mesh_.voxel_count()) -
                              rvox.begin();
    shell_mask_ = shell;
    res_dir_valid_ = false;
    ck(cudaMemcpyAsync(shell_values_, shell_vals.data(), sizeof(double) * S, cudaMemcpyHostToDevice, st), "shell");
    ck(cudaStreamSynchronize(st), "sync");
    invalidate_graphs();
}

void DeviceSession::set_agents(const AgentPopulation& agents)
{
    set_agents_multi({&agents});
    agents_ = agents;
}

void DeviceSession::upload(const double* values, std::int64_t count)
{
    if (count != value_count()) throw state_error("density field size does not match the mesh");
    ck(cudaSetDevice(device_), "cudaSetDevice");
    ck(cudaMemcpyAsync(rho_, values, sizeof(double) * count, cudaMemcpyHostToDevice,
                       static_cast<cudaStream_t>(stream_)),
       "upload");
}

void DeviceSession::fill(const double* initial)
{
    ck(cudaSetDevice(device_), "cudaSetDevice");
    auto st = static_cast<cudaStream_t>(stream_);
    double* d = dalloc_copy(initial, static_cast<std::size_t>(S_), st);
    begin_kernel(kAux);
    kernels::fill_field<<<sm_count_ * 8, 256, 0, st>>>(rho_, value_count(), d, S_);
    end_kernel(kAux);
    ck(cudaStreamSynchronize(st), "sync");
    cudaFree(d);
}

void DeviceSession::download(double* values, std::int64_t count)
{
    if (count != value_count()) throw state_error("density field size does not match the mesh");
    ck(cudaSetDevice(device_), "cudaSetDevice");
    auto st = static_cast<cudaStream_t>(stream_);
    ck(cudaMemcpyAsync(values, rho_, sizeof(double) * count, cudaMemcpyDeviceToHost, st), "download");
    ck(cudaStreamSynchronize(st), "sync");
}

void DeviceSession::download_range(double* values, std::int64_t offset, std::int64_t count)
{
    if (offset < 0 || count < 0 || offset + count > value_count())
        throw std::invalid_argument("field range out of bounds");
    ck(cudaSetDevice(device_), "cudaSetDevice");
    auto st = static_cast<cudaStream_t>(stream_);
    ck(cudaMemcpyAsync(values, rho_ + offset, sizeof(double) * count, cudaMemcpyDeviceToHost, st), "download");
    ck(cudaStreamSynchronize(st), "sync");
}

void DeviceSession::synchronize()
{
    ck(cudaSetDevice(device_), "cudaSetDevice");
    ck(cudaStreamSynchronize(static_cast<cudaStream_t>(stream_)), "cudaStreamSynchronize");
}

void DeviceSession::event_record(int slot)
{
    if (slot < 0 || slot >= 16) throw std::invalid_argument("event slot must be 0..15");
    ck(cudaSetDevice(device_), "cudaSetDevice");
    if (!slots_[slot]) {
        cudaEvent_t e;
        ck(cudaEventCreate(&e), "cudaEventCreate");
        slots_[slot] = e;
    }
    ck(cudaEventRecord(static_cast<cudaEvent_t>(slots_[slot]), static_cast<cudaStream_t>(stream_)), "cudaEventRecord");
}

double DeviceSession::event_elapsed(int begin, int end)
{
    if (begin < 0 || begin >= 16 || end < 0 || end >= 16 || !slots_[begin] || !slots_[end])
        throw std::invalid_argument("event slot not recorded");
    ck(cudaEventSynchronize(static_cast<cudaEvent_t>(slots_[end])), "cudaEventSynchronize");
    float ms = 0.f;
    ck(cudaEventElapsedTime(&ms, static_cast<cudaEvent_t>(slots_[begin]), static_cast<cudaEvent_t>(slots_[end])),
       "cudaEventElapsedTime");
    return ms;
}

void DeviceSession::check_ready(Axis axis) const
{
    if (!ws_[static_cast<int>(axis)].active) throw state_error("solver workspace for this axis not set");
}

void DeviceSession::begin_kernel(int cls)
{
    ++launches_;
    if (!timing_) return;
    cudaEvent_t a, b;
    if (event_pool_.size() >= 2) {
        a = static_cast<cudaEvent_t>(event_pool_.back());
        event_pool_.pop_back();
        b = static_cast<cudaEvent_t>(event_pool_.back());
        event_pool_.pop_back();
    } else {
        ck(cudaEventCreate(&a), "cudaEventCreate");
        ck(cudaEventCreate(&b), "cudaEventCreate");
    }
    ck(cudaEventRecord(a, static_cast<cudaStream_t>(stream_)), "cudaEventRecord");
    pending_events_.push_back({cls, {a, b}});
}

void DeviceSession::end_kernel(int cls)
{
    (void)cls;
    ck(cudaGetLastError(), "kernel launch");
    if (!timing_) return;
    ck(cudaEventRecord(static_cast<cudaEvent_t>(pending_events_.back().second.second),
                       static_cast<cudaStream_t>(stream_)),
       "cudaEventRecord");
}

void DeviceSession::set_kernel_timing(bool on)
{
    synchronize();
    timing_ = on;
    for (int c = 0; c < kNumKernelClasses; ++c) {
        class_launches_[c] = 0;
        class_ms_[c] = 0.0;
    }
    for (auto& pe : pending_events_) {
        event_pool_.push_back(pe.second.first);
        event_pool_.push_back(pe.second.second);
    }
    pending_events_.clear();
}

void DeviceSession::kernel_times(std::int64_t* launches, double* ms)
{
    synchronize();
    for (auto& pe : pending_events_) {
        float t = 0.f;
        ck(cudaEventElapsedTime(&t, static_cast<cudaEvent_t>(pe.second.first),
                                static_cast<cudaEvent_t>(pe.second.second)),
           "cudaEventElapsedTime");
        class_launches_[pe.first] += 1;
        class_ms_[pe.first] += t;
        event_pool_.push_back(pe.second.first);
        event_pool_.push_back(pe.second.second);
    }
    pending_events_.clear();
    for (int c = 0; c < kNumKernelClasses; ++c) {
        launches[c] = class_launches_[c];
        ms[c] = class_ms_[c];
    }
}

void DeviceSession::launch_sweep(Axis axis, bool clamp)
{
    const int ax = static_cast<int>(axis);
    const DeviceWorkspace& w = ws_[ax];
    auto st = static_cast<cudaStream_t>(stream_);
    const int S = S_;
    const int rowlen = mesh_.nx * S;
    kernels::Clamp cl{shell_values_, clamp ? shell_mask_ : 0ull, z0_, nzg_};
    const bool do_clamp = clamp && shell_mask_ != 0;
    const SweepPath p = path_[ax];
    // per-replica settle rows only for ring2 (one replica per tile)
    const kernels::Coef coef{w.q,        w.dinv, w.cb, w.dconst, w.cconst, w.settle, static_cast<long long>(w.n) * S,
                             w.dinvT, w.cbT, w.n, p == SweepPath::smem_ring2 ? w.settle_r : nullptr};
    const bool bulk = p == SweepPath::smem_bulk;
    begin_kernel(ax);
    if (p == SweepPath::global) {
        kernels::GlobalSweep g{rho_, w.q, w.dinv, w.cb, ax, mesh_.nx, mesh_.ny, mesh_.nz, S, w.n, 0, cl};
        g.chains = mesh_.voxel_count() * S / w.n;
        const int block = 128;
        const long long grid = (g.chains + block - 1) / block;
        if (do_clamp)
            kernels::sweep_global<true><<<static_cast<unsigned>(grid), block, 0, st>>>(g);
        else
            kernels::sweep_global<false><<<static_cast<unsigned>(grid), block, 0, st>>>(g);
        end_kernel(ax);
        return;
    }
    if (p == SweepPath::smem_ring2) {
        launch_ring2(ax, do_clamp, cl, coef);
        end_kernel(ax);
        return;
    }
    const bool ring = p == SweepPath::smem_ring;
    const int smem = ring ? ring_smem_bytes(ax) : sweep_smem_bytes(ax, bulk);
    const int n_ax = ax == 0 ? mesh_.nx : ax == 1 ? mesh_.ny : mesh_.nz;
    const kernels::Ring rg{ring_slots(ax), (n_ax + kernels::kChunk - 1) / kernels::kChunk,
                           std::atoi(env_or("BIODIFF_L2_HINTS", "0"))};
    // Persistent grid: as many CTAs as fit on the device at this smem size.
    auto persistent_grid = [&](const void* fn, long long tiles) {
        ck(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem), "smem attr");
        int per_sm = 0;
        ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kernels::kLanes, smem), "occupancy");
        const long long g = static_cast<long long>(std::max(per_sm, 1)) * sm_count_;
        return static_cast<unsigned>(std::min(g, tiles));
    };
    if (ax == 0) {
        kernels::XSweep x{};
        x.rho = rho_;
        x.coef = coef;
        x.lines_per_rep = static_cast<long long>(mesh_.ny) * mesh_.nz;
        x.lines = x.lines_per_rep * replicas_;
        x.nx = mesh_.nx;
        x.ny = mesh_.ny;
        x.nz = mesh_.nz;
        x.S = S;
        x.rowlen = rowlen;
        const int pad = ((S + 1) / 2) * 2;
        x.cpitch = kernels::kChunk * S + pad;
        x.pitch = ((rowlen + 15) / 16) * 16 + pad;
        x.L = std::max(1, kernels::kLanes / S);
        x.tiles = (x.lines + x.L - 1) / x.L;
        x.clamp = cl;
        if (ring) {
            if (ring_persist_x_) {
                auto k = do_clamp ? kernels::sweep_x_pring<true> : kernels::sweep_x_pring<false>;
                const unsigned grid = persistent_grid(reinterpret_cast<const void*>(k), x.tiles);
                k<<<grid, kernels::kLanes, smem, st>>>(x, rg);
            } else {
                auto k = do_clamp ? kernels::sweep_x_ring<true> : kernels::sweep_x_ring<false>;
                ck(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem), "smem attr");
                k<<<static_cast<unsigned>(x.tiles), kernels::kLanes, smem, st>>>(x, rg);
            }
        } else if (bulk) {
            auto k = do_clamp ? kernels::sweep_x_bulk<true> : kernels::sweep_x_bulk<false>;
            const unsigned grid = persistent_grid(reinterpret_cast<const void*>(k), x.tiles);
            k<<<grid, kernels::kLanes, smem, st>>>(x);
        } else {
            ck(cudaFuncSetAttribute(kernels::sweep_x_plain, cudaFuncAttributeMaxDynamicSharedMemorySize, smem),
               "smem attr");
            kernels::sweep_x_plain<<<static_cast<unsigned>(x.tiles), kernels::kLanes, smem, st>>>(x, do_clamp);
        }
        end_kernel(ax);
        return;
    }
    kernels::StridedSweep y{};
    y.rho = rho_;
    y.coef = coef;
    y.axis = ax;
    const long long row = rowlen;
    const long long plane = row * mesh_.ny;
    y.stride = ax == 1 ? row : plane;
    y.outer_stride = ax == 1 ? plane : row;
    y.n_outer = ax == 1 ? mesh_.nz : mesh_.ny;
    y.n = w.n;
    y.rowlen = rowlen;
    y.tiles_per_row = (rowlen + kernels::kLanes - 1) / kernels::kLanes;
    y.reps = replicas_;
    y.tiles = y.tiles_per_row * y.n_outer * replicas_;
    y.S = S;
    y.nx = mesh_.nx;
    y.clamp = cl;
    y.exp_bottom = (slab_ && ax == 2) ? plane_bottom_ : nullptr;
    y.exp_top = (slab_ && ax == 2) ? plane_top_ : nullptr;
    if (ring) {
        const CUtensorMap& tm = *reinterpret_cast<const CUtensorMap*>(tmap_[ax]);
        if (ring_persist_yz_) {
            auto k = do_clamp ? kernels::sweep_yz_pring<true> : kernels::sweep_yz_pring<false>;
            const unsigned grid = persistent_grid(reinterpret_cast<const void*>(k), y.tiles);
            k<<<grid, kernels::kLanes, smem, st>>>(tm, y, rg);
        } else {
            auto k = do_clamp ? kernels::sweep_yz_ring<true> : kernels::sweep_yz_ring<false>;
            ck(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem), "smem attr");
            k<<<static_cast<unsigned>(y.tiles), kernels::kLanes, smem, st>>>(tm, y, rg);
        }
    } else if (bulk) {
        const CUtensorMap& tm = *reinterpret_cast<const CUtensorMap*>(tmap_[ax]);
        auto k = do_clamp ? kernels::sweep_yz_tma<true> : kernels::sweep_yz_tma<false>;
        const unsigned grid = persistent_grid(reinterpret_cast<const void*>(k), y.tiles);
        k<<<grid, kernels::kLanes, smem, st>>>(tm, y);
    } else {
        ck(cudaFuncSetAttribute(kernels::sweep_yz_plain, cudaFuncAttributeMaxDynamicSharedMemorySize, smem),
           "smem attr");
        kernels::sweep_yz_plain<<<static_cast<unsigned>(y.tiles), kernels::kLanes, smem, st>>>(y, do_clamp);
    }
    end_kernel(ax);
}

bool DeviceSession::xy_fusable() const
{
    if (!(xy_fused_ && ws_[1].active && path_[0] == SweepPath::smem_ring2 && path_[1] == SweepPath::smem_ring2))
        return false;
    return xy_mode_ != -1 || xy_cluster_pays();
}

// Plane clusters pay off when each of a cluster's 32 warps has an x and a y
// item per plane (C3: 32 + 32 items) and the planes the ~37 clusters hold at
// once stay in L2 (C3: 37 x 2 MB; C4's 32 MB planes would not).
bool DeviceSession::xy_cluster_pays() const
{
    if (replicas_ > 1 || !ws_[2].active) return false;
    const int L = kernels::kLanes / S_;
    const int xi = (mesh_.ny + L - 1) / L;
    const int yi = (mesh_.nx * S_ + kernels::kLanes - 1) / kernels::kLanes;
    const double plane_mb = static_cast<double>(mesh_.nx) * mesh_.ny * S_ * 8.0 / 1e6;
    const double clusters = std::min(static_cast<double>(mesh_.nz), sm_count_ / 4.0);
    // Measured only to pay at S = 4 (C3: 0.587 vs 0.622 ms per step); at S = 2
    // the same 256^2 planes run slower fused (0.46 vs 0.33 ms, r02
    // tools/shard_probe.py), at S = 1 the x items are too few.
    return S_ == 4 && xi >= 16 && yi >= 16 && plane_mb * clusters <= 80.0;
}

namespace {

template <int NS>
const void* xyc_pick_s(int S, bool three)
{
    if (three) {
        if (S == 1) return reinterpret_cast<const void*>(kernels::sweep_xyz_cluster<NS, 1>);
        if (S == 2) return reinterpret_cast<const void*>(kernels::sweep_xyz_cluster<NS, 2>);
        return reinterpret_cast<const void*>(kernels::sweep_xyz_cluster<NS, 4>);
    }
    if (S == 1) return reinterpret_cast<const void*>(kernels::sweep_xy_cluster<NS, 1>);
    if (S == 2) return reinterpret_cast<const void*>(kernels::sweep_xy_cluster<NS, 2>);
    return reinterpret_cast<const void*>(kernels::sweep_xy_cluster<NS, 4>);
}

} // namespace

// x+y of each plane by one thread-block cluster through L2 (xyc.cuh); with
// `three` (ensembles) x, y and z of each replica, the z phase with the
// Dirichlet shell clamp.
void DeviceSession::launch_xy_cluster(bool three)
{
    auto st = static_cast<cudaStream_t>(stream_);
    const int S = S_;
    const DeviceWorkspace& wx = ws_[0];
    const DeviceWorkspace& wy = ws_[1];
    kernels::XYCluster a{};
    a.xcoef = kernels::Coef{wx.q,     wx.dinv, wx.cb, wx.dconst, wx.cconst, wx.settle, static_cast<long long>(wx.n) * S,
                            wx.dinvT, wx.cbT, wx.n, wx.settle_r};
    a.nx = mesh_.nx;
    a.ny = mesh_.ny;
    a.nz = mesh_.nz;
    a.S = S;
    a.rowlen = mesh_.nx * S;
    a.planes = three ? replicas_ : mesh_.nz * replicas_;
    const int L = kernels::kLanes / S;
    a.xi = (mesh_.ny + L - 1) / L;
    a.yi = (a.rowlen + kernels::kLanes - 1) / kernels::kLanes;
    kernels::StridedSweep& y = a.y;
    y.coef = kernels::Coef{wy.q,     wy.dinv, wy.cb, wy.dconst, wy.cconst, wy.settle, static_cast<long long>(wy.n) * S,
                           wy.dinvT, wy.cbT, wy.n, wy.settle_r};
    y.axis = 1;
    y.n = mesh_.ny;
    y.n_outer = mesh_.nz;
    y.rowlen = a.rowlen;
    y.S = S;
    y.nx = mesh_.nx;
    y.clamp = kernels::Clamp{shell_values_, 0ull, z0_, nzg_};
    if (three) {
        const DeviceWorkspace& wz = ws_[2];
        kernels::StridedSweep& z = a.z;
        z.coef = kernels::Coef{wz.q,     wz.dinv, wz.cb, wz.dconst, wz.cconst, wz.settle,
                               static_cast<long long>(wz.n) * S, wz.dinvT, wz.cbT, wz.n, wz.settle_r};
        z.axis = 2;
        z.n = mesh_.nz;
        z.n_outer = mesh_.ny;
        z.rowlen = a.rowlen;
        z.S = S;
        z.nx = mesh_.nx;
        z.clamp = kernels::Clamp{shell_values_, shell_mask_, z0_, nzg_};
    }
    // Three slots; two when no line of a 3-phase unit has more than two
    // chunks (C5: 2.785 vs 2.819 ms per step) — no reloads either way.
    const int nmax = std::max({mesh_.nx, mesh_.ny, three ? mesh_.nz : 0});
    const char* ns_dflt = three && nmax <= 2 * kernels::kChunk ? "2" : "3";
    const int ns = std::max(2, std::min(3, std::atoi(env_or("BIODIFF_XYC_SLOTS", ns_dflt))));
    // 8 CTAs x 4 warps per cluster (32 warps: one x and one y item each at
    // C3), two CTAs of DIFFERENT clusters per SM: their plane phases and
    // barriers drift apart, so one cluster's x (DRAM) phase overlaps the
    // other's y (L2) phase — 388 -> 378 us vs 4 CTAs x 8 warps (one CTA per
    // SM); 2 x 16 and 1 x 16 (non-portable sizes) measured 410 / 409 us.
    const int wpc = std::max(1, std::min(8, std::atoi(env_or("BIODIFF_XYC_WARPS", "4"))));
    const int cl = std::max(1, std::min(16, std::atoi(env_or("BIODIFF_XYC_CLUSTER", "8"))));
    const int nch = (std::max(mesh_.nx * S / (2 * S) * 2 / 2, mesh_.ny) + kernels::kChunk - 1) / kernels::kChunk;
    const int nchx = (mesh_.nx + kernels::kChunk - 1) / kernels::kChunk;
    const int nchm = std::max({nch, nchx, three ? (mesh_.nz + kernels::kChunk - 1) / kernels::kChunk : 0});
    // Odd clusters start ~half an x item later (~50 ns per x position): the
    // two clusters sharing an SM then keep their DRAM-fed x phases and
    // L2-fed y phases apart instead of starting in lockstep. C3: 381 -> 363
    // us (0 / 9 / 12 / 15 us: 381 / 366 / 363 / 363; 3-8 groups no better).
    a.stagger_ns = std::atoi(env_or("BIODIFF_XYC_STAGGER_NS", std::to_string(50 * mesh_.nx).c_str()));
    a.stagger_groups = std::atoi(env_or("BIODIFF_XYC_STAGGER_GROUPS", "2"));
    a.plane_ctr = std::atoi(env_or("BIODIFF_XYC_DYNAMIC", "1")) ? xyc_ctr_ : nullptr;
    if (a.plane_ctr) ck(cudaMemsetAsync(xyc_ctr_, 0, sizeof(unsigned), st), "memset plane counter");
    a.warp_bytes = ((ns * kernels::kChunk * kernels::kLanes * 8 + 128 + nchm * kernels::kLanes * 8 + 1023) / 1024) * 1024;
    const int smem = 1024 + wpc * a.warp_bytes;
    const void* fn = ns == 2 ? xyc_pick_s<2>(S, three) : xyc_pick_s<3>(S, three);
    ck(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem), "smem attr");
    if (cl > 8) ck(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1), "cluster 16");
    cudaLaunchConfig_t cfg{};
    cfg.blockDim = dim3(32 * wpc);
    cfg.dynamicSmemBytes = static_cast<std::size_t>(smem);
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(cl);
    int max_clusters = 0;
    ck(cudaOccupancyMaxActiveClusters(&max_clusters, fn, &cfg), "max active clusters");
    // Planes are visited from the top and the y results of the lowest planes
    // (~64 MB) stay in L2 (evict_normal instead of evict_first): they are the
    // last ones written and the first ones the z sweep reads. C3: z 207.8 ->
    // 202.0 us (reverse alone 204.5; 32 / 48 / 64 kept planes alike).
    const double plane_bytes = static_cast<double>(mesh_.nx) * mesh_.ny * S * 8.0;
    a.reverse = three ? 0 : std::atoi(env_or("BIODIFF_XYC_REVERSE", "1"));
    a.keep_planes = three ? 0
                          : std::atoi(env_or("BIODIFF_XYC_KEEP_PLANES",
                                             std::to_string(static_cast<int>(64e6 / plane_bytes)).c_str()));
    const int cap = std::atoi(env_or("BIODIFF_XYC_MAX_CLUSTERS", "0"));
    const int clusters = std::max(1, std::min({max_clusters, a.planes, cap > 0 ? cap : max_clusters}));
    cfg.gridDim = dim3(clusters * cl);
    cfg.numAttrs = pdl_ ? 2 : 1;
    const KernelClass kc = three ? kSweepXYZ : kSweepXY;
    begin_kernel(kc);
    void* args2[] = {tmap_[0], tmap_[1], &a};
    void* args3[] = {tmap_[0], tmap_[1], tmap_[2], &a};
    ck(cudaLaunchKernelExC(&cfg, fn, three ? args3 : args2), "launch xy cluster");
    end_kernel(kc);
}

// Ensembles: one cluster per replica for all three sweeps. Opt-in
// (BIODIFF_XYZ_CLUSTER=1): with per-replica settle rows the separate ring2
// sweeps are faster at C5 (2.613 vs 2.659 ms per step; before them the
// clusters led, 2.785 vs 2.98 ms). "auto" would take it when every warp of a
// cluster has an item per phase and the in-flight replicas roughly fit L2.
bool DeviceSession::xyz_cluster_pays() const
{
    const std::string m = env_or("BIODIFF_XYZ_CLUSTER", "0");
    if (m == "0") return false;
    if (replicas_ <= 1 || !ws_[1].active || !ws_[2].active || slab_ || batch_replicas_ > 0) return false;
    if (!(S_ == 1 || S_ == 2 || S_ == 4)) return false;
    for (int ax = 0; ax < 3; ++ax)
        if (path_[ax] != SweepPath::smem_ring2) return false;
    if (m == "1") return true;
    const int L = kernels::kLanes / S_;
    const long long xi = static_cast<long long>((mesh_.ny + L - 1) / L) * mesh_.nz;
    const long long yi = static_cast<long long>((mesh_.nx * S_ + kernels::kLanes - 1) / kernels::kLanes);
    const double replica_mb = static_cast<double>(mesh_.voxel_count()) * S_ * 8.0 / 1e6;
    return xi >= 32 && yi * mesh_.nz >= 32 && yi * mesh_.ny >= 32 && replica_mb * (sm_count_ / 4.0) <= 160.0;
}

namespace {

#ifdef BIODIFF_EXPERIMENTAL
template <int NS>
const void* xy2_pick_s(int S)
{
    if (S == 1) return reinterpret_cast<const void*>(kernels::sweep_xy2<NS, 1>);
    if (S == 2) return reinterpret_cast<const void*>(kernels::sweep_xy2<NS, 2>);
    return reinterpret_cast<const void*>(kernels::sweep_xy2<NS, 4>);
}

const void* xy2_pick(int ns, int S)
{
    switch (ns) {
    case 1: return xy2_pick_s<1>(S);
    case 2: return xy2_pick_s<2>(S);
    case 3: return xy2_pick_s<3>(S);
    default: return xy2_pick_s<4>(S);
    }
}
#endif

} // namespace

// Lag (planes) between X(p) and Y(p) in the fused ticket order: enough
// tickets that every x item of plane p has finished when Y(p) is handed out
// (one resident wave ~ one item time, BIODIFF_XY_LAG_WAVES), or
// BIODIFF_XY_LAG planes.
static int xy_lag_for(long long resident, int xi, int yi, int planes)
{
    const double f = std::atof(env_or("BIODIFF_XY_LAG_WAVES", "1.25"));
    long long lag = static_cast<long long>(std::ceil(f * static_cast<double>(resident) / (xi + yi)));
    if (const char* e = std::getenv("BIODIFF_XY_LAG")) lag = std::atoll(e);
    return static_cast<int>(std::max(1LL, std::min(lag, static_cast<long long>(planes))));
}

// x then y sweep of a 3-D step (no clamp: z is the last sweep): two ring
// sweeps, or the fused x+y kernel through L2 (xy2.cuh) when
// BIODIFF_XY_FUSED=1 (opt-in: measured slower on C3).
void DeviceSession::launch_xy_sweeps()
{
    if (!xy_fusable()) {
        launch_sweep(Axis::x, false);
        if (ws_[1].active) launch_sweep(Axis::y, false);
        return;
    }
    if (xy_mode_ == 1)
        launch_xy2();
    else
        launch_xy_cluster(false);
}

namespace {

template <int NS, bool CLAMP>
const void* yz_ring2_fn()
{
    return reinterpret_cast<const void*>(kernels::sweep_yz_ring2<NS, CLAMP>);
}

template <int NS, int S, bool CLAMP>
const void* x_ring2_fn()
{
    return reinterpret_cast<const void*>(kernels::sweep_x_ring2<NS, S, CLAMP>);
}

// short: two slot sets for lines of <= ns/2 chunks (solve_short2); only
// ns = 2 (one-chunk lines) and ns = 4 (two-chunk lines) occur.
template <bool CLAMP>
const void* yz_ring2_pick(int ns, bool short_lines)
{
    if (short_lines)
        return ns == 2 ? reinterpret_cast<const void*>(kernels::sweep_yz_ring2<2, CLAMP, true>)
                       : reinterpret_cast<const void*>(kernels::sweep_yz_ring2<4, CLAMP, true>);
    switch (ns) {
    case 1: return yz_ring2_fn<1, CLAMP>(); // one-chunk lines
#ifdef BIODIFF_EXPERIMENTAL
    case 4: return yz_ring2_fn<4, CLAMP>();
#endif
    case 2: return yz_ring2_fn<2, CLAMP>();
    default: return yz_ring2_fn<3, CLAMP>();
    }
}

template <int S, bool CLAMP>
const void* x_ring2_pick_ns(int ns, bool short_lines)
{
    if (short_lines)
        return ns == 2 ? reinterpret_cast<const void*>(kernels::sweep_x_ring2<2, S, CLAMP, true>)
                       : reinterpret_cast<const void*>(kernels::sweep_x_ring2<4, S, CLAMP, true>);
    switch (ns) {
    case 1: return x_ring2_fn<1, S, CLAMP>(); // one-chunk lines
#ifdef BIODIFF_EXPERIMENTAL
    case 4: return x_ring2_fn<4, S, CLAMP>();
#endif
    case 2: return x_ring2_fn<2, S, CLAMP>();
    default: return x_ring2_fn<3, S, CLAMP>();
    }
}

template <bool CLAMP>
const void* x_ring2_pick(int ns, int S, bool short_lines)
{
    if (S == 1) return x_ring2_pick_ns<1, CLAMP>(ns, short_lines);
    if (S == 2) return x_ring2_pick_ns<2, CLAMP>(ns, short_lines);
    return x_ring2_pick_ns<4, CLAMP>(ns, short_lines);
}

} // namespace

// Long lines (C4: 32 chunks, ~300 MB between a chunk's first read and its
// reload): the first loads of the later half of the reloaded chunks are
// kept in L2 (hint bit 2), the rest stream — C4 43.5 -> 42.7 ms per step;
// at C3's 8-chunk lines the same hint is slower (z 202 -> 213 us).
int DeviceSession::long_line_hint(int nch) const
{
    const int from = std::atoi(env_or("BIODIFF_L2_LONG_CHUNKS", "16"));
    return (from > 0 && nch >= from) ? 4 : 0;
}

// Kernel launch on the session stream, with programmatic dependent launch
// (PDL: the kernel's CTAs may be scheduled while the previous kernel drains;
// every step kernel starts with griddepcontrol.wait) when pdl_ is on.
void DeviceSession::launch_k(const void* fn, unsigned grid, unsigned block, void** args, std::size_t smem, const char* what)
{
    auto st = static_cast<cudaStream_t>(stream_);
    if (!pdl_) {
        ck(cudaLaunchKernel(fn, dim3(grid), dim3(block), args, smem, st), what);
        return;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    ck(cudaLaunchKernelExC(&cfg, fn, args), what);
}

// ring2 launch (ring2.cuh): x persistent over per-plane line tiles (next
// tile's chunks prefetched), y / z one tile per CTA unless
// BIODIFF_RING_PERSIST=all.
void DeviceSession::launch_ring2(int ax, bool do_clamp, const kernels::Clamp& cl, const kernels::Coef& coef)
{
    auto st = static_cast<cudaStream_t>(stream_);
    const int ns = ring_slots(ax);
    const int smem = ring2_smem_bytes(ax);
    const int rowlen = mesh_.nx * S_;
    const CUtensorMap& tm = *reinterpret_cast<const CUtensorMap*>(tmap_[ax]);
    auto occupancy_grid = [&](const void* fn, long long tiles) {
        ck(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem), "smem attr");
        int per_sm = 0;
        ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kernels::kLanes, smem), "occupancy");
        const long long g = static_cast<long long>(std::max(per_sm, 1)) * sm_count_;
        return static_cast<unsigned>(std::min(g, tiles));
    };
    if (ax == 0) {
        kernels::XSweep2 x{};
        x.coef = coef;
        x.nx = mesh_.nx;
        x.ny = mesh_.ny;
        x.nz = mesh_.nz;
        x.S = S_;
        x.planes = mesh_.nz * batch_nr();
        x.P0 = (rbn_ ? rb0_ : 0) * mesh_.nz;
        x.hints = l2_hints_ | long_line_hint((mesh_.nx + kernels::kChunk - 1) / kernels::kChunk);
        x.keep_from8 = l2_keep_from8_;
        const int L = kernels::kLanes / S_;
        x.xi = (mesh_.ny + L - 1) / L;
        x.tiles = static_cast<long long>(x.xi) * x.planes;
        x.clamp = cl;
        const int nchx = (mesh_.nx + kernels::kChunk - 1) / kernels::kChunk;
        const bool short_lines = 2 * nchx <= ns && (ns == 2 || ns == 4);
        const void* fn = do_clamp ? x_ring2_pick<true>(ns, S_, short_lines) : x_ring2_pick<false>(ns, S_, short_lines);
        const unsigned grid = ring_persist_x_ ? occupancy_grid(fn, x.tiles) : static_cast<unsigned>(x.tiles);
        if (!ring_persist_x_) ck(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem), "smem attr");
        void* args[] = {const_cast<CUtensorMap*>(&tm), &x};
        launch_k(fn, grid, kernels::kLanes, args, smem, "launch x ring2");
        return;
    }
    kernels::StridedSweep y{};
    y.rho = rho_;
    y.coef = coef;
    y.axis = ax;
    y.n = ax == 1 ? mesh_.ny : mesh_.nz;
    y.n_outer = ax == 1 ? mesh_.nz : mesh_.ny;
    y.rowlen = rowlen;
    y.tiles_per_row = (rowlen + kernels::kLanes - 1) / kernels::kLanes;
    y.reps = replicas_;
    y.r0 = rbn_ ? rb0_ : 0;
    y.hints = l2_hints_ | long_line_hint((y.n + kernels::kChunk - 1) / kernels::kChunk);
    y.keep_from8 = l2_keep_from8_;
    y.tiles = y.tiles_per_row * y.n_outer * batch_nr();
    y.S = S_;
    y.nx = mesh_.nx;
    y.clamp = cl;
    y.exp_bottom = nullptr; // z-slabs: interface values come from zslab_interface
    y.exp_top = nullptr;
    y.in_lo = ax == 2 ? z_in_lo_ : nullptr;
    y.in_hi = ax == 2 ? z_in_hi_ : nullptr;
    const int nch = (y.n + kernels::kChunk - 1) / kernels::kChunk;
    const bool short_lines = 2 * nch <= ns && (ns == 2 || ns == 4);
    const void* fn = do_clamp ? yz_ring2_pick<true>(ns, short_lines) : yz_ring2_pick<false>(ns, short_lines);
    unsigned grid;
    if (ring_persist_yz_ || short_lines) { // short lines: persistent, next tile prefetched (solve_short2)
        grid = occupancy_grid(fn, y.tiles);
    } else {
        ck(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem), "smem attr");
        grid = static_cast<unsigned>(y.tiles);
    }
    void* args[] = {const_cast<CUtensorMap*>(&tm), &y};
    launch_k(fn, grid, kernels::kLanes, args, smem, "launch yz ring2");
}

#ifdef BIODIFF_EXPERIMENTAL
// Fused x+y on ring2 (xy2.cuh).
void DeviceSession::launch_xy2()
{
    auto st = static_cast<cudaStream_t>(stream_);
    const int S = S_;
    const DeviceWorkspace& wx = ws_[0];
    const DeviceWorkspace& wy = ws_[1];
    kernels::XYFused2 a{};
    a.xcoef = kernels::Coef{wx.q,     wx.dinv, wx.cb, wx.dconst, wx.cconst, wx.settle, static_cast<long long>(wx.n) * S,
                            wx.dinvT, wx.cbT, wx.n, wx.settle_r};
    a.ycoef = kernels::Coef{wy.q,     wy.dinv, wy.cb, wy.dconst, wy.cconst, wy.settle, static_cast<long long>(wy.n) * S,
                            wy.dinvT, wy.cbT, wy.n, wy.settle_r};
    a.nx = mesh_.nx;
    a.ny = mesh_.ny;
    a.nz = mesh_.nz;
    a.S = S;
    a.rowlen = mesh_.nx * S;
    a.planes = mesh_.nz * replicas_;
    const int L = kernels::kLanes / S;
    a.xi = (mesh_.ny + L - 1) / L;
    a.yi = (a.rowlen + kernels::kLanes - 1) / kernels::kLanes;
    kernels::StridedSweep& y = a.y;
    y.coef = a.ycoef;
    y.axis = 1;
    y.n = mesh_.ny;
    y.n_outer = mesh_.nz;
    y.rowlen = a.rowlen;
    y.S = S;
    y.nx = mesh_.nx;
    y.clamp = kernels::Clamp{shell_values_, 0ull, z0_, nzg_};
    int ns = std::min(3, (std::max(mesh_.nx, mesh_.ny) + kernels::kChunk - 1) / kernels::kChunk);
    if (const char* e = std::getenv("BIODIFF_XY_SLOTS")) ns = std::max(1, std::min(4, std::atoi(e)));
    const int nch = (std::max(mesh_.nx, mesh_.ny) + kernels::kChunk - 1) / kernels::kChunk;
    const int smem = kernels::ring2_smem_bytes(ns, nch) - 1024 + smem_align_slack_;
    const void* fn = xy2_pick(ns, S);
    ck(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem), "smem attr");
    int per_sm = 0;
    ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kernels::kLanes, smem), "occupancy");
    per_sm = std::max(per_sm, 1);
    if (const char* e = std::getenv("BIODIFF_XY_CTAS_PER_SM")) per_sm = std::max(1, std::min(per_sm, std::atoi(e)));
    const long long resident = static_cast<long long>(per_sm) * sm_count_;
    const long long items = static_cast<long long>(a.planes) * (a.xi + a.yi);
    a.lag = xy_lag_for(resident, a.xi, a.yi, a.planes);
    xy_lag_ = a.lag;
    a.ctr = xy_ctr_;
    ck(cudaMemsetAsync(xy_ctr_, 0, sizeof(unsigned) * (1 + static_cast<std::size_t>(a.planes)), st), "memset");
    const unsigned grid = static_cast<unsigned>(std::min(resident, items));
    begin_kernel(kSweepXY);
    void* args[] = {tmap_[0], tmap_[1], &a};
    ck(cudaLaunchKernel(fn, dim3(grid), dim3(kernels::kLanes), args, smem, st), "launch xy2");
    end_kernel(kSweepXY);
}
#else
void DeviceSession::launch_xy2() { throw state_error("built without EXPERIMENTAL=1"); }
#endif

void DeviceSession::launch_residual_dirichlet(bool all_entries)
{
    std::int64_t count = all_entries ? dir_all_count_ : dir_res_count_;
    std::int64_t first = 0;
    if (!all_entries && rbn_ && !dir_res_rep_off_.empty()) { // this replica batch's entries only
        first = dir_res_rep_off_[rb0_];
        count = dir_res_rep_off_[rb0_ + rbn_] - first;
    }
    if (count == 0) return;
    const long long total = count * S_;
    const int block = 256;
    begin_kernel(kDirichlet);
    {
        double* rho = rho_;
        int S = S_;
        long long cnt = count;
        const int64_t* vox = (all_entries ? dir_all_voxel_ : dir_res_voxel_) + first;
        const unsigned char* mask = (all_entries ? dir_all_mask_ : dir_res_mask_) + first * S_;
        const double* vals = (all_entries ? dir_all_values_ : dir_res_values_) + first * S_;
        void* args[] = {&rho, &S, &cnt, &vox, &mask, &vals};
        launch_k(reinterpret_cast<const void*>(kernels::dirichlet_entries),
                 static_cast<unsigned>((total + block - 1) / block), block, args, 0, "dirichlet entries");
    }
    end_kernel(kDirichlet);
}

// (Re)computes the per-agent update factors when dt changes. Outside any
// graph capture: advance() calls it before capturing.
void DeviceSession::ensure_source_factors(double dt)
{
    std::uint64_t bits;
    std::memcpy(&bits, &dt, sizeof(bits));
    if (n_agents_ == 0 || (factors_valid_ && bits == factors_dt_bits_)) return;
    const double inv_voxel_volume = 1.0 / mesh_.voxel_volume(); // agents.cpp:82
    const long long total = n_agents_ * S_;
    const int block = 256;
    begin_kernel(kAux);
    kernels::sources_factors<<<static_cast<unsigned>((total + block - 1) / block), block, 0,
                               static_cast<cudaStream_t>(stream_)>>>(S_, n_agents_, agent_volume_, agent_secretion_,
                                                                      agent_uptake_, agent_saturation_, dt,
                                                                      inv_voxel_volume, agent_add_, agent_den_);
    end_kernel(kAux);
    factors_dt_bits_ = bits;
    factors_valid_ = true;
}

// Launched over the agent capacity; the kernel reads the group count of the
// last (device) rebuild, so graphs stay valid across rebuilds.
void DeviceSession::launch_sources(double dt)
{
    if (n_agents_ == 0) return;
    ensure_source_factors(dt);
    // Groups of this replica batch (all replicas outside a batch); the grid
    // covers the batch's agent count, an upper bound of its groups.
    const int r0 = rbn_ ? rb0_ : 0, nr = batch_nr();
    std::int64_t cap = n_agents_;
    if (rbn_ && static_cast<int>(rep_agents_.size()) == replicas_) {
        cap = 0;
        for (int r = r0; r < r0 + nr; ++r) cap += rep_agents_[r];
        if (cap == 0) return;
    }
    const long long total = cap * S_;
    const int block = 128;
    begin_kernel(kSources);
    {
        double* rho = rho_;
        int S = S_;
        const int64_t* glo = rep_groups_ + r0;
        const int64_t* ghi = rep_groups_ + r0 + nr;
        const int64_t* gv = group_voxel_;
        const int64_t* go = group_offsets_;
        const double* add = agent_add_;
        const double* den = agent_den_;
        void* args[] = {&rho, &S, &glo, &ghi, &gv, &go, &add, &den};
        launch_k(reinterpret_cast<const void*>(kernels::sources_groups),
                 static_cast<unsigned>((total + block - 1) / block), block, args, 0, "sources");
    }
    end_kernel(kSources);
}

// Ensembles: `steps` steps as batch visits — each batch of batch_replicas_
// replicas (sized to stay in L2) advances batch_steps_ steps before the next
// batch starts. Replicas are independent, so this is exactly `steps`
// whole-ensemble steps, bit for bit.
void DeviceSession::step_body_batches(bool with_sources, double dt, std::int64_t steps)
{
    const int nb = batch_replicas_;
    for (std::int64_t s0 = 0; s0 < steps; s0 += batch_steps_) {
        const std::int64_t s1 = std::min<std::int64_t>(steps, s0 + batch_steps_);
        for (int b = 0; b < replicas_; b += nb) {
            rb0_ = b;
            rbn_ = std::min(nb, replicas_ - b);
            for (std::int64_t s = s0; s < s1; ++s) step_body(with_sources, dt);
        }
    }
    rb0_ = 0;
    rbn_ = 0;
}

// ---- resident multi-step kernel (resident.cuh) -----------------------------

// Pivots of the three axes (dinv, cb), kept in shared memory by the kernel.
int DeviceSession::resident_coef_doubles() const { return 2 * (mesh_.nx + mesh_.ny + mesh_.nz) * S_; }

// Shared memory per warp: one 32-chain column block of the longest axis.
int DeviceSession::resident_smem_per_warp() const
{
    const int nmax = std::max(mesh_.nx, std::max(mesh_.ny, mesh_.nz));
    const long long rows = 4LL * ((nmax + 3) / 4); // TMA boxes of ceil(n/4) rows, zero-filled past n
    return static_cast<int>(std::min<long long>(rows * kernels::kLanes * 8, 1 << 30));
}

// 3-D single fields (every axis active, >= 2 points) whose lines fit a warp's
// shared-memory column block and, by default, whose field fits comfortably in
// L2 (BIODIFF_RESIDENT_MB, default 32 MB: C1 1 MB, C2 16 MB).
// BIODIFF_RESIDENT=0 / 1 forces it off / on (where supported).
bool DeviceSession::resident_path() const
{
    if (resident_mode_ == 0 || replicas_ != 1 || slab_ || S_ > kernels::kLanes) return false;
    for (int ax = 0; ax < 3; ++ax)
        if (!ws_[ax].active || ws_[ax].n < 2) return false;
    if (resident_smem_per_warp() + 8 * resident_coef_doubles() > 227 * 1024) return false;
    if (resident_mode_ == 1) return true;
    const double mb = static_cast<double>(value_count()) * 8.0 / 1e6;
    return mb <= std::atof(env_or("BIODIFF_RESIDENT_MB", "32"));
}

// Per-z-tile CSR of items [lo, hi) by voxel: count, scan, fill (item order
// inside a tile is irrelevant: one item per voxel, distinct voxels commute).
void DeviceSession::build_resident_list(const std::int64_t* vox, const std::int64_t* lo, const std::int64_t* hi,
                                        std::int64_t cap, int* off, int* idx, int* tile)
{
    auto st = static_cast<cudaStream_t>(stream_);
    const int tpr = resident_tpr();
    const int tiles = tpr * mesh_.ny;
    ck(cudaMemsetAsync(res_tile_cnt_, 0, sizeof(int) * tiles, st), "memset");
    const int block = 256;
    const unsigned grid = static_cast<unsigned>(std::max<std::int64_t>(1, (cap + block - 1) / block));
    begin_kernel(kAux);
    kernels::res_list_count<<<grid, block, 0, st>>>(vox, lo, hi, cap, mesh_.nx, mesh_.ny, S_, tpr, res_tile_cnt_);
    end_kernel(kAux);
    begin_kernel(kAux);
    kernels::res_list_scan<<<1, 1024, 0, st>>>(res_tile_cnt_, off, tiles);
    end_kernel(kAux);
    begin_kernel(kAux);
    kernels::res_list_fill<<<grid, block, 0, st>>>(vox, lo, hi, cap, mesh_.nx, mesh_.ny, S_, tpr, res_tile_cnt_, idx,
                                                    tile);
    end_kernel(kAux);
}

void DeviceSession::launch_resident(std::int64_t steps, double dt, bool with_sources)
{
    auto st = static_cast<cudaStream_t>(stream_);
    kernels::Resident a{};
    a.rho = rho_;
    a.nx = mesh_.nx;
    a.ny = mesh_.ny;
    a.nz = mesh_.nz;
    a.S = S_;
    a.tpr = resident_tpr();
    for (int ax = 0; ax < 3; ++ax) {
        const DeviceWorkspace& w = ws_[ax];
        a.ax[ax] = kernels::ResAxis{w.q, w.dinv, w.cb, w.dconst, w.cconst, w.settle, w.n};
    }
    a.clamp = kernels::Clamp{shell_values_, shell_mask_, z0_, nzg_};
    const std::int64_t tiles = static_cast<std::int64_t>(a.tpr) * mesh_.ny;
    a.dirichlet = dir_res_count_ > 0 ? 1 : 0;
    if (a.dirichlet) {
        if (!res_dir_valid_) {
            dfree(res_dir_idx_);
            ck(cudaMalloc(&res_dir_idx_, sizeof(int) * 2 * dir_res_count_), "cudaMalloc");
            build_resident_list(dir_res_voxel_, nullptr, nullptr, dir_res_count_, res_dir_off_, res_dir_idx_, nullptr);
            res_dir_valid_ = true;
        }
        a.zdir_off = res_dir_off_;
        a.zdir_idx = res_dir_idx_;
        a.dir_voxel = dir_res_voxel_;
        a.dir_mask = dir_res_mask_;
        a.dir_values = dir_res_values_;
    }
    a.sources = with_sources && n_agents_ > 0 ? 1 : 0;
    if (a.sources) {
        ensure_source_factors(dt);
        if (!res_grp_valid_) {
            if (res_grp_cap_ < 2 * n_agents_) {
                dfree(res_grp_idx_);
                dfree(res_grp_tile_);
                dfree(res_grp_desc_);
                res_grp_cap_ = 2 * n_agents_;
                ck(cudaMalloc(&res_grp_idx_, sizeof(int) * res_grp_cap_), "cudaMalloc");
                ck(cudaMalloc(&res_grp_tile_, sizeof(int) * res_grp_cap_), "cudaMalloc");
                ck(cudaMalloc(&res_grp_desc_, sizeof(kernels::ResSrc) * res_grp_cap_), "cudaMalloc");
            }
            build_resident_list(group_voxel_, rep_groups_, rep_groups_ + 1, n_agents_, res_grp_off_, res_grp_idx_,
                                res_grp_tile_);
            const int tiles_z = a.tpr * mesh_.ny;
            begin_kernel(kAux);
            kernels::res_src_desc<<<static_cast<unsigned>((res_grp_cap_ + 255) / 256), 256, 0, st>>>(
                res_grp_idx_, res_grp_off_ + tiles_z, group_voxel_, group_offsets_, static_cast<kernels::ResSrc*>(res_grp_desc_));
            end_kernel(kAux);
            res_grp_valid_ = true;
        }
        a.zgrp_off = res_grp_off_;
        a.zgrp_idx = res_grp_idx_;
        a.zgrp_tile = res_grp_tile_;
        a.zsrc = static_cast<const kernels::ResSrc*>(res_grp_desc_);
        a.group_voxel = group_voxel_;
        a.group_offsets = group_offsets_;
        a.add = agent_add_;
        a.den = agent_den_;
    }
    a.steps = steps;
    a.cnt = res_cnt_;
    const int per_warp = resident_smem_per_warp();
    a.buf_doubles = per_warp / 8;
    a.coef_doubles = resident_coef_doubles();
    a.coef_doubles = (a.coef_doubles + 15) / 16 * 16; // keeps the column blocks 128-byte aligned
    const int kWarps = std::max(1, std::min(4, (227 * 1024 - 512 - a.coef_doubles * 8) / per_warp));
    const int block = kWarps * kernels::kLanes;
    const int smem = 128 * kWarps + a.coef_doubles * 8 + kWarps * per_warp;
    a.tma = res_tmap_ok_ ? 1 : 0;
    const void* fn = reinterpret_cast<const void*>(kernels::step_resident);
    ck(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem), "smem attr");
    int per_sm = 0;
    ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, block, smem), "occupancy");
    if (per_sm < 1) throw state_error("resident kernel does not fit an SM");
    // One warp tile per CTA first (warp rank = warp-in-block * grid + block),
    // at most what is co-resident.
    const long long L = kernels::kLanes / S_;
    long long max_tiles = (static_cast<long long>(mesh_.ny) * mesh_.nz + L - 1) / L;
    max_tiles = std::max(max_tiles, static_cast<long long>(a.tpr) * std::max(mesh_.ny, mesh_.nz));
    const long long grid = std::max<long long>(1, std::min<long long>(static_cast<long long>(per_sm) * sm_count_, max_tiles));
    (void)tiles;
    ck(cudaMemsetAsync(res_cnt_, 0,
                       sizeof(unsigned) * kernels::kCntPad * (static_cast<std::size_t>(mesh_.nz) + a.tpr + 2 * mesh_.ny), st),
       "counter reset");
    const char* trace_path = std::getenv("BIODIFF_RES_TRACE"); // design probe: per-tile phase stamps
    std::size_t trace_n = 0;
    if (trace_path) {
        a.trace_tiles = std::max<long long>(max_tiles, (n_agents_ * 2 + 31) / 32);
        trace_n = static_cast<std::size_t>(8 * 4 * a.trace_tiles * 6);
        ck(cudaMalloc(&a.trace, trace_n * 8), "cudaMalloc");
        ck(cudaMemsetAsync(a.trace, 0, trace_n * 8, st), "memset");
    }
    void* args[] = {res_tmap_[0], res_tmap_[1], &a};
    begin_kernel(kResident);
    ck(cudaLaunchCooperativeKernel(fn, dim3(static_cast<unsigned>(grid)), dim3(block), args, smem, st),
       "resident launch");
    end_kernel(kResident);
    if (trace_path) {
        std::vector<unsigned long long> h(trace_n);
        ck(cudaMemcpyAsync(h.data(), a.trace, trace_n * 8, cudaMemcpyDeviceToHost, st), "download");
        ck(cudaStreamSynchronize(st), "sync");
        cudaFree(a.trace);
        if (FILE* f = std::fopen(trace_path, "wb")) {
            const long long hdr[4] = {a.trace_tiles, grid, block, smem};
            std::fwrite(hdr, sizeof(hdr), 1, f);
            std::fwrite(h.data(), 8, trace_n, f);
            std::fclose(f);
        }
    }
}

// ---- one-cluster kernel for fields that fit a cluster's shared memory (small.cuh)

// Shared row pitch of the one-cluster / slab-grid kernel: the TMA box is
// `pitch` doubles wide (columns past the row zero-filled on load, clipped on
// store), chosen so the (line, substrate) lanes of the x chains spread over
// the bank pairs: pitch = S (mod 16) for even S (conflict-free), 2 (mod 16)
// for odd S (the box width must stay a multiple of 16 bytes).
static int small_pitch(int rowlen, int S)
{
    const int want = S % 2 == 0 ? S % 16 : 2;
    return rowlen + ((want - rowlen) % 16 + 16) % 16;
}

// Cluster size, planes per CTA, row pitch and dynamic smem of the one-cluster
// kernel, or false when the field does not fit (or the mode is off).
bool DeviceSession::small_config(int& cl, int& planes, int& pitch, int& smem_bytes, bool& grid) const
{
    grid = false;
    if (small_mode_ == 0 || resident_mode_ == 0 || replicas_ != 1 || slab_ || S_ > kernels::kLanes) return false;
    for (int ax = 0; ax < 3; ++ax)
        if (!ws_[ax].active || ws_[ax].n < 2) return false;
    constexpr int kThreads = 256;
    const int rowlen = mesh_.nx * S_;
    const int coef = (resident_coef_doubles() + 15) / 16 * 16;
    for (int c : {16, 8}) {
        planes = (mesh_.nz + c - 1) / c;
        // TMA slab moves need 16-byte rows and a box of <= 256 x 256; the
        // rows are then dense (pitch = rowlen), else padded to S mod 16.
        pitch = small_pitch(rowlen, S_);
        const bool tma = rowlen % 2 == 0 && pitch <= 256 && planes * mesh_.ny <= 256;
        if (!tma) continue; // slab moves by TMA only (the one-cluster kernel's supported shapes)
        const long long slab = std::max<long long>(static_cast<long long>(planes) * mesh_.ny * pitch,
                                                   static_cast<long long>(mesh_.nz) * kThreads);
        const long long bytes = (16 + coef + slab) * 8;
        if (bytes <= 227 * 1024) {
            cl = c;
            smem_bytes = static_cast<int>(bytes);
            return true;
        }
    }
    // Grid mode: one CTA per slab of planes, all co-resident (one per SM),
    // grid barriers instead of cluster barriers.
    for (planes = std::max(1, (mesh_.nz + sm_count_ - 1) / sm_count_); planes * mesh_.ny <= 256; ++planes) {
        pitch = small_pitch(rowlen, S_);
        if (rowlen % 2 != 0 || pitch > 256) break;
        const long long slab = std::max<long long>(static_cast<long long>(planes) * mesh_.ny * pitch,
                                                   static_cast<long long>(mesh_.nz) * kThreads);
        const long long bytes = (16 + coef + slab) * 8;
        if (bytes > 227 * 1024) continue;
        cl = (mesh_.nz + planes - 1) / planes;
        smem_bytes = static_cast<int>(bytes);
        grid = true;
        return true;
    }
    return false;
}

bool DeviceSession::small_path() const
{
    int cl, planes, pitch, smem;
    bool grid;
    if (!small_config(cl, planes, pitch, smem, grid)) return false;
    if (small_mode_ == 1) return true;
    // auto: where it measured faster than the L2 dataflow kernel — the
    // one-cluster mode (C1: 19.0 vs 27.3 us per step) and the slab-grid mode
    // (C2: 41.4 vs 43.4 us) — for fields up to BIODIFF_SMALL_MB (32 MB).
    return static_cast<double>(value_count()) * 8.0 / 1e6 <= std::atof(env_or("BIODIFF_SMALL_MB", "32"));
}

void DeviceSession::launch_small(std::int64_t steps, double dt, bool with_sources)
{
    auto st = static_cast<cudaStream_t>(stream_);
    int cl = 0, planes = 0, pitch = 0, smem = 0;
    bool grid = false;
    if (!small_config(cl, planes, pitch, smem, grid)) throw state_error("field does not fit the one-cluster kernel");
    kernels::Small a{};
    a.rho = rho_;
    a.nx = mesh_.nx;
    a.ny = mesh_.ny;
    a.nz = mesh_.nz;
    a.S = S_;
    a.pitch = pitch;
    a.planes = planes;
    for (int ax = 0; ax < 3; ++ax) {
        const DeviceWorkspace& w = ws_[ax];
        a.ax[ax] = kernels::ResAxis{w.q, w.dinv, w.cb, w.dconst, w.cconst, w.settle, w.n};
    }
    a.clamp = kernels::Clamp{shell_values_, shell_mask_, z0_, nzg_};
    a.dir_count = dir_res_count_;
    a.dir_voxel = dir_res_voxel_;
    a.dir_mask = dir_res_mask_;
    a.dir_values = dir_res_values_;
    a.sources = with_sources && n_agents_ > 0 ? 1 : 0;
    if (a.sources) {
        ensure_source_factors(dt);
        a.g_lo = rep_groups_;
        a.g_hi = rep_groups_ + 1;
        a.group_voxel = group_voxel_;
        a.group_offsets = group_offsets_;
        a.add = agent_add_;
        a.den = agent_den_;
    }
    a.steps = steps;
    a.coef_doubles = (resident_coef_doubles() + 15) / 16 * 16;
    a.slab_doubles = smem / 8 - 16 - a.coef_doubles;
    const long long rowlen = static_cast<long long>(mesh_.nx) * S_;
    a.tma = rowlen % 2 == 0 ? std::atoi(env_or("BIODIFF_SMALL_TMA_MASK", "3")) : 0;
    alignas(64) unsigned char tmap[128] = {};
    if (a.tma) { // 4-D view (row, (plane, j) row index, 1, 1), box (rowlen, planes * ny)
        void* efn = nullptr;
        cudaDriverEntryPointQueryResult q;
        ck(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &efn, cudaEnableDefault, &q), "driver entry point");
        using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
        const cuuint64_t dims[4] = {static_cast<cuuint64_t>(rowlen),
                                    static_cast<cuuint64_t>(mesh_.ny) * static_cast<cuuint64_t>(mesh_.nz), 1, 1};
        const cuuint64_t total = static_cast<cuuint64_t>(rowlen) * mesh_.ny * mesh_.nz * 8;
        const cuuint64_t strides[3] = {static_cast<cuuint64_t>(rowlen) * 8, total, total};
        const cuuint32_t box[4] = {static_cast<cuuint32_t>(pitch), static_cast<cuuint32_t>(planes * mesh_.ny), 1, 1};
        const cuuint32_t estr[4] = {1, 1, 1, 1};
        if (reinterpret_cast<Encode>(efn)(reinterpret_cast<CUtensorMap*>(tmap), CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4,
                                          rho_, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            throw state_error("slab tensor map");
    }
    a.grid = grid ? 1 : 0;
    a.bar = res_cnt_; // grid mode: two words of the resident kernel's counter block
    const void* fn = reinterpret_cast<const void*>(kernels::step_small);
    ck(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem), "smem attr");
    if (!grid && cl > 8) ck(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1), "cluster 16");
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(cl);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = static_cast<std::size_t>(smem);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const char* trace_path = std::getenv("BIODIFF_RES_TRACE"); // design probe: per-CTA phase stamps
    const std::size_t trace_n = static_cast<std::size_t>(8) * cl * 12;
    if (trace_path) {
        ck(cudaMalloc(&a.trace, trace_n * 8), "cudaMalloc");
        ck(cudaMemsetAsync(a.trace, 0, trace_n * 8, st), "memset");
    }
    void* args[] = {tmap, &a};
    begin_kernel(kResident);
    if (grid) {
        ck(cudaMemsetAsync(res_cnt_, 0, 2 * sizeof(unsigned), st), "barrier reset");
        ck(cudaLaunchCooperativeKernel(fn, dim3(static_cast<unsigned>(cl)), dim3(256), args, static_cast<std::size_t>(smem),
                                       st),
           "launch slab-grid kernel");
    } else {
        ck(cudaLaunchKernelExC(&cfg, fn, args), "launch one-cluster kernel");
    }
    end_kernel(kResident);
    if (trace_path) {
        std::vector<unsigned long long> h(trace_n);
        ck(cudaMemcpyAsync(h.data(), a.trace, trace_n * 8, cudaMemcpyDeviceToHost, st), "download");
        ck(cudaStreamSynchronize(st), "sync");
        cudaFree(a.trace);
        if (FILE* f = std::fopen(trace_path, "wb")) {
            const long long hdr[4] = {-1, cl, 256, smem}; // -1: one-cluster trace layout
            std::fwrite(hdr, sizeof(hdr), 1, f);
            std::fwrite(h.data(), 8, trace_n, f);
            std::fclose(f);
        }
    }
}

void DeviceSession::sweep(Axis axis)
{
    ck(cudaSetDevice(device_), "cudaSetDevice");
    check_ready(axis);
    launch_sweep(axis, false);
}

void DeviceSession::apply_dirichlet()
{
    ck(cudaSetDevice(device_), "cudaSetDevice");
    launch_residual_dirichlet(true);
}

// solver.cpp:289-299 with the clamp fused into the last active sweep.
void DeviceSession::step_body(bool with_sources, double dt)
{
    if (slab_ && remote_) { // one slab per rank: exchanges on this stream (slab.cu)
        slab_step_nccl(with_sources, dt);
        return;
    }
    if (slab_ && (prev_slab_ || next_slab_))
        throw state_error("in-process z-slabs advance together: use the group advance");
    const Axis last = ws_[2].active ? Axis::z : ws_[1].active ? Axis::y : Axis::x;
    if (last == Axis::z && xyz_cluster_pays()) {
        launch_xy_cluster(true);
        launch_residual_dirichlet(false);
        if (with_sources) launch_sources(dt);
        return;
    }
    if (last == Axis::z) {
        launch_xy_sweeps();
    } else {
        launch_sweep(Axis::x, last == Axis::x);
        if (ws_[1].active) launch_sweep(Axis::y, last == Axis::y);
    }
    if (ws_[2].active) launch_sweep(Axis::z, last == Axis::z);
    launch_residual_dirichlet(false);
    if (with_sources) launch_sources(dt);
}

void DeviceSession::diffuse_decay_step()
{
    ck(cudaSetDevice(device_), "cudaSetDevice");
    check_ready(Axis::x);
    step_body(false, 0.0);
}

void DeviceSession::sources(double dt)
{
    if (!(dt > 0.0)) throw std::invalid_argument("reaction step size must be positive");
    ck(cudaSetDevice(device_), "cudaSetDevice");
    launch_sources(dt);
}

// The body advance() runs (or captures) for n steps.
void DeviceSession::advance_body(std::int64_t n, double dt, bool with_sources)
{
    const bool batched = batch_replicas_ > 0 && !slab_ && path_[0] == SweepPath::smem_ring2 &&
                         (!ws_[1].active || path_[1] == SweepPath::smem_ring2) &&
                         (!ws_[2].active || path_[2] == SweepPath::smem_ring2) && !xy_fusable();
    if (batched)
        step_body_batches(with_sources, dt, n);
    else
        for (std::int64_t s = 0; s < n; ++s) step_body(with_sources, dt);
}

bool DeviceSession::uses_graphs() const { return !(timing_ || slab_ || std::getenv("BIODIFF_NO_GRAPH")); }

// The instantiated graph of n steps (captured on first use).
std::pair<void*, int>& DeviceSession::graph_for(std::int64_t n, double dt, bool with_sources)
{
    std::uint64_t bits;
    std::memcpy(&bits, &dt, sizeof(bits));
    GraphKey key{n, with_sources, bits};
    auto it = graphs_.find(key);
    if (it == graphs_.end()) {
        auto st = static_cast<cudaStream_t>(stream_);
        const std::int64_t before = launches_;
        cudaGraph_t graph;
        ck(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal), "begin capture");
        advance_body(n, dt, with_sources);
        ck(cudaStreamEndCapture(st, &graph), "end capture");
        cudaGraphExec_t exec;
        ck(cudaGraphInstantiate(&exec, graph, 0), "graph instantiate");
        cudaGraphDestroy(graph);
        const int kernels_in_graph = static_cast<int>(launches_ - before);
        launches_ = before;
        it = graphs_.emplace(key, std::make_pair(static_cast<void*>(exec), kernels_in_graph)).first;
    }
    return it->second;
}

void DeviceSession::check_advance(std::int64_t steps, double dt) const
{
    if (steps < 0) throw std::invalid_argument("step count must be non-negative");
    if (!(dt > 0.0)) throw std::invalid_argument("reaction step size must be positive");
    check_ready(Axis::x);
    if (std::memcmp(&dt, &dt_, sizeof(double)) != 0)
        throw state_error("advance dt does not match the solver workspace dt");
}

// Captures and instantiates every graph advance(steps, dt, with_sources)
// would replay, without running anything: a caller that times advance()
// excludes the one-time capture cost.
void DeviceSession::prepare_advance(std::int64_t steps, double dt, bool with_sources)
{
    if (steps == 0) return;
    ck(cudaSetDevice(device_), "cudaSetDevice");
    check_advance(steps, dt);
    if (with_sources) ensure_source_factors(dt);
    if (!uses_graphs() || resident_path() || small_path()) return;
    if (steps / kGraphSteps) graph_for(kGraphSteps, dt, with_sources);
    if (steps % kGraphSteps) graph_for(steps % kGraphSteps, dt, with_sources);
}

void DeviceSession::advance(std::int64_t steps, double dt, bool with_sources)
{
    if (steps < 0) throw std::invalid_argument("step count must be non-negative");
    if (steps == 0) return;
    ck(cudaSetDevice(device_), "cudaSetDevice");
    check_advance(steps, dt);
    auto st = static_cast<cudaStream_t>(stream_);
    if (with_sources) ensure_source_factors(dt); // not inside the graph capture
    if (small_path()) { // every step in one launch of one cluster (field in shared memory)
        launch_small(steps, dt, with_sources);
        return;
    }
    if (resident_path()) { // every step in one cooperative launch
        launch_resident(steps, dt, with_sources);
        return;
    }
    if (!uses_graphs()) {
        advance_body(steps, dt, with_sources);
        return;
    }
    // Replay captured graphs of up to kGraphSteps steps (launch gaps vanish).
    auto run_chunk = [&](std::int64_t n) {
        auto& g = graph_for(n, dt, with_sources);
        ck(cudaGraphLaunch(static_cast<cudaGraphExec_t>(g.first), st), "graph launch");
        launches_ += g.second;
    };
    const std::int64_t full = steps / kGraphSteps;
    for (std::int64_t c = 0; c < full; ++c) run_chunk(kGraphSteps);
    if (steps % kGraphSteps) run_chunk(steps % kGraphSteps);
}

bool DeviceSession::all_finite()
{
    ck(cudaSetDevice(device_), "cudaSetDevice");
    auto st = static_cast<cudaStream_t>(stream_);
    int* flag = nullptr;
    ck(cudaMalloc(&flag, sizeof(int)), "cudaMalloc");
    ck(cudaMemsetAsync(flag, 0, sizeof(int), st), "memset");
    begin_kernel(kAux);
    kernels::any_nonfinite<<<sm_count_ * 4, 256, 0, st>>>(rho_, value_count(), flag);
    end_kernel(kAux);
    int h = 0;
    ck(cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, st), "D2H");
    ck(cudaStreamSynchronize(st), "sync");
    cudaFree(flag);
    return h == 0;
}

void DeviceSession::cross_check(const double* other, std::int64_t count, double abs_tol, double rel_tol,
                                double* max_abs, double* max_rel, std::int64_t* worst, bool* pass)
{
    if (count != value_count()) throw std::invalid_argument("cross_check fields have different shapes");
    if (abs_tol < 0.0 || rel_tol < 0.0) throw std::invalid_argument("cross_check tolerances must be non-negative");
    ck(cudaSetDevice(device_), "cudaSetDevice");
    auto st = static_cast<cudaStream_t>(stream_);
    double* b = nullptr;
    unsigned long long* scratch = nullptr;
    ck(cudaMalloc(&b, sizeof(double) * count), "cudaMalloc");
    ck(cudaMalloc(&scratch, 4 * sizeof(unsigned long long)), "cudaMalloc");
    const unsigned long long init[4] = {0ull, 0ull, ~0ull, 0ull};
    ck(cudaMemcpyAsync(scratch, init, sizeof(init), cudaMemcpyHostToDevice, st), "H2D");
    ck(cudaMemcpyAsync(b, other, sizeof(double) * count, cudaMemcpyHostToDevice, st), "H2D");
    begin_kernel(kAux);
    kernels::cross_check_max<<<148 * 4, 256, 0, st>>>(rho_, b, count, scratch, scratch + 1, abs_tol, rel_tol,
                                                      reinterpret_cast<int*>(scratch + 3));
    end_kernel(kAux);
    begin_kernel(kAux);
    kernels::cross_check_argmax<<<148 * 4, 256, 0, st>>>(rho_, b, count, scratch, scratch + 2);
    end_kernel(kAux);
    unsigned long long out[4];
    ck(cudaMemcpyAsync(out, scratch, sizeof(out), cudaMemcpyDeviceToHost, st), "D2H");
    ck(cudaStreamSynchronize(st), "sync");
    cudaFree(b);
    cudaFree(scratch);
    std::memcpy(max_abs, &out[0], sizeof(double));
    std::memcpy(max_rel, &out[1], sizeof(double));
    *worst = out[2] == ~0ull ? -1 : static_cast<std::int64_t>(out[2]);
    *pass = (out[3] & 1ull) == 0;
}

// ---- DeviceBackend (host.hpp) --------------------------------------------

DeviceBackend::DeviceBackend(int device) : device_(device) {}
DeviceBackend::~DeviceBackend() = default;

void DeviceBackend::attach(const Microenvironment& env, const SolverWorkspaces& ws, const AgentPopulation* agents)
{
    session_ = std::make_unique<DeviceSession>(env.mesh, env.substrate_count(), device_);
    session_->set_workspaces(ws);
    session_->set_dirichlet(env.dirichlet);
    if (agents) attach_agents(*agents);
    session_->upload(env.field.values.data(), static_cast<std::int64_t>(env.field.values.size()));
}

void DeviceBackend::attach_agents(const AgentPopulation& agents)
{
    if (!session_) throw state_error("device backend not attached");
    session_->set_agents(agents);
    agents_from_ = &agents;
}

void DeviceBackend::upload(const DensityField& field)
{
    if (!session_) throw state_error("device backend not attached");
    session_->upload(field.values.data(), static_cast<std::int64_t>(field.values.size()));
}

void DeviceBackend::download(DensityField& field)
{
    if (!session_) throw state_error("device backend not attached");
    field.values.resize(static_cast<std::size_t>(session_->value_count()));
    field.substrates = session_->substrates();
    session_->download(field.values.data(), static_cast<std::int64_t>(field.values.size()));
}

void DeviceBackend::upload(const NestedDensity& nested)
{
    if (!session_) throw state_error("device backend not attached");
    const DensityField flat = translate_vector_to_array(nested);
    if (flat.substrates != session_->substrates() && !nested.empty())
        throw state_error("nested density substrate count does not match the session");
    session_->upload(flat.values.data(), static_cast<std::int64_t>(flat.values.size()));
}

void DeviceBackend::download(NestedDensity& nested)
{
    DensityField flat;
    download(flat);
    nested = translate_array_to_vector(flat);
}

void diffuse_decay_step(Microenvironment& env, const SolverWorkspaces& workspaces, DeviceBackend& backend)
{
    if (!workspaces.x) throw state_error("solver workspaces not built");
    (void)env;
    backend.session().diffuse_decay_step();
}

void cell_sources_sinks_step(DensityField& field, const AgentPopulation& agents, const CartesianMesh& mesh, double dt,
                             DeviceBackend& backend)
{
    (void)field;
    (void)mesh;
    if (!(dt > 0.0)) throw std::invalid_argument("reaction step size must be positive");
    if (agents.empty()) return;
    // Re-upload when the caller hands a different population than the one
    // attached (agents are static between grouping rebuilds).
    if (backend.attached_agents() != &agents || backend.session().agents().size() != agents.size())
        backend.attach_agents(agents);
    backend.session().sources(dt);
}

} // namespace biodiff_b200

#ifdef BIODIFF_XYC_TRACE
// Design probe (variant builds only): copies the plane-cluster phase stamps.
extern "C" int biodiff_debug_xyc_trace(unsigned long long* out, long long n)
{
    return static_cast<int>(cudaMemcpyFromSymbol(out, biodiff_b200::kernels::g_xyc_trace, n * 8));
}
#endif
