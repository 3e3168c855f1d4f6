// z-slab decomposition of the LOD step across GPUs.
//
// Slab p owns global planes [z0, z1) and the GLOBAL factorisation rows of
// its planes. The x and y sweeps are local. One read of the slab
// (zslab_interface) gives, with zero inflow at its ends, the forward value of
// its last row (dhat) and the back-substituted value of its first row
// (xhat_0). D_{p-1} (the true forward value of the previous slab's last row)
// and X_{p+1} (the true final value of the next slab's first row) then follow
// exactly from two plane recurrences across the slabs (phi / Phi / Psi: the
// slab's host-precomputed responses to unit inflows):
//   forward : D_p = dhat_p + phi_p(last row) * D_{p-1}           p -> p+1
//   backward: X_p = xhat_0,p + Phi_p(0) * D_{p-1} + Psi_p(0) * X_{p+1}   p -> p-1
// Finally the z sweep runs the global recurrence on the slab with D_{p-1} as
// the inflow into row 0 and X_{p+1} into the last row — no correction pass.
// No coupling is truncated, so there is no minimum slab thickness; the result
// differs from the single-domain solve only by rounding (the interface values
// are formed in a different order). Per step a slab reads its field once more
// (8 B/vsu) than a single domain, and each interface moves two nx*ny*S planes
// (33.6 MB at 1024^2 x 4), pipelined in pieces.
// Transports: NCCL send/recv on the session stream (one slab per rank, the
// multi-GPU path) or device/peer copies between sessions of one process.
#include "device.hpp"
#include "kernels.cuh"

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>

namespace biodiff_b200 {

namespace {

void ck(cudaError_t e, const char* what)
{
    if (e != cudaSuccess) throw state_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

// NCCL is resolved at run time (the process may already hold torch's copy);
// the library has no link-time NCCL dependency.
struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    std::string error;
};

NcclApi& nccl()
{
    static NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            a.error = std::string("cannot load libnccl.so.2: ") + dlerror();
            return a;
        }
        auto sym = [&](const char* n) { return dlsym(h, n); };
        a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
        a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
        a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
        a.Send = reinterpret_cast<decltype(a.Send)>(sym("ncclSend"));
        a.Recv = reinterpret_cast<decltype(a.Recv)>(sym("ncclRecv"));
        a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
        a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
        a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
        if (!a.GetUniqueId || !a.CommInitRank || !a.Send || !a.Recv || !a.GroupStart || !a.GroupEnd)
            a.error = "libnccl.so.2 lacks the point-to-point API";
        return a;
    }();
    return api;
}

void nck(ncclResult_t r, const char* what)
{
    if (r != ncclSuccess)
        throw state_error(std::string("NCCL error in ") + what + ": " +
                          (nccl().GetErrorString ? nccl().GetErrorString(r) : "?"));
}

} // namespace

void nccl_unique_id(unsigned char* out)
{
    NcclApi& a = nccl();
    if (!a.error.empty()) throw state_error(a.error);
    ncclUniqueId id;
    nck(a.GetUniqueId(&id), "ncclGetUniqueId");
    static_assert(sizeof(id) == NCCL_UNIQUE_ID_BYTES, "unexpected ncclUniqueId size");
    std::memcpy(out, &id, sizeof(id));
}

void DeviceSession::configure_slab(int nz_global, int z0)
{
    if (slab_) throw state_error("session is already a z-slab");
    if (z0 < 0 || z0 + mesh_.nz > nz_global) throw config_error("z-slab outside the global mesh");
    if (ws_[0].active || ws_[1].active || ws_[2].active)
        throw state_error("configure the z-slab before setting workspaces");
    ck(cudaSetDevice(device_), "cudaSetDevice");
    slab_ = true;
    nzg_ = nz_global;
    z0_ = z0;
    const std::size_t bytes = sizeof(double) * plane_count();
    for (double** p : {&plane_bottom_, &plane_top_, &plane_din_, &plane_dout_, &plane_xin_, &plane_xtop_}) {
        ck(cudaMalloc(p, bytes), "cudaMalloc plane");
        ck(cudaMemsetAsync(*p, 0, bytes, static_cast<cudaStream_t>(stream_)), "cudaMemset plane");
    }
    choose_paths();
    if (nz_global > 1 && path_[2] != SweepPath::smem_ring2)
        throw config_error("z-slab needs the ring2 z-sweep (rows with an even number of doubles)");
}

bool DeviceSession::is_boundary_local(int i, int j, int k_local) const
{
    const int k = k_local + z0_;
    return i == 0 || i == mesh_.nx - 1 || j == 0 || j == mesh_.ny - 1 || k == 0 || k == nzg_ - 1;
}

std::int64_t DeviceSession::boundary_count_local() const
{
    std::int64_t n = 0;
    const std::int64_t face = static_cast<std::int64_t>(mesh_.nx) * mesh_.ny;
    const std::int64_t inner = static_cast<std::int64_t>(std::max(mesh_.nx - 2, 0)) * std::max(mesh_.ny - 2, 0);
    for (int k = 0; k < mesh_.nz; ++k) {
        const int kg = k + z0_;
        n += (kg == 0 || kg == nzg_ - 1) ? face : face - inner;
    }
    return n;
}

void DeviceSession::set_slab_spikes(const double* Phi, const double* psi, const double* phi_last)
{
    if (!slab_) throw state_error("not a z-slab session");
    ck(cudaSetDevice(device_), "cudaSetDevice");
    auto st = static_cast<cudaStream_t>(stream_);
    const std::size_t n = static_cast<std::size_t>(mesh_.nz) * S_;
    if (!slab_phi_) ck(cudaMalloc(&slab_phi_, sizeof(double) * n), "cudaMalloc");
    if (!slab_psi_) ck(cudaMalloc(&slab_psi_, sizeof(double) * n), "cudaMalloc");
    if (!slab_philast_) ck(cudaMalloc(&slab_philast_, sizeof(double) * S_), "cudaMalloc");
    ck(cudaMemcpyAsync(slab_phi_, Phi, sizeof(double) * n, cudaMemcpyHostToDevice, st), "H2D");
    ck(cudaMemcpyAsync(slab_psi_, psi, sizeof(double) * n, cudaMemcpyHostToDevice, st), "H2D");
    ck(cudaMemcpyAsync(slab_philast_, phi_last, sizeof(double) * S_, cudaMemcpyHostToDevice, st), "H2D");
    ck(cudaStreamSynchronize(st), "sync");
}

void DeviceSession::connect_nccl(const unsigned char* unique_id, int nranks, int rank)
{
    if (!slab_) throw state_error("not a z-slab session");
    if (nranks < 1 || rank < 0 || rank >= nranks) throw config_error("bad NCCL rank / size");
    NcclApi& a = nccl();
    if (!a.error.empty()) throw state_error(a.error);
    ck(cudaSetDevice(device_), "cudaSetDevice");
    ncclUniqueId id;
    std::memcpy(&id, unique_id, sizeof(id));
    if (remote_ || prev_slab_ || next_slab_) throw state_error("z-slab transport already connected");
    ncclComm_t comm;
    nck(a.CommInitRank(&comm, nranks, id, rank), "ncclCommInitRank");
    nccl_comm_ = comm;
    nccl_rank_ = rank;
    nccl_ranks_ = nranks;
    remote_ = true;
}

void DeviceSession::connect_host_transport(int nranks, int rank, HostExchange fn, void* user)
{
    if (!slab_) throw state_error("not a z-slab session");
    if (nranks < 1 || rank < 0 || rank >= nranks) throw config_error("bad transport rank / size");
    if (!fn) throw std::invalid_argument("null exchange callback");
    if (remote_ || prev_slab_ || next_slab_) throw state_error("z-slab transport already connected");
    ck(cudaSetDevice(device_), "cudaSetDevice");
    const std::size_t bytes = sizeof(double) * plane_count();
    ck(cudaMallocHost(&host_send_, bytes), "cudaMallocHost");
    ck(cudaMallocHost(&host_recv_, bytes), "cudaMallocHost");
    host_xchg_ = fn;
    host_xchg_user_ = user;
    nccl_rank_ = rank;
    nccl_ranks_ = nranks;
    remote_ = true;
}

// The one exchange primitive of slab_step_remote: NCCL send/recv on the
// session stream, or — host transport — the stream is drained, the send
// piece staged to pinned memory, the callback moves it, and the received
// piece is queued back onto the stream (same order, same pieces).
void DeviceSession::nccl_exchange(double* send, int send_peer, double* recv, int recv_peer, std::int64_t count)
{
    if (!send && !recv) return;
    auto st0 = static_cast<cudaStream_t>(stream_);
    if (!nccl_comm_) {
        const std::size_t bytes = sizeof(double) * static_cast<std::size_t>(count);
        if (send) ck(cudaMemcpyAsync(host_send_, send, bytes, cudaMemcpyDeviceToHost, st0), "D2H plane");
        ck(cudaStreamSynchronize(st0), "sync");
        if (host_xchg_(host_xchg_user_, send ? host_send_ : nullptr, send_peer, recv ? host_recv_ : nullptr, recv_peer,
                       count) != 0)
            throw state_error("z-slab plane exchange callback failed");
        if (recv) {
            ck(cudaMemcpyAsync(recv, host_recv_, bytes, cudaMemcpyHostToDevice, st0), "H2D plane");
            ck(cudaStreamSynchronize(st0), "sync"); // the staging buffer is reused by the next exchange
        }
        return;
    }
    NcclApi& a = nccl();
    auto comm = static_cast<ncclComm_t>(nccl_comm_);
    auto st = static_cast<cudaStream_t>(stream_);
    nck(a.GroupStart(), "ncclGroupStart");
    if (send) nck(a.Send(send, static_cast<size_t>(count), ncclFloat64, send_peer, comm, st), "ncclSend");
    if (recv) nck(a.Recv(recv, static_cast<size_t>(count), ncclFloat64, recv_peer, comm, st), "ncclRecv");
    nck(a.GroupEnd(), "ncclGroupEnd");
}

// The interface chains are serial over slabs; splitting each plane into
// pieces (whole columns of S values, >= 1 MB) pipelines them: slab p+1 works
// on piece 1 while piece 2 of slab p is still in flight.
std::vector<std::pair<std::int64_t, std::int64_t>> DeviceSession::plane_pieces() const
{
    const std::int64_t plane = plane_count();
    int want = std::max(1, std::atoi(std::getenv("BIODIFF_ZSLAB_PIECES") ? std::getenv("BIODIFF_ZSLAB_PIECES") : "8"));
    const char* mp = std::getenv("BIODIFF_ZSLAB_MIN_PIECE"); // doubles per piece (tests: force several pieces)
    const std::int64_t min_piece = std::max<std::int64_t>(S_, mp ? std::atoll(mp) : (1 << 20) / 8);
    want = static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>(want, plane / min_piece)));
    std::vector<std::pair<std::int64_t, std::int64_t>> pieces;
    const std::int64_t cols = plane / S_;
    for (int i = 0; i < want; ++i) {
        const std::int64_t c0 = cols * i / want, c1 = cols * (i + 1) / want;
        if (c1 > c0) pieces.push_back({c0 * S_, (c1 - c0) * S_});
    }
    return pieces;
}

void DeviceSession::link_local(const std::vector<DeviceSession*>& slabs)
{
    for (std::size_t p = 0; p < slabs.size(); ++p) {
        DeviceSession* s = slabs[p];
        if (!s->slab_) throw state_error("link_local needs z-slab sessions");
        if (s->remote_) throw state_error("z-slab transport already connected");
        if (p + 1 < slabs.size() && s->z0_ + s->mesh_.nz != slabs[p + 1]->z0_)
            throw config_error("z-slabs must be contiguous and in order");
        s->prev_slab_ = p > 0 ? slabs[p - 1] : nullptr;
        s->next_slab_ = p + 1 < slabs.size() ? slabs[p + 1] : nullptr;
    }
}

// x, y sweeps (local), then one read of the slab for its interface values
// with zero inflow: dhat -> plane_bottom_, xhat0 -> plane_top_.
void DeviceSession::slab_phase_xy()
{
    check_ready(Axis::x);
    if (!ws_[2].active) {
        launch_sweep(Axis::x, false);
        if (ws_[1].active) launch_sweep(Axis::y, false);
        return;
    }
    launch_xy_sweeps();
    if (!has_prev() && !has_next()) return;
    const DeviceWorkspace& w = ws_[2];
    const long long plane = plane_count();
    begin_kernel(kAux);
    kernels::zslab_interface<<<sm_count_ * 8, 256, 0, static_cast<cudaStream_t>(stream_)>>>(
        rho_, plane, mesh_.nz, S_, w.q, w.dinv, w.cb, plane_bottom_, plane_top_);
    end_kernel(kAux);
}

// D_p = dhat_p + phi_last * D_{p-1} (needed only when a next slab exists).
void DeviceSession::slab_phase_fwdfix(std::int64_t off, std::int64_t count)
{
    if (!has_next()) return;
    if (!slab_philast_) throw state_error("z-slab spikes not set");
    const int block = 256;
    begin_kernel(kAux);
    kernels::zslab_fwdfix<<<static_cast<unsigned>((count + block - 1) / block), block, 0,
                            static_cast<cudaStream_t>(stream_)>>>(plane_dout_ + off, plane_bottom_ + off,
                                                                  plane_din_ + off, slab_philast_, count, S_);
    end_kernel(kAux);
}

// X_p = xhat0 + Phi_0 * D_{p-1} + Psi_0 * X_{p+1} (needed only when a previous slab exists).
void DeviceSession::slab_phase_topfix(std::int64_t off, std::int64_t count)
{
    if (!has_prev()) return;
    if (!slab_phi_) throw state_error("z-slab spikes not set");
    const int block = 256;
    begin_kernel(kAux);
    kernels::zslab_topfix<<<static_cast<unsigned>((count + block - 1) / block), block, 0,
                            static_cast<cudaStream_t>(stream_)>>>(plane_xtop_ + off, plane_top_ + off,
                                                                  plane_din_ + off, plane_xin_ + off, slab_phi_,
                                                                  slab_psi_, count, S_);
    end_kernel(kAux);
}

// The global recurrence on the slab: row 0 continues from D_{p-1}, the last
// row is back-substituted from X_{p+1}; the shell clamp is fused as usual.
void DeviceSession::slab_phase_z()
{
    if (!ws_[2].active) return;
    if (path_[2] != SweepPath::smem_ring2) throw state_error("z-slab inflows need the ring2 z-sweep");
    z_in_lo_ = has_prev() ? plane_din_ : nullptr;
    z_in_hi_ = has_next() ? plane_xin_ : nullptr;
    launch_sweep(Axis::z, true);
    z_in_lo_ = nullptr;
    z_in_hi_ = nullptr;
}

void DeviceSession::slab_phase_finish(bool with_sources, double dt)
{
    launch_residual_dirichlet(false);
    if (with_sources) launch_sources(dt);
}

// One slab per rank: the two plane chains run on this stream through the
// rank transport (NCCL, or the host callback), pipelined over plane pieces.
void DeviceSession::slab_step_nccl(bool with_sources, double dt)
{
    slab_phase_xy();
    const auto pieces = plane_pieces();
    for (const auto& [off, cnt] : pieces) { // forward chain D_0 -> D_{P-1}
        nccl_exchange(nullptr, 0, has_prev() ? plane_din_ + off : nullptr, nccl_rank_ - 1, cnt);
        slab_phase_fwdfix(off, cnt);
        nccl_exchange(has_next() ? plane_dout_ + off : nullptr, nccl_rank_ + 1, nullptr, 0, cnt);
    }
    for (const auto& [off, cnt] : pieces) { // backward chain X_{P-1} -> X_0
        nccl_exchange(nullptr, 0, has_next() ? plane_xin_ + off : nullptr, nccl_rank_ + 1, cnt);
        slab_phase_topfix(off, cnt);
        nccl_exchange(has_prev() ? plane_xtop_ + off : nullptr, nccl_rank_ - 1, nullptr, 0, cnt);
    }
    slab_phase_z();
    slab_phase_finish(with_sources, dt);
}

// In-process slabs (one or several GPUs driven by one host thread): the same
// phases, with the chains walked slab by slab and the planes moved by device
// (or peer) copies ordered by events between the slab streams.
void DeviceSession::group_advance(const std::vector<DeviceSession*>& slabs, std::int64_t steps, double dt,
                                  bool with_sources)
{
    const std::size_t P = slabs.size();
    if (steps < 0) throw std::invalid_argument("step count must be non-negative");
    if (P == 0 || steps == 0) return;
    if (!(dt > 0.0)) throw std::invalid_argument("reaction step size must be positive");
    // The checks advance() makes, for every slab.
    for (auto* s : slabs) {
        if (!s->slab_) throw state_error("group advance needs z-slab sessions");
        ck(cudaSetDevice(s->device_), "cudaSetDevice");
        s->check_ready(Axis::x);
        if (std::memcmp(&dt, &s->dt_, sizeof(double)) != 0)
            throw state_error("advance dt does not match the solver workspace dt");
    }
    // Events are released on every exit path (a failed launch throws).
    struct Events {
        std::vector<cudaEvent_t> ev;
        std::vector<int> dev;
        ~Events()
        {
            for (std::size_t p = 0; p < ev.size(); ++p)
                if (ev[p]) {
                    cudaSetDevice(dev[p]);
                    cudaEventDestroy(ev[p]);
                }
        }
    } events;
    events.ev.assign(P, nullptr);
    events.dev.assign(P, 0);
    std::vector<cudaEvent_t>& ev = events.ev;
    for (std::size_t p = 0; p < P; ++p) {
        ck(cudaSetDevice(slabs[p]->device_), "cudaSetDevice");
        events.dev[p] = slabs[p]->device_;
        ck(cudaEventCreateWithFlags(&ev[p], cudaEventDisableTiming), "cudaEventCreate");
        if (with_sources) slabs[p]->ensure_source_factors(dt);
    }
    auto stream = [&](std::size_t p) { return static_cast<cudaStream_t>(slabs[p]->stream_); };
    auto bytes = [&](std::size_t p) { return sizeof(double) * slabs[p]->plane_count(); };
    auto on = [&](std::size_t p) { ck(cudaSetDevice(slabs[p]->device_), "cudaSetDevice"); };
    auto mark = [&](std::size_t p) { ck(cudaEventRecord(ev[p], stream(p)), "cudaEventRecord"); };
    auto wait_on = [&](std::size_t p, std::size_t q) { ck(cudaStreamWaitEvent(stream(p), ev[q], 0), "wait"); };
    for (std::int64_t step = 0; step < steps; ++step) {
        for (std::size_t p = 0; p < P; ++p) {
            on(p);
            slabs[p]->slab_phase_xy();
        }
        for (std::size_t p = 0; p < P; ++p) { // forward chain D_0 -> D_{P-1}
            on(p);
            if (p > 0) {
                wait_on(p, p - 1);
                ck(cudaMemcpyPeerAsync(slabs[p]->plane_din_, slabs[p]->device_, slabs[p - 1]->plane_dout_,
                                       slabs[p - 1]->device_, bytes(p), stream(p)),
                   "copy D");
            }
            slabs[p]->slab_phase_fwdfix(0, slabs[p]->plane_count());
            mark(p);
        }
        for (std::size_t pp = P; pp-- > 0;) { // backward chain X_{P-1} -> X_0
            on(pp);
            if (pp + 1 < P) {
                wait_on(pp, pp + 1);
                ck(cudaMemcpyPeerAsync(slabs[pp]->plane_xin_, slabs[pp]->device_, slabs[pp + 1]->plane_xtop_,
                                       slabs[pp + 1]->device_, bytes(pp), stream(pp)),
                   "copy X");
            }
            slabs[pp]->slab_phase_topfix(0, slabs[pp]->plane_count());
            mark(pp);
        }
        for (std::size_t p = 0; p < P; ++p) {
            on(p);
            slabs[p]->slab_phase_z();
            slabs[p]->slab_phase_finish(with_sources, dt);
            mark(p);
        }
        for (std::size_t p = 0; p < P; ++p) { // next pre-pass overwrites planes the neighbours read
            on(p);
            for (std::size_t q : {p - 1, p + 1})
                if (q < P) wait_on(p, q);
        }
    }
    for (std::size_t p = 0; p < P; ++p) {
        on(p);
        ck(cudaStreamSynchronize(stream(p)), "sync");
    }
}

void DeviceSession::release_slab()
{
    for (double** p : {&plane_bottom_, &plane_top_, &plane_din_, &plane_dout_, &plane_xin_, &plane_xtop_, &slab_phi_,
                       &slab_psi_, &slab_philast_}) {
        if (*p) cudaFree(*p);
        *p = nullptr;
    }
    if (nccl_comm_ && nccl().CommDestroy) nccl().CommDestroy(static_cast<ncclComm_t>(nccl_comm_));
    nccl_comm_ = nullptr;
    if (host_send_) cudaFreeHost(host_send_);
    if (host_recv_) cudaFreeHost(host_recv_);
    host_send_ = host_recv_ = nullptr;
    host_xchg_ = nullptr;
    remote_ = false;
}

void DeviceSession::set_agents_range(const AgentPopulation& agents, const CartesianMesh& global_mesh,
                                     std::int64_t vox_lo, std::int64_t vox_hi)
{
    // Every agent is kept on the device (they may move between slabs); each
    // rebuild groups those whose GLOBAL voxel lies in [vox_lo, vox_hi), with
    // slab-local voxel indices, in (voxel, id) order.
    agent_filter_ = true;
    filter_lo_ = vox_lo;
    filter_hi_ = vox_hi;
    agent_mesh_ = global_mesh;
    agent_mesh_set_ = true;
    set_agents(agents);
}

} // namespace biodiff_b200
