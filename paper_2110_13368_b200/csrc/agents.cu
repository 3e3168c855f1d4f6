// On-device agent grouping: the reference's
// AgentPopulation::rebuild_voxel_grouping (agents.cpp:56-73) — cache each
// agent's voxel with CartesianMesh::nearest_voxel (mesh.cpp:72-88), order the
// agents by (voxel, id), cut one group per voxel — as a device pipeline, so
// agents that move between steps (set_position, agents.cpp:45-54) are
// regrouped without a host round trip:
//
//   agent_keys     one thread per agent, in ascending-id rank order: domain
//                  check (mesh.cpp:66-70) + voxel key (replica offset for
//                  ensembles, slab-local / sentinel for z-slabs)
//   radix sort     stable by key over the id-ranked sequence => (key, id)
//                  order, exactly the reference's comparator
//   group_flags    group starts; exclusive scan -> group index
//   group_write    CSR: group voxel, offsets, group and agent counts
//   agent_gather   per-agent parameters into group order
//
// The source kernel reads the group count from device memory and is
// launched over the agent capacity, so CUDA graphs captured before a rebuild
// stay valid after it. Every set_agents goes through this pipeline.
#include "device.hpp"
#include "kernels.cuh"

#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstring>
#include <numeric>

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
void dalloc(T*& p, std::size_t count)
{
    dfree(p);
    if (count) ck(cudaMalloc(&p, sizeof(T) * count), "cudaMalloc agents");
}

struct AgentMesh {
    double lo[3], hi[3], h[3];
    int n[3];
    long long nvox;     // voxels of one replica of the (global) mesh
    long long vox_lo;   // slab filter: keep voxels in [vox_lo, vox_hi), key = voxel - vox_lo
    long long vox_hi;
    long long key_span; // keys per replica (vox_hi - vox_lo)
    long long sentinel; // key of a filtered-out agent (sorts last)
};

// mesh.cpp:78-86: floor((v - lo) / h) clamped to [0, n - 1].
__device__ __forceinline__ int cell_of(double v, double lo, double h, int n)
{
    const int i = static_cast<int>(floor(__ddiv_rn(__dsub_rn(v, lo), h)));
    return min(max(i, 0), n - 1);
}

__global__ void agent_keys(const double* pos, const int* rep, long long N, AgentMesh m, const int64_t* id_order,
                           int64_t* keys, unsigned long long* bad)
{
    const long long r = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= N) return;
    const long long a = id_order[r];
    const double p0 = pos[3 * a], p1 = pos[3 * a + 1], p2 = pos[3 * a + 2];
    // mesh.cpp:66-70 (NaN fails every comparison, as on the host).
    const bool inside = p0 >= m.lo[0] && p0 <= m.hi[0] && p1 >= m.lo[1] && p1 <= m.hi[1] && p2 >= m.lo[2] &&
                        p2 <= m.hi[2];
    if (!inside) {
        atomicMin(bad, static_cast<unsigned long long>(a));
        keys[r] = m.sentinel;
        return;
    }
    const int i = cell_of(p0, m.lo[0], m.h[0], m.n[0]);
    const int j = cell_of(p1, m.lo[1], m.h[1], m.n[1]);
    const int k = cell_of(p2, m.lo[2], m.h[2], m.n[2]);
    const long long v = static_cast<long long>(i) + static_cast<long long>(m.n[0]) * (j + static_cast<long long>(m.n[1]) * k);
    if (v < m.vox_lo || v >= m.vox_hi) {
        keys[r] = m.sentinel;
        return;
    }
    keys[r] = (v - m.vox_lo) + static_cast<long long>(rep ? rep[a] : 0) * m.key_span;
}

__global__ void group_flags(const int64_t* keys, long long N, long long sentinel, int* flags)
{
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= N) return;
    flags[i] = keys[i] != sentinel && (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

// The live grouping arrays are written only when no agent lies outside the
// domain (bad == ~0): a failed rebuild leaves them as they were, without a
// host round trip between the key pass and the writes.
__global__ void group_reset(const unsigned long long* bad, int64_t* counts, int64_t* group_offsets)
{
    if (*bad != ~0ull) return;
    counts[0] = 0;
    counts[1] = 0;
    group_offsets[0] = 0;
}

// counts[0] = groups, counts[1] = grouped agents (keys before the first sentinel).
__global__ void group_write(const int64_t* keys, const int* flags, const int64_t* gidx, long long N,
                            long long sentinel, int64_t* group_voxel, int64_t* group_offsets, int64_t* counts,
                            const unsigned long long* bad)
{
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= N || *bad != ~0ull) return;
    if (flags[i]) {
        group_voxel[gidx[i]] = keys[i];
        group_offsets[gidx[i]] = i;
    }
    const bool valid = keys[i] != sentinel;
    const bool last_valid = valid && (i == N - 1 || keys[i + 1] == sentinel);
    if (last_valid) {
        const long long G = gidx[i] + flags[i];
        counts[0] = G;
        counts[1] = i + 1;
        group_offsets[G] = i + 1;
    }
}

// Per-agent source factors of one (agent, substrate) for step dt — the
// expressions of sources_factors (kernels.cuh), computed in the gather so a
// regrouping leaves them ready (fac.add == nullptr: not computed here).
struct FactorOut {
    double* add;
    double* den;
    double dt;
    double inv_voxel_volume;
};
__device__ __forceinline__ void gather_factors(const FactorOut& fo, long long t, double volume, double sec, double upt,
                                               double sat)
{
    const double f = __dmul_rn(__dmul_rn(fo.dt, volume), fo.inv_voxel_volume);
    fo.add[t] = __dmul_rn(__dmul_rn(f, sec), sat);
    fo.den[t] = __dadd_rn(1.0, __dmul_rn(f, __dadd_rn(sec, upt)));
}

__global__ void agent_gather(const int64_t* order, long long N, int S, const double* vol, const double* sec,
                             const double* upt, const double* sat, double* vol_g, double* sec_g, double* upt_g,
                             double* sat_g, const unsigned long long* bad, int64_t* rank, FactorOut fo)
{
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= N * S || *bad != ~0ull) return;
    const long long i = t / S;
    const int s = static_cast<int>(t % S);
    const long long a = order[i];
    const double v = vol[a];
    if (s == 0) {
        vol_g[i] = v;
        rank[a] = i; // inverse of the (voxel, id) order: agent -> sorted position
    }
    const double se = sec[a * S + s], up = upt[a * S + s], sa = sat[a * S + s];
    sec_g[t] = se;
    upt_g[t] = up;
    sat_g[t] = sa;
    if (fo.add) gather_factors(fo, t, v, se, up, sa);
}

// rep_groups[r] = first group of replica r (groups are sorted by key, keys of
// replica r start at r * key_span); rep_groups[R] = G.
__global__ void rep_group_bounds(const int64_t* group_voxel, const int64_t* counts, long long key_span, int R,
                                 int64_t* rep_groups, const unsigned long long* bad, long long* host_out)
{
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r == 0 && host_out) { // [bad, groups, grouped agents] straight to the page-locked host buffer
        host_out[0] = static_cast<long long>(*bad);
        host_out[1] = counts[0];
        host_out[2] = counts[1];
    }
    if (r > R || *bad != ~0ull) return;
    const long long G = counts[0];
    const long long key = static_cast<long long>(r) * key_span;
    long long lo = 0, hi = G;
    while (lo < hi) {
        const long long mid = (lo + hi) / 2;
        if (group_voxel[mid] < key)
            lo = mid + 1;
        else
            hi = mid;
    }
    rep_groups[r] = r == R ? G : lo;
}

// Grid-stride copy of `count` doubles from a device-mapped host buffer
// (16-byte aligned), 16 bytes per load.
__global__ void copy_from_mapped(const double* __restrict__ src, double* __restrict__ dst, long long count)
{
    const long long pairs = count / 2;
    const double2* s2 = reinterpret_cast<const double2*>(src);
    double2* d2 = reinterpret_cast<double2*>(dst);
    for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < pairs;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        d2[i] = s2[i];
    if (count % 2 && blockIdx.x == 0 && threadIdx.x == 0) dst[count - 1] = src[count - 1];
}

// The densities each agent senses (its cached voxel's values, the
// reference's field.values[agent.voxel * S + s]), in agent-index order:
// thread (a, s) looks up a's sorted position, so the output is written
// contiguously (into a device buffer, or straight into a mapped host
// buffer). Agents outside this session's voxels (other z-slabs) read NaN.
__global__ void agent_sample(const int64_t* keys_sorted, const int64_t* rank, const int64_t* counts, long long N,
                             int S, const double* rho, double* out)
{
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= N * S) return;
    const long long i = rank[t / S];
    const int s = static_cast<int>(t % S);
    out[t] = i < counts[1] ? rho[keys_sorted[i] * S + s] : __longlong_as_double(-1LL);
}

// Small populations (one replica, no slab filter, N <= kSmallRegroup): the
// whole pipeline above in ONE CTA — keys (same domain check and voxel rule),
// a bitonic sort of (key << 32 | id rank) in shared memory (= the stable
// radix sort's (key, id) order), group flags, a block scan, the CSR, the
// gather — so a regroup costs one launch and one read-back instead of ~12
// launches and two. An agent outside the domain leaves every live array
// untouched (the reference's failed rebuild keeps the old grouping).
constexpr long long kSmallRegroup = 2048; // measured: C1 (1000 agents) 65.6 -> 44.7 us per regroup; at 10k agents the one-CTA sort loses to CUB (304 us)

__global__ void __launch_bounds__(1024) regroup_small(const double* pos, long long N, AgentMesh m,
                                                      const int64_t* id_order, int S, const double* vol,
                                                      const double* sec, const double* upt, const double* sat,
                                                      int64_t* keys_sorted, int64_t* order, int64_t* group_voxel,
                                                      int64_t* group_offsets, int64_t* counts, int64_t* rep_groups,
                                                      double* vol_g, double* sec_g, double* upt_g, double* sat_g,
                                                      unsigned long long* bad, long long* host_out, int64_t* rank,
                                                      FactorOut fo)
{
    // host_out (page-locked, device-mapped, or nullptr): [bad, groups,
    // grouped agents] written straight to the host — no read-back copies.
    extern __shared__ unsigned long long sk[]; // [P] packed keys, then [1024] scan partials
    __shared__ unsigned long long s_bad;
    const int tid = threadIdx.x, nt = blockDim.x;
    long long P = 1;
    while (P < N) P <<= 1;
    unsigned long long* part = sk + P;
    if (tid == 0) s_bad = ~0ull;
    __syncthreads();
    for (long long r = tid; r < P; r += nt) {
        if (r >= N) {
            sk[r] = ~0ull;
            continue;
        }
        const long long a = id_order[r];
        const double p0 = pos[3 * a], p1 = pos[3 * a + 1], p2 = pos[3 * a + 2];
        const bool inside = p0 >= m.lo[0] && p0 <= m.hi[0] && p1 >= m.lo[1] && p1 <= m.hi[1] && p2 >= m.lo[2] &&
                            p2 <= m.hi[2];
        if (!inside) {
            atomicMin(&s_bad, static_cast<unsigned long long>(a));
            sk[r] = ~0ull;
            continue;
        }
        const int i = cell_of(p0, m.lo[0], m.h[0], m.n[0]);
        const int j = cell_of(p1, m.lo[1], m.h[1], m.n[1]);
        const int k = cell_of(p2, m.lo[2], m.h[2], m.n[2]);
        const unsigned long long v = static_cast<unsigned long long>(i) +
                                     static_cast<unsigned long long>(m.n[0]) * (j + static_cast<unsigned long long>(m.n[1]) * k);
        sk[r] = (v << 32) | static_cast<unsigned long long>(r);
    }
    __syncthreads();
    if (s_bad != ~0ull) {
        if (tid == 0) {
            *bad = s_bad;
            if (host_out) host_out[0] = static_cast<long long>(s_bad);
        }
        return;
    }
    for (long long size = 2; size <= P; size <<= 1) // bitonic sort, ascending
        for (long long stride = size >> 1; stride > 0; stride >>= 1) {
            for (long long t = tid; t < P / 2; t += nt) {
                const long long lo = 2 * t - (t & (stride - 1));
                const long long hi = lo + stride;
                const bool up = (lo & size) == 0;
                const unsigned long long x = sk[lo], y = sk[hi];
                if ((x > y) == up) {
                    sk[lo] = y;
                    sk[hi] = x;
                }
            }
            __syncthreads();
        }
    // group flags + exclusive scan (each thread a contiguous run of `per` entries)
    const long long per = (N + nt - 1) / nt, b = tid * per, e = min(N, b + per);
    unsigned long long run = 0;
    for (long long i = b; i < e; ++i) run += (i == 0 || (sk[i] >> 32) != (sk[i - 1] >> 32)) ? 1 : 0;
    part[tid] = run;
    __syncthreads();
    for (int d = 1; d < nt; d <<= 1) {
        const unsigned long long add = tid >= d ? part[tid - d] : 0;
        __syncthreads();
        part[tid] += add;
        __syncthreads();
    }
    long long g = static_cast<long long>(part[tid] - run);
    for (long long i = b; i < e; ++i) {
        const long long key = static_cast<long long>(sk[i] >> 32);
        const long long a = id_order[sk[i] & 0xffffffffull];
        keys_sorted[i] = key;
        order[i] = a;
        rank[a] = i;
        if (i == 0 || key != static_cast<long long>(sk[i - 1] >> 32)) {
            group_voxel[g] = key;
            group_offsets[g] = i;
            ++g;
        }
        if (S > 0) {
            const double v = vol[a];
            vol_g[i] = v;
            for (int s = 0; s < S; ++s) {
                const double se = sec[a * S + s], up = upt[a * S + s], sa = sat[a * S + s];
                sec_g[i * S + s] = se;
                upt_g[i * S + s] = up;
                sat_g[i * S + s] = sa;
                if (fo.add) gather_factors(fo, i * S + s, v, se, up, sa);
            }
        }
    }
    if (tid == nt - 1) {
        const long long G = static_cast<long long>(part[nt - 1]);
        group_offsets[G] = N;
        counts[0] = G;
        counts[1] = N;
        rep_groups[0] = 0;
        rep_groups[1] = G;
        *bad = ~0ull;
        if (host_out) {
            host_out[0] = -1; // ~0: no agent outside
            host_out[1] = G;
            host_out[2] = N;
        }
    }
}

int bits_for(long long v)
{
    int b = 1;
    while (b < 63 && (1LL << b) <= v) ++b;
    return b;
}

unsigned blocks(long long n, int block) { return static_cast<unsigned>(std::max(1LL, (n + block - 1) / block)); }

} // namespace

void DeviceSession::release_agents()
{
    for (auto** p : {&in_ids_, &id_order_, &keys_a_, &keys_b_, &vals_b_, &keys_c_, &vals_c_, &agent_rank_, &scan_, &group_voxel_, &group_offsets_,
                     &agent_counts_, &rep_groups_})
        dfree(*p);
    for (auto** p : {&in_pos_, &in_vol_, &in_sec_, &in_upt_, &in_sat_, &agent_volume_, &agent_secretion_,
                     &agent_uptake_, &agent_saturation_, &agent_add_, &agent_den_, &agent_sample_})
        dfree(*p);
    dfree(in_rep_);
    dfree(flags_);
    dfree(agent_bad_);
    if (cub_tmp_) cudaFree(cub_tmp_);
    cub_tmp_ = nullptr;
    cub_bytes_ = 0;
    n_agents_ = 0;
    groups_ = 0;
    grouped_agents_ = 0;
    res_grp_valid_ = false;
    destroy_regroup_graphs();
    sort_parity_ = 0; // the sort buffers are freed with the population
    id_index_.clear();
    rep_agents_.clear();
}

// Ensembles: population r lives in replica r (keys offset by r * voxels).
// Input order = the populations' agents concatenated (replica-major).
void DeviceSession::set_agents_multi(const std::vector<const AgentPopulation*>& pops)
{
    ck(cudaSetDevice(device_), "cudaSetDevice");
    auto st = static_cast<cudaStream_t>(stream_);
    ck(cudaStreamSynchronize(st), "sync");
    if (static_cast<int>(pops.size()) > replicas_) throw state_error("more agent populations than replicas");
    const int S = S_;
    std::vector<std::int64_t> ids;
    std::vector<double> pos, vol, sec, upt, sat;
    std::vector<int> rep;
    for (std::size_t r = 0; r < pops.size(); ++r)
        for (const CellAgent& a : pops[r]->agents()) {
            if (a.secretion_rates.size() != static_cast<std::size_t>(S) ||
                a.uptake_rates.size() != static_cast<std::size_t>(S) ||
                a.saturation_densities.size() != static_cast<std::size_t>(S))
                throw state_error("agent rate vectors do not match the substrate count");
            ids.push_back(a.id);
            pos.insert(pos.end(), a.position.begin(), a.position.end());
            vol.push_back(a.volume);
            sec.insert(sec.end(), a.secretion_rates.begin(), a.secretion_rates.end());
            upt.insert(upt.end(), a.uptake_rates.begin(), a.uptake_rates.end());
            sat.insert(sat.end(), a.saturation_densities.begin(), a.saturation_densities.end());
            rep.push_back(static_cast<int>(r));
        }
    const std::int64_t N = static_cast<std::int64_t>(ids.size());
    std::vector<std::int64_t> per_rep(replicas_, 0);
    for (int r : rep) ++per_rep[r];
    // Ascending-id rank order (the tie-break of the (voxel, id) sort).
    std::vector<std::int64_t> order(N);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](std::int64_t l, std::int64_t r) { return ids[l] < ids[r]; });

    invalidate_graphs(); // buffers are reallocated below
    release_agents();
    factors_valid_ = false;
    n_agents_ = N;
    rep_agents_ = per_rep;
    if (replicas_ == 1)
        for (std::int64_t a = 0; a < N; ++a) id_index_[ids[a]] = a;
    if (N == 0) return;
    auto up = [&](auto*& d, const auto& h) {
        dalloc(d, h.size());
        ck(cudaMemcpyAsync(d, h.data(), sizeof(h[0]) * h.size(), cudaMemcpyHostToDevice, st), "upload agents");
    };
    up(in_ids_, ids);
    up(in_pos_, pos);
    up(in_vol_, vol);
    up(in_sec_, sec);
    up(in_upt_, upt);
    up(in_sat_, sat);
    if (replicas_ > 1) up(in_rep_, rep);
    up(id_order_, order);
    dalloc(keys_a_, N);
    dalloc(keys_b_, N);
    dalloc(vals_b_, N);
    dalloc(keys_c_, N);
    dalloc(vals_c_, N);
    dalloc(agent_rank_, N);
    dalloc(flags_, N);
    dalloc(scan_, N);
    dalloc(group_voxel_, N);
    dalloc(group_offsets_, N + 1);
    dalloc(agent_counts_, 2);
    dalloc(rep_groups_, replicas_ + 1);
    dalloc(agent_bad_, 1);
    dalloc(agent_volume_, N);
    dalloc(agent_secretion_, N * S);
    dalloc(agent_uptake_, N * S);
    dalloc(agent_saturation_, N * S);
    dalloc(agent_add_, N * S);
    dalloc(agent_den_, N * S);
    // CUB scratch for the sort and the scan (sized once per population).
    std::size_t sort_bytes = 0, scan_bytes = 0;
    ck(cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, keys_a_, keys_b_, id_order_, vals_b_, N, 0, 63, st),
       "cub sort size");
    ck(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, flags_, scan_, N, st), "cub scan size");
    cub_bytes_ = std::max(sort_bytes, scan_bytes);
    ck(cudaMalloc(&cub_tmp_, cub_bytes_), "cudaMalloc cub");
    rebuild_voxel_grouping();
}

// After a successful rebuild: the factors the gather wrote (for dt_) are
// current; else they must be recomputed before the next sources step.
void DeviceSession::mark_factors(bool computed)
{
    factors_valid_ = computed;
    if (computed) std::memcpy(&factors_dt_bits_, &dt_, sizeof(factors_dt_bits_));
}

void DeviceSession::destroy_regroup_graphs()
{
    for (auto& g : regroup_graphs_) {
        if (g.exec) cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(g.exec));
        g = RegroupGraph{};
    }
}

void DeviceSession::rebuild_voxel_grouping()
{
    ck(cudaSetDevice(device_), "cudaSetDevice");
    const std::int64_t N = n_agents_;
    if (N == 0) return;
    auto st = static_cast<cudaStream_t>(stream_);
    const CartesianMesh& gm = agent_mesh_set_ ? agent_mesh_ : mesh_;
    AgentMesh m{};
    m.lo[0] = gm.x_min;
    m.lo[1] = gm.y_min;
    m.lo[2] = gm.z_min;
    m.hi[0] = gm.x_max;
    m.hi[1] = gm.y_max;
    m.hi[2] = gm.z_max;
    m.h[0] = gm.dx;
    m.h[1] = gm.dy;
    m.h[2] = gm.dz;
    m.n[0] = gm.nx;
    m.n[1] = gm.ny;
    m.n[2] = gm.nz;
    m.nvox = gm.voxel_count();
    m.vox_lo = agent_filter_ ? filter_lo_ : 0;
    m.vox_hi = agent_filter_ ? filter_hi_ : m.nvox;
    m.key_span = m.vox_hi - m.vox_lo;
    m.sentinel = m.key_span * replicas_;
    const int end_bit = bits_for(m.sentinel);
    if (!host_pin_) ck(cudaMallocHost(&host_pin_, 64), "cudaMallocHost"); // pinned: the two read-backs below
    // The read-back buffer is device-mapped (UVA): the last kernel of the
    // pipeline writes it directly, no copies.
    long long* pin_dev = nullptr;
    if (cudaHostGetDevicePointer(reinterpret_cast<void**>(&pin_dev), host_pin_, 0) != cudaSuccess) {
        cudaGetLastError();
        pin_dev = nullptr;
    }
    // The source factors for the session's dt come out of the gather (the
    // step would otherwise recompute them after every regrouping).
    const bool with_factors = dt_ > 0.0;
    const FactorOut fo{with_factors ? agent_add_ : nullptr, agent_den_, dt_, 1.0 / mesh_.voxel_volume()};
    if (replicas_ == 1 && !agent_filter_ && N <= kSmallRegroup && m.nvox < (1LL << 31) &&
        std::getenv("BIODIFF_REGROUP_CUB") == nullptr) { // one launch, one read-back
        long long P = 1;
        while (P < N) P <<= 1;
        const int smem = static_cast<int>((P + 1024) * sizeof(unsigned long long));
        ck(cudaFuncSetAttribute(regroup_small, cudaFuncAttributeMaxDynamicSharedMemorySize, smem), "smem attr");
        begin_kernel(kAux);
        regroup_small<<<1, 1024, smem, st>>>(in_pos_, N, m, id_order_, S_, in_vol_, in_sec_, in_upt_, in_sat_,
                                             keys_b_, vals_b_, group_voxel_, group_offsets_, agent_counts_,
                                             rep_groups_, agent_volume_, agent_secretion_, agent_uptake_,
                                             agent_saturation_, agent_bad_, pin_dev, agent_rank_, fo);
        end_kernel(kAux);
        auto* pin = static_cast<long long*>(host_pin_);
        if (!pin_dev) {
            ck(cudaMemcpyAsync(pin, agent_bad_, sizeof(long long), cudaMemcpyDeviceToHost, st), "download");
            ck(cudaMemcpyAsync(pin + 1, agent_counts_, 2 * sizeof(long long), cudaMemcpyDeviceToHost, st), "download");
        }
        ck(cudaStreamSynchronize(st), "sync");
        const unsigned long long bad = static_cast<unsigned long long>(pin[0]);
        if (bad != ~0ull) {
            double p[3];
            ck(cudaMemcpy(p, in_pos_ + 3 * bad, sizeof(p), cudaMemcpyDeviceToHost), "download");
            throw std::domain_error("position (" + format_double(p[0]) + "," + format_double(p[1]) + "," +
                                    format_double(p[2]) + ") outside the simulation domain");
        }
        mark_factors(with_factors);
        res_grp_valid_ = false;
        groups_ = pin[1];
        grouped_agents_ = pin[2];
        return;
    }
    auto* pin = static_cast<long long*>(host_pin_);
    auto issue = [&] {
        ck(cudaMemsetAsync(agent_bad_, 0xff, sizeof(unsigned long long), st), "reset"); // ~0: no agent outside
        const int block = 256;
        begin_kernel(kAux);
        agent_keys<<<blocks(N, block), block, 0, st>>>(in_pos_, in_rep_, N, m, id_order_, keys_a_, agent_bad_);
        end_kernel(kAux);
        // The sort goes to the spare (keys, order) pair and every write of a live
        // array is conditional on the domain check (group_reset / group_write /
        // agent_gather / rep_group_bounds skip when an agent is outside), so the
        // pipeline runs with ONE read-back at its end; a failed rebuild keeps the
        // previous grouping, as the reference does (its nearest_voxel throws
        // before groups_ is reassigned, agents.cpp:56-73).
        std::size_t bytes = cub_bytes_;
        ck(cub::DeviceRadixSort::SortPairs(cub_tmp_, bytes, keys_a_, keys_c_, id_order_, vals_c_, N, 0, end_bit, st),
           "cub sort");
        begin_kernel(kAux);
        group_flags<<<blocks(N, block), block, 0, st>>>(keys_c_, N, m.sentinel, flags_);
        end_kernel(kAux);
        bytes = cub_bytes_;
        ck(cub::DeviceScan::ExclusiveSum(cub_tmp_, bytes, flags_, scan_, N, st), "cub scan");
        begin_kernel(kAux);
        group_reset<<<1, 1, 0, st>>>(agent_bad_, agent_counts_, group_offsets_);
        end_kernel(kAux);
        begin_kernel(kAux);
        group_write<<<blocks(N, block), block, 0, st>>>(keys_c_, flags_, scan_, N, m.sentinel, group_voxel_,
                                                        group_offsets_, agent_counts_, agent_bad_);
        end_kernel(kAux);
        begin_kernel(kAux);
        agent_gather<<<blocks(N * S_, block), block, 0, st>>>(vals_c_, N, S_, in_vol_, in_sec_, in_upt_, in_sat_,
                                                              agent_volume_, agent_secretion_, agent_uptake_,
                                                              agent_saturation_, agent_bad_, agent_rank_, fo);
        end_kernel(kAux);
        begin_kernel(kAux);
        rep_group_bounds<<<blocks(replicas_ + 1, block), block, 0, st>>>(group_voxel_, agent_counts_, m.key_span,
                                                                          replicas_, rep_groups_, agent_bad_, pin_dev);
        end_kernel(kAux);
        if (!pin_dev) {
            ck(cudaMemcpyAsync(pin, agent_bad_, sizeof(long long), cudaMemcpyDeviceToHost, st), "download");
            ck(cudaMemcpyAsync(pin + 1, agent_counts_, 2 * sizeof(long long), cudaMemcpyDeviceToHost, st), "download");
        }
    };
    // The pipeline is static for a population (sizes, buffers, mesh): it is
    // captured once per sort-output buffer and replayed (one launch instead
    // of ~12); kernel timing runs it eagerly.
    const char* rg = std::getenv("BIODIFF_REGROUP_GRAPH");
    if (!timing_ && (rg == nullptr || std::atoi(rg) != 0)) {
        RegroupGraph& g = regroup_graphs_[sort_parity_];
        if (!g.exec || g.n != N || g.end_bit != end_bit || g.keys != keys_c_) {
            if (g.exec) cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(g.exec));
            g.exec = nullptr;
            const std::int64_t before = launches_;
            cudaGraph_t graph;
            ck(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal), "begin capture");
            issue();
            ck(cudaStreamEndCapture(st, &graph), "end capture");
            cudaGraphExec_t exec;
            ck(cudaGraphInstantiate(&exec, graph, 0), "graph instantiate");
            cudaGraphDestroy(graph);
            g = RegroupGraph{exec, N, end_bit, keys_c_, static_cast<int>(launches_ - before)};
            launches_ = before;
        }
        ck(cudaGraphLaunch(static_cast<cudaGraphExec_t>(g.exec), st), "graph launch");
        launches_ += g.kernels;
    } else {
        issue();
    }
    ck(cudaStreamSynchronize(st), "sync");
    const unsigned long long bad = static_cast<unsigned long long>(pin[0]);
    if (bad != ~0ull) {
        // mesh.cpp:74-76 (nearest_voxel's std::domain_error, same message).
        double p[3];
        ck(cudaMemcpy(p, in_pos_ + 3 * bad, sizeof(p), cudaMemcpyDeviceToHost), "download");
        throw std::domain_error("position (" + format_double(p[0]) + "," + format_double(p[1]) + "," +
                                format_double(p[2]) + ") outside the simulation domain");
    }
    std::swap(keys_b_, keys_c_);
    sort_parity_ ^= 1;
    std::swap(vals_b_, vals_c_);
    mark_factors(with_factors);
    res_grp_valid_ = false;
    groups_ = pin[1];
    grouped_agents_ = pin[2];
}

void DeviceSession::sample_agent_densities(double* out, std::int64_t count)
{
    if (count != n_agents_ * S_) throw std::invalid_argument("sample buffer size does not match agents x substrates");
    if (count == 0) return;
    ck(cudaSetDevice(device_), "cudaSetDevice");
    auto st = static_cast<cudaStream_t>(stream_);
    // A page-locked, device-mapped caller buffer is written by the kernel
    // directly (contiguous 8-byte stores over PCIe); any other buffer gets a
    // device buffer and one copy.
    cudaPointerAttributes attr{};
    const bool mapped = zc_positions_ && cudaPointerGetAttributes(&attr, out) == cudaSuccess &&
                        attr.type == cudaMemoryTypeHost && attr.devicePointer != nullptr;
    cudaGetLastError();
    if (!mapped && !agent_sample_) dalloc(agent_sample_, count);
    double* dst = mapped ? static_cast<double*>(attr.devicePointer) : agent_sample_;
    const int block = 256;
    begin_kernel(kAux);
    agent_sample<<<blocks(count, block), block, 0, st>>>(keys_b_, agent_rank_, agent_counts_, n_agents_, S_, rho_,
                                                         dst);
    end_kernel(kAux);
    if (!mapped)
        ck(cudaMemcpyAsync(out, agent_sample_, sizeof(double) * count, cudaMemcpyDeviceToHost, st), "download");
    ck(cudaStreamSynchronize(st), "sync");
}

void DeviceSession::set_agent_positions(const double* xyz, std::int64_t n)
{
    if (n != n_agents_) throw std::invalid_argument("position count does not match the agent count");
    if (n == 0) return;
    ck(cudaSetDevice(device_), "cudaSetDevice");
    auto st = static_cast<cudaStream_t>(stream_);
    // Page-locked, device-mapped caller buffers (cudaHostAlloc / pin_memory)
    // are read by a copy kernel (zero-copy loads over PCIe) instead of a DMA
    // copy: BIODIFF_ZC_POSITIONS=0 forces the DMA path.
    cudaPointerAttributes attr{};
    const bool mapped = zc_positions_ && cudaPointerGetAttributes(&attr, xyz) == cudaSuccess &&
                        attr.type == cudaMemoryTypeHost && attr.devicePointer != nullptr &&
                        reinterpret_cast<std::uintptr_t>(attr.devicePointer) % 16 == 0;
    cudaGetLastError();
    if (mapped) {
        const long long pairs = (3 * n + 1) / 2;
        begin_kernel(kAux);
        copy_from_mapped<<<static_cast<unsigned>(std::min<long long>((pairs + 255) / 256, 4LL * sm_count_)), 256, 0,
                           st>>>(static_cast<const double*>(attr.devicePointer), in_pos_, 3 * n);
        end_kernel(kAux);
    } else {
        ck(cudaMemcpyAsync(in_pos_, xyz, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, st), "upload positions");
    }
    ck(cudaStreamSynchronize(st), "sync");
}

// AgentPopulation::set_position (agents.cpp:45-54): the id must exist.
void DeviceSession::set_agent_position(std::int64_t id, const double* xyz)
{
    if (replicas_ > 1) throw state_error("set_position by id needs a single-replica session (ids repeat across replicas)");
    auto it = id_index_.find(id);
    if (it == id_index_.end()) throw std::invalid_argument("no agent with id " + std::to_string(id));
    ck(cudaSetDevice(device_), "cudaSetDevice");
    auto st = static_cast<cudaStream_t>(stream_);
    ck(cudaMemcpyAsync(in_pos_ + 3 * it->second, xyz, 3 * sizeof(double), cudaMemcpyHostToDevice, st), "upload");
    ck(cudaStreamSynchronize(st), "sync");
}

std::int64_t DeviceSession::download_grouping(std::int64_t* group_voxel, std::int64_t* group_offsets,
                                              std::int64_t* order)
{
    ck(cudaSetDevice(device_), "cudaSetDevice");
    synchronize();
    if (groups_ == 0) {
        if (group_offsets) group_offsets[0] = 0;
        return 0;
    }
    if (group_voxel)
        ck(cudaMemcpy(group_voxel, group_voxel_, sizeof(long long) * groups_, cudaMemcpyDeviceToHost), "download");
    if (group_offsets)
        ck(cudaMemcpy(group_offsets, group_offsets_, sizeof(long long) * (groups_ + 1), cudaMemcpyDeviceToHost),
           "download");
    if (order)
        ck(cudaMemcpy(order, vals_b_, sizeof(long long) * grouped_agents_, cudaMemcpyDeviceToHost), "download");
    return groups_;
}

void DeviceSession::download_agents(std::int64_t* ids, double* pos, double* vol, double* sec, double* upt,
                                    double* sat)
{
    ck(cudaSetDevice(device_), "cudaSetDevice");
    synchronize();
    const std::size_t N = static_cast<std::size_t>(n_agents_), S = static_cast<std::size_t>(S_);
    if (N == 0) return;
    auto down = [&](void* h, const void* d, std::size_t bytes) {
        if (h) ck(cudaMemcpy(h, d, bytes, cudaMemcpyDeviceToHost), "download agents");
    };
    down(ids, in_ids_, 8 * N);
    down(pos, in_pos_, 24 * N);
    down(vol, in_vol_, 8 * N);
    down(sec, in_sec_, 8 * N * S);
    down(upt, in_upt_, 8 * N * S);
    down(sat, in_sat_, 8 * N * S);
}

} // namespace biodiff_b200
