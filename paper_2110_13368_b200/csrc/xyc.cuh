// x+y sweeps of a plane by one thread-block cluster (3-D steps).
//
// A plane's y lines need every x line of that plane — and nothing else. A
// cluster of CL CTAs x WPC warps (32 warps: one x item of L lines and one y
// item of 32 columns each, at 256^2 x 4) owns a plane at a time:
//   x phase : every warp sweeps its x item (ring2, TMA in / out);
//   cluster barrier (stores completed, release / acquire at cluster scope);
//   y phase : every warp sweeps its y item, reading the plane the x phase
//             has just written — still in L2.
// The plane's x results are overwritten by the y results before they leave
// L2, so x+y cost one HBM read and one HBM write per value instead of two
// (the lagged ticket scheme of xy2.cuh needed a window of planes too large
// for L2 because y items waited on the slowest x item of their plane; here a
// phase ends when the cluster's own 32 items end). Numerics: the same
// per-chain operations as the separate sweeps — bit-identical.
#pragma once

#include "ring2.cuh"

namespace biodiff_b200 {
namespace kernels {

struct XYCluster {
    Coef xcoef;
    StridedSweep y;  // y coefficients / geometry for make_chain_yz (axis 1)
    StridedSweep z;  // z (axis 2; 3-phase kernel only, with the Dirichlet shell clamp)
    int nx, ny, nz, S;
    int planes;      // work units: planes (nz * replicas; 2-phase) or replicas (3-phase)
    int xi, yi;      // x / y items per plane
    int rowlen;
    int warp_bytes;  // shared memory per warp (1024-aligned)
    int stagger_ns;  // cluster c starts (c % stagger_groups) * stagger_ns later (phase offset; 0 = off)
    int stagger_groups;
    unsigned* plane_ctr; // dynamic plane scheduling (zeroed before the launch), or nullptr: static P += clusters
    int reverse;         // 2-phase: visit planes from the top (unit U = plane planes-1-U)
    int keep_planes;     // 2-phase: y results of planes k < keep_planes stay in L2 (evict_normal) for the z sweep
};

__device__ __forceinline__ uint32_t cluster_ctarank()
{
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cluster_id_x()
{
    uint32_t r;
    asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t ncluster_x()
{
    uint32_t r;
    asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cluster_nctarank()
{
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}
// Reads an int from the shared memory of CTA `rank` of this cluster (DSMEM).
__device__ __forceinline__ int ld_cluster_int(const int* p, uint32_t rank)
{
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(ptx::smem_addr(p)), "r"(rank));
    int v;
    asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(v) : "r"(r) : "memory");
    return v;
}
__device__ __forceinline__ void cluster_sync()
{
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Layout of either item kind in one form (so the cluster kernel holds ONE
// copy of the ring2 chunk code): off(u) = row + t[u % P] + (u / P) * L * 16.
//   x item: LayoutX<S> (swizzled rows of 16 doubles);
//   y item: [position][lane] = lane + 32 u, i.e. row = lane, t[j] = 32 j
//           (P * 32 = 16 * L doubles per piece step).
template <int S>
struct LayoutU {
    static constexpr int L = kLanes / S;
    static constexpr int P = 16 / S;
    int row;
    int t[P];
    __device__ __forceinline__ void set_x(int l, int s)
    {
        const LayoutX<S> x(l, s);
        row = x.row;
#pragma unroll
        for (int j = 0; j < P; ++j) t[j] = x.t[j];
    }
    __device__ __forceinline__ void set_y(int lane)
    {
        row = lane;
#pragma unroll
        for (int j = 0; j < P; ++j) t[j] = 32 * j;
    }
    __device__ __forceinline__ int off(int u) const { return row + t[u % P] + (u / P) * (L * 16); }
};

// Geometry of one item. 2-phase (plane units, THREE = false): x = lines
// it*L.. of plane U, y = columns it*32.. of plane U. 3-phase (replica
// units): x item it = (plane it / xi, line block it % xi), y item = (plane
// it / yi, column block it % yi), z item = (row it / yi, column block
// it % yi) of replica U. x: plane index P and line block j; y / z: replica
// rep, outer index o (plane for y, row for z), column block eb.
struct XycGeom {
    int P, j, rep, o, eb;
};

template <bool THREE>
__device__ __forceinline__ XycGeom xyc_geom(const XYCluster& a, int kind, int U, int it)
{
    XycGeom g;
    if constexpr (THREE) {
        g.P = U * a.nz + it / a.xi;
        g.j = it % a.xi;
        g.rep = U;
        g.o = it / a.yi;
        g.eb = it % a.yi;
    } else {
        const int Pp = a.reverse ? a.planes - 1 - U : U;
        g.P = Pp;
        g.j = it;
        g.rep = Pp / a.nz;
        g.o = Pp % a.nz;
        g.eb = it;
    }
    (void)kind;
    return g;
}

// Issues chunk k of an item into `slot` (lane 0).
template <int S, bool THREE>
__device__ __forceinline__ void xyc_issue(const CUtensorMap* tmap_x, const CUtensorMap* tmap_y,
                                          const CUtensorMap* tmap_z, const Ring2Smem& sm, int kind, const XycGeom& g,
                                          int k, int slot)
{
    constexpr int kSlot = kChunk * kLanes;
    constexpr int L = kLanes / S;
    ptx::mbar_arrive_expect_tx(&sm.bars[slot], kSlot * 8);
    if (kind == 0)
        ptx::tma_load_4d(sm.slots + slot * kSlot, tmap_x, 0, g.j * L, g.P, k * 2 * S, &sm.bars[slot]);
    else if (THREE && kind == 2)
        ptx::tma_load_4d(sm.slots + slot * kSlot, tmap_z, g.eb * kLanes, g.o, k * kChunk, g.rep, &sm.bars[slot]);
    else
        ptx::tma_load_4d(sm.slots + slot * kSlot, tmap_y, g.eb * kLanes, k * kChunk, g.o, g.rep, &sm.bars[slot]);
}

// One item (kind 0 x, 1 y, 2 z). Issues its first chunks unless the
// warp's previous item prefetched them; prefetches the warp's next item
// (kind tk, unit tU, item tit >= 0: the next item of the same phase, or the
// next unit's first x item after the last phase) into the slots it frees.
// Returns whether it did.
template <int NS, int S, bool THREE>
__device__ __forceinline__ bool xyc_item(const CUtensorMap* tmap_x, const CUtensorMap* tmap_y,
                                         const CUtensorMap* tmap_z, const XYCluster& a, const Ring2Smem& sm,
                                         uint32_t& parity, int kind, int U, int it, bool prefetched, int tk, int tU,
                                         int tit)
{
    constexpr int kSlot = kChunk * kLanes;
    constexpr int L = kLanes / S;
    const int lane = threadIdx.x & 31;
    const bool is_x = kind == 0;
    auto nch_of = [&](int kd) {
        const int n = kd == 0 ? a.nx : (THREE && kd == 2 ? a.nz : a.ny);
        return (n + kChunk - 1) / kChunk;
    };
    const int nch = nch_of(kind);
    const XycGeom g = xyc_geom<THREE>(a, kind, U, it);
    if (lane == 0 && !prefetched)
        for (int k = 0; k < min(NS, nch); ++k) xyc_issue<S, THREE>(tmap_x, tmap_y, tmap_z, sm, kind, g, k, k);
    __syncwarp();
    LayoutU<S> lay;
    Chain c;
    bool active;
    if (is_x) {
        int xl, xs;
        x_lane<S>(lane, xl, xs);
        lay.set_x(xl, xs);
        Clamp none{nullptr, 0ull, 0, a.nz};
        c = make_chain(a.xcoef, S, xs, a.nx, none, false, g.rep);
        active = g.j * L + xl < a.ny;
    } else {
        lay.set_y(lane);
        const int e0 = g.eb * kLanes;
        active = lane < min(kLanes, a.rowlen - e0);
        const int e = e0 + (active ? lane : 0);
        c = make_chain_yz(THREE && kind == 2 ? a.z : a.y, e % S, e / S, g.o, g.rep);
    }
    const int tnch = tit >= 0 ? min(NS, nch_of(tk)) : 0;
    const bool pf = tit >= 0 && tnch <= min(NS, nch);
    // x (and, 3-phase, y) results are read again by the next phase: keep them
    // in L2; the last phase's results stream out.
    const uint64_t pol = (is_x || (THREE && kind == 1)) ? ptx::policy_evict_last()
                         : (!THREE && g.o < a.keep_planes) ? ptx::policy_evict_normal()
                                                           : ptx::policy_evict_first();
    solve_ring2<NS, THREE>(
        c, active, sm.bars, sm.slots, kSlot, sm.ckpt, lane, parity, [&] { return pf; }, lay,
        [&](int rel, int k, int slot, bool) {
            if (!rel)
                xyc_issue<S, THREE>(tmap_x, tmap_y, tmap_z, sm, kind, g, k, slot);
            else if (k < tnch)
                xyc_issue<S, THREE>(tmap_x, tmap_y, tmap_z, sm, tk, xyc_geom<THREE>(a, tk, tU, tit), k, slot);
        },
        [&](int k, int slot) {
            if (is_x)
                ptx::tma_store_4d_hint(tmap_x, 0, g.j * L, g.P, k * 2 * S, sm.slots + slot * kSlot, pol);
            else if (THREE && kind == 2)
                ptx::tma_store_4d_hint(tmap_z, g.eb * kLanes, g.o, k * kChunk, g.rep, sm.slots + slot * kSlot, pol);
            else
                ptx::tma_store_4d_hint(tmap_y, g.eb * kLanes, k * kChunk, g.o, g.rep, sm.slots + slot * kSlot, pol);
        },
        nullptr);
    return pf;
}

__device__ __forceinline__ unsigned long long xyc_clock()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

#ifdef BIODIFF_XYC_TRACE
// Design probe (variant builds only): per (plane, cluster warp) globaltimer
// stamps at x start, x end, after the cluster barrier, y end.
__device__ unsigned long long g_xyc_trace[4096 * 32 * 4];
__device__ __forceinline__ unsigned long long xyc_now()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define XYC_STAMP(P, gw, i)                                                                                            \
    if (lane == 0 && (P) < 4096 && (gw) < 32) g_xyc_trace[((P) * 32 + (gw)) * 4 + (i)] = xyc_now();
#else
#define XYC_STAMP(P, gw, i)
#endif

template <int NS, int S, bool THREE>
__device__ __forceinline__ void xyc_body(const CUtensorMap* tmap_x, const CUtensorMap* tmap_y,
                                         const CUtensorMap* tmap_z, const XYCluster& a, unsigned char* smem_xyc)
{
    constexpr int kSlot = kChunk * kLanes;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wpc = blockDim.x >> 5;
    const int gw = static_cast<int>(cluster_ctarank()) * wpc + warp; // warp index in the cluster
    const int nw = static_cast<int>(cluster_nctarank()) * wpc;       // warps per cluster
    const uint32_t base = ptx::smem_addr(smem_xyc);
    unsigned char* mine = smem_xyc + (((base + 1023u) & ~1023u) - base) + static_cast<size_t>(warp) * a.warp_bytes;
    ptx::griddep_wait();
    ptx::griddep_launch();
    Ring2Smem sm;
    sm.slots = reinterpret_cast<double*>(mine);
    sm.bars = reinterpret_cast<uint64_t*>(mine + NS * kSlot * 8);
    sm.ckpt = reinterpret_cast<double*>(mine + NS * kSlot * 8 + 128);
    if (lane == 0) {
        if (warp == 0) {
            ptx::tma_prefetch_desc(tmap_x);
            ptx::tma_prefetch_desc(tmap_y);
            if (THREE) ptx::tma_prefetch_desc(tmap_z);
        }
        for (int s = 0; s < NS; ++s) ptx::mbar_init(&sm.bars[s], 1);
        ptx::fence_mbar_init();
    }
    __syncwarp();
    uint32_t parity = 0;
    const int P0 = static_cast<int>(cluster_id_x()), dP = static_cast<int>(ncluster_x());
    if (a.stagger_ns > 0 && a.stagger_groups > 1 && P0 % a.stagger_groups) {
        const unsigned long long wait = static_cast<unsigned long long>(a.stagger_ns) * (P0 % a.stagger_groups);
        const unsigned long long t0 = xyc_clock();
        while (xyc_clock() - t0 < wait) __nanosleep(1000);
    }
    // Plane scheduling: the first plane is the cluster's index; with
    // a.plane_ctr the cluster's leader thread fetches the next one from a
    // global counter during the x phase and publishes it in its shared memory
    // (double-buffered by round), read by every warp after the x/y barrier —
    // clusters that started late (stagger) or ran slow take fewer planes.
    __shared__ int s_next[2];
    const bool leader = cluster_ctarank() == 0 && threadIdx.x == 0;
    bool prefetched = false;
    int round = 0;
    for (int P = P0; P < a.planes; ++round) {
        int Pn = P + dP, itn = -1;
        constexpr int nph = THREE ? 3 : 2;
        const int xitems = THREE ? a.xi * a.nz : a.xi;
        if (a.plane_ctr && leader) s_next[round & 1] = dP + static_cast<int>(atomicAdd(a.plane_ctr, 1u));
        // Phase 0: this warp's x items of plane P; phase 1: its y items (the
        // last one prefetches the next plane's first x item). One loop, one
        // copy of the chunk code.
#pragma unroll 1
        for (int ph = 0; ph < nph; ++ph) {
            if (!THREE) {
                XYC_STAMP(P, gw, ph == 0 ? 0 : 1)
            }
            if (ph >= 1) {
                // The plane's x results must be complete and visible before
                // any warp of the cluster reads them through TMA.
                if (lane == 0) {
                    ptx::bulk_wait_all();
                    ptx::fence_proxy_async_global();
                }
                __syncwarp();
                cluster_sync();
                if (lane == 0) ptx::fence_proxy_async_global();
                if (ph == 1 && a.plane_ctr) {
                    int v = 0;
                    if (lane == 0) v = ld_cluster_int(&s_next[round & 1], 0);
                    Pn = __shfl_sync(0xffffffffu, v, 0);
                }
                itn = (Pn < a.planes && gw < xitems) ? gw : -1;
                __syncwarp();
                if (!THREE) {
                    XYC_STAMP(P, gw, 2)
                }
            }
            const bool is_x = ph == 0;
            const int items = is_x ? xitems : (THREE ? a.yi * (ph == 1 ? a.nz : a.ny) : a.yi);
#pragma unroll 1
            for (int it = gw; it < items; it += nw) {
                // prefetch target: this warp's next item of the phase, else
                // (last phase) its first x item of the next unit
                int tk = ph, tU = P, tit = it + nw;
                if (tit >= items) {
                    tk = 0;
                    tU = Pn;
                    tit = ph == nph - 1 ? itn : -1;
                }
                prefetched = xyc_item<NS, S, THREE>(tmap_x, tmap_y, tmap_z, a, sm, parity, ph, P, it, prefetched, tk,
                                                    tU, tit);
            }
        }
        if (!THREE) {
            XYC_STAMP(P, gw, 3)
        }
        P = Pn;
    }
    if (lane == 0) ptx::bulk_wait_all();
    // No CTA may exit while another CTA of its cluster can still read its
    // s_next through DSMEM (compute-sanitizer racecheck, r02).
    cluster_sync();
}

template <int NS, int S>
__global__ void __launch_bounds__(256) sweep_xy_cluster(const __grid_constant__ CUtensorMap tmap_x,
                                                        const __grid_constant__ CUtensorMap tmap_y, XYCluster a)
{
    extern __shared__ __align__(1024) unsigned char smem_xyc[];
    xyc_body<NS, S, false>(&tmap_x, &tmap_y, &tmap_y, a, smem_xyc);
}

// Ensembles: one cluster advances one replica through x, y and z (three
// phases, two cluster barriers) while the replica stays in L2; the z phase
// applies the fused Dirichlet shell like the separate z sweep.
template <int NS, int S>
__global__ void __launch_bounds__(256) sweep_xyz_cluster(const __grid_constant__ CUtensorMap tmap_x,
                                                         const __grid_constant__ CUtensorMap tmap_y,
                                                         const __grid_constant__ CUtensorMap tmap_z, XYCluster a)
{
    extern __shared__ __align__(1024) unsigned char smem_xyc[];
    xyc_body<NS, S, true>(&tmap_x, &tmap_y, &tmap_z, a, smem_xyc);
}

} // namespace kernels
} // namespace biodiff_b200
