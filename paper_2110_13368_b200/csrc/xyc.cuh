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
    int nx, ny, nz, S;
    int planes;      // nz * replicas
    int xi, yi;      // x / y items per plane
    int rowlen;
    int warp_bytes;  // shared memory per warp (1024-aligned)
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
__device__ __forceinline__ void cluster_sync()
{
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// One x item (lines j0 .. j0+L-1 of plane P). The item's first min(NS, nch) chunks are issued here unless the previous
// item prefetched them (`prefetched`).
template <int NS, int S>
__device__ __forceinline__ void xyc_x_item(const CUtensorMap* tmap_x, const XYCluster& a, const Ring2Smem& sm,
                                        uint32_t& parity, int P, int it, bool prefetched)
{
    constexpr int kSlot = kChunk * kLanes;
    constexpr int L = kLanes / S;
    const int lane = threadIdx.x & 31;
    const int nchx = (a.nx + kChunk - 1) / kChunk;
    const int j0 = it * L;
    auto issue = [&](int k, int slot) {
        ptx::mbar_arrive_expect_tx(&sm.bars[slot], kSlot * 8);
        ptx::tma_load_4d(sm.slots + slot * kSlot, tmap_x, 0, j0, P, k * 2 * S, &sm.bars[slot]);
    };
    if (lane == 0 && !prefetched)
        for (int k = 0; k < min(NS, nchx); ++k) issue(k, k);
    __syncwarp();
    int xl, xs;
    x_lane<S>(lane, xl, xs);
    const LayoutX<S> lay(xl, xs);
    Clamp none{nullptr, 0ull, 0, a.nz};
    const Chain c = make_chain(a.xcoef, S, xs, a.nx, none, false, P / a.nz);
    solve_ring2<NS, false>(
        c, j0 + xl < a.ny, sm.bars, sm.slots, kSlot, sm.ckpt, lane, parity, [] { return false; }, lay,
        [&](int, int k, int slot, bool) { issue(k, slot); },
        [&](int k, int slot) {
            ptx::tma_store_4d_hint(tmap_x, 0, j0, P, k * 2 * S, sm.slots + slot * kSlot, ptx::policy_evict_last());
        },
        nullptr);
}

// One y item (columns e0 .. e0+31 of plane P). While its slots drain it
// prefetches the warp's next x item (plane Pn, item itn; itn < 0: none),
// whose data does not depend on anything still running.
template <int NS, int S>
__device__ __forceinline__ bool xyc_y_item(const CUtensorMap* tmap_y, const CUtensorMap* tmap_x, const XYCluster& a,
                                        const Ring2Smem& sm, uint32_t& parity, int P, int it, int Pn, int itn)
{
    constexpr int kSlot = kChunk * kLanes;
    constexpr int L = kLanes / S;
    const int lane = threadIdx.x & 31;
    const int nchy = (a.ny + kChunk - 1) / kChunk;
    const int nchx = (a.nx + kChunk - 1) / kChunk;
    const int rep = P / a.nz, kk = P % a.nz;
    const int e0 = it * kLanes;
    auto issue = [&](int k, int slot) {
        ptx::mbar_arrive_expect_tx(&sm.bars[slot], kSlot * 8);
        ptx::tma_load_4d(sm.slots + slot * kSlot, tmap_y, e0, k * kChunk, kk, rep, &sm.bars[slot]);
    };
    if (lane == 0)
        for (int k = 0; k < min(NS, nchy); ++k) issue(k, k);
    __syncwarp();
    const int width = min(kLanes, a.rowlen - e0);
    const bool active = lane < width;
    const int e = e0 + (active ? lane : 0);
    const Chain c = make_chain_yz(a.y, e % S, e / S, kk, rep);
    const LayoutYZ lay{lane};
    // Next x item's chunk j goes to slot j (j < min(NS, nch_y)) as the y
    // item's slots free up; only when both items have the same chunk count
    // limits (else the x item issues its own loads).
    const bool pf = itn >= 0 && min(NS, nchx) <= min(NS, nchy);
    solve_ring2<NS, false>(
        c, active, sm.bars, sm.slots, kSlot, sm.ckpt, lane, parity, [&] { return pf; }, lay,
        [&](int rel, int k, int slot, bool) {
            if (!rel) {
                issue(k, slot);
            } else if (k < min(NS, nchx)) {
                ptx::mbar_arrive_expect_tx(&sm.bars[slot], kSlot * 8);
                ptx::tma_load_4d(sm.slots + slot * kSlot, tmap_x, 0, itn * L, Pn, k * 2 * S, &sm.bars[slot]);
            }
        },
        [&](int k, int slot) {
            ptx::tma_store_4d_hint(tmap_y, e0, k * kChunk, kk, rep, sm.slots + slot * kSlot, ptx::policy_evict_first());
        },
        nullptr);
    return pf;
}

template <int NS, int S>
__global__ void __launch_bounds__(256) sweep_xy_cluster(const __grid_constant__ CUtensorMap tmap_x,
                                                        const __grid_constant__ CUtensorMap tmap_y, XYCluster a)
{
    extern __shared__ __align__(1024) unsigned char smem_xyc[];
    constexpr int kSlot = kChunk * kLanes;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wpc = blockDim.x >> 5;
    const int gw = static_cast<int>(cluster_ctarank()) * wpc + warp; // warp index in the cluster
    const int nw = static_cast<int>(cluster_nctarank()) * wpc;       // warps per cluster
    const uint32_t base = ptx::smem_addr(smem_xyc);
    unsigned char* mine = smem_xyc + (((base + 1023u) & ~1023u) - base) + static_cast<size_t>(warp) * a.warp_bytes;
    Ring2Smem sm;
    sm.slots = reinterpret_cast<double*>(mine);
    sm.bars = reinterpret_cast<uint64_t*>(mine + NS * kSlot * 8);
    sm.ckpt = reinterpret_cast<double*>(mine + NS * kSlot * 8 + 128);
    if (lane == 0) {
        if (warp == 0) {
            ptx::tma_prefetch_desc(&tmap_x);
            ptx::tma_prefetch_desc(&tmap_y);
        }
        for (int s = 0; s < NS; ++s) ptx::mbar_init(&sm.bars[s], 1);
        ptx::fence_mbar_init();
    }
    __syncwarp();
    uint32_t parity = 0;
    const int P0 = static_cast<int>(cluster_id_x()), dP = static_cast<int>(ncluster_x());
    bool prefetched = false;
    for (int P = P0; P < a.planes; P += dP) {
        // ---- x phase: this warp's x items of plane P ----------------------
        for (int it = gw; it < a.xi; it += nw) {
            xyc_x_item<NS, S>(&tmap_x, a, sm, parity, P, it, prefetched && it == gw);
            prefetched = false;
        }
        // The plane's x results must be complete and visible before any warp
        // of the cluster reads them through TMA.
        if (lane == 0) {
            ptx::bulk_wait_all();
            ptx::fence_proxy_async_global();
        }
        __syncwarp();
        cluster_sync();
        if (lane == 0) ptx::fence_proxy_async_global();
        __syncwarp();
        // ---- y phase; the last y item prefetches the next plane's first x item
        const int Pn = P + dP;
        const int itn = (Pn < a.planes && gw < a.xi) ? gw : -1;
        for (int it = gw; it < a.yi; it += nw) {
            const bool last = it + nw >= a.yi;
            prefetched = xyc_y_item<NS, S>(&tmap_y, &tmap_x, a, sm, parity, P, it, Pn, last ? itn : -1);
        }
    }
    if (lane == 0) ptx::bulk_wait_all();
}

} // namespace kernels
} // namespace biodiff_b200
