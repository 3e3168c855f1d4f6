// Fused x+y sweeps through L2 on the ring2 machinery (default 3-D path).
//
// Same scheme as xy.cuh (lagged ticket order X(0..D-1), X(D) Y(0), ...,
// per-plane release/acquire counters, bit-identical to separate sweeps), with
// the item-boundary costs that made the first version slower than two
// separate sweeps removed:
//   * the next ticket is taken when an item starts (its latency hides behind
//     the item's forward pass) and its first chunks are prefetched into the
//     slots the back substitution frees, exactly like the persistent tile
//     kernels — for a Y item only if its plane is already published
//     (non-blocking check);
//   * an X item's plane is published after the first forward chunk of the
//     warp's next item, by which time its bulk stores have long completed,
//     instead of blocking on them at the item boundary.
// Deadlock freedom: a warp only ever blocks on a plane counter at the start
// of a Y item, after publishing whatever it still owed; every item it waits
// for holds a smaller ticket and belongs to a running warp.
#pragma once

#include "ring2.cuh"

namespace biodiff_b200 {
namespace kernels {

struct XYFused2 {
    Coef xcoef, ycoef;
    int nx, ny, nz, S;
    int planes;      // NP = nz * replicas
    int xi, yi;      // items per plane
    int lag;         // D (1 <= D <= NP)
    int rowlen;
    unsigned* ctr;   // [0] ticket, [1 + P] finished x items of plane P (zeroed before each launch)
    StridedSweep y;  // for make_chain_yz (axis 1)
};

struct XYItem {
    int kind; // 0 = X, 1 = Y, -1 = none
    int P, it;
};

__device__ __forceinline__ XYItem xy2_decode(const XYFused2& a, unsigned T)
{
    XYItem r;
    const unsigned xi = a.xi, yi = a.yi, D = a.lag, NP = a.planes;
    if (T >= NP * (xi + yi)) {
        r.kind = -1;
        r.P = r.it = 0;
        return r;
    }
    const unsigned A = D * xi;
    if (T < A) {
        r.kind = 0;
        r.P = T / xi;
        r.it = T % xi;
        return r;
    }
    T -= A;
    const unsigned B = (NP - D) * (xi + yi);
    if (T < B) {
        const unsigned b = T / (xi + yi), q = T % (xi + yi);
        if (q < xi) {
            r.kind = 0;
            r.P = D + b;
            r.it = q;
        } else {
            r.kind = 1;
            r.P = b;
            r.it = q - xi;
        }
        return r;
    }
    T -= B;
    r.kind = 1;
    r.P = (NP - D) + T / yi;
    r.it = T % yi;
    return r;
}

template <int NS, int S>
__global__ void __launch_bounds__(kLanes) sweep_xy2(const __grid_constant__ CUtensorMap tmap_x,
                                                    const __grid_constant__ CUtensorMap tmap_y, XYFused2 a)
{
    extern __shared__ __align__(1024) unsigned char smem_r2[];
    constexpr int kSlot = kChunk * kLanes;
    constexpr int L = kLanes / S;
    const Ring2Smem sm = ring2_carve<NS>(smem_r2);
    const int lane = threadIdx.x;
    const int nchx = (a.nx + kChunk - 1) / kChunk;
    const int nchy = (a.ny + kChunk - 1) / kChunk;
    auto nch_of = [&](const XYItem& it) { return it.kind == 0 ? nchx : nchy; };
    auto issue = [&](const XYItem& it, int k, int slot) {
        ptx::mbar_arrive_expect_tx(&sm.bars[slot], kSlot * 8);
        if (it.kind == 0)
            ptx::tma_load_4d(sm.slots + slot * kSlot, &tmap_x, 0, it.it * L, it.P, k * 2 * S, &sm.bars[slot]);
        else
            ptx::tma_load_4d(sm.slots + slot * kSlot, &tmap_y, it.it * kLanes, k * kChunk, it.P % a.nz, it.P / a.nz,
                             &sm.bars[slot]);
    };
    auto ready = [&](const XYItem& it) { // lane 0: Y item's plane published?
        return ptx::ld_acquire(a.ctr + 1 + it.P) >= static_cast<unsigned>(a.xi);
    };
    if (lane == 0) {
        ptx::tma_prefetch_desc(&tmap_x);
        ptx::tma_prefetch_desc(&tmap_y);
        for (int s = 0; s < NS; ++s) ptx::mbar_init(&sm.bars[s], 1);
        ptx::fence_mbar_init();
    }
    __syncwarp();

    uint32_t parity = 0;
    int pending = -1;      // plane this warp still has to publish
    unsigned tk = 0;
    if (lane == 0) tk = atomicAdd(a.ctr, 1u);
    XYItem cur = xy2_decode(a, __shfl_sync(0xffffffffu, tk, 0));
    int issued = 0; // chunks of `cur` already issued (prefetched by the previous item)
    auto publish = [&]() {
        if (pending >= 0 && lane == 0) {
            ptx::bulk_wait_all();
            ptx::fence_proxy_async_global();
            ptx::red_release_add(a.ctr + 1 + pending, 1u);
        }
        pending = -1;
    };
    while (cur.kind >= 0) {
        const int nch = nch_of(cur);
        // Issue what the previous item did not prefetch (a Y item first
        // publishes what this warp owes, then waits for its plane).
        if (issued < min(NS, nch)) {
            if (cur.kind == 1 && issued == 0) {
                publish();
                if (lane == 0) {
                    while (!ready(cur)) __nanosleep(100);
                    ptx::fence_proxy_async_global();
                }
            }
            if (lane == 0)
                for (int k = issued; k < min(NS, nch); ++k) issue(cur, k, k);
        }
        __syncwarp();
        // Next ticket now; used (by lane 0) when the first slot frees up.
        if (lane == 0) tk = atomicAdd(a.ctr, 1u);
        XYItem nxt;
        nxt.kind = -2; // lane 0: decoded lazily
        bool pf = false;
        auto has_next = [&]() {
            if (nxt.kind == -2) {
                nxt = xy2_decode(a, tk);
                pf = nxt.kind == 0 || (nxt.kind == 1 && nxt.P != pending && ready(nxt));
                if (pf && nxt.kind == 1) ptx::fence_proxy_async_global();
            }
            return pf;
        };
        auto load = [&](int rel, int k, int slot, bool) {
            if (!rel)
                issue(cur, k, slot);
            else if (k < min(NS, nch_of(nxt)))
                issue(nxt, k, slot);
        };
        auto after = [&](int k) {
            if (k == 0 && pending >= 0) publish();
        };
        if (cur.kind == 0) {
            const int j0 = cur.it * L;
            int l, sub;
            x_lane<S>(lane, l, sub);
            const int rep = cur.P / a.nz, kk = cur.P % a.nz;
            const int j = j0 + l;
            const LayoutX<S> lay(l, sub);
            Clamp cl{nullptr, 0ull, 0, a.nz};
            const Chain c = make_chain(a.xcoef, S, sub, a.nx, cl, false, rep);
            (void)kk;
            solve_ring2<NS, false>(
                c, j < a.ny, sm.bars, sm.slots, kSlot, sm.ckpt, lane, parity, has_next, lay, load,
                [&](int k, int slot) { ptx::tma_store_4d(&tmap_x, 0, j0, cur.P, k * 2 * S, sm.slots + slot * kSlot); },
                nullptr, after);
        } else {
            const int e0 = cur.it * kLanes;
            const int rep = cur.P / a.nz, kk = cur.P % a.nz;
            const int width = min(kLanes, a.rowlen - e0);
            const bool active = lane < width;
            const int e = e0 + (active ? lane : 0);
            const int s = e % S, i = e / S;
            const Chain c = make_chain_yz(a.y, s, i, kk, rep);
            const LayoutYZ lay{lane};
            solve_ring2<NS, false>(
                c, active, sm.bars, sm.slots, kSlot, sm.ckpt, lane, parity, has_next, lay, load,
                [&](int k, int slot) { ptx::tma_store_4d(&tmap_y, e0, k * kChunk, kk, rep, sm.slots + slot * kSlot); },
                nullptr, after);
        }
        if (cur.kind == 0) {
            publish(); // (only if the hook did not run: nch == 0 never happens; keeps the invariant simple)
            pending = cur.P;
        }
        // Broadcast lane 0's view of the next item and whether it was prefetched.
        if (lane == 0) has_next();
        const unsigned T = __shfl_sync(0xffffffffu, tk, 0);
        const int pfl = __shfl_sync(0xffffffffu, pf ? 1 : 0, 0);
        const XYItem n2 = xy2_decode(a, T);
        issued = pfl ? min(min(NS, nch), min(NS, nch_of(n2))) : 0;
        cur = n2;
    }
    publish();
    if (lane == 0) ptx::bulk_wait_all();
}

} // namespace kernels
} // namespace biodiff_b200
