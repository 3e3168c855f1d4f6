// Persistent ring sweeps (default tile path since r01-late).
//
// Same numerics and smem layout as solve_ring in kernels.cuh (ring of NS
// chunk slots, per-chunk forward checkpoints, bit-identical backward
// recompute of reloaded chunks), but each CTA walks tiles t, t+G, t+2G, ...
// and the slots freed at the end of tile t's back substitution immediately
// receive tile t+G's first chunks. For short lines (nch <= NS: the C5
// ensemble's 64-point lines, C1/C2) every chunk of the next tile is in flight
// while the current tile finishes, so no tile starts on a cold load.
#pragma once

#include "kernels.cuh"

namespace biodiff_b200 {
namespace kernels {

// One tile of a persistent ring CTA. load(rel, k, slot, keep): lane 0 issues
// chunk k of the current (rel = 0) or next (rel = 1) tile into `slot`.
// `parity` carries the per-slot mbarrier phases across tiles.
template <bool CLAMP, class Ptr, class Load, class Store>
__device__ __forceinline__ void solve_ring_tile(const Chain& c, bool active, int step, int NS, uint64_t* bars,
                                                double* ckpt, int lane, uint32_t& parity, bool has_next, Ptr ptr,
                                                Load load, Store store, const SlabExport* exp)
{
    const int n = c.n;
    const int nch = (n + kChunk - 1) / kChunk;
    auto wait_slot = [&](int s) {
        ptx::mbar_wait(&bars[s], (parity >> s) & 1u);
        parity ^= (1u << s);
    };

    double prev = 0.0;
    for (int k = 0; k < nch; ++k) {
        const int s = k % NS;
        wait_slot(s);
        const int m0 = k * kChunk;
        const int m1 = min(n, m0 + kChunk);
        if (active) {
            double* p = ptr(s);
            int m = m0;
            if (m == 0) {
                prev = fwd_first(p[0], __ldg(c.dinv));
                p[0] = prev;
                m = 1;
                p += step;
            }
            if (m >= c.settle && m1 <= n - 1)
                prev = fwd_seg<true>(c, p, step, m, m1, prev);
            else
                prev = fwd_seg<false>(c, p, step, m, m1, prev);
            ckpt[k * kLanes + lane] = prev;
        }
        if (k + NS < nch) {
            ptx::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) load(0, k + NS, s, k + NS < nch - NS);
        }
    }
    if (exp && active && exp->bottom) exp->bottom[exp->idx] = prev;

    double next = prev;
    const int first_reloaded = nch - NS - 1;
    if (CLAMP && active && c.clamp_s && (c.face || c.face_hi))
        ptr((nch - 1) % NS)[((n - 1) - (nch - 1) * kChunk) * step] = c.clamp_v;
    for (int k = nch - 1; k >= 0; --k) {
        const int s = k % NS;
        const int m0 = k * kChunk;
        const int m1 = min(n, m0 + kChunk);
        if (k <= first_reloaded) {
            wait_slot(s);
            if (active) {
                double* p = ptr(s);
                int m = m0;
                double f;
                if (m == 0) {
                    f = fwd_first(p[0], __ldg(c.dinv));
                    p[0] = f;
                    m = 1;
                    p += step;
                } else {
                    f = ckpt[(k - 1) * kLanes + lane];
                }
                if (m >= c.settle && m1 <= n - 1)
                    fwd_seg<true>(c, p, step, m, m1, f);
                else
                    fwd_seg<false>(c, p, step, m, m1, f);
            }
        }
        int mtop = m1 - 1;
        if (k == nch - 1) --mtop;
        if (active && mtop >= m0) {
            if (m0 >= c.settle)
                next = bwd_seg<true, CLAMP>(c, ptr(s), step, mtop, m0, next);
            else
                next = bwd_seg<false, CLAMP>(c, ptr(s), step, mtop, m0, next);
        }
        ptx::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
            store(k, s);
            ptx::bulk_commit();
            // The store of chunk j = k+1 (issued one step earlier) has read
            // its slot: refill it with this tile's chunk j-NS (recompute) or,
            // once no reload needs it, the next tile's chunk j.
            const int j = k + 1;
            if (j < nch) {
                if (j - NS >= 0 && j - NS <= first_reloaded) {
                    ptx::bulk_wait_read<1>();
                    load(0, j - NS, (j - NS) % NS, false);
                } else if (j < NS && has_next) {
                    ptx::bulk_wait_read<1>();
                    load(1, j, j, j < nch - NS);
                }
            }
        }
    }
    if (exp && active && exp->top) exp->top[exp->idx] = next;
    if (lane == 0) {
        ptx::bulk_wait_read<0>();
        if (has_next) load(1, 0, 0, 0 < nch - NS); // slot 0 last
    }
    __syncwarp();
}

template <bool CLAMP>
__global__ void __launch_bounds__(kLanes) sweep_yz_pring(const __grid_constant__ CUtensorMap tmap, StridedSweep a,
                                                         Ring rg)
{
    extern __shared__ __align__(128) unsigned char smem[];
    constexpr int kSlot = kChunk * kLanes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
    double* slots = reinterpret_cast<double*>(smem + bar_bytes(rg.ns));
    double* ckpt = slots + rg.ns * kSlot;
    const int lane = threadIdx.x;
    const int G = gridDim.x;
    int t = blockIdx.x;
    if (t >= a.tiles) return;
    // Tile -> (row element e0, outer index, replica) and its TMA box of chunk k.
    auto box = [&](int tile, int k, int& e0, int& c1, int& c2, int& r) {
        e0 = (tile % a.tiles_per_row) * kLanes;
        const int outer_all = tile / a.tiles_per_row;
        r = outer_all / a.n_outer;
        const int outer = outer_all % a.n_outer;
        c1 = a.axis == 2 ? outer : k * kChunk;
        c2 = a.axis == 2 ? k * kChunk : outer;
    };
    auto issue = [&](int tile, int k, int slot) {
        int e0, c1, c2, r;
        box(tile, k, e0, c1, c2, r);
        ptx::mbar_arrive_expect_tx(&bars[slot], kSlot * 8);
        ptx::tma_load_4d(slots + slot * kSlot, &tmap, e0, c1, c2, r, &bars[slot]);
    };
    const int nch = (a.n + kChunk - 1) / kChunk;
    if (lane == 0) {
        ptx::tma_prefetch_desc(&tmap);
        for (int s = 0; s < rg.ns; ++s) ptx::mbar_init(&bars[s], 1);
        ptx::fence_mbar_init();
        for (int k = 0; k < min(rg.ns, nch); ++k) issue(t, k, k);
    }
    __syncwarp();
    uint32_t parity = 0;
    for (; t < a.tiles; t += G) {
        const int tn = t + G;
        const bool has_next = tn < a.tiles;
        int e0, c1u, c2u, r;
        box(t, 0, e0, c1u, c2u, r);
        const int outer = (t / a.tiles_per_row) % a.n_outer;
        const int width = min(kLanes, a.rowlen - e0);
        const bool active = lane < width;
        const int e = e0 + (active ? lane : 0);
        const int s = e % a.S, i = e / a.S;
        const Chain c = make_chain_yz(a, s, i, outer, r);
        const SlabExport ex{a.exp_bottom, a.exp_top, static_cast<long long>(outer) * a.rowlen + e};
        solve_ring_tile<CLAMP>(
            c, active, kLanes, rg.ns, bars, ckpt, lane, parity, has_next,
            [&](int slot) { return slots + slot * kSlot + lane; },
            [&](int rel, int k, int slot, bool) { issue(rel ? tn : t, k, slot); },
            [&](int k, int slot) {
                int e0s, c1, c2, rs;
                box(t, k, e0s, c1, c2, rs);
                ptx::tma_store_4d(&tmap, e0s, c1, c2, rs, slots + slot * kSlot);
            },
            &ex);
    }
}

template <bool CLAMP>
__global__ void __launch_bounds__(kLanes) sweep_x_pring(XSweep a, Ring rg)
{
    extern __shared__ __align__(128) unsigned char smem[];
    const int S = a.S;
    const int slot_sz = a.L * a.cpitch;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
    double* slots = reinterpret_cast<double*>(smem + bar_bytes(rg.ns));
    double* ckpt = slots + rg.ns * slot_sz;
    const int lane = threadIdx.x;
    const long long G = gridDim.x;
    long long t = blockIdx.x;
    if (t >= a.tiles) return;
    auto lines_in = [&](long long tile) {
        return static_cast<int>(min(static_cast<long long>(a.L), a.lines - tile * a.L));
    };
    auto bytes_of = [&](int k) { return static_cast<uint32_t>(min(kChunk, a.nx - k * kChunk) * S * 8); };
    auto move = [&](long long tile, int k, int slot, bool load) {
        const int nl = lines_in(tile);
        const uint32_t bytes = bytes_of(k);
        double* g = a.rho + tile * a.L * a.rowlen + static_cast<long long>(k) * kChunk * S;
        double* sm = slots + slot * slot_sz;
        if (load) ptx::mbar_arrive_expect_tx(&bars[slot], nl * bytes);
        for (int l = 0; l < nl; ++l) {
            if (load)
                ptx::bulk_g2s(sm + l * a.cpitch, g + static_cast<long long>(l) * a.rowlen, bytes, &bars[slot]);
            else
                ptx::bulk_s2g(g + static_cast<long long>(l) * a.rowlen, sm + l * a.cpitch, bytes);
        }
    };
    const int nch = (a.nx + kChunk - 1) / kChunk;
    if (lane == 0) {
        for (int s = 0; s < rg.ns; ++s) ptx::mbar_init(&bars[s], 1);
        ptx::fence_mbar_init();
        for (int k = 0; k < min(rg.ns, nch); ++k) move(t, k, k, true);
    }
    __syncwarp();
    uint32_t parity = 0;
    for (; t < a.tiles; t += G) {
        const long long tn = t + G;
        const bool has_next = tn < a.tiles;
        const int nl = lines_in(t);
        const bool active = lane < nl * S;
        const int l = active ? lane / S : 0;
        const int sub = active ? lane % S : 0;
        const long long line = t * a.L + l;
        const int rep = static_cast<int>(line / a.lines_per_rep);
        const long long rline = line % a.lines_per_rep;
        const int j = static_cast<int>(rline % a.ny), kk = static_cast<int>(rline / a.ny);
        const Chain c =
            make_chain(a.coef, S, sub, a.nx, a.clamp, j == 0 || j == a.ny - 1 || kface(kk, a.clamp), rep);
        solve_ring_tile<CLAMP>(
            c, active, S, rg.ns, bars, ckpt, lane, parity, has_next,
            [&](int slot) { return slots + slot * slot_sz + l * a.cpitch + sub; },
            [&](int rel, int k, int slot, bool) { move(rel ? tn : t, k, slot, true); },
            [&](int k, int slot) { move(t, k, slot, false); }, nullptr);
    }
}

} // namespace kernels
} // namespace biodiff_b200
