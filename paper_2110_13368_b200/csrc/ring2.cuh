// Ring sweeps, register-chunk form (default tile path).
//
// Same algorithm and numerics as solve_ring / solve_ring_tile (ring of NS
// chunk slots in shared memory, one forward checkpoint per chunk, the chunks
// that left the ring reloaded and their forward values recomputed bit for
// bit before the back substitution), rebuilt around the measured bottleneck
// of those kernels: per-warp instruction latency, not DRAM (ncu r01: ~40
// warp instructions per position, 22% of them issuing per-line bulk copies,
// 'wait' the top stall reason). Here
//   * a chunk (32 positions of the 32 chains of a warp) is processed fully
//     unrolled out of registers: 32 independent shared-memory loads, the
//     dependent FP64 chain, 32 stores;
//   * a reloaded chunk's recompute and back substitution run on the same
//     registers (no intermediate store/reload of the recomputed values);
//   * forward values of chunks that will be reloaded are never stored;
//   * NS is a compile-time constant (slot arithmetic folds);
//   * x chunks move with ONE 4-D TMA box per chunk (16 doubles x L lines x
//     1 plane x 2S pieces, 128-byte swizzle) instead of one bulk copy per
//     line; the swizzle makes the (line, substrate) lane pattern conflict-free.
// The FP64 operations and their order are exactly the reference's
// (fwd_first / fwd / bwd of kernels.cuh), so results stay bit-identical.
#pragma once

#include "kernels.cuh"

namespace biodiff_b200 {
namespace kernels {

// y / z chunk slot: [position u][lane], 32 x 32 doubles (TMA box 32 x 32 x 1 x 1).
struct LayoutYZ {
    int lane;
    __device__ __forceinline__ int off(int u) const { return lane + u * kLanes; }
};

// x chunk slot: TMA box (16 doubles, L lines, 1 plane, 2S pieces) with the
// 128-byte swizzle: smem [piece][line][16 doubles], the 16-byte granule g of
// row r stored at granule g ^ (r & 7). Row r = piece * L + l, and L is a
// multiple of 8, so r & 7 = l & 7. Element (position u, substrate s) of line
// l is double e = u*S + s of the chunk: piece e / 16, column e % 16.
template <int S>
struct LayoutX {
    static constexpr int L = kLanes / S;
    static constexpr int P = 16 / S; // positions per piece
    int row;                         // l * 16
    int t[P];                        // swizzled column of position j (u % P == j)
    __device__ __forceinline__ LayoutX(int l, int s)
    {
        row = l * 16;
#pragma unroll
        for (int j = 0; j < P; ++j) {
            const int col = j * S + s;
            t[j] = ((((col >> 1) ^ (l & 7))) << 1) | (col & 1);
        }
    }
    __device__ __forceinline__ int off(int u) const { return row + t[u % P] + (u / P) * (L * 16); }
};

// Lane -> (line, substrate) of an x tile. With the swizzle above, lines l
// and l^1 share a 32-byte granule pair at every position, so they must not
// sit in the same half-warp (64-bit shared accesses are served per 16 lanes):
// at S = 4 the half-warps take the even and the odd lines (ncu: the plain
// lane/S mapping measured 4 bank-conflict wavefronts per load). S <= 2
// needs no remap (at S = 2 a half-warp's 8 lines hit 8 distinct granules).
template <int S>
__device__ __forceinline__ void x_lane(int lane, int& l, int& s)
{
    s = lane % S;
    const int q = lane / S;
    l = S == 4 ? (((q & 3) << 1) | (q >> 2)) : q;
}

// Forward elimination over positions u < cnt of one chunk (line positions
// m0 + u). `first`: position 0 of the line (fwd_first). `constc`: every row
// of the chunk is in the settled region. `lastc`: the line's last chunk with
// every row but n-1 settled — row n-1 uses `dlast` (= dT[n-1], loaded before
// the chunk's wait), so the chunk needs no per-row coefficient loads (ncu:
// chunks that load them ran ~2.3x slower). `keep`: store the forward values
// (chunks that stay resident for the back substitution).
template <bool FULL, class Lay>
__device__ __forceinline__ double fwd_chunk(const Chain& c, double* sl, const Lay& lay, int m0, int cnt, bool first,
                                            bool constc, bool keep, double prev, bool lastc = false,
                                            double dlast = 0.0)
{
    double v[kChunk];
#pragma unroll
    for (int u = 0; u < kChunk; ++u)
        if (FULL || u < cnt) v[u] = sl[lay.off(u)];
    if (constc) {
#pragma unroll
        for (int u = 0; u < kChunk; ++u)
            if (FULL || u < cnt) {
                prev = fwd(v[u], prev, c.q, c.dc);
                v[u] = prev;
            }
    } else if (lastc) {
#pragma unroll
        for (int u = 0; u < kChunk; ++u)
            if (FULL || u < cnt) {
                prev = fwd(v[u], prev, c.q, (FULL ? u == kChunk - 1 : u == cnt - 1) ? dlast : c.dc);
                v[u] = prev;
            }
    } else {
#pragma unroll
        for (int u = 0; u < kChunk; ++u)
            if (FULL || u < cnt) {
                const double d = __ldg(c.dT + m0 + u);
                prev = (u == 0 && first) ? fwd_first(v[u], d) : fwd(v[u], prev, c.q, d);
                v[u] = prev;
            }
    }
    if (keep) {
#pragma unroll
        for (int u = 0; u < kChunk; ++u)
            if (FULL || u < cnt) sl[lay.off(u)] = v[u];
    }
    return prev;
}

__device__ __forceinline__ bool clamped_at(const Chain& c, int m)
{
    return c.clamp_s && (c.face || (m == 0 && c.face_lo) || (m == c.n - 1 && c.face_hi));
}

// Back-substitution chain over v[u], u = hi .. 0 (compile-time bounds when
// FULL), storing the (optionally clamped) result in place. Interior rows
// clamp iff the chain's line lies on a face (`cl_all`); row 0 of the line
// (m0 == 0) also when its low end is a face.
template <bool FULL, bool CLAMP, bool CONSTB>
__device__ __forceinline__ double bwd_regs(const Chain& c, double (&v)[kChunk], int m0, int hi, bool skip_top,
                                           double next)
{
    const bool cl_all = CLAMP && c.clamp_s && c.face;
#pragma unroll
    for (int u = kChunk - 1; u >= 0; --u) {
        if (!FULL && u > hi) continue;
        if (FULL && skip_top && u == kChunk - 1) continue;
        const double b = CONSTB ? c.cc : __ldg(c.cT + m0 + u);
        next = bwd(v[u], next, b);
        v[u] = cl_all ? c.clamp_v : next;
    }
    if (CLAMP && m0 == 0 && c.clamp_s && c.face_lo && !(FULL ? false : hi < 0)) v[0] = c.clamp_v;
    return next;
}

// Back substitution of a resident chunk (smem holds its forward values).
// Processes u = cnt-1-top .. 0 (top: the line's last chunk, whose position
// n-1 keeps its forward value); position cnt-1 of the top chunk is rewritten
// with the clamp when it applies. The recurrence carries unclamped values.
template <bool FULL, bool CLAMP, class Lay>
__device__ __forceinline__ double bwd_chunk(const Chain& c, double* sl, const Lay& lay, int m0, int cnt, bool top,
                                            bool constc, double next)
{
    double v[kChunk];
#pragma unroll
    for (int u = 0; u < kChunk; ++u)
        if (FULL || u < cnt) v[u] = sl[lay.off(u)];
    const int hi = cnt - 1 - (top ? 1 : 0);
    if (constc)
        next = bwd_regs<FULL, CLAMP, true>(c, v, m0, hi, top, next);
    else
        next = bwd_regs<FULL, CLAMP, false>(c, v, m0, hi, top, next);
    if (CLAMP && top && clamped_at(c, c.n - 1)) {
#pragma unroll
        for (int u = 0; u < kChunk; ++u)
            if (u == cnt - 1) v[u] = c.clamp_v;
    }
#pragma unroll
    for (int u = 0; u < kChunk; ++u)
        if (FULL || u < cnt) sl[lay.off(u)] = v[u];
    return next;
}

// Reloaded (always full, never the top) chunk: recompute the forward values
// from the previous chunk's checkpoint in registers, then back-substitute.
template <bool CLAMP, class Lay>
__device__ __forceinline__ double rbwd_chunk(const Chain& c, double* sl, const Lay& lay, int m0, bool first,
                                             bool constf, bool constb, double fprev, double next)
{
    double v[kChunk];
#pragma unroll
    for (int u = 0; u < kChunk; ++u) v[u] = sl[lay.off(u)];
    if (constf) {
#pragma unroll
        for (int u = 0; u < kChunk; ++u) {
            fprev = fwd(v[u], fprev, c.q, c.dc);
            v[u] = fprev;
        }
    } else {
#pragma unroll
        for (int u = 0; u < kChunk; ++u) {
            const double d = __ldg(c.dT + m0 + u);
            fprev = (u == 0 && first) ? fwd_first(v[u], d) : fwd(v[u], fprev, c.q, d);
            v[u] = fprev;
        }
    }
    if (constb)
        next = bwd_regs<true, CLAMP, true>(c, v, m0, kChunk - 1, false, next);
    else
        next = bwd_regs<true, CLAMP, false>(c, v, m0, kChunk - 1, false, next);
#pragma unroll
    for (int u = 0; u < kChunk; ++u) sl[lay.off(u)] = v[u];
    return next;
}

// One line tile through a ring of NS slots. The first min(NS, nch) chunks
// must already be issued into slots 0.. (by the caller or the previous
// tile). load(rel, k, slot): lane 0 issues chunk k of this (rel 0) or the
// next (rel 1) tile; store(k, slot): lane 0 writes chunk k back.
// has_next(): evaluated by lane 0 only, when the first slot frees up in the
// back substitution — whether to prefetch the next tile's first chunks.
// after_fwd(k): called on every lane after forward chunk k. `parity`
// carries the per-slot mbarrier phases across tiles.
struct NoHook {
    __device__ __forceinline__ void operator()(int) const {}
};

template <int NS, bool CLAMP, class Lay, class Next, class Load, class Store, class After = NoHook>
__device__ __forceinline__ void solve_ring2(const Chain& c, bool active, uint64_t* bars, double* slots, int slot_doubles,
                                            double* ckpt, int lane, uint32_t& parity, Next has_next, const Lay& lay,
                                            Load load, Store store, const SlabExport* exp, After after_fwd = NoHook())
{
    const int n = c.n;
    const int nch = (n + kChunk - 1) / kChunk;
    auto wait_slot = [&](int s) {
        ptx::mbar_wait(&bars[s], (parity >> s) & 1u);
        parity ^= (1u << s);
    };
    const int first_reloaded = nch - NS - 1; // chunks <= this are reloaded in the back substitution

    // z-slab inflow: row 0 continues the previous slab's forward recurrence
    // (fwd with D_{p-1} instead of fwd_first), the last row is back-substituted
    // from X_{p+1} instead of keeping its forward value.
    double prev = c.has_lo ? c.lo_val : 0.0;
    for (int k = 0; k < nch; ++k) {
        const int s = k % NS;
        const int m0 = k * kChunk;
        const int cnt = min(kChunk, n - m0);
        const bool constc = k > 0 && m0 >= c.settle && m0 + cnt <= n - 1;
        const bool lastc = k > 0 && m0 >= c.settle && m0 + cnt == n;
        const double dlast = lastc && active ? __ldg(c.dT + n - 1) : 0.0;
        wait_slot(s);
        if (active) {
            double* sl = slots + s * slot_doubles;
            const bool keep = k > first_reloaded;
            const bool first = k == 0 && !c.has_lo;
            if (cnt == kChunk)
                prev = fwd_chunk<true>(c, sl, lay, m0, cnt, first, constc, keep, prev, lastc, dlast);
            else
                prev = fwd_chunk<false>(c, sl, lay, m0, cnt, first, constc, keep, prev, lastc, dlast);
            ckpt[k * kLanes + lane] = prev;
        }
        after_fwd(k);
        if (k + NS < nch) { // recycle the slot for chunk k+NS (chunk k will be reloaded)
            ptx::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) load(0, k + NS, s, false);
        }
    }
    if (exp && active && exp->bottom) exp->bottom[exp->idx] = prev;

    double next = c.has_hi ? c.hi_val : prev; // without inflow: final (unclamped) value of position n-1
    for (int k = nch - 1; k >= 0; --k) {
        const int s = k % NS;
        const int m0 = k * kChunk;
        const int cnt = min(kChunk, n - m0);
        double* sl = slots + s * slot_doubles;
        if (k <= first_reloaded) {
            wait_slot(s);
            if (active) {
                const double f = k > 0 ? ckpt[(k - 1) * kLanes + lane] : (c.has_lo ? c.lo_val : 0.0);
                next = rbwd_chunk<CLAMP>(c, sl, lay, m0, k == 0 && !c.has_lo, k > 0 && m0 >= c.settle,
                                         m0 >= c.settle, f, next);
            }
        } else if (active) {
            const bool top = k == nch - 1 && !c.has_hi;
            const bool constb = m0 >= c.settle && !(k == nch - 1 && c.has_hi); // row n-1's own c_back
            if (cnt == kChunk)
                next = bwd_chunk<true, CLAMP>(c, sl, lay, m0, cnt, top, constb, next);
            else
                next = bwd_chunk<false, CLAMP>(c, sl, lay, m0, cnt, top, constb, next);
        }
        ptx::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
            store(k, s);
            ptx::bulk_commit();
            // The store of chunk j = k+1 (issued one step earlier) has read
            // its slot: refill it with this tile's chunk j-NS (reload) or,
            // once no reload needs it, the next tile's chunk j.
            const int j = k + 1;
            if (j < nch) {
                if (j - NS >= 0 && j - NS <= first_reloaded) {
                    ptx::bulk_wait_read<1>();
                    load(0, j - NS, (j - NS) % NS, true);
                } else if (j < NS && has_next()) {
                    ptx::bulk_wait_read<1>();
                    load(1, j, j, false);
                }
            }
        }
    }
    if (exp && active && exp->top) exp->top[exp->idx] = next;
    if (lane == 0) {
        ptx::bulk_wait_read<0>();
        if (has_next()) load(1, 0, 0, false);
    }
    __syncwarp();
}

// Short lines (2 * nch <= NS, e.g. the C5 ensemble's 64-point lines): every
// chunk of a tile stays resident (no reloads) and the slots form two sets
// used by alternate tiles, so the NEXT tile's chunks are issued when this
// tile starts — its load latency hides behind a whole tile of work instead of
// the last chunk's back substitution. `base` = first slot of this tile's set.
template <int NS, bool CLAMP, class Lay, class Next, class Load, class Store>
__device__ __forceinline__ void solve_short2(const Chain& c, bool active, uint64_t* bars, double* slots,
                                             int slot_doubles, int lane, uint32_t& parity, int base, Next has_next,
                                             const Lay& lay, Load load, Store store, const SlabExport* exp)
{
    const int n = c.n;
    const int nch = (n + kChunk - 1) / kChunk;
    const int other = nch - base;
    auto wait_slot = [&](int s) {
        ptx::mbar_wait(&bars[s], (parity >> s) & 1u);
        parity ^= (1u << s);
    };
    if (lane == 0 && has_next()) {
        ptx::bulk_wait_read<0>(); // the previous tile's stores out of the other set
        for (int k = 0; k < nch; ++k) load(1, k, other + k, false);
    }
    __syncwarp();
    double prev = c.has_lo ? c.lo_val : 0.0;
    for (int k = 0; k < nch; ++k) {
        const int m0 = k * kChunk;
        const int cnt = min(kChunk, n - m0);
        const bool constc = k > 0 && m0 >= c.settle && m0 + cnt <= n - 1;
        const bool lastc = k > 0 && m0 >= c.settle && m0 + cnt == n;
        const double dlast = lastc && active ? __ldg(c.dT + n - 1) : 0.0;
        wait_slot(base + k);
        if (active) {
            double* sl = slots + (base + k) * slot_doubles;
            const bool first = k == 0 && !c.has_lo;
            if (cnt == kChunk)
                prev = fwd_chunk<true>(c, sl, lay, m0, cnt, first, constc, true, prev, lastc, dlast);
            else
                prev = fwd_chunk<false>(c, sl, lay, m0, cnt, first, constc, true, prev, lastc, dlast);
        }
    }
    if (exp && active && exp->bottom) exp->bottom[exp->idx] = prev;
    double next = c.has_hi ? c.hi_val : prev;
    for (int k = nch - 1; k >= 0; --k) {
        const int m0 = k * kChunk;
        const int cnt = min(kChunk, n - m0);
        if (active) {
            double* sl = slots + (base + k) * slot_doubles;
            const bool top = k == nch - 1 && !c.has_hi;
            const bool constb = m0 >= c.settle && !(k == nch - 1 && c.has_hi);
            if (cnt == kChunk)
                next = bwd_chunk<true, CLAMP>(c, sl, lay, m0, cnt, top, constb, next);
            else
                next = bwd_chunk<false, CLAMP>(c, sl, lay, m0, cnt, top, constb, next);
        }
        ptx::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
            store(k, base + k);
            ptx::bulk_commit();
        }
    }
    if (exp && active && exp->top) exp->top[exp->idx] = next;
    __syncwarp();
}

// Dynamic smem of the ring2 kernels: 1024-byte aligned slots (the x box
// uses the 128-byte swizzle), then mbarriers, then checkpoints.
__host__ __device__ constexpr int ring2_smem_bytes(int ns, int nch)
{
    return 1024 + ns * kChunk * kLanes * 8 + 128 + nch * kLanes * 8;
}

struct Ring2Smem {
    double* slots;
    uint64_t* bars;
    double* ckpt;
};

template <int NS>
__device__ __forceinline__ Ring2Smem ring2_carve(unsigned char* smem)
{
    const uint32_t base = ptx::smem_addr(smem);
    unsigned char* p = smem + (((base + 1023u) & ~1023u) - base);
    Ring2Smem r;
    r.slots = reinterpret_cast<double*>(p);
    r.bars = reinterpret_cast<uint64_t*>(p + NS * kChunk * kLanes * 8);
    r.ckpt = reinterpret_cast<double*>(p + NS * kChunk * kLanes * 8 + 128);
    return r;
}

// y / z sweep: tile t = (32-double column block e0 of a row, outer index,
// replica); persistent over t, t + G, ... (G = grid; one tile per CTA when
// the grid covers every tile).
template <int NS, bool CLAMP, bool SHORT = false>
__global__ void __launch_bounds__(kLanes) sweep_yz_ring2(const __grid_constant__ CUtensorMap tmap, StridedSweep a)
{
    extern __shared__ __align__(1024) unsigned char smem_r2[];
    constexpr int kSlot = kChunk * kLanes;
    const Ring2Smem sm = ring2_carve<NS>(smem_r2);
    const int lane = threadIdx.x;
    const int G = gridDim.x;
    int t = blockIdx.x;
    if (t >= a.tiles) return;
    ptx::griddep_wait();
    ptx::griddep_launch();
    struct TileAt {
        int e0, outer, r;
    };
    auto decode = [&](int tile) {
        TileAt d;
        d.e0 = (tile % a.tiles_per_row) * kLanes;
        const int outer_all = tile / a.tiles_per_row;
        d.r = a.r0 + outer_all / a.n_outer;
        d.outer = outer_all % a.n_outer;
        return d;
    };
    const int nch = (a.n + kChunk - 1) / kChunk;
    // L2 hints (a.hints bit 0): first loads of chunks the back substitution
    // will reload stay (evict_last); reloads and the other loads stream.
    // Bit 2: only the later ones (k >= keep_from8/8 of them: the reloads with
    // the shortest reuse distance) stay.
    const uint64_t keep_pol = ptx::policy_evict_last(), stream_pol = ptx::policy_evict_first();
    auto issue = [&](const TileAt& d, int k, int slot, bool reload = false) {
        const int c1 = a.axis == 2 ? d.outer : k * kChunk;
        const int c2 = a.axis == 2 ? k * kChunk : d.outer;
        ptx::mbar_arrive_expect_tx(&sm.bars[slot], kSlot * 8);
        if (a.hints & 5)
            ptx::tma_load_4d_hint(sm.slots + slot * kSlot, &tmap, d.e0, c1, c2, d.r, &sm.bars[slot],
                                  (!reload && k < nch - NS && (!(a.hints & 4) || 8 * k >= a.keep_from8 * (nch - NS))) ? keep_pol
                                                                                                     : stream_pol);
        else
            ptx::tma_load_4d(sm.slots + slot * kSlot, &tmap, d.e0, c1, c2, d.r, &sm.bars[slot]);
    };
    if (lane == 0) {
        ptx::tma_prefetch_desc(&tmap);
        for (int s = 0; s < NS; ++s) ptx::mbar_init(&sm.bars[s], 1);
        ptx::fence_mbar_init();
        const TileAt d0 = decode(t);
        for (int k = 0; k < min(NS, nch); ++k) issue(d0, k, k);
    }
    __syncwarp();
    uint32_t parity = 0;
    int it = 0;
    const LayoutYZ lay{lane};
    for (; t < a.tiles; t += G) {
        const int tn = t + G;
        const TileAt dc = decode(t), dn = decode(tn);
        const int e0 = dc.e0, outer = dc.outer, r = dc.r;
        const int width = min(kLanes, a.rowlen - e0);
        const bool active = lane < width;
        const int e = e0 + (active ? lane : 0);
        const int s = e % a.S, i = e / a.S;
        Chain c = make_chain_yz(a, s, i, outer, r);
        const long long pidx = static_cast<long long>(outer) * a.rowlen + e; // column's index in a z plane
        if (a.in_lo) {
            c.has_lo = true;
            c.lo_val = a.in_lo[pidx];
        }
        if (a.in_hi) {
            c.has_hi = true;
            c.hi_val = a.in_hi[pidx];
        }
        const SlabExport ex{a.exp_bottom, a.exp_top, pidx};
        auto has_next = [&] { return tn < a.tiles; };
        auto load = [&](int rel, int k, int slot, bool reload) { issue(rel ? dn : dc, k, slot, reload); };
        auto store = [&](int k, int slot) {
            const int c1 = a.axis == 2 ? outer : k * kChunk;
            const int c2 = a.axis == 2 ? k * kChunk : outer;
            if (a.hints & 2)
                ptx::tma_store_4d_hint(&tmap, e0, c1, c2, r, sm.slots + slot * kSlot, stream_pol);
            else
                ptx::tma_store_4d(&tmap, e0, c1, c2, r, sm.slots + slot * kSlot);
        };
        if constexpr (SHORT) // host guarantees 2 * nch <= NS
            solve_short2<NS, CLAMP>(c, active, sm.bars, sm.slots, kSlot, lane, parity, (it & 1) ? nch : 0, has_next,
                                    lay, load, store, &ex);
        else
            solve_ring2<NS, CLAMP>(c, active, sm.bars, sm.slots, kSlot, sm.ckpt, lane, parity, has_next, lay, load,
                                   store, &ex);
        ++it;
    }
}

// x sweep over the swizzled 4-D map (16 doubles, j, plane, piece): tile t =
// (plane P = t / xi, lines j0 = (t % xi) * L .. j0 + L - 1). Persistent.
struct XSweep2 {
    Coef coef;
    int nx, ny, nz, S;
    int planes; // nz * replicas (of this launch's replica batch)
    int P0;     // first plane (replica batch r0: r0 * nz)
    int hints;  // L2 cache hints: bit 0 loads, bit 1 stores, bit 2 near reloads only (BIODIFF_L2_HINTS)
    int keep_from8;
    int xi;     // tiles per plane
    long long tiles;
    Clamp clamp;
};

template <int NS, int S, bool CLAMP, bool SHORT = false>
__global__ void __launch_bounds__(kLanes) sweep_x_ring2(const __grid_constant__ CUtensorMap tmap, XSweep2 a)
{
    extern __shared__ __align__(1024) unsigned char smem_r2[];
    constexpr int kSlot = kChunk * kLanes;
    constexpr int L = kLanes / S;
    const Ring2Smem sm = ring2_carve<NS>(smem_r2);
    const int lane = threadIdx.x;
    const long long G = gridDim.x;
    long long t = blockIdx.x;
    if (t >= a.tiles) return;
    ptx::griddep_wait();
    ptx::griddep_launch();
    const int nch = (a.nx + kChunk - 1) / kChunk;
    const uint64_t keep_pol = ptx::policy_evict_last(), stream_pol = ptx::policy_evict_first();
    auto issue = [&](int P, int j0, int k, int slot, bool reload = false) {
        ptx::mbar_arrive_expect_tx(&sm.bars[slot], kSlot * 8);
        if (a.hints & 5)
            ptx::tma_load_4d_hint(sm.slots + slot * kSlot, &tmap, 0, j0, P, k * 2 * S, &sm.bars[slot],
                                  (!reload && k < nch - NS && (!(a.hints & 4) || 8 * k >= a.keep_from8 * (nch - NS))) ? keep_pol
                                                                                                     : stream_pol);
        else
            ptx::tma_load_4d(sm.slots + slot * kSlot, &tmap, 0, j0, P, k * 2 * S, &sm.bars[slot]);
    };
    if (lane == 0) {
        ptx::tma_prefetch_desc(&tmap);
        for (int s = 0; s < NS; ++s) ptx::mbar_init(&sm.bars[s], 1);
        ptx::fence_mbar_init();
        for (int k = 0; k < min(NS, nch); ++k)
            issue(a.P0 + static_cast<int>(t / a.xi), static_cast<int>(t % a.xi) * L, k, k);
    }
    __syncwarp();
    uint32_t parity = 0;
    int it = 0;
    int l, sub;
    x_lane<S>(lane, l, sub);
    const LayoutX<S> lay(l, sub);
    for (; t < a.tiles; t += G) {
        const long long tn = t + G;
        const int P = a.P0 + static_cast<int>(t / a.xi), j0 = static_cast<int>(t % a.xi) * L;
        const int Pn = a.P0 + static_cast<int>(tn / a.xi), j0n = static_cast<int>(tn % a.xi) * L;
        const int rep = P / a.nz, kk = P % a.nz;
        const int j = j0 + l;
        const bool active = j < a.ny;
        const Chain c = make_chain(a.coef, S, sub, a.nx, a.clamp, j == 0 || j == a.ny - 1 || kface(kk, a.clamp), rep);
        auto has_next = [&] { return tn < a.tiles; };
        auto load = [&](int rel, int k, int slot, bool reload) {
            if (rel)
                issue(Pn, j0n, k, slot);
            else
                issue(P, j0, k, slot, reload);
        };
        auto store = [&](int k, int slot) {
            if (a.hints & 2)
                ptx::tma_store_4d_hint(&tmap, 0, j0, P, k * 2 * S, sm.slots + slot * kSlot, stream_pol);
            else
                ptx::tma_store_4d(&tmap, 0, j0, P, k * 2 * S, sm.slots + slot * kSlot);
        };
        if constexpr (SHORT) // host guarantees 2 * nch <= NS
            solve_short2<NS, CLAMP>(c, active, sm.bars, sm.slots, kSlot, lane, parity, (it & 1) ? nch : 0, has_next,
                                    lay, load, store, nullptr);
        else
            solve_ring2<NS, CLAMP>(c, active, sm.bars, sm.slots, kSlot, sm.ckpt, lane, parity, has_next, lay, load,
                                   store, nullptr);
        ++it;
    }
}

} // namespace kernels
} // namespace biodiff_b200
