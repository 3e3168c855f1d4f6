// sm_100a FP64 kernels of the LOD diffusion step and the cell source/sink
// step. Bitwise contract: every arithmetic operation
// is an explicitly rounded __dmul_rn / __dadd_rn / __ddiv_rn in the
// reference's operand order, so no FMA contraction can change a bit:
//   forward  first: v*dinv                 (solver.cpp:17 fwd_first)
//   forward       : (v + q*prev)*dinv      (solver.cpp:18 fwd)
//   backward      : v + cb*next            (solver.cpp:19 bwd)
//   sources       : (r + (f*sec)*target) / (1 + f*(sec+upt)),  f = (dt*V)*inv_vox
//                                          (agents.cpp:102-107)
#pragma once

#include "ptx.cuh"

#include <cuda.h>
#include <cstdint>

namespace biodiff_b200 {
namespace kernels {

constexpr int kLanes = 32;   // chains per CTA (one warp)
constexpr int kChunk = 32;   // positions per mbarrier chunk along the sweep axis

__host__ __device__ constexpr int bar_bytes(int nch) { return ((nch * 8 + 127) / 128) * 128; }

struct Clamp {
    const double* values;    // [S] shell clamp values
    unsigned long long mask; // bit s: substrate s clamped on every boundary voxel
    int k0;                  // global z index of local plane 0 (z-slab), else 0
    int nzg;                 // global nz
};

// Is local plane k on a global z face?
__device__ __forceinline__ bool kface(int k_local, const Clamp& cl)
{
    const int k = k_local + cl.k0;
    return k == 0 || k == cl.nzg - 1;
}

// Thomas coefficients of one axis. The precomputed pivots settle to
// bit-constant values a few dozen rows into the line (SURVEY.md §7 hard part
// 3): rows in [settle, n-2] use dconst[s] / cconst[s] from registers instead
// of a load. `settle` is the max over substrates (warp-uniform) and is
// verified on the host bit for bit; settle = n disables the shortcut.
struct Coef {
    const double* q;      // [S]
    const double* dinv;   // [n*S]
    const double* cb;     // [n*S]
    const double* dconst; // [S]
    const double* cconst; // [S]
    int settle;
    long long rstride;    // ensembles: doubles between replicas' dinv/cb sets (n*S); q/dconst/cconst step S
    const double* dinvT = nullptr; // [R][S][n]: the same bits per substrate row-contiguous (ring2:
    const double* cbT = nullptr;   // row m0 + u of a chunk is an immediate offset from one base)
    int n = 0;
    const int* settle_r = nullptr; // [R] per-replica settle rows (ring2 / cluster chains), or nullptr: settle
};

__device__ __forceinline__ double fwd_first(double v, double d) { return __dmul_rn(v, d); }
#ifndef BIODIFF_FMA
__device__ __forceinline__ double fwd(double v, double prev, double q, double d)
{
    return __dmul_rn(__dadd_rn(v, __dmul_rn(q, prev)), d);
}
__device__ __forceinline__ double bwd(double v, double next, double cb) { return __dadd_rn(v, __dmul_rn(cb, next)); }
#else
// Contracted variant (one rounding instead of two in v + q*prev and
// v + cb*next): shorter dependent chains, not bit-identical to the reference.
__device__ __forceinline__ double fwd(double v, double prev, double q, double d)
{
    return __dmul_rn(__fma_rn(q, prev, v), d);
}
__device__ __forceinline__ double bwd(double v, double next, double cb) { return __fma_rn(cb, next, v); }
#endif

// Per-lane constants of one chain (line x substrate).
struct Chain {
    int S;
    const double* dinv; // coefficient column of this lane's substrate (stride S)
    const double* cb;
    const double* dT;   // the same column, contiguous (Coef::dinvT / cbT), or nullptr
    const double* cT;
    double q, dc, cc;
    int settle, n;
    bool clamp_s, face;     // clamped substrate; lane's line lies on a mesh face
    bool face_lo, face_hi;  // line positions 0 / n-1 lie on a mesh face (false at interior z-slab cuts)
    double clamp_v;
    bool has_lo = false, has_hi = false; // z-slab inflows (ring2): row 0 continues the previous slab's
    double lo_val = 0.0, hi_val = 0.0;   // forward recurrence, row n-1 the next slab's back substitution
    int s = 0, ts = 0;                   // substrate; stride between substrate columns of dT / cT
};

// Forward elimination over positions [m0, m1) (m0 >= 1); position m lives
// at p[(m - m0) * step].
template <bool CONSTC>
__device__ __forceinline__ double fwd_seg(const Chain& c, double* p, int step, int m0, int m1, double prev)
{
    int m = m0;
    for (; m + 8 <= m1; m += 8, p += 8 * step) {
        double v[8], d[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            v[u] = p[u * step];
            d[u] = CONSTC ? c.dc : __ldg(c.dinv + (m + u) * c.S);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            prev = fwd(v[u], prev, c.q, d[u]);
            p[u * step] = prev;
        }
    }
    for (; m < m1; ++m, p += step) {
        prev = fwd(*p, prev, c.q, CONSTC ? c.dc : __ldg(c.dinv + m * c.S));
        *p = prev;
    }
    return prev;
}

// Back substitution over positions mtop down to m0; position m lives at
// p[(m - m0) * step]. Stores the (optionally clamped) result while the
// recurrence carries the unclamped one: the clamp is applied after all
// sweeps (solver.cpp:298), so it must not feed back into this sweep.
template <bool CONSTC, bool CLAMP>
__device__ __forceinline__ double bwd_seg(const Chain& c, double* p, int step, int mtop, int m0, double next)
{
    int m = mtop;
    double* q = p + (mtop - m0) * step;
    for (; m - 7 >= m0; m -= 8, q -= 8 * step) {
        double v[8], b[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            v[u] = q[-u * step];
            b[u] = CONSTC ? c.cc : __ldg(c.cb + (m - u) * c.S);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            next = bwd(v[u], next, b[u]);
            double out = next;
            if (CLAMP && c.clamp_s && (c.face || ((m - u) == 0 && c.face_lo))) out = c.clamp_v;
            q[-u * step] = out;
        }
    }
    for (; m >= m0; --m, q -= step) {
        next = bwd(*q, next, CONSTC ? c.cc : __ldg(c.cb + m * c.S));
        double out = next;
        if (CLAMP && c.clamp_s && (c.face || (m == 0 && c.face_lo))) out = c.clamp_v;
        *q = out;
    }
    return next;
}

// The Thomas solve of one chain whose line is split in chunks of kChunk
// positions; chunk k starts at ptr(k) (stride `step`). wait(k) blocks until
// chunk k is in shared memory; flush(k) runs (on every lane) once chunk k
// holds its final values.
template <bool CLAMP, class Ptr, class Wait, class Flush>
__device__ __forceinline__ void solve_chunked(const Chain& c, bool active, int step, Ptr ptr, Wait wait, Flush flush)
{
    const int n = c.n;
    const int nch = (n + kChunk - 1) / kChunk;
    double prev = 0.0;
    for (int k = 0; k < nch; ++k) {
        wait(k);
        const int m0 = k * kChunk;
        const int m1 = min(n, m0 + kChunk);
        if (active) {
            double* p = ptr(k);
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
        }
    }
    double next = prev; // final value of position n-1
    if (CLAMP && active && c.clamp_s && (c.face || c.face_hi))
        ptr(nch - 1)[(n - 1 - (nch - 1) * kChunk) * step] = c.clamp_v;
    for (int k = nch - 1; k >= 0; --k) {
        const int m0 = k * kChunk;
        int mtop = min(n, m0 + kChunk) - 1;
        if (k == nch - 1) --mtop;
        if (active && mtop >= m0) {
            if (m0 >= c.settle)
                next = bwd_seg<true, CLAMP>(c, ptr(k), step, mtop, m0, next);
            else
                next = bwd_seg<false, CLAMP>(c, ptr(k), step, mtop, m0, next);
        }
        flush(k);
    }
}

// ---------------------------------------------------------------------------
// y / z sweep: persistent CTAs (one warp each, a few per SM) stream "tiles"
// of 32 contiguous doubles of a row — 32 (i,s) chains — times the whole
// line along the sweep axis. The line sits in shared memory as nch chunk
// slots of 32 positions x 32 chains (8 KB), moved by 3-D tiled TMA
// (UTMALDG / UTMASTG), one mbarrier per slot. HBM traffic: one read + one
// write per value.
//
// Slot recycling: the back substitution finishes chunks top-down, and each
// finished chunk's slot (once its TMA store has read it) immediately
// receives the NEXT tile's chunk nch-1-k — the next tile's chunks therefore
// arrive bottom-up while this tile is still being finished, and the next
// forward pass starts without a cold-load bubble. Tiles alternate between
// the identity and the reversed slot order.
// ---------------------------------------------------------------------------
struct StridedSweep {
    double* rho;
    Coef coef;
    int axis;    // 1 = y (outer k), 2 = z (outer j)
    int n;       // line length
    int n_outer; // number of outer indices (nz for y, ny for z)
    int rowlen;  // nx*S
    int tiles_per_row;
    int tiles;   // tiles_per_row * n_outer * reps
    int reps;    // ensemble replicas stacked along the 4th tensor dimension (ring kernel)
    int r0;      // first replica of this launch (ring2 replica batches), else 0
    int hints;   // ring2 L2 cache hints: bit 0 loads, bit 1 stores, bit 2 loads of near reloads only (BIODIFF_L2_HINTS)
    int keep_from8; // bit 2: first loads of reloaded chunks k >= keep_from8/8 of them stay in L2
    int S;
    int nx;
    long long stride;       // (plain kernel) doubles between positions along the axis
    long long outer_stride; // (plain kernel) doubles between outer indices
    Clamp clamp;
    double* exp_bottom;     // z-slab plane exports (ring kernel, z axis), or nullptr
    double* exp_top;
    const double* in_lo = nullptr; // z-slab inflows (ring2, z axis): D_{p-1} into row 0,
    const double* in_hi = nullptr; // X_{p+1} into the last row; nullptr at a global face
};

__device__ __forceinline__ Chain make_chain(const Coef& coef, int S, int s, int n, const Clamp& cl, bool face, int r = 0)
{
    Chain c;
    c.S = S;
    c.dinv = coef.dinv + r * coef.rstride + s;
    c.cb = coef.cb + r * coef.rstride + s;
    c.dT = coef.dinvT ? coef.dinvT + (static_cast<long long>(r) * S + s) * coef.n : nullptr;
    c.cT = coef.cbT ? coef.cbT + (static_cast<long long>(r) * S + s) * coef.n : nullptr;
    c.q = coef.q[r * S + s];
    c.dc = coef.dconst[r * S + s];
    c.cc = coef.cconst[r * S + s];
    c.settle = coef.settle_r ? __ldg(coef.settle_r + r) : coef.settle;
    c.n = n;
    c.s = s;
    c.ts = coef.n;
    c.clamp_s = (cl.mask >> s) & 1ull;
    c.clamp_v = c.clamp_s ? cl.values[s] : 0.0;
    c.face = face;
    c.face_lo = true;
    c.face_hi = true;
    return c;
}

// Chain of a y/z tile lane: column (i, s) at outer index `outer` (k for y,
// j for z). Along z the line ends are global faces only on the first/last slab.
__device__ __forceinline__ Chain make_chain_yz(const StridedSweep& a, int s, int i, int outer, int r = 0)
{
    const bool outer_face = a.axis == 2 ? (outer == 0 || outer == a.n_outer - 1) : kface(outer, a.clamp);
    Chain c = make_chain(a.coef, a.S, s, a.n, a.clamp, i == 0 || i == a.nx - 1 || outer_face, r);
    if (a.axis == 2) {
        c.face_lo = a.clamp.k0 == 0;
        c.face_hi = a.clamp.k0 + a.n == a.clamp.nzg;
    }
    return c;
}

template <bool CLAMP>
static __global__ void __launch_bounds__(kLanes) sweep_yz_tma(const __grid_constant__ CUtensorMap tmap, StridedSweep a)
{
    extern __shared__ __align__(128) unsigned char smem[];
    constexpr int kSlot = kChunk * kLanes; // doubles per slot
    const int nch = (a.n + kChunk - 1) / kChunk;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
    double* slots = reinterpret_cast<double*>(smem + bar_bytes(nch));
    const int lane = threadIdx.x;
    int t = blockIdx.x;
    if (t >= a.tiles) return;

    // Box coordinates (dim0 = row element, dim1 = j, dim2 = k) of chunk k of tile t.
    auto issue_load = [&](int tile, int k, int slot) {
        const int e0 = (tile % a.tiles_per_row) * kLanes;
        const int outer = tile / a.tiles_per_row;
        const int c1 = a.axis == 2 ? outer : k * kChunk;
        const int c2 = a.axis == 2 ? k * kChunk : outer;
        ptx::mbar_arrive_expect_tx(&bars[slot], kSlot * 8);
        ptx::tma_load_4d(slots + slot * kSlot, &tmap, e0, c1, c2, 0, &bars[slot]);
    };
    if (lane == 0) {
        ptx::tma_prefetch_desc(&tmap);
        for (int k = 0; k < nch; ++k) ptx::mbar_init(&bars[k], 1);
        ptx::fence_mbar_init();
        for (int k = 0; k < nch; ++k) issue_load(t, k, k);
    }
    __syncwarp();

    for (int it = 0; t < a.tiles; ++it) {
        const int tnext = t + gridDim.x;
        const bool rev = it & 1;
        const uint32_t phase = it & 1;
        auto slot_of = [&](int k) { return rev ? nch - 1 - k : k; };
        const int e0 = (t % a.tiles_per_row) * kLanes;
        const int outer = t / a.tiles_per_row;
        const int width = min(kLanes, a.rowlen - e0);
        const bool active = lane < width;
        const int e = e0 + (active ? lane : 0);
        const int s = e % a.S, i = e / a.S;
        const Chain c = make_chain_yz(a, s, i, outer);
        solve_chunked<CLAMP>(
            c, active, kLanes, [&](int k) { return slots + slot_of(k) * kSlot + lane; },
            [&](int k) { ptx::mbar_wait(&bars[slot_of(k)], phase); },
            [&](int k) {
                ptx::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    const int c1 = a.axis == 2 ? outer : k * kChunk;
                    const int c2 = a.axis == 2 ? k * kChunk : outer;
                    ptx::tma_store_4d(&tmap, e0, c1, c2, 0, slots + slot_of(k) * kSlot);
                    ptx::bulk_commit();
                    if (tnext < a.tiles) {
                        // The store of chunk k+1 (issued one step earlier) has
                        // read its slot: recycle it for the next tile.
                        if (k < nch - 1) {
                            ptx::bulk_wait_read<1>();
                            issue_load(tnext, nch - 1 - (k + 1), slot_of(k + 1));
                        }
                        if (k == 0) {
                            ptx::bulk_wait_read<0>();
                            issue_load(tnext, nch - 1, slot_of(0));
                        }
                    }
                }
            });
        t = tnext;
    }
    if (lane == 0) ptx::bulk_wait_read<0>();
}

// Whole line in shared memory without TMA (rows with an odd number of
// doubles cannot be described by a tensor map: strides must be 16-byte
// multiples). One tile per CTA.
static __global__ void __launch_bounds__(kLanes) sweep_yz_plain(StridedSweep a, bool clamp)
{
    extern __shared__ __align__(128) unsigned char smem[];
    double* tile = reinterpret_cast<double*>(smem);
    const int lane = threadIdx.x;
    const int e0 = static_cast<int>(blockIdx.x % a.tiles_per_row) * kLanes;
    const int outer = static_cast<int>(blockIdx.x / a.tiles_per_row);
    const int width = min(kLanes, a.rowlen - e0);
    double* base = a.rho + outer * a.outer_stride + e0;
    const bool active = lane < width;
    for (int m = 0; m < a.n; ++m)
        if (active) tile[m * kLanes + lane] = base[m * a.stride + lane];
    __syncwarp();
    const int e = e0 + (active ? lane : 0);
    const int s = e % a.S, i = e / a.S;
    const Chain c = make_chain_yz(a, s, i, outer);
    auto ptr = [&](int k) { return tile + k * kChunk * kLanes + lane; };
    auto none = [](int) {};
    if (clamp)
        solve_chunked<true>(c, active, kLanes, ptr, none, none);
    else
        solve_chunked<false>(c, active, kLanes, ptr, none, none);
    __syncwarp();
    for (int m = 0; m < a.n; ++m)
        if (active) base[m * a.stride + lane] = tile[m * kLanes + lane];
}

// ---------------------------------------------------------------------------
// x sweep: persistent CTAs stream tiles of L whole x-lines (contiguous in
// HBM). Lane -> (line l, substrate s). Chunk k (voxels 32k..32k+31 of every
// line) sits in slot `slot_of(k)` as [l][cpitch], cpitch = 32*S padded so
// the lanes of a half-warp hit distinct banks; lane 0 moves a chunk with one
// bulk copy per line (1 KB at S=4). Same slot recycling as the y/z kernel.
// ---------------------------------------------------------------------------
struct XSweep {
    double* rho;
    Coef coef;
    long long lines; // ny*nz
    long long tiles; // ceil(lines / L)
    long long lines_per_rep; // ny*nz (ensembles stack replicas along the lines)
    int nx, ny, nz, S;
    int rowlen;      // nx*S
    int cpitch;      // smem doubles per line within a chunk slot
    int pitch;       // (plain kernel) smem doubles per whole line
    int L;           // lines per tile (L*S <= 32)
    Clamp clamp;
};

template <bool CLAMP>
static __global__ void __launch_bounds__(kLanes) sweep_x_bulk(XSweep a)
{
    extern __shared__ __align__(128) unsigned char smem[];
    const int nch = (a.nx + kChunk - 1) / kChunk;
    const int S = a.S;
    const int slot_sz = a.L * a.cpitch;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
    double* slots = reinterpret_cast<double*>(smem + bar_bytes(nch));
    const int lane = threadIdx.x;
    long long t = blockIdx.x;
    if (t >= a.tiles) return;

    auto lines_in = [&](long long tile) {
        return static_cast<int>(min(static_cast<long long>(a.L), a.lines - tile * a.L));
    };
    auto issue = [&](long long tile, int k, int slot, bool load) {
        const int nl = lines_in(tile);
        const int cnt = min(kChunk, a.nx - k * kChunk);
        const int off = k * kChunk * S;
        const uint32_t bytes = static_cast<uint32_t>(cnt * S * 8);
        double* g = a.rho + tile * a.L * a.rowlen + off;
        double* sm = slots + slot * slot_sz;
        if (load) ptx::mbar_arrive_expect_tx(&bars[slot], nl * bytes);
        for (int l = 0; l < nl; ++l) {
            if (load)
                ptx::bulk_g2s(sm + l * a.cpitch, g + static_cast<long long>(l) * a.rowlen, bytes, &bars[slot]);
            else
                ptx::bulk_s2g(g + static_cast<long long>(l) * a.rowlen, sm + l * a.cpitch, bytes);
        }
    };
    if (lane == 0) {
        for (int k = 0; k < nch; ++k) ptx::mbar_init(&bars[k], 1);
        ptx::fence_mbar_init();
        for (int k = 0; k < nch; ++k) issue(t, k, k, true);
    }
    __syncwarp();

    for (int it = 0; t < a.tiles; ++it) {
        const long long tnext = t + gridDim.x;
        const bool rev = it & 1;
        const uint32_t phase = it & 1;
        auto slot_of = [&](int k) { return rev ? nch - 1 - k : k; };
        const int nl = lines_in(t);
        const bool active = lane < nl * S;
        const int l = active ? lane / S : 0;
        const int s = active ? lane % S : 0;
        const long long line = t * a.L + l;
        const int j = static_cast<int>(line % a.ny), kk = static_cast<int>(line / a.ny);
        const Chain c = make_chain(a.coef, S, s, a.nx, a.clamp, j == 0 || j == a.ny - 1 || kface(kk, a.clamp));
        solve_chunked<CLAMP>(
            c, active, S, [&](int k) { return slots + slot_of(k) * slot_sz + l * a.cpitch + s; },
            [&](int k) { ptx::mbar_wait(&bars[slot_of(k)], phase); },
            [&](int k) {
                ptx::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    issue(t, k, slot_of(k), false);
                    ptx::bulk_commit();
                    if (tnext < a.tiles) {
                        if (k < nch - 1) {
                            ptx::bulk_wait_read<1>();
                            issue(tnext, nch - 1 - (k + 1), slot_of(k + 1), true);
                        }
                        if (k == 0) {
                            ptx::bulk_wait_read<0>();
                            issue(tnext, nch - 1, slot_of(0), true);
                        }
                    }
                }
            });
        t = tnext;
    }
    if (lane == 0) ptx::bulk_wait_read<0>();
}

// Whole lines in shared memory without bulk copies (odd nx*S). One tile per CTA.
static __global__ void __launch_bounds__(kLanes) sweep_x_plain(XSweep a, bool clamp)
{
    extern __shared__ __align__(128) unsigned char smem[];
    double* tile = reinterpret_cast<double*>(smem);
    const int lane = threadIdx.x;
    const long long line0 = static_cast<long long>(blockIdx.x) * a.L;
    const int nl = static_cast<int>(min(static_cast<long long>(a.L), a.lines - line0));
    const int S = a.S;
    double* base = a.rho + line0 * a.rowlen;
    for (int idx = lane; idx < nl * a.rowlen; idx += kLanes)
        tile[(idx / a.rowlen) * a.pitch + idx % a.rowlen] = base[idx];
    __syncwarp();
    const bool active = lane < nl * S;
    const int l = active ? lane / S : 0;
    const int s = active ? lane % S : 0;
    const long long line = line0 + l;
    const int j = static_cast<int>(line % a.ny), kk = static_cast<int>(line / a.ny);
    const Chain c = make_chain(a.coef, S, s, a.nx, a.clamp, j == 0 || j == a.ny - 1 || kface(kk, a.clamp));
    auto ptr = [&](int k) { return tile + l * a.pitch + k * kChunk * S + s; };
    auto none = [](int) {};
    if (clamp)
        solve_chunked<true>(c, active, S, ptr, none, none);
    else
        solve_chunked<false>(c, active, S, ptr, none, none);
    __syncwarp();
    for (int idx = lane; idx < nl * a.rowlen; idx += kLanes)
        base[idx] = tile[(idx / a.rowlen) * a.pitch + idx % a.rowlen];
}

// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// Ring-buffered sweeps with backward recompute (default tile path).
//
// The resident-line kernels above keep a whole line per chain in shared
// memory, which caps residency at ~3 warps per SM (64 KB per 32 chains at
// n = 256) and leaves the FP64 recurrences latency-bound. Here a warp keeps
// only a ring of NS chunk slots (8 KB each) plus one checkpoint per chunk:
//   forward : chunks stream through the ring (TMA / bulk loads, NS deep);
//             the forward value at each chunk end is checkpointed;
//   backward: the last NS chunks are still resident (their forward values
//             are in the ring); every earlier chunk is reloaded (an L2 hit:
//             it was read a few microseconds earlier) and its forward values
//             recomputed from the previous chunk's checkpoint — the same
//             operations in the same order, so the result is bit-identical —
//             then back-substituted and stored.
// HBM traffic stays one read + one write per value; L2 serves the reloads.
// ---------------------------------------------------------------------------
// Boundary-plane exports of the z-slab decomposition (nullptr members = off):
// bottom[idx] <- forward value of the last row, top[idx] <- unclamped final
// value of row 0.
struct SlabExport {
    double* bottom;
    double* top;
    long long idx;
};

template <bool CLAMP, class Ptr, class Load, class Store>
__device__ __forceinline__ void solve_ring(const Chain& c, bool active, int step, int NS, uint64_t* bars, double* ckpt,
                                           int lane, Ptr ptr, Load load, Store store,
                                           const SlabExport* exp = nullptr)
{
    const int n = c.n;
    const int nch = (n + kChunk - 1) / kChunk;
    uint32_t parity = 0; // expected phase parity per slot
    auto wait_slot = [&](int s) {
        ptx::mbar_wait(&bars[s], (parity >> s) & 1u);
        parity ^= (1u << s);
    };
    // Forward loads of chunks that will be reloaded are kept in L2
    // (evict_last); everything else streams (evict_first).
    if (lane == 0)
        for (int k = 0; k < min(NS, nch); ++k) load(k, k, k < nch - NS);
    __syncwarp();

    // Forward elimination with per-chunk checkpoints.
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
        if (k + NS < nch) { // recycle the slot for chunk k+NS (chunk k will be recomputed)
            ptx::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) load(k + NS, s, k + NS < nch - NS);
        }
    }

    // z-slab: the forward value of the last row goes to the next slab.
    if (exp && active && exp->bottom) exp->bottom[exp->idx] = prev;

    // Back substitution, top chunk first.
    double next = prev; // final value of position n-1
    const int first_reloaded = nch - NS - 1; // highest chunk that must be reloaded
    if (CLAMP && active && c.clamp_s && (c.face || c.face_hi))
        ptr((nch - 1) % NS)[((n - 1) - (nch - 1) * kChunk) * step] = c.clamp_v;
    for (int k = nch - 1; k >= 0; --k) {
        const int s = k % NS;
        const int m0 = k * kChunk;
        const int m1 = min(n, m0 + kChunk);
        if (k <= first_reloaded) {
            wait_slot(s);
            if (active) { // recompute the forward values of chunk k
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
            // The store of chunk k+1 (one step earlier) has read its slot by
            // now: reload chunk k+1-NS into it for the recompute.
            const int kr = k + 1 - NS;
            if (k + 1 < nch && kr >= 0 && kr <= first_reloaded) {
                ptx::bulk_wait_read<1>();
                load(kr, kr % NS, false);
            }
        }
    }
    // z-slab: the unclamped back-substituted value of row 0 goes to the previous slab.
    if (exp && active && exp->top) exp->top[exp->idx] = next;
    if (lane == 0) ptx::bulk_wait_read<0>();
}

struct Ring {
    int ns;    // slots
    int nch;   // chunks per line
    int hints; // use L2 eviction-priority hints
};

template <bool CLAMP>
static __global__ void __launch_bounds__(kLanes) sweep_yz_ring(const __grid_constant__ CUtensorMap tmap, StridedSweep a, Ring rg)
{
    extern __shared__ __align__(128) unsigned char smem[];
    constexpr int kSlot = kChunk * kLanes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
    double* slots = reinterpret_cast<double*>(smem + bar_bytes(rg.ns));
    double* ckpt = slots + rg.ns * kSlot;
    const int lane = threadIdx.x;
    const int t = blockIdx.x;
    const int e0 = (t % a.tiles_per_row) * kLanes;
    const int outer_all = t / a.tiles_per_row;
    const int r = outer_all / a.n_outer; // ensemble replica
    const int outer = outer_all % a.n_outer;
    const int width = min(kLanes, a.rowlen - e0);
    if (lane == 0) {
        ptx::tma_prefetch_desc(&tmap);
        for (int s = 0; s < rg.ns; ++s) ptx::mbar_init(&bars[s], 1);
        ptx::fence_mbar_init();
    }
    __syncwarp();
    auto box = [&](int k, int& c1, int& c2) {
        c1 = a.axis == 2 ? outer : k * kChunk;
        c2 = a.axis == 2 ? k * kChunk : outer;
    };
    const bool active = lane < width;
    const int e = e0 + (active ? lane : 0);
    const int s = e % a.S, i = e / a.S;
    const Chain c = make_chain_yz(a, s, i, outer, r);
    const uint64_t keep_pol = ptx::policy_evict_last(), stream_pol = ptx::policy_evict_first();
    // Plane index of this column for the z-slab exports (z axis: outer = j).
    const SlabExport ex{a.exp_bottom, a.exp_top, static_cast<long long>(outer) * a.rowlen + e};
    solve_ring<CLAMP>(
        c, active, kLanes, rg.ns, bars, ckpt, lane, [&](int slot) { return slots + slot * kSlot + lane; },
        [&](int k, int slot, bool keep) {
            int c1, c2;
            box(k, c1, c2);
            ptx::mbar_arrive_expect_tx(&bars[slot], kSlot * 8);
            if (rg.hints)
                ptx::tma_load_4d_hint(slots + slot * kSlot, &tmap, e0, c1, c2, r, &bars[slot],
                                      keep ? keep_pol : stream_pol);
            else
                ptx::tma_load_4d(slots + slot * kSlot, &tmap, e0, c1, c2, r, &bars[slot]);
        },
        [&](int k, int slot) {
            int c1, c2;
            box(k, c1, c2);
            if (rg.hints)
                ptx::tma_store_4d_hint(&tmap, e0, c1, c2, r, slots + slot * kSlot, stream_pol);
            else
                ptx::tma_store_4d(&tmap, e0, c1, c2, r, slots + slot * kSlot);
        },
        &ex);
}

template <bool CLAMP>
static __global__ void __launch_bounds__(kLanes) sweep_x_ring(XSweep a, Ring r)
{
    extern __shared__ __align__(128) unsigned char smem[];
    const int S = a.S;
    const int slot_sz = a.L * a.cpitch;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
    double* slots = reinterpret_cast<double*>(smem + bar_bytes(r.ns));
    double* ckpt = slots + r.ns * slot_sz;
    const int lane = threadIdx.x;
    const long long t = blockIdx.x;
    const int nl = static_cast<int>(min(static_cast<long long>(a.L), a.lines - t * a.L));
    if (lane == 0) {
        for (int s = 0; s < r.ns; ++s) ptx::mbar_init(&bars[s], 1);
        ptx::fence_mbar_init();
    }
    __syncwarp();
    double* gbase = a.rho + t * a.L * a.rowlen;
    const bool active = lane < nl * S;
    const int l = active ? lane / S : 0;
    const int sub = active ? lane % S : 0;
    const long long line = t * a.L + l;
    const int rep = static_cast<int>(line / a.lines_per_rep); // ensemble replica of this lane's line
    const long long rline = line % a.lines_per_rep;
    const int j = static_cast<int>(rline % a.ny), kk = static_cast<int>(rline / a.ny);
    const Chain c = make_chain(a.coef, S, sub, a.nx, a.clamp, j == 0 || j == a.ny - 1 || kface(kk, a.clamp), rep);
    const uint64_t keep_pol = ptx::policy_evict_last(), stream_pol = ptx::policy_evict_first();
    auto bytes_of = [&](int k) { return static_cast<uint32_t>(min(kChunk, a.nx - k * kChunk) * S * 8); };
    solve_ring<CLAMP>(
        c, active, S, r.ns, bars, ckpt, lane, [&](int slot) { return slots + slot * slot_sz + l * a.cpitch + sub; },
        [&](int k, int slot, bool keep) {
            const uint32_t bytes = bytes_of(k);
            ptx::mbar_arrive_expect_tx(&bars[slot], nl * bytes);
            const uint64_t pol = keep ? keep_pol : stream_pol;
            for (int ll = 0; ll < nl; ++ll) {
                double* d = slots + slot * slot_sz + ll * a.cpitch;
                const double* g = gbase + static_cast<long long>(ll) * a.rowlen + k * kChunk * S;
                if (r.hints)
                    ptx::bulk_g2s_hint(d, g, bytes, &bars[slot], pol);
                else
                    ptx::bulk_g2s(d, g, bytes, &bars[slot]);
            }
        },
        [&](int k, int slot) {
            const uint32_t bytes = bytes_of(k);
            for (int ll = 0; ll < nl; ++ll) {
                double* g = gbase + static_cast<long long>(ll) * a.rowlen + k * kChunk * S;
                const double* d = slots + slot * slot_sz + ll * a.cpitch;
                if (r.hints)
                    ptx::bulk_s2g_hint(g, d, bytes, stream_pol);
                else
                    ptx::bulk_s2g(g, d, bytes);
            }
        });
}

// Any-axis sweep straight from global memory, one thread per chain. Used for
// lines too long for a shared-memory tile. The forward intermediates are
// written in place and re-read by the backward pass (L2-resident when the
// in-flight set of lines fits in L2).
// ---------------------------------------------------------------------------
struct GlobalSweep {
    double* rho;
    const double* q;
    const double* dinv;
    const double* cb;
    int axis;
    int nx, ny, nz, S;
    int n;            // line length
    long long chains; // total chains
    Clamp clamp;
};

template <bool CLAMP>
static __global__ void __launch_bounds__(128) sweep_global(GlobalSweep a)
{
    const long long chain = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (chain >= a.chains) return;
    const int S = a.S;
    const long long row = static_cast<long long>(a.nx) * S;
    const long long plane = row * a.ny;
    long long base_off, stride;
    int i = 0, j = 0, k = 0, s;
    if (a.axis == 0) {
        const long long line = chain / S;
        s = static_cast<int>(chain % S);
        base_off = line * row + s;
        stride = S;
        j = static_cast<int>(line % a.ny);
        k = static_cast<int>(line / a.ny);
    } else {
        const long long e = chain % row;
        const long long outer = chain / row;
        s = static_cast<int>(e % S);
        i = static_cast<int>(e / S);
        if (a.axis == 1) {
            k = static_cast<int>(outer);
            base_off = outer * plane + e;
            stride = row;
        } else {
            j = static_cast<int>(outer);
            base_off = outer * row + e;
            stride = plane;
        }
    }
    double* p = a.rho + base_off;
    const double qs = a.q[s];
    const double* dinv = a.dinv + s;
    const double* cb = a.cb + s;
    const int n = a.n;

    double prev = fwd_first(p[0], __ldg(dinv));
    p[0] = prev;
    int m = 1;
    for (; m + 8 <= n; m += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = p[(m + u) * stride];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            prev = fwd(v[u], prev, qs, __ldg(dinv + (m + u) * S));
            p[(m + u) * stride] = prev;
        }
    }
    for (; m < n; ++m) {
        prev = fwd(p[m * stride], prev, qs, __ldg(dinv + m * S));
        p[m * stride] = prev;
    }

    bool clamp_s = false;
    double clamp_v = 0.0;
    if (CLAMP) {
        clamp_s = (a.clamp.mask >> s) & 1ull;
        clamp_v = a.clamp.values[s];
    }
    auto is_face = [&](int mm) {
        int ii = i, jj = j, kk = k;
        if (a.axis == 0) ii = mm;
        else if (a.axis == 1) jj = mm;
        else kk = mm;
        return ii == 0 || ii == a.nx - 1 || jj == 0 || jj == a.ny - 1 || kface(kk, a.clamp);
    };
    double next = prev;
    if (CLAMP && clamp_s && is_face(n - 1)) p[(n - 1) * stride] = clamp_v;
    m = n - 2;
    for (; m - 7 >= 0; m -= 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = p[(m - u) * stride];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            next = bwd(v[u], next, __ldg(cb + (m - u) * S));
            p[(m - u) * stride] = (CLAMP && clamp_s && is_face(m - u)) ? clamp_v : next;
        }
    }
    for (; m >= 0; --m) {
        next = bwd(p[m * stride], next, __ldg(cb + m * S));
        p[m * stride] = (CLAMP && clamp_s && is_face(m)) ? clamp_v : next;
    }
}

// Masked overwrite of Dirichlet entries (solver.cpp:267-275); one thread per
// (entry, substrate). Entries are unique voxels, so order is irrelevant.
static __global__ void dirichlet_entries(double* rho, int S, long long count, const int64_t* voxel,
                                  const unsigned char* mask, const double* values)
{
    ptx::griddep_wait();
    ptx::griddep_launch();
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= count * S) return;
    if (mask[t]) rho[voxel[t / S] * S + (t % S)] = values[t];
}

// cell_sources_sinks_step (agents.cpp:75-112): one thread per (voxel group,
// substrate); the group's agents are applied in ascending-id order. The
// substrates of one agent update independently, so (group, s) threads
// reproduce the reference's agent-outer / substrate-inner loop bitwise.
// Per-agent, per-substrate factors of the implicit update for one dt:
// add = (f*sec)*target and den = 1 + f*(sec+upt), f = (dt*V)*inv_vox
// (agents.cpp:102-107). They do not depend on the density, so computing them
// once per dt and reusing them is bit-identical to the reference.
static __global__ void sources_factors(int S, long long agents, const double* volume, const double* secretion,
                                const double* uptake, const double* saturation, double dt, double inv_voxel_volume,
                                double* add, double* den)
{
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= agents * S) return;
    const long long m = t / S;
    const double f = __dmul_rn(__dmul_rn(dt, volume[m]), inv_voxel_volume);
    const double sec = secretion[t];
    add[t] = __dmul_rn(__dmul_rn(f, sec), saturation[t]);
    den[t] = __dadd_rn(1.0, __dmul_rn(f, __dadd_rn(sec, uptake[t])));
}

// One thread per (voxel group, substrate); the group's agents are applied in
// ascending-id order: x <- (x + add) / den. Agents of distinct voxels commute
// and substrates are independent, so (group, s) threads reproduce the
// reference's agent-outer / substrate-inner loop bitwise. Groups are in
// (voxel) order, built on the device (agents.cu); [*g_lo, *g_hi) is the group
// range to apply — all groups of the last rebuild, or one replica batch's —
// read from device memory (the grid covers the agent capacity of the range).
static __global__ void sources_groups(double* rho, int S, const int64_t* g_lo, const int64_t* g_hi,
                               const int64_t* group_voxel, const int64_t* group_offsets, const double* add,
                               const double* den)
{
    ptx::griddep_wait();
    ptx::griddep_launch();
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const long long g0 = *g_lo;
    if (t >= (*g_hi - g0) * S) return;
    const long long g = g0 + t / S;
    const int s = static_cast<int>(t % S);
    double* r = rho + group_voxel[g] * S + s;
    double x = *r;
    long long m = group_offsets[g];
    const long long a1 = group_offsets[g + 1];
    for (; m + 4 <= a1; m += 4) {
        double a[4], d[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            a[u] = add[(m + u) * S + s];
            d[u] = den[(m + u) * S + s];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) x = __ddiv_rn(__dadd_rn(x, a[u]), d[u]);
    }
    for (; m < a1; ++m) x = __ddiv_rn(__dadd_rn(x, add[m * S + s]), den[m * S + s]);
    *r = x;
}

// ---------------------------------------------------------------------------
// z-slab partitioned solve. With zero inflow at its ends a
// slab's z-lines have forward value dhat at the last row and back-substituted
// value xhat0 at row 0 (zslab_interface, one read of the slab). By linearity,
// with d_in = D_{p-1} (the true forward value of the previous slab's last row)
// and x_in = X_{p+1} (the true final value of the next slab's first row):
//   forward value at the last row = dhat + phi_last * d_in,
//   final value at row 0          = xhat0 + Phi_0 * d_in + Psi_0 * x_in,
// with phi / Phi / Psi the slab's RHS-independent responses to unit inflows
// (host-computed). The two plane chains below give every D and X exactly (no
// truncation of cross-slab couplings); the z sweep then runs the global
// recurrence itself on the slab with D_{p-1} / X_{p+1} as boundary values
// (StridedSweep::in_lo / in_hi), so no correction pass over the slab is
// needed: per step a slab moves 8 B/vsu more than a single domain, not 16.
// ---------------------------------------------------------------------------

// Exact interface recurrences (two plane chains across the slabs):
//   D_p = dhat_p(last row) + phi_p(last row) * D_{p-1}          (forward, p = 0..P-1)
//   X_p = xhat_p(row 0) + Phi_p(row 0) * D_{p-1} + Psi_p(row 0) * X_{p+1}   (backward)
// D_{-1} = X_P = 0. D_p is the true forward value of slab p's last row, X_p
// the true unclamped final value of its first row.
static __global__ void zslab_fwdfix(double* d_out, const double* dhat_bottom, const double* d_in,
                                    const double* phi_last, long long plane, int S)
{
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= plane) return;
    d_out[t] = __dadd_rn(dhat_bottom[t], __dmul_rn(phi_last[t % S], d_in[t]));
}

static __global__ void zslab_topfix(double* x_out, const double* xhat_top, const double* d_in, const double* x_in,
                                    const double* Phi, const double* Psi, long long plane, int S)
{
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= plane) return;
    const int s = static_cast<int>(t % S);
    x_out[t] = __dadd_rn(__dadd_rn(xhat_top[t], __dmul_rn(Phi[s], d_in[t])), __dmul_rn(Psi[s], x_in[t]));
}

// Interface pre-pass of a slab, one thread per column (i, j, s), zero
// inflow at both slab ends, ONE read of the slab:
//   dhat  = forward value of the last row (the zero-inflow recurrence);
//   xhat0 = back-substituted value of row 0 = sum_m (prod_{k<m} cb_k) f_m,
// the back substitution x_m = f_m + cb_m x_{m+1} (x_{n-1} = f_{n-1}) unrolled
// into the forward pass (all terms share the field's sign: no cancellation).
static __global__ void zslab_interface(const double* rho, long long plane, int n, int S, const double* q,
                                       const double* dinv, const double* cb, double* dhat, double* xhat0)
{
    for (long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; t < plane;
         t += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int s = static_cast<int>(t % S);
        const double qs = q[s];
        double f = 0.0, acc = 0.0, prod = 1.0;
#pragma unroll 8
        for (int m = 0; m < n; ++m) {
            const double v = rho[m * plane + t];
            const double d = __ldg(dinv + static_cast<long long>(m) * S + s);
            f = m == 0 ? fwd_first(v, d) : fwd(v, f, qs, d);
            acc = __dadd_rn(acc, __dmul_rn(prod, f));
            prod = __dmul_rn(prod, __ldg(cb + static_cast<long long>(m) * S + s));
        }
        dhat[t] = f;
        xhat0[t] = acc;
    }
}


// DensityField::all_finite (mesh.cpp:95-99): flag = 1 if any value is NaN/inf.
static __global__ void any_nonfinite(const double* a, long long n, int* flag)
{
    int bad = 0;
    for (long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; t < n;
         t += static_cast<long long>(gridDim.x) * blockDim.x)
        bad |= !isfinite(a[t]);
    bad = __any_sync(0xffffffffu, bad);
    if (bad && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

// values[v*S + s] = initial[s] for every voxel (grid-stride).
static __global__ void fill_field(double* rho, long long total, const double* initial, int S)
{
    for (long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
         t += static_cast<long long>(gridDim.x) * blockDim.x)
        rho[t] = initial[t % S];
}

// cross_check (validation.cpp:112-137) reductions. Non-negative doubles
// order like their bit patterns, so atomicMax on the bits is exact. NaN
// differences behave as in the reference: every comparison with NaN is false,
// so they neither fail the check nor enter max_abs / max_rel (fmax drops NaN
// exactly like std::max(current, NaN) keeps `current`).
static __global__ void cross_check_max(const double* a, const double* b, long long n, unsigned long long* max_abs_bits,
                                unsigned long long* max_rel_bits, double abs_tol, double rel_tol, int* fail)
{
    double my_abs = 0.0, my_rel = 0.0;
    int my_fail = 0;
    for (long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; t < n;
         t += static_cast<long long>(gridDim.x) * blockDim.x) {
        const double av = a[t], bv = b[t];
        const double diff = fabs(av - bv);
        const double mag = fmax(fabs(av), fabs(bv));
        const double rel = (diff == 0.0 || mag == 0.0) ? 0.0 : diff / mag;
        my_abs = fmax(my_abs, diff);
        my_rel = fmax(my_rel, rel);
        if (diff > abs_tol + rel_tol * mag) my_fail = 1;
    }
    for (int o = 16; o > 0; o >>= 1) {
        my_abs = fmax(my_abs, __shfl_xor_sync(0xffffffffu, my_abs, o));
        my_rel = fmax(my_rel, __shfl_xor_sync(0xffffffffu, my_rel, o));
        my_fail |= __shfl_xor_sync(0xffffffffu, my_fail, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(max_abs_bits, static_cast<unsigned long long>(__double_as_longlong(my_abs)));
        atomicMax(max_rel_bits, static_cast<unsigned long long>(__double_as_longlong(my_rel)));
        if (my_fail) atomicOr(fail, 1);
    }
}

static __global__ void cross_check_argmax(const double* a, const double* b, long long n, const unsigned long long* max_abs_bits,
                                   unsigned long long* worst)
{
    const double target = __longlong_as_double(static_cast<long long>(*max_abs_bits));
    for (long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; t < n;
         t += static_cast<long long>(gridDim.x) * blockDim.x) {
        const double diff = fabs(a[t] - b[t]);
        if (diff == target && target > 0.0) atomicMin(worst, static_cast<unsigned long long>(t));
    }
}

} // namespace kernels
} // namespace biodiff_b200
