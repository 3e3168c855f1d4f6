// Resident multi-step kernel for grids that live in L2 (the paper's own
// 50^3 / 100^3 workloads, BASELINE.json configs[0..1]).
//
// At these sizes a step is not bound by HBM (the whole field, 1-16 MB, sits
// in the 126 MB L2) but by the three dependent sweeps' chain latency and by
// launch gaps. ONE cooperative launch runs all `steps` steps of an advance(),
// with no grid-wide barrier: every warp tile waits only for the tiles it
// reads, through counters (one per 128-byte line, polled with relaxed loads
// and back-off, acquired once):
//
//   x tile (32/S lines)   waits: the previous step's z tiles and sources of
//                         each line's row j; signals cnt_x[k] += its lines of plane k
//   y tile (plane k, 32 (i,s) columns)  waits: cnt_x[k] == ny lines this step;
//                         signals cnt_y[r] += 1
//   z tile (row j, 32 (i,s) columns)    waits: cnt_y[r] == nz planes this step;
//                         shell clamp fused, then the residual Dirichlet
//                         entries of its voxels; signals cnt_z[j] += 1
//   sources chunk (32/S listed (z tile, group) entries, one item per lane)
//                         waits: the z tiles of its rows; signals cnt_src[j]
//
// Tiles are assigned statically (warp rank = warp-in-block * grid + block,
// so consecutive tiles land on different SMs) and every warp walks its tiles
// in (step, phase) order; a tile only ever waits on tiles of an earlier
// (step, phase), so the dataflow cannot deadlock among co-resident warps.
// Every lane owns one chain (line x substrate) in a private shared-memory
// column c[m*32]: y / z tiles arrive by four TMA boxes (one mbarrier each, so
// the forward pass starts when the first quarter has landed), x tiles by
// LDGSTS in four commit groups; the forward values stay in the column and
// the back substitution reads them (no recompute). The chains run in
// branch-free register blocks of 8 positions; the pivots live in shared memory.
//
// Numerics are the reference's, in its order (kernels.cuh fwd_first / fwd /
// bwd = solver.cpp:17-19; rows of the settled region use the host-verified
// bit-constant pivots; the shell clamp on the stored value after the last
// sweep, residual Dirichlet entries, then the sources in ascending agent id
// per (voxel, substrate): solver.cpp:289-299, agents.cpp:97-109). Per voxel
// that is the reference's order (clamp, Dirichlet, sources), and distinct
// voxels / substrates commute, so results are bit-identical to the reference.
//
// Design probe: BIODIFF_RES_TRACE=<file> records per-tile globaltimer stamps
// of the first 8 steps (tools/resident_trace_probe.py).
#pragma once

#include "kernels.cuh"

namespace biodiff_b200 {
namespace kernels {

struct ResAxis {
    const double* q;      // [S]
    const double* dinv;   // [n*S]
    const double* cb;     // [n*S]
    const double* dconst; // [S] rows [settle, n-2]
    const double* cconst; // [S]
    int settle;
    int n;
};

struct Resident {
    double* rho;
    int nx, ny, nz, S;
    int tpr;                  // 32-wide (i, s) ranges per row: ceil(nx*S / 32)
    ResAxis ax[3];
    Clamp clamp;
    // Residual Dirichlet entries and agent groups, listed per z tile (j, r)
    // (res_list_* kernels): tile t's items are idx[off[t] .. off[t+1]).
    int dirichlet;
    const int* zdir_off;
    const int* zdir_idx;
    const int64_t* dir_voxel;
    const unsigned char* dir_mask;
    const double* dir_values;
    int sources;
    const int* zgrp_off;
    const int* zgrp_idx;
    const int* zgrp_tile;     // z tile of each listed group entry
    const struct ResSrc* zsrc; // descriptor of each listed group entry
    const int64_t* group_voxel;
    const int64_t* group_offsets;
    const double* add;        // per-agent factors (sources_factors), group order
    const double* den;
    long long steps;
    unsigned* cnt;            // [nz] x lines per plane | [tpr] y tiles per range | [ny] z tiles per row |
                              // [ny] source entries per row, kCntPad apart; zeroed before the launch
    int buf_doubles;          // shared doubles per warp: 32 * max(nx, ny, nz)
    int coef_doubles;         // every axis' dinv / cb, copied into shared memory at launch
    int tma;                  // y / z tiles load through the tensor maps (rows of 16-byte multiples)
    unsigned long long* trace; // design probe (BIODIFF_RES_TRACE): [step<8][x,y,z,src][tile][6] globaltimer stamps
    long long trace_tiles;
};

__device__ __forceinline__ unsigned long long res_clock()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define RES_STAMP(AX, I)                                                                                            \
    if (a.trace && st < 8 && lane == 0) a.trace[((st * 4 + (AX)) * a.trace_tiles + t) * 6 + (I)] = res_clock();
#define RES_TS(AX) (a.trace && st < 8 && lane == 0 ? a.trace + ((st * 4 + (AX)) * a.trace_tiles + t) * 6 : nullptr)

// Counters, one per 128-byte line: polls of different counters then hit
// different L2 lines (slices) instead of hammering one.
constexpr int kCntPad = 32;
__device__ __forceinline__ unsigned* cnt_x(const Resident& a, long long k) { return a.cnt + k * kCntPad; }
__device__ __forceinline__ unsigned* cnt_y(const Resident& a, int r) { return a.cnt + (a.nz + r) * kCntPad; }
__device__ __forceinline__ unsigned* cnt_zr(const Resident& a, int j)
{
    return a.cnt + static_cast<long long>(a.nz + a.tpr + j) * kCntPad;
}
__device__ __forceinline__ unsigned* cnt_src(const Resident& a, int j)
{
    return a.cnt + static_cast<long long>(a.nz + a.tpr + a.ny + j) * kCntPad;
}

// Polls with relaxed loads (a gpu-scope acquire per poll would flush the
// SM's L1 every time: CCTL.IVALL, B300_MICROARCH.md "L1 data cache") and
// acquires once when the count is reached.
__device__ __forceinline__ void res_wait(const unsigned* c, unsigned target)
{
    unsigned v, ns = 32;
    for (;;) {
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(c) : "memory");
        if (static_cast<int>(v - target) >= 0) break;
        __nanosleep(ns);
        ns = min(2 * ns, 256u); // back off: thousands of waiting warps must not saturate the counters' L2 slices
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

// Issues the LDGSTS copies of one lane's chain (positions [0, n) at g[m*gst])
// into its shared column c[m*32], in four commit groups of P positions.
// y / z tiles with tensor maps (rows of 16-byte multiples): lane 0 issues
// four TMA boxes of (32 columns x P positions) into the warp's column block
// (box order = c[m*32 + lane]; columns past the row end and positions past n
// are zero-filled), each completing on its own mbarrier so the forward pass
// starts when the first quarter has landed.
// `phases` (warp-uniform) holds each barrier's next phase parity; the
// parities this tile waits on are returned, and the issued barriers flip
// (a short axis may leave its last barrier unused).
__device__ __forceinline__ uint32_t res_issue_tma(double* buf, const void* tmap, uint64_t* bars, int n, int P, int c0,
                                                  int fixed, bool z, int lane, uint32_t& phases)
{
    ptx::fence_proxy_async_smem(); // this warp's generic writes of the previous tile before the async overwrite
    __syncwarp();
    const uint32_t wait = phases;
    for (int g = 0; g < 4 && g * P < n; ++g) {
        if (lane == 0) {
            ptx::mbar_arrive_expect_tx(bars + g, static_cast<uint32_t>(kLanes) * P * 8);
            if (z) ptx::tma_load_4d(buf + g * P * kLanes, tmap, c0, fixed, g * P, 0, bars + g);
            else ptx::tma_load_4d(buf + g * P * kLanes, tmap, c0, g * P, fixed, 0, bars + g);
        }
        phases ^= 1u << g;
    }
    return wait;
}

__device__ __forceinline__ void res_issue(double* c, const double* g, long long gst, int n, int P, bool active,
                                          int W = kLanes)
{
#pragma unroll
    for (int G = 0; G < 4; ++G) {
        if (active) {
            const int m1 = min(n, (G + 1) * P);
            for (int m = G * P; m < m1; ++m) ptx::cp_async8(c + m * W, g + m * gst);
        }
        ptx::cp_async_commit();
    }
}

// The LDGSTS copies of a chain land in four commit groups of P positions;
// need(upto) waits until positions [0, upto) have landed.
struct ResLanded {
    int landed = 0, pend = 4, P, n;
    uint64_t* bars = nullptr; // TMA tiles: group g completes on bars[g], phase parity bit g of `parity`
    uint32_t parity = 0;
    __device__ __forceinline__ void need(int upto)
    {
        if (bars) {
            while (landed < upto) {
                ptx::mbar_wait(bars + (4 - pend), (parity >> (4 - pend)) & 1u);
                --pend;
                landed = pend == 0 ? n : landed + P;
            }
            return;
        }
        while (landed < upto) {
            --pend;
            switch (pend) {
            case 3: ptx::cp_async_wait<3>(); break;
            case 2: ptx::cp_async_wait<2>(); break;
            case 1: ptx::cp_async_wait<1>(); break;
            default: ptx::cp_async_wait<0>(); break;
            }
            landed = pend == 0 ? n : landed + P;
        }
    }
};

constexpr int kResB = 8; // positions per register block of the chains

// Shared-memory copies of every axis' pivots (derived from the kernel's
// dynamic shared array, so the chains issue LDS, not generic loads).
struct ResCoef {
    const double* dinv[3];
    const double* cb[3];
};

// Thomas solve of one lane's chain (substrate s) held in shared memory at
// c[m*W] (W = 32: column blocks; W = S: x-tile rows); dinv / cb point at the shared-memory copies of this axis'
// pivots (offset by s). Full blocks of kResB positions of the settled region
// (bit-constant pivots in registers, every row but the line's first ~settle
// and its last) run branch-free: 8 shared loads, the dependent FP64 chain,
// 8 stores; the unsettled rows run the same blocks with their pivots loaded
// alongside; leftovers go one position at a time. The final values go to
// the shared column (TO_SMEM: the z tile's Dirichlet entries and store pass
// follow) or straight to global memory (g, stride gst). clamp_any /
// clamp_all: the shell clamp of the line's ends / of every position (stored
// values only; the recurrence runs on the unclamped values).
template <bool TO_SMEM>
__device__ __forceinline__ void res_chain(double* c, int W, double* g, long long gst, int n, int P, int s, int S,
                                          const ResAxis& A, const double* dinv, const double* cb, bool clamp_any,
                                          bool clamp_all, double cv, unsigned long long* ts = nullptr,
                                          uint64_t* bars = nullptr, uint32_t parity = 0)
{
    if (ts) ts[3] = res_clock();
    constexpr int B = kResB;
    const double q = A.q[s];
    const double dc = A.dconst[s], cc = A.cconst[s];
    const int a = max(1, min(A.settle, n - 1)); // rows [1, a) load their pivot, [a, n-2] are settled
    ResLanded ld;
    ld.P = P;
    ld.n = n;
    ld.bars = bars;
    ld.parity = parity;
    // ---- forward elimination
    ld.need(1);
    double prev = fwd_first(c[0], dinv[0]);
    c[0] = prev;
    int m = 1;
    for (; m + B <= a; m += B) {
        ld.need(m + B);
        double v[B], d[B];
#pragma unroll
        for (int u = 0; u < B; ++u) {
            v[u] = c[(m + u) * W];
            d[u] = dinv[(m + u) * S];
        }
#pragma unroll
        for (int u = 0; u < B; ++u) {
            prev = fwd(v[u], prev, q, d[u]);
            c[(m + u) * W] = prev;
        }
    }
    for (; m < a; ++m) {
        ld.need(m + 1);
        prev = fwd(c[m * W], prev, q, dinv[m * S]);
        c[m * W] = prev;
    }
    for (; m + B <= n - 1; m += B) {
        ld.need(m + B);
        double v[B];
#pragma unroll
        for (int u = 0; u < B; ++u) v[u] = c[(m + u) * W];
#pragma unroll
        for (int u = 0; u < B; ++u) {
            prev = fwd(v[u], prev, q, dc);
            c[(m + u) * W] = prev;
        }
    }
    for (; m < n - 1; ++m) {
        ld.need(m + 1);
        prev = fwd(c[m * W], prev, q, dc);
        c[m * W] = prev;
    }
    ld.need(n);
    prev = fwd(c[(n - 1) * W], prev, q, dinv[(n - 1) * S]);
    if (ts) ts[4] = res_clock();
    // ---- back substitution; c_back rows [b, n-2] settled
    double next = prev; // final (unclamped) value of position n-1
    double* gq = g + (n - 1) * gst;
    if (TO_SMEM) c[(n - 1) * W] = clamp_any ? cv : prev; else *gq = clamp_any ? cv : prev;
    gq -= gst;
    const int b = max(A.settle, 0);
    m = n - 2;
    for (; m - (B - 1) >= b; m -= B) {
        double v[B];
#pragma unroll
        for (int u = 0; u < B; ++u) v[u] = c[(m - u) * W];
#pragma unroll
        for (int u = 0; u < B; ++u) {
            next = bwd(v[u], next, cc);
            const double o = clamp_all ? cv : next;
            if (TO_SMEM) c[(m - u) * W] = o; else { *gq = o; gq -= gst; }
        }
    }
    for (; m >= b; --m) {
        next = bwd(c[m * W], next, cc);
        const double o = clamp_all ? cv : next;
        if (TO_SMEM) c[m * W] = o; else { *gq = o; gq -= gst; }
    }
    for (; m - (B - 1) >= 0; m -= B) {
        double v[B], d[B];
#pragma unroll
        for (int u = 0; u < B; ++u) {
            v[u] = c[(m - u) * W];
            d[u] = cb[(m - u) * S];
        }
#pragma unroll
        for (int u = 0; u < B; ++u) {
            next = bwd(v[u], next, d[u]);
            const double o = clamp_all ? cv : next;
            if (TO_SMEM) c[(m - u) * W] = o; else { *gq = o; gq -= gst; }
        }
    }
    for (; m >= 0; --m) {
        next = bwd(c[m * W], next, cb[m * S]);
        const double o = clamp_all ? cv : next;
        if (TO_SMEM) c[m * W] = o; else { *gq = o; gq -= gst; }
    }
    if (clamp_any) {
        if (TO_SMEM) c[0] = cv; else g[0] = cv;
    }
    if (ts) ts[5] = res_clock();
}

__device__ __forceinline__ void res_x_tile(const Resident& a, const ResCoef& cf, double* buf, long long t, long long st,
                                           int lane)
{
    const int S = a.S, L = kLanes / S;
    const long long rowlen = static_cast<long long>(a.nx) * S;
    const long long nlines = static_cast<long long>(a.ny) * a.nz;
    const long long g0 = t * L;
    const int nl = static_cast<int>(min(static_cast<long long>(L), nlines - g0));
    const int l = lane / S, s = lane % S;
    const bool active = lane < L * S && l < nl;
    RES_STAMP(0, 0)
    if (st > 0 && active && s == 0) {
        const int j = static_cast<int>((g0 + l) % a.ny);
        res_wait(cnt_zr(a, j), static_cast<unsigned>(a.tpr * st));
        if (a.sources) {
            const long long items = a.zgrp_off[(j + 1) * a.tpr] - a.zgrp_off[j * a.tpr];
            res_wait(cnt_src(a, j), static_cast<unsigned>(items * st));
        }
    }
    __syncwarp();
    RES_STAMP(0, 1)
    const int n = a.nx;
    double* g = a.rho + (g0 + l) * rowlen + s;
    {
        // Column blocks via LDGSTS (measured faster than coalesced row copies
        // into padded rows, whose per-element index math costs more than the
        // 32-line gathers, and than per-line bulk copies, which serialise on
        // the TMA unit).
        const int P = (n + 3) / 4;
        double* c = buf + lane;
        res_issue(c, g, S, n, P, active);
        if (active)
            res_chain<false>(c, kLanes, g, S, n, P, s, S, a.ax[0], cf.dinv[0] + s, cf.cb[0] + s, false, false, 0.0,
                             RES_TS(0));
    }
    __syncwarp();
    RES_STAMP(0, 2)
    if (lane == 0) {
        const long long k0 = g0 / a.ny, k1 = (g0 + nl - 1) / a.ny;
        for (long long k = k0; k <= k1; ++k) {
            const long long lo = max(g0, k * a.ny), hi = min(g0 + nl, (k + 1) * a.ny);
            ptx::red_release_add(cnt_x(a, k), static_cast<unsigned>(hi - lo));
        }
    }
}

__device__ __forceinline__ void res_y_tile(const Resident& a, const ResCoef& cf, double* buf, long long t, long long st,
                                           int lane, const void* tmap, uint64_t* bars, uint32_t& phases)
{
    const int S = a.S;
    const long long rowlen = static_cast<long long>(a.nx) * S;
    const int k = static_cast<int>(t / a.tpr), r = static_cast<int>(t % a.tpr);
    const long long e = static_cast<long long>(r) * kLanes + lane;
    const bool active = e < rowlen;
    RES_STAMP(1, 0)
    if (lane == 0) res_wait(cnt_x(a, k), static_cast<unsigned>(static_cast<long long>(a.ny) * (st + 1)));
    __syncwarp();
    RES_STAMP(1, 1)
    const int n = a.ny, P = (n + 3) / 4;
    double* g = a.rho + static_cast<long long>(k) * a.ny * rowlen + e;
    double* c = buf + lane;
    uint32_t parity = 0;
    if (tmap) parity = res_issue_tma(buf, tmap, bars, n, P, r * kLanes, k, false, lane, phases);
    else res_issue(c, g, rowlen, n, P, active);
    if (active) {
        const int s = static_cast<int>(e % S);
        res_chain<false>(c, kLanes, g, rowlen, n, P, s, S, a.ax[1], cf.dinv[1] + s, cf.cb[1] + s, false, false, 0.0, RES_TS(1),
                         tmap ? bars : nullptr, parity);
    }
    __syncwarp();
    RES_STAMP(1, 2)
    if (lane == 0) ptx::red_release_add(cnt_y(a, r), 1u);
}

__device__ __forceinline__ void res_z_tile(const Resident& a, const ResCoef& cf, double* buf, long long t, long long st,
                                           int lane, const void* tmap, uint64_t* bars, uint32_t& phases)
{
    const int S = a.S;
    const long long rowlen = static_cast<long long>(a.nx) * S;
    const long long plane = static_cast<long long>(a.ny) * rowlen;
    const int j = static_cast<int>(t / a.tpr), r = static_cast<int>(t % a.tpr);
    const int e0 = r * kLanes;
    const long long e = e0 + lane;
    const bool active = e < rowlen;
    RES_STAMP(2, 0)
    if (lane == 0) res_wait(cnt_y(a, r), static_cast<unsigned>(static_cast<long long>(a.nz) * (st + 1)));
    __syncwarp();
    RES_STAMP(2, 1)
    const int n = a.nz, P = (n + 3) / 4;
    double* g = a.rho + static_cast<long long>(j) * rowlen + e;
    double* c = buf + lane;
    uint32_t parity = 0;
    if (tmap) parity = res_issue_tma(buf, tmap, bars, n, P, e0, j, true, lane, phases);
    else res_issue(c, g, plane, n, P, active);
    if (active) {
        const int i = static_cast<int>(e / S), s = static_cast<int>(e % S);
        const bool cs = (a.clamp.mask >> s) & 1ull;
        const bool face = i == 0 || i == a.nx - 1 || j == 0 || j == a.ny - 1;
        const double cv = cs ? a.clamp.values[s] : 0.0;
        if (a.dirichlet)
            res_chain<true>(c, kLanes, g, plane, n, P, s, S, a.ax[2], cf.dinv[2] + s, cf.cb[2] + s, cs, cs && face, cv, RES_TS(2),
                            tmap ? bars : nullptr, parity);
        else
            res_chain<false>(c, kLanes, g, plane, n, P, s, S, a.ax[2], cf.dinv[2] + s, cf.cb[2] + s, cs, cs && face, cv, RES_TS(2),
                             tmap ? bars : nullptr, parity);
    }
    __syncwarp();
    if (a.dirichlet) { // residual entries after the clamp (solver.cpp:298), before the sources
        const long long nxy = static_cast<long long>(a.nx) * a.ny;
        const int o0 = a.zdir_off[t], items = (a.zdir_off[t + 1] - o0) * S;
        for (int it = lane; it < items; it += kLanes) {
            const int q = a.zdir_idx[o0 + it / S], s = it % S;
            const long long v = a.dir_voxel[q];
            const int ee = static_cast<int>(v % a.nx) * S + s - e0;
            if (ee >= 0 && ee < kLanes && a.dir_mask[static_cast<long long>(q) * S + s])
                buf[(v / nxy) * kLanes + ee] = a.dir_values[static_cast<long long>(q) * S + s];
        }
        __syncwarp();
        if (active) {
#pragma unroll 4
            for (int m = 0; m < n; ++m) g[m * plane] = c[m * kLanes];
        }
        __syncwarp();
    }
    RES_STAMP(2, 2)
    if (lane == 0) ptx::red_release_add(cnt_zr(a, j), 1u);
}

// cell_sources_sinks_step over a chunk of listed (z tile, group) entries,
// one (entry, substrate) item per lane (agents.cpp:97-109: per (voxel,
// substrate) the group's agents in ascending id, x <- (x + add) / den), after
// the z tiles of the chunk's rows. Chunks balance the work (a tumour's core
// rows hold most of the groups); each entry carries a descriptor (voxel,
// agent range, z tile) so an item costs two dependent L2 round trips.
struct ResSrc {
    long long voxel;
    int m0, m1; // the group's agents [m0, m1) in group order (factor arrays)
};
__device__ __forceinline__ void res_src_tile(const Resident& a, long long t, long long st, int lane, int total)
{
    const int S = a.S, per = kLanes / S;
    const int q0 = static_cast<int>(t) * per, q1 = min(total, q0 + per);
    const int j0 = a.zgrp_tile[q0] / a.tpr, j1 = a.zgrp_tile[q1 - 1] / a.tpr;
    RES_STAMP(3, 0)
    for (int j = j0 + lane; j <= j1; j += kLanes) res_wait(cnt_zr(a, j), static_cast<unsigned>(a.tpr * (st + 1)));
    __syncwarp();
    RES_STAMP(3, 1)
    const int q = q0 + lane / S, s = lane % S;
    if (lane < per * S && q < q1) {
        const ResSrc d = a.zsrc[q];
        const int tile = a.zgrp_tile[q];
        if ((static_cast<int>(d.voxel % a.nx) * S + s) / kLanes == tile % a.tpr) { // else: the other tile's entry
            double* p = a.rho + d.voxel * S + s;
            double x = *p;
            int m = d.m0;
            for (; m + 4 <= d.m1; m += 4) { // the factors' loads off the dependent divide chain
                double ad[4], de[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    ad[u] = a.add[static_cast<long long>(m + u) * S + s];
                    de[u] = a.den[static_cast<long long>(m + u) * S + s];
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) x = __ddiv_rn(__dadd_rn(x, ad[u]), de[u]);
            }
            for (; m < d.m1; ++m)
                x = __ddiv_rn(__dadd_rn(x, a.add[static_cast<long long>(m) * S + s]), a.den[static_cast<long long>(m) * S + s]);
            *p = x;
        }
    }
    __syncwarp();
    RES_STAMP(3, 2)
    if (lane == 0)
        for (int j = j0; j <= j1; ++j) {
            const int lo = max(q0, a.zgrp_off[j * a.tpr]), hi = min(q1, a.zgrp_off[(j + 1) * a.tpr]);
            if (hi > lo) ptx::red_release_add(cnt_src(a, j), static_cast<unsigned>(hi - lo));
        }
}

// Descriptors of the listed group entries (after res_list_fill).
__global__ void res_src_desc(const int* idx, const int* off_end, const int64_t* group_voxel,
                             const int64_t* group_offsets, ResSrc* out)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= *off_end) return;
    const int gi = idx[t];
    out[t] = ResSrc{group_voxel[gi], static_cast<int>(group_offsets[gi]), static_cast<int>(group_offsets[gi + 1])};
}

__global__ void __launch_bounds__(128, 1) step_resident(const __grid_constant__ CUtensorMap tmap_y,
                                                       const __grid_constant__ CUtensorMap tmap_z, Resident a)
{
    extern __shared__ __align__(128) double smem_res[];
    const int lane = threadIdx.x % kLanes;
    const int wib = threadIdx.x / kLanes;
    const long long W = static_cast<long long>(gridDim.x) * (blockDim.x / kLanes);
    const long long rank = static_cast<long long>(wib) * gridDim.x + blockIdx.x;
    // [4 mbarriers per warp, 128 B][coefficients][per-warp column blocks, 128-byte aligned]
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_res) + 4 * wib;
    double* buf = smem_res + 16 * (blockDim.x / kLanes) + a.coef_doubles + static_cast<long long>(wib) * a.buf_doubles;
    if (lane == 0)
        for (int g = 0; g < 4; ++g) ptx::mbar_init(bars + g, 1);
    ptx::fence_mbar_init();
    __syncwarp();
    uint32_t phases = 0; // next phase parity of each of the warp's 4 mbarriers
    // The pivots of unsettled rows are read inside the chains: keep them on chip.
    ResCoef cf;
    {
        double* cs = smem_res + 16 * (blockDim.x / kLanes);
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
            const int len = a.ax[ax].n * a.S;
            for (int i = threadIdx.x; i < len; i += blockDim.x) {
                cs[i] = a.ax[ax].dinv[i];
                cs[len + i] = a.ax[ax].cb[i];
            }
            cf.dinv[ax] = cs;
            cf.cb[ax] = cs + len;
            cs += 2 * len;
        }
        __syncthreads();
    }
    const long long L = kLanes / a.S;
    const long long tx = (static_cast<long long>(a.ny) * a.nz + L - 1) / L;
    const long long ty = static_cast<long long>(a.tpr) * a.nz;
    const long long tz = static_cast<long long>(a.tpr) * a.ny;
    const int entries = a.sources ? a.zgrp_off[tz] : 0;
    const long long ts = (entries + kLanes / a.S - 1) / (kLanes / a.S);
    for (long long st = 0; st < a.steps; ++st) {
        for (long long t = rank; t < tx; t += W) res_x_tile(a, cf, buf, t, st, lane);
        for (long long t = rank; t < ty; t += W)
            res_y_tile(a, cf, buf, t, st, lane, a.tma ? &tmap_y : nullptr, bars, phases);
        for (long long t = rank; t < tz; t += W)
            res_z_tile(a, cf, buf, t, st, lane, a.tma ? &tmap_z : nullptr, bars, phases);
        for (long long t = rank; t < ts; t += W) res_src_tile(a, t, st, lane, entries);
    }
}

// ---- per-z-tile item lists (residual Dirichlet entries, agent groups) -----
// Item q of [lo, hi) (lo / hi read from device memory when given: the group
// range of the last device rebuild) with voxel vox[q] belongs to the z tiles
// (j, r) whose 32-wide (i, s) range holds one of its S entries.
__global__ void res_list_count(const int64_t* vox, const int64_t* lo_p, const int64_t* hi_p, long long cap, int nx,
                               int ny, int S, int tpr, int* cnt)
{
    const long long lo = lo_p ? *lo_p : 0, hi = hi_p ? *hi_p : cap;
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= hi - lo) return;
    const long long v = vox[lo + t];
    const int i = static_cast<int>(v % nx), j = static_cast<int>((v / nx) % ny);
    for (int r = (i * S) / kLanes; r <= (i * S + S - 1) / kLanes; ++r) atomicAdd(cnt + j * tpr + r, 1);
}

// Exclusive scan of cnt[0, n) into off[0, n]; cnt becomes the fill cursor.
__global__ void __launch_bounds__(1024) res_list_scan(int* cnt, int* off, int n)
{
    __shared__ int part[1024];
    const int per = (n + 1023) / 1024;
    const int b = threadIdx.x * per, e = min(n, b + per);
    int sum = 0;
    for (int i = b; i < e; ++i) sum += cnt[i];
    part[threadIdx.x] = sum;
    __syncthreads();
    for (int d = 1; d < 1024; d <<= 1) {
        const int v = threadIdx.x >= d ? part[threadIdx.x - d] : 0;
        __syncthreads();
        part[threadIdx.x] += v;
        __syncthreads();
    }
    int run = part[threadIdx.x] - sum;
    for (int i = b; i < e; ++i) {
        const int c = cnt[i];
        off[i] = run;
        cnt[i] = run;
        run += c;
    }
    if (threadIdx.x == 1023) off[n] = part[1023];
}

__global__ void res_list_fill(const int64_t* vox, const int64_t* lo_p, const int64_t* hi_p, long long cap, int nx,
                              int ny, int S, int tpr, int* cursor, int* idx, int* tile)
{
    const long long lo = lo_p ? *lo_p : 0, hi = hi_p ? *hi_p : cap;
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= hi - lo) return;
    const long long v = vox[lo + t];
    const int i = static_cast<int>(v % nx), j = static_cast<int>((v / nx) % ny);
    for (int r = (i * S) / kLanes; r <= (i * S + S - 1) / kLanes; ++r) {
        const int pos = atomicAdd(cursor + j * tpr + r, 1);
        idx[pos] = static_cast<int>(lo + t);
        if (tile) tile[pos] = j * tpr + r;
    }
}

} // namespace kernels
} // namespace biodiff_b200
