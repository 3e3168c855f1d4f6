// sm_100a FP64 kernels of the LOD diffusion step and the cell source/sink
// step. Bitwise contract: every arithmetic operation
// is an explicitly rounded __dmul_rn / __dadd_rn / __ddiv_rn in the
// reference's operand order, so no FMA contraction can change a bit:
//   forward  first: v*dinv                 (solver.cpp:17 fwd_first)
//   forward       : (v + q*prev)*dinv      (solver.cpp:18 fwd)
//   backward      : v + cb*next            (solver.cpp:19 bwd)
//   sources       : (r + (f*sec)*target) / (1 + f*(sec+upt)),  f = (dt*V)*inv_vox
//                                          (agents.cpp:538-543)
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
};

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
};

__device__ __forceinline__ double fwd_first(double v, double d) { return __dmul_rn(v, d); }
__device__ __forceinline__ double fwd(double v, double prev, double q, double d)
{
    return __dmul_rn(__dadd_rn(v, __dmul_rn(q, prev)), d);
}
__device__ __forceinline__ double bwd(double v, double next, double cb) { return __dadd_rn(v, __dmul_rn(cb, next)); }

// Per-lane view of one chain (line x substrate) resident in shared memory:
// element m lives at col[m*step].
// Per-lane view of one chain (line x substrate). Positions [0, ns) live in
// shared memory at col[m*step]; positions [ns, n) (at most RMAX of them)
// live in registers, loaded from / stored to HBM at gcol[m*gstep].
// Keeping the tail of every line in registers shrinks the shared-memory tile
// so more chains are resident per SM (the recurrences are latency-bound:
// 3 dependent FP64 ops per forward element, 2 per backward element).
struct Chain {
    double* col;
    int step;
    const double* gcol;
    long long gstep;
    int S;
    const double* dinv; // coefficient column of this lane's substrate (stride S)
    const double* cb;
    double q, dc, cc;
    int settle, n, ns;
    bool clamp_s, face;
    double clamp_v;
};

// Forward elimination over shared-memory positions [m0, m1) (m0 >= 1).
template <bool CONSTC>
__device__ __forceinline__ double fwd_range(const Chain& c, int m0, int m1, double prev)
{
    int m = m0;
    for (; m + 8 <= m1; m += 8) {
        double v[8], d[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            v[u] = c.col[(m + u) * c.step];
            d[u] = CONSTC ? c.dc : __ldg(c.dinv + (m + u) * c.S);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            prev = fwd(v[u], prev, c.q, d[u]);
            c.col[(m + u) * c.step] = prev;
        }
    }
    for (; m < m1; ++m) {
        prev = fwd(c.col[m * c.step], prev, c.q, CONSTC ? c.dc : __ldg(c.dinv + m * c.S));
        c.col[m * c.step] = prev;
    }
    return prev;
}

// Back substitution over shared-memory positions mtop down to m0, storing
// the (optionally clamped) result while the recurrence carries the
// unclamped one (the clamp happens after all sweeps, solver.cpp:380).
template <bool CONSTC, bool CLAMP>
__device__ __forceinline__ double bwd_range(const Chain& c, int mtop, int m0, double next)
{
    int m = mtop;
    for (; m - 7 >= m0; m -= 8) {
        double v[8], b[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            v[u] = c.col[(m - u) * c.step];
            b[u] = CONSTC ? c.cc : __ldg(c.cb + (m - u) * c.S);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            next = bwd(v[u], next, b[u]);
            double out = next;
            if (CLAMP && c.clamp_s && (c.face || (m - u) == 0)) out = c.clamp_v;
            c.col[(m - u) * c.step] = out;
        }
    }
    for (; m >= m0; --m) {
        next = bwd(c.col[m * c.step], next, CONSTC ? c.cc : __ldg(c.cb + m * c.S));
        double out = next;
        if (CLAMP && c.clamp_s && (c.face || m == 0)) out = c.clamp_v;
        c.col[m * c.step] = out;
    }
    return next;
}

__device__ __forceinline__ double coef_at(const Chain& c, const double* arr, double cst, int m)
{
    return (m >= c.settle && m < c.n - 1) ? cst : __ldg(arr + m * c.S);
}

// The full Thomas solve of one chain. wait(ch) blocks until shared-memory
// chunk ch has landed; flush(ch) is called by every lane once the chunk's
// final values are in shared memory, to write it back.
template <bool CLAMP, int RMAX, class Wait, class Flush>
__device__ __forceinline__ void solve_chain(const Chain& c, bool active, Wait wait, Flush flush)
{
    const int n = c.n, ns = c.ns;
    const int R = n - ns; // register-resident positions (<= RMAX)
    const int nchs = (ns + kChunk - 1) / kChunk;
    double rv[RMAX > 0 ? RMAX : 1];
    if (RMAX > 0 && active) {
#pragma unroll
        for (int r = 0; r < RMAX; ++r)
            if (r < R) rv[r] = __ldcs(c.gcol + static_cast<long long>(ns + r) * c.gstep);
    }

    // Forward elimination: shared-memory chunks, then the register tail.
    double prev = 0.0;
    for (int ch = 0; ch < nchs; ++ch) {
        wait(ch);
        const int m0 = ch * kChunk;
        const int m1 = min(ns, m0 + kChunk);
        if (active) {
            int m = m0;
            if (m == 0) {
                prev = fwd_first(c.col[0], __ldg(c.dinv));
                c.col[0] = prev;
                m = 1;
            }
            if (m >= c.settle && m1 <= n - 1)
                prev = fwd_range<true>(c, m, m1, prev);
            else
                prev = fwd_range<false>(c, m, m1, prev);
        }
    }
    if (RMAX > 0 && active) {
#pragma unroll
        for (int r = 0; r < RMAX; ++r) {
            if (r < R) {
                const int m = ns + r;
                const double d = coef_at(c, c.dinv, c.dc, m);
                prev = (m == 0) ? fwd_first(rv[r], d) : fwd(rv[r], prev, c.q, d);
                rv[r] = prev;
            }
        }
    }

    // Back substitution: register tail (stored straight to HBM), then the
    // shared-memory chunks from the top.
    double next = prev; // final value of position n-1
    if (active) {
        const double top = (CLAMP && c.clamp_s) ? c.clamp_v : next; // position n-1 is always a face
        if (R > 0)
            __stcs(const_cast<double*>(c.gcol) + static_cast<long long>(n - 1) * c.gstep, top);
        else
            c.col[(n - 1) * c.step] = top;
    }
    if (RMAX > 0 && active) {
#pragma unroll
        for (int r = RMAX - 1; r >= 0; --r) {
            if (r < R - 1) {
                const int m = ns + r;
                next = bwd(rv[r], next, coef_at(c, c.cb, c.cc, m));
                double out = next;
                if (CLAMP && c.clamp_s && (c.face || m == 0)) out = c.clamp_v;
                __stcs(const_cast<double*>(c.gcol) + static_cast<long long>(m) * c.gstep, out);
            }
        }
    }
    for (int ch = nchs - 1; ch >= 0; --ch) {
        const int m0 = ch * kChunk;
        int mtop = min(ns, m0 + kChunk) - 1;
        if (R == 0 && ch == nchs - 1) --mtop; // n-1 already final
        if (active && mtop >= m0) {
            if (m0 >= c.settle)
                next = bwd_range<true, CLAMP>(c, mtop, m0, next);
            else
                next = bwd_range<false, CLAMP>(c, mtop, m0, next);
        }
        flush(ch);
    }
}

// ---------------------------------------------------------------------------
// y / z sweep with TMA. A CTA (one warp) owns 32 contiguous doubles of one
// row — 32 (i,s) chains — and the whole line along the sweep axis. Line
// positions [0, ns) sit in shared memory, tile[m*32 + lane]: one elected
// lane issues 3-D tiled TMA loads of 32 x 32-position boxes (one mbarrier
// each) so the forward recurrence starts on the first box, and TMA-stores
// each finished box during the backward recurrence. Positions [ns, n) sit in
// registers (coalesced 256-byte rows). HBM traffic: one read + one write per
// value. Partial tiles at the row end / line end are handled by TMA bounds
// (zero fill on load, clipped stores).
// ---------------------------------------------------------------------------
struct StridedSweep {
    double* rho;
    Coef coef;
    long long stride;       // doubles between consecutive positions along the axis
    long long outer_stride; // doubles between consecutive outer indices
    int axis;               // 1 = y (outer k), 2 = z (outer j)
    int n;                  // line length
    int ns;                 // positions kept in shared memory (multiple of kChunk, or n)
    int n_outer;            // number of outer indices (ny for z, nz for y)
    int rowlen;             // nx*S
    int tiles_per_row;
    int S;
    int nx;
    Clamp clamp;
};

__device__ __forceinline__ Chain make_chain_yz(const StridedSweep& a, double* tile, int lane, int e0,
                                               long long outer, bool active)
{
    const int e = e0 + (active ? lane : 0);
    const int s = e % a.S;
    const int i = e / a.S;
    Chain c;
    c.col = tile + lane;
    c.step = kLanes;
    c.gcol = a.rho + outer * a.outer_stride + e;
    c.gstep = a.stride;
    c.S = a.S;
    c.dinv = a.coef.dinv + s;
    c.cb = a.coef.cb + s;
    c.q = a.coef.q[s];
    c.dc = a.coef.dconst[s];
    c.cc = a.coef.cconst[s];
    c.settle = a.coef.settle;
    c.n = a.n;
    c.ns = a.ns;
    c.clamp_s = (a.clamp.mask >> s) & 1ull;
    c.clamp_v = c.clamp_s ? a.clamp.values[s] : 0.0;
    c.face = (i == 0 || i == a.nx - 1 || outer == 0 || outer == a.n_outer - 1);
    return c;
}

template <bool CLAMP, int RMAX>
__global__ void __launch_bounds__(kLanes) sweep_yz_tma(const __grid_constant__ CUtensorMap tmap, StridedSweep a)
{
    extern __shared__ __align__(128) unsigned char smem[];
    const int nchs = (a.ns + kChunk - 1) / kChunk;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
    double* tile = reinterpret_cast<double*>(smem + bar_bytes(nchs));
    const int lane = threadIdx.x;
    const int et = static_cast<int>(blockIdx.x % a.tiles_per_row);
    const int outer = static_cast<int>(blockIdx.x / a.tiles_per_row);
    const int e0 = et * kLanes;
    const int width = min(kLanes, a.rowlen - e0);
    // Tensor coordinates (dim0 = row element, dim1 = j, dim2 = k) of box ch.
    auto coords = [&](int ch, int& c1, int& c2) {
        if (a.axis == 2) {
            c1 = outer;
            c2 = ch * kChunk;
        } else {
            c1 = ch * kChunk;
            c2 = outer;
        }
    };
    if (lane == 0 && nchs > 0) {
        ptx::tma_prefetch_desc(&tmap);
        for (int ch = 0; ch < nchs; ++ch) ptx::mbar_init(&bars[ch], 1);
        ptx::fence_mbar_init();
        for (int ch = 0; ch < nchs; ++ch) {
            int c1, c2;
            coords(ch, c1, c2);
            ptx::mbar_arrive_expect_tx(&bars[ch], kLanes * kChunk * 8);
            ptx::tma_load_3d(tile + ch * kChunk * kLanes, &tmap, e0, c1, c2, &bars[ch]);
        }
    }
    __syncwarp();
    const bool active = lane < width;
    const Chain c = make_chain_yz(a, tile, lane, e0, outer, active);
    solve_chain<CLAMP, RMAX>(
        c, active, [&](int ch) { ptx::mbar_wait(&bars[ch], 0); },
        [&](int ch) {
            ptx::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
                int c1, c2;
                coords(ch, c1, c2);
                ptx::tma_store_3d(&tmap, e0, c1, c2, tile + ch * kChunk * kLanes);
                ptx::bulk_commit();
            }
        });
    if (lane == 0) ptx::bulk_wait_read_all();
}

// Same tile without TMA (rows with an odd number of doubles cannot be
// described by a tensor map: strides must be 16-byte multiples).
__global__ void __launch_bounds__(kLanes) sweep_yz_plain(StridedSweep a, bool clamp)
{
    extern __shared__ __align__(128) unsigned char smem[];
    double* tile = reinterpret_cast<double*>(smem);
    const int lane = threadIdx.x;
    const int et = static_cast<int>(blockIdx.x % a.tiles_per_row);
    const int outer = static_cast<int>(blockIdx.x / a.tiles_per_row);
    const int e0 = et * kLanes;
    const int width = min(kLanes, a.rowlen - e0);
    double* base = a.rho + outer * a.outer_stride + e0;
    const bool active = lane < width;
    for (int m = 0; m < a.n; ++m)
        if (active) tile[m * kLanes + lane] = base[m * a.stride + lane];
    __syncwarp();
    StridedSweep b = a;
    b.ns = a.n;
    const Chain c = make_chain_yz(b, tile, lane, e0, outer, active);
    auto none = [](int) {};
    if (clamp)
        solve_chain<true, 0>(c, active, none, none);
    else
        solve_chain<false, 0>(c, active, none, none);
    __syncwarp();
    for (int m = 0; m < a.n; ++m)
        if (active) base[m * a.stride + lane] = tile[m * kLanes + lane];
}

// ---------------------------------------------------------------------------
// x sweep, tile of L whole x-lines (contiguous in HBM). Lane -> (line l,
// substrate s). Positions [0, ns) sit in shared memory at
// tile[l*pitch + i*S + s], pitch padded so the lanes of a half-warp hit
// distinct banks; lane 0 issues one bulk copy per (line, chunk) — 1 KB at
// S=4 — and the stores of each finished chunk. Positions [ns, nx) sit in
// registers.
// ---------------------------------------------------------------------------
struct XSweep {
    double* rho;
    Coef coef;
    long long lines; // ny*nz
    int nx, ny, nz, S;
    int ns;          // positions kept in shared memory (multiple of kChunk, or nx)
    int rowlen;      // nx*S
    int pitch;       // smem doubles per line
    int L;           // lines per tile (L*S <= 32)
    Clamp clamp;
};

__device__ __forceinline__ Chain make_chain_x(const XSweep& a, double* tile, int lane, long long line0, bool active)
{
    const int l = active ? lane / a.S : 0;
    const int s = active ? lane % a.S : 0;
    const long long line = line0 + l;
    const int j = static_cast<int>(line % a.ny), k = static_cast<int>(line / a.ny);
    Chain c;
    c.col = tile + l * a.pitch + s;
    c.step = a.S;
    c.gcol = a.rho + line * a.rowlen + s;
    c.gstep = a.S;
    c.S = a.S;
    c.dinv = a.coef.dinv + s;
    c.cb = a.coef.cb + s;
    c.q = a.coef.q[s];
    c.dc = a.coef.dconst[s];
    c.cc = a.coef.cconst[s];
    c.settle = a.coef.settle;
    c.n = a.nx;
    c.ns = a.ns;
    c.clamp_s = (a.clamp.mask >> s) & 1ull;
    c.clamp_v = c.clamp_s ? a.clamp.values[s] : 0.0;
    c.face = (j == 0 || j == a.ny - 1 || k == 0 || k == a.nz - 1);
    return c;
}

template <bool CLAMP, bool BULK, int RMAX>
__global__ void __launch_bounds__(kLanes) sweep_x_smem(XSweep a)
{
    extern __shared__ __align__(128) unsigned char smem[];
    const int ns = BULK ? a.ns : a.nx;
    const int nchs = (ns + kChunk - 1) / kChunk;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
    double* tile = reinterpret_cast<double*>(smem + bar_bytes(nchs));
    const int lane = threadIdx.x;
    const long long line0 = static_cast<long long>(blockIdx.x) * a.L;
    const int nl = static_cast<int>(min(static_cast<long long>(a.L), a.lines - line0));
    const int S = a.S;
    double* base = a.rho + line0 * a.rowlen;

    if (BULK) {
        if (lane == 0 && nchs > 0) {
            for (int ch = 0; ch < nchs; ++ch) ptx::mbar_init(&bars[ch], 1);
            ptx::fence_mbar_init();
            for (int ch = 0; ch < nchs; ++ch) {
                const int cnt = min(kChunk, ns - ch * kChunk);
                const int off = ch * kChunk * S;
                ptx::mbar_arrive_expect_tx(&bars[ch], static_cast<uint32_t>(nl * cnt * S * 8));
                for (int l = 0; l < nl; ++l)
                    ptx::bulk_g2s(tile + l * a.pitch + off, base + static_cast<long long>(l) * a.rowlen + off,
                                  static_cast<uint32_t>(cnt * S * 8), &bars[ch]);
            }
        }
        __syncwarp();
    } else {
        for (int idx = lane; idx < nl * a.rowlen; idx += kLanes) {
            const int l = idx / a.rowlen, o = idx % a.rowlen;
            tile[l * a.pitch + o] = base[idx];
        }
        __syncwarp();
    }

    const bool active = lane < nl * S;
    XSweep b = a;
    b.ns = ns;
    const Chain c = make_chain_x(b, tile, lane, line0, active);
    auto wait = [&](int ch) {
        if (BULK) ptx::mbar_wait(&bars[ch], 0);
    };
    auto flush = [&](int ch) {
        if (!BULK) return;
        ptx::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
            const int i0 = ch * kChunk;
            const int cnt = min(kChunk, ns - i0);
            const int off = i0 * S;
            for (int l = 0; l < nl; ++l)
                ptx::bulk_s2g(base + static_cast<long long>(l) * a.rowlen + off, tile + l * a.pitch + off,
                              static_cast<uint32_t>(cnt * S * 8));
            ptx::bulk_commit();
        }
    };
    solve_chain<CLAMP, BULK ? RMAX : 0>(c, active, wait, flush);
    if (BULK) {
        if (lane == 0) ptx::bulk_wait_read_all();
    } else {
        __syncwarp();
        for (int idx = lane; idx < nl * a.rowlen; idx += kLanes) {
            const int ll = idx / a.rowlen, o = idx % a.rowlen;
            base[idx] = tile[ll * a.pitch + o];
        }
    }
}

// ---------------------------------------------------------------------------
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
__global__ void __launch_bounds__(128) sweep_global(GlobalSweep a)
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
        return ii == 0 || ii == a.nx - 1 || jj == 0 || jj == a.ny - 1 || kk == 0 || kk == a.nz - 1;
    };
    double next = prev;
    if (CLAMP && clamp_s) p[(n - 1) * stride] = clamp_v;
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

// Masked overwrite of Dirichlet entries (solver.cpp:349-357); one thread per
// (entry, substrate). Entries are unique voxels, so order is irrelevant.
__global__ void dirichlet_entries(double* rho, int S, long long count, const int64_t* voxel,
                                  const unsigned char* mask, const double* values)
{
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= count * S) return;
    if (mask[t]) rho[voxel[t / S] * S + (t % S)] = values[t];
}

// cell_sources_sinks_step (agents.cpp:511-548): one thread per (voxel group,
// substrate); the group's agents are applied in ascending-id order. The
// substrates of one agent update independently, so (group, s) threads
// reproduce the reference's agent-outer / substrate-inner loop bitwise.
__global__ void sources_groups(double* rho, int S, long long groups, const int64_t* group_voxel,
                               const int64_t* group_offsets, const double* volume, const double* secretion,
                               const double* uptake, const double* saturation, double dt, double inv_voxel_volume)
{
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= groups * S) return;
    const long long g = t / S;
    const int s = static_cast<int>(t % S);
    double* r = rho + group_voxel[g] * S + s;
    double x = *r;
    const long long a1 = group_offsets[g + 1];
    for (long long m = group_offsets[g]; m < a1; ++m) {
        const double f = __dmul_rn(__dmul_rn(dt, volume[m]), inv_voxel_volume);
        const double sec = secretion[m * S + s];
        const double upt = uptake[m * S + s];
        const double num = __dadd_rn(x, __dmul_rn(__dmul_rn(f, sec), saturation[m * S + s]));
        const double den = __dadd_rn(1.0, __dmul_rn(f, __dadd_rn(sec, upt)));
        x = __ddiv_rn(num, den);
    }
    *r = x;
}

// cross_check (validation.cpp:112-137) reductions. Non-negative doubles
// order like their bit patterns, so atomicMax on the bits is exact.
__global__ void cross_check_max(const double* a, const double* b, long long n, unsigned long long* max_abs_bits,
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
        if (diff > abs_tol + rel_tol * mag || diff != diff) my_fail = 1;
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

__global__ void cross_check_argmax(const double* a, const double* b, long long n, const unsigned long long* max_abs_bits,
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
