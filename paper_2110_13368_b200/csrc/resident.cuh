// Resident multi-step kernel for grids that live in L2 (the paper's own
// 50^3 / 100^3 workloads, BASELINE.json configs[0..1]).
//
// At these sizes a step is not bound by HBM (the whole field, 1-16 MB, sits
// in the 126 MB L2) but by launch gaps and the three dependent sweeps: the
// ring kernels spend ~7 us per sweep launch on 2,500-20,000 chains. Here ONE
// cooperative launch runs all `steps` steps of an advance():
//   for each step: x sweep | y sweep | z sweep + shell clamp
//                  | residual Dirichlet entries | cell sources
// with a grid-wide barrier after each phase (the next phase reads what other
// CTAs wrote). Each phase hands out warp tiles of 32 chains; a tile's lines
// are copied whole into the warp's shared memory with LDGSTS (cp.async, one
// L2 round trip for the tile), solved there thread-per-chain — the forward
// values stay resident, so the back substitution needs no recompute — and
// written back with coalesced stores.
//
// Numerics are the reference's, in its order (kernels.cuh fwd_first / fwd /
// bwd = solver.cpp:17-19; rows of the settled region use the host-verified
// bit-constant pivots; clamp after the sweeps, solver.cpp:295-298; sources
// per (voxel group, substrate) in ascending agent id, agents.cpp:97-109), so
// the results are bit-identical to the reference and to the ring kernels.
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
    int active;
};

struct Resident {
    double* rho;
    int nx, ny, nz, S;
    ResAxis ax[3];
    int last;                 // last active axis: the shell clamp is fused into its stores
    Clamp clamp;
    long long dir_count;      // residual Dirichlet entries (interior clamps, partial masks)
    const int64_t* dir_voxel;
    const unsigned char* dir_mask;
    const double* dir_values;
    int sources;              // cell_sources_sinks_step after every diffusion step
    const int64_t* g_lo;      // group range [*g_lo, *g_hi) of the last (device) rebuild
    const int64_t* g_hi;
    const int64_t* group_voxel;
    const int64_t* group_offsets;
    const double* add;        // per-agent factors (sources_factors), group order
    const double* den;
    long long steps;
    unsigned* bar;            // [2] arrival count, generation; zeroed before the launch
    int xrow;                 // smem doubles per x line: >= nx*S, xrow % 16 == S % 16 (conflict-free lanes)
    int warp_doubles;         // smem doubles per warp
};

// Grid-wide barrier of a cooperative launch (all CTAs co-resident). Thread 0
// of each CTA arrives with release semantics (cumulative over the CTA's
// writes through the preceding bar.sync) and spins with acquire loads, which
// also invalidate this SM's L1 so the next phase reads other CTAs' results.
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned& gen)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned nb = gridDim.x;
        if (ptx::atom_acq_rel_add(&bar[0], 1u) == nb - 1) {
            atomicExch(&bar[0], 0u);
            ptx::st_release(&bar[1], gen + 1);
        } else {
            while (ptx::ld_acquire(&bar[1]) == gen) {
            }
        }
        ++gen;
    }
    __syncthreads();
}

// Thomas solve of one chain held in shared memory (position m at p[m*st]),
// substrate s; `clamp_any` / `clamp_all`: the shell clamp of the line's ends /
// of every position (the stored value only; the recurrence runs unclamped).
__device__ __forceinline__ void res_solve(double* p, int st, int n, int s, int S, const ResAxis& A, bool clamp_any,
                                          bool clamp_all, double clamp_v)
{
    const double q = A.q[s];
    const double dc = A.dconst[s], cc = A.cconst[s];
    const double* dinv = A.dinv + s;
    const double* cb = A.cb + s;
    const int a = max(1, min(A.settle, n - 1)); // rows [1, a) load their pivot, [a, n-2] are settled
    double prev = fwd_first(p[0], __ldg(dinv));
    p[0] = prev;
    int m = 1;
#pragma unroll 4
    for (; m < a; ++m) {
        prev = fwd(p[m * st], prev, q, __ldg(dinv + m * S));
        p[m * st] = prev;
    }
#pragma unroll 8
    for (; m < n - 1; ++m) {
        prev = fwd(p[m * st], prev, q, dc);
        p[m * st] = prev;
    }
    if (n > 1) prev = fwd(p[(n - 1) * st], prev, q, __ldg(dinv + (n - 1) * S));
    double next = prev; // final (unclamped) value of position n-1
    p[(n - 1) * st] = clamp_any ? clamp_v : prev;
    const int b = max(A.settle, 0); // c_back rows [settle, n-2] settled
    m = n - 2;
#pragma unroll 8
    for (; m >= b; --m) {
        next = bwd(p[m * st], next, cc);
        p[m * st] = clamp_all ? clamp_v : next;
    }
#pragma unroll 4
    for (; m >= 0; --m) {
        next = bwd(p[m * st], next, __ldg(cb + m * S));
        p[m * st] = clamp_all ? clamp_v : next;
    }
    if (clamp_any) p[0] = clamp_v;
}

// One phase: every x line / y / z column tile of the grid, one warp per tile.
__device__ __forceinline__ void res_sweep(const Resident& a, int axis, double* buf, int gwarp, int nwarps, int lane)
{
    const ResAxis& A = a.ax[axis];
    const int S = a.S;
    const int rowlen = a.nx * S;
    const bool clamp = axis == a.last;
    if (axis == 0) {
        const int L = kLanes / S;
        const long long nlines = static_cast<long long>(a.ny) * a.nz;
        const long long tiles = (nlines + L - 1) / L;
        const int l = lane / S, s = lane % S;
        for (long long t = gwarp; t < tiles; t += nwarps) {
            const long long g0 = t * L;
            const int nl = static_cast<int>(min(static_cast<long long>(L), nlines - g0));
            double* base = a.rho + g0 * rowlen;
            for (int ll = 0; ll < nl; ++ll)
                for (int off = lane; off < rowlen; off += kLanes)
                    ptx::cp_async8(buf + ll * a.xrow + off, base + static_cast<long long>(ll) * rowlen + off);
            ptx::cp_async_wait_all();
            __syncwarp();
            if (l < nl) {
                const long long g = g0 + l;
                const int j = static_cast<int>(g % a.ny), k = static_cast<int>(g / a.ny);
                const bool cs = clamp && ((a.clamp.mask >> s) & 1ull);
                const bool face = j == 0 || j == a.ny - 1 || k == 0 || k == a.nz - 1;
                res_solve(buf + l * a.xrow + s, S, a.nx, s, S, A, cs, cs && face, cs ? a.clamp.values[s] : 0.0);
            }
            __syncwarp();
            for (int ll = 0; ll < nl; ++ll)
                for (int off = lane; off < rowlen; off += kLanes)
                    base[static_cast<long long>(ll) * rowlen + off] = buf[ll * a.xrow + off];
            __syncwarp();
        }
        return;
    }
    // y (axis 1, outer k) / z (axis 2, outer j): 32 consecutive (i, s) columns.
    const int tpr = (rowlen + kLanes - 1) / kLanes;
    const int n = A.n;
    const int n_outer = axis == 1 ? a.nz : a.ny;
    const long long tiles = static_cast<long long>(tpr) * n_outer;
    const long long plane = static_cast<long long>(a.ny) * rowlen;
    const long long step = axis == 1 ? rowlen : plane;
    for (long long t = gwarp; t < tiles; t += nwarps) {
        const int e = static_cast<int>(t % tpr) * kLanes + lane;
        const int outer = static_cast<int>(t / tpr);
        const bool active = e < rowlen;
        double* col = a.rho + (axis == 1 ? outer * plane : static_cast<long long>(outer) * rowlen) + e;
        if (active)
            for (int m = 0; m < n; ++m) ptx::cp_async8(buf + m * kLanes + lane, col + m * step);
        ptx::cp_async_wait_all();
        __syncwarp();
        if (active) {
            const int i = e / S, s = e % S;
            const bool cs = clamp && ((a.clamp.mask >> s) & 1ull);
            const bool oface = axis == 1 ? (outer == 0 || outer == a.nz - 1) : (outer == 0 || outer == a.ny - 1);
            const bool face = i == 0 || i == a.nx - 1 || oface;
            res_solve(buf + lane, kLanes, n, s, S, A, cs, cs && face, cs ? a.clamp.values[s] : 0.0);
            for (int m = 0; m < n; ++m) col[m * step] = buf[m * kLanes + lane];
        }
        __syncwarp();
    }
}

__global__ void __launch_bounds__(128) step_resident(Resident a)
{
    extern __shared__ __align__(16) double smem_res[];
    const int lane = threadIdx.x % kLanes;
    const int wib = threadIdx.x / kLanes;
    const int wpb = blockDim.x / kLanes;
    const int gwarp = blockIdx.x * wpb + wib;
    const int nwarps = gridDim.x * wpb;
    double* buf = smem_res + static_cast<long long>(wib) * a.warp_doubles;
    const long long tid = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const long long nthreads = static_cast<long long>(gridDim.x) * blockDim.x;
    unsigned gen = 0;
    for (long long st = 0; st < a.steps; ++st) {
        for (int axis = 0; axis < 3; ++axis) {
            if (!a.ax[axis].active) continue;
            res_sweep(a, axis, buf, gwarp, nwarps, lane);
            grid_barrier(a.bar, gen);
        }
        if (a.dir_count) {
            for (long long t = tid; t < a.dir_count * a.S; t += nthreads)
                if (a.dir_mask[t]) a.rho[a.dir_voxel[t / a.S] * a.S + (t % a.S)] = a.dir_values[t];
            grid_barrier(a.bar, gen);
        }
        if (a.sources) {
            const long long g0 = *a.g_lo;
            const long long total = (*a.g_hi - g0) * a.S;
            for (long long t = tid; t < total; t += nthreads) {
                const long long g = g0 + t / a.S;
                const int s = static_cast<int>(t % a.S);
                double* r = a.rho + a.group_voxel[g] * a.S + s;
                double x = *r;
                for (long long m = a.group_offsets[g]; m < a.group_offsets[g + 1]; ++m)
                    x = __ddiv_rn(__dadd_rn(x, a.add[m * a.S + s]), a.den[m * a.S + s]);
                *r = x;
            }
            grid_barrier(a.bar, gen);
        }
    }
}

} // namespace kernels
} // namespace biodiff_b200
