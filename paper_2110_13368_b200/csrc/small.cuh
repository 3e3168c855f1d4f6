// One-cluster kernel for fields that fit a thread-block cluster's shared
// memory (the paper's own 50^3 case, BASELINE.json configs[0]; SURVEY.md §8
// row a9; VERDICT r01 "small-grid path").
//
// A cluster of C CTAs (16, non-portable, else 8) runs every step of an
// advance() in one launch. CTA c owns the z-planes [k0, k1) and keeps them in
// shared memory (dense rows of nx*S doubles):
//
//   x sweep, y sweep   on the CTA's own planes, in shared memory; x -> y is a
//                      CTA barrier (both axes lie inside a plane)
//   slab -> L2         one 2-D TMA store box; cluster barrier (release /
//                      acquire at cluster scope, also invalidates L1)
//   z sweep            the cluster's nx*ny*S columns split over the CTAs;
//                      each thread LDGSTS-copies its column into the (now
//                      free) slab memory and runs the chain, storing the
//                      clamped results to L2; cluster barrier
//   events             residual Dirichlet entries, then the cell sources, on
//                      the L2 copy, spread over every thread of the cluster
//                      (a tumour's core planes hold most groups); barrier
//   L2 -> slab         one 2-D TMA load box
//
// Three cluster barriers per step, no grid barrier, no launch gaps. The
// chains are the resident kernel's (res_chain: 8-position register blocks,
// pivots in shared memory), so numerics and order are the reference's:
// bit-identical. Supported: rows of 16-byte multiples, a CTA's box <= 256 x
// 256 (small_config); other shapes take the L2 dataflow kernel.
//
// Design probe: BIODIFF_RES_TRACE=<file> records per-CTA phase stamps
// (tools/resident_trace_probe.py).
#pragma once

#include "resident.cuh"
#include "xyc.cuh" // cluster_ctarank / cluster_nctarank / cluster_sync

namespace biodiff_b200 {
namespace kernels {

struct Small {
    double* rho;
    int nx, ny, nz, S;
    int pitch;          // shared row length (doubles) of a (plane, j) row, >= nx*S
    int planes;         // planes per CTA (ceil(nz / C))
    ResAxis ax[3];
    Clamp clamp;
    long long dir_count; // residual Dirichlet entries (voxel order)
    const int64_t* dir_voxel;
    const unsigned char* dir_mask;
    const double* dir_values;
    int sources;
    const int64_t* g_lo;  // group range of the last device rebuild (voxel order)
    const int64_t* g_hi;
    const int64_t* group_voxel;
    const int64_t* group_offsets;
    const double* add;
    const double* den;
    long long steps;
    int slab_doubles;   // max(planes*ny*pitch, nz*blockDim) doubles
    int coef_doubles;
    int tma;            // slab moves by one 2-D TMA box of pitch x rows (columns past rowlen: zero-filled on
                        // load, clipped on store)
    int grid;           // 1: cooperative grid of slab CTAs with grid barriers (else one cluster)
    unsigned* bar;      // grid mode: [arrivals, generation], zeroed before the launch
    unsigned long long* trace; // design probe: [step<8][cta][8] globaltimer stamps (thread 0 of each CTA)
};
#define SMALL_STAMP(I)                                                                                            \
    if (a.trace && st < 8 && tid == 0) a.trace[(st * C + cr) * 12 + (I)] = res_clock();

__global__ void __launch_bounds__(256, 1) step_small(const __grid_constant__ CUtensorMap tmap_slab, Small a)
{
    extern __shared__ __align__(128) double smem_small[];
    const int tid = threadIdx.x, nt = blockDim.x;
    const int lane = tid % kLanes, warp = tid / kLanes, nw = nt / kLanes;
    // Cluster mode: one cluster, cluster barriers. Grid mode (a.grid): a
    // cooperative launch of one CTA per slab of planes (fields too large for
    // one cluster's shared memory, e.g. C2), grid barriers.
    const int C = a.grid ? static_cast<int>(gridDim.x) : static_cast<int>(cluster_nctarank());
    const int cr = a.grid ? static_cast<int>(blockIdx.x) : static_cast<int>(cluster_ctarank());
    unsigned gen = 0;
    auto sync_all = [&]() {
        if (!a.grid) {
            cluster_sync();
            return;
        }
        __syncthreads();
        if (tid == 0) { // arrival counter + generation word; acquire also invalidates this SM's L1
            if (ptx::atom_acq_rel_add(a.bar, 1u) == static_cast<unsigned>(C) - 1) {
                atomicExch(a.bar, 0u);
                ptx::st_release(a.bar + 1, gen + 1);
            } else {
                while (ptx::ld_acquire(a.bar + 1) == gen) __nanosleep(32);
            }
            ++gen;
        }
        __syncthreads();
    };
    const int S = a.S;
    const long long rowlen = static_cast<long long>(a.nx) * S;
    const long long plane = static_cast<long long>(a.ny) * rowlen;
    const int k0 = min(a.nz, cr * a.planes), k1 = min(a.nz, k0 + a.planes), nkl = k1 - k0;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem_small); // slab TMA mbarrier (16 doubles reserved)
    double* cs = smem_small + 16;
    ResCoef cf;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
        const int len = a.ax[ax].n * S;
        for (int i = tid; i < len; i += nt) {
            cs[i] = a.ax[ax].dinv[i];
            cs[len + i] = a.ax[ax].cb[i];
        }
        cf.dinv[ax] = cs;
        cf.cb[ax] = cs + len;
        cs += 2 * len;
    }
    double* slab = smem_small + 16 + a.coef_doubles;
    if (tid == 0) ptx::mbar_init(bar, 1);
    ptx::fence_mbar_init();
    __syncthreads(); // the barrier (and the pivots) before any wait / chain
    uint32_t phase = 0;
    // Slab <-> L2: one 2-D TMA box (rowlen x planes*ny rows; rows past the
    // field are zero-filled / clipped) when the rows are 16-byte multiples,
    // else coalesced LDGSTS / store loops.
    auto load_slab = [&]() {
        if (a.tma & 1) {
            if (tid == 0) {
                ptx::fence_proxy_async_global(); // other CTAs' generic writes (z, sources) before the async read
                ptx::mbar_arrive_expect_tx(bar, static_cast<uint32_t>(a.planes * a.ny * a.pitch * 8));
                ptx::tma_load_4d(slab, &tmap_slab, 0, k0 * a.ny, 0, 0, bar);
            }
            ptx::mbar_wait(bar, phase);
            phase ^= 1u;
        } else {
            for (int r = warp; r < nkl * a.ny; r += nw) {
                const double* src = a.rho + (k0 * plane) + r * rowlen;
                for (int o = lane; o < rowlen; o += kLanes) ptx::cp_async8(slab + r * a.pitch + o, src + o);
            }
            ptx::cp_async_wait_all();
        }
        __syncthreads();
    };
    auto store_slab = [&]() {
        if (a.tma & 2) ptx::fence_proxy_async_smem(); // the chains' generic smem writes before the async read
        __syncthreads();
        if (a.tma & 2) {
            if (tid == 0) {
                ptx::tma_store_4d(&tmap_slab, 0, k0 * a.ny, 0, 0, slab);
                ptx::bulk_commit();
                ptx::bulk_wait_all();
                ptx::fence_proxy_async_global(); // visible to the generic-proxy z loads
            }
        } else {
            for (int r = warp; r < nkl * a.ny; r += nw) {
                double* dst = a.rho + (k0 * plane) + r * rowlen;
                for (int o = lane; o < rowlen; o += kLanes) dst[o] = slab[r * a.pitch + o];
            }
        }
    };
    const long long gt = static_cast<long long>(cr) * nt + tid, G = static_cast<long long>(C) * nt;
    load_slab();
    for (long long st = 0; st < a.steps; ++st) {
        SMALL_STAMP(0)
        // ---- x: chains (line (j, plane), substrate), thread per chain
        {
            const int nch = nkl * a.ny * S;
            const int n = a.nx;
            for (int q = tid; q < nch; q += nt) {
                const int s = q % S, r = q / S; // r = kl * ny + j
                double* c = slab + r * a.pitch + s;
                res_chain<true>(c, S, nullptr, 0, n, n, s, S, a.ax[0], cf.dinv[0] + s, cf.cb[0] + s, false, false,
                                0.0);
            }
        }
        __syncthreads();
        SMALL_STAMP(1)
        // ---- y: chains ((i, s), plane)
        {
            const int nch = nkl * static_cast<int>(rowlen);
            const int n = a.ny;
            for (int q = tid; q < nch; q += nt) {
                const int e = q % static_cast<int>(rowlen), kl = q / static_cast<int>(rowlen);
                const int s = e % S;
                double* c = slab + kl * a.ny * a.pitch + e;
                res_chain<true>(c, a.pitch, nullptr, 0, n, n, s, S, a.ax[1], cf.dinv[1] + s, cf.cb[1] + s, false,
                                false, 0.0);
            }
        }
        SMALL_STAMP(2)
        store_slab();
        SMALL_STAMP(8)
        sync_all();
        SMALL_STAMP(3)
        // ---- z: the cluster's columns (j, e), C-way split; column block of
        // the CTA's threads in the free slab memory ([m][thread]).
        {
            const long long ncol = static_cast<long long>(a.ny) * rowlen;
            const int n = a.nz, P = (n + 3) / 4;
            for (long long q0 = static_cast<long long>(cr) * nt; q0 < ncol; q0 += static_cast<long long>(C) * nt) {
                const long long q = q0 + tid;
                const bool active = q < ncol;
                const int j = static_cast<int>(q / rowlen), e = static_cast<int>(q % rowlen);
                double* g = a.rho + q; // (i, s) = e of row j, plane 0
                double* c = slab + tid;
                res_issue(c, g, plane, n, P, active, nt);
                if (active) {
                    const int i = e / S, s = e % S;
                    const bool csb = (a.clamp.mask >> s) & 1ull;
                    const bool face = i == 0 || i == a.nx - 1 || j == 0 || j == a.ny - 1;
                    res_chain<false>(c, nt, g, plane, n, P, s, S, a.ax[2], cf.dinv[2] + s, cf.cb[2] + s, csb,
                                     csb && face, csb ? a.clamp.values[s] : 0.0);
                }
                __syncthreads(); // the column block is reused by the next round
            }
            ptx::fence_proxy_async_smem(); // generic writes of the column block before the slab's TMA refill
        }
        SMALL_STAMP(4)
        sync_all();
        SMALL_STAMP(5)
        // ---- residual Dirichlet entries (solver.cpp:298), then the sources
        // (agents.cpp:97-109), on the L2 copy, spread over every thread of
        // the cluster (a tumour's core planes hold most of the groups).
        if (a.dir_count) {
            for (long long it = gt; it < a.dir_count * S; it += G) {
                const long long q = it / S;
                const int s = static_cast<int>(it % S);
                if (a.dir_mask[q * S + s]) a.rho[a.dir_voxel[q] * S + s] = a.dir_values[q * S + s];
            }
            if (a.sources) sync_all();
        }
        if (a.sources) {
            const long long glo = *a.g_lo, ghi = *a.g_hi;
            for (long long it = gt; it < (ghi - glo) * S; it += G) {
                const long long gi = glo + it / S;
                const int s = static_cast<int>(it % S);
                double* p = a.rho + a.group_voxel[gi] * S + s;
                double x = *p;
                long long m = a.group_offsets[gi];
                const long long m1 = a.group_offsets[gi + 1];
                for (; m + 4 <= m1; m += 4) {
                    double ad[4], de[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        ad[u] = a.add[(m + u) * S + s];
                        de[u] = a.den[(m + u) * S + s];
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u) x = __ddiv_rn(__dadd_rn(x, ad[u]), de[u]);
                }
                for (; m < m1; ++m) x = __ddiv_rn(__dadd_rn(x, a.add[m * S + s]), a.den[m * S + s]);
                *p = x;
            }
        }
        if (a.dir_count || a.sources) sync_all();
        SMALL_STAMP(6)
        load_slab();
        SMALL_STAMP(7)
    }
    // The field already sits in L2 after the last step's events (no store).
}

} // namespace kernels
} // namespace biodiff_b200
