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

#include <cstdint>

namespace biodiff_b200 {
namespace kernels {

constexpr int kLanes = 32;   // chains per CTA (one warp)
constexpr int kChunk = 32;   // positions per mbarrier chunk along the sweep axis

__host__ __device__ constexpr int bar_bytes(int nch) { return ((nch * 8 + 127) / 128) * 128; }

struct Clamp {
    const double* values;   // [S] shell clamp values
    unsigned long long mask; // bit s: substrate s clamped on every boundary voxel
};

__device__ __forceinline__ double fwd_first(double v, double d) { return __dmul_rn(v, d); }
__device__ __forceinline__ double fwd(double v, double prev, double q, double d)
{
    return __dmul_rn(__dadd_rn(v, __dmul_rn(q, prev)), d);
}
__device__ __forceinline__ double bwd(double v, double next, double cb) { return __dadd_rn(v, __dmul_rn(cb, next)); }

// ---------------------------------------------------------------------------
// y / z sweep, shared-memory resident tile.
// A CTA (one warp) owns 32 contiguous doubles of one row (32 (i,s) chains)
// and the whole line along the sweep axis: tile[m*32 + lane]. Rows arrive
// by cp.async.bulk in chunks of kChunk rows (one mbarrier each) so the
// forward recurrence starts on the first chunk; the backward recurrence
// writes each finished chunk straight back with bulk stores. HBM traffic is
// one read + one write per value (the line never leaves the SM in between).
// ---------------------------------------------------------------------------
struct StridedSweep {
    double* rho;
    const double* q;
    const double* dinv;
    const double* cb;
    long long stride;       // doubles between consecutive positions along the axis
    long long outer_stride; // doubles between consecutive outer indices
    int n;                  // line length
    int n_outer;            // number of outer indices (ny for z, nz for y)
    int rowlen;             // nx*S
    int tiles_per_row;
    int S;
    int nx;
    Clamp clamp;
};

template <bool CLAMP, bool BULK>
__global__ void __launch_bounds__(kLanes) sweep_strided_smem(StridedSweep a)
{
    extern __shared__ __align__(128) unsigned char smem[];
    const int nch = (a.n + kChunk - 1) / kChunk;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
    double* tile = reinterpret_cast<double*>(smem + bar_bytes(nch));
    const int lane = threadIdx.x;
    const int et = static_cast<int>(blockIdx.x % a.tiles_per_row);
    const long long outer = blockIdx.x / a.tiles_per_row;
    const int e0 = et * kLanes;
    const int width = min(kLanes, a.rowlen - e0);
    double* base = a.rho + outer * a.outer_stride + e0;

    if (BULK) {
        if (lane == 0) {
            for (int c = 0; c < nch; ++c) ptx::mbar_init(&bars[c], 1);
            ptx::fence_mbar_init();
            for (int c = 0; c < nch; ++c) {
                const int rows = min(kChunk, a.n - c * kChunk);
                ptx::mbar_arrive_expect_tx(&bars[c], static_cast<uint32_t>(rows * width * 8));
            }
        }
        __syncwarp();
        for (int m = lane; m < a.n; m += kLanes)
            ptx::bulk_g2s(tile + m * kLanes, base + m * a.stride, static_cast<uint32_t>(width * 8),
                          &bars[m / kChunk]);
    } else {
        for (int m = 0; m < a.n; ++m)
            if (lane < width) tile[m * kLanes + lane] = base[m * a.stride + lane];
        __syncwarp();
    }

    const bool active = lane < width;
    const int e = e0 + (active ? lane : 0);
    const int s = e % a.S;
    const int i = e / a.S;
    const double qs = a.q[s];
    const double* dinv = a.dinv + s;
    const double* cb = a.cb + s;
    const int S = a.S;
    bool clamp_s = false, lane_face = false;
    double clamp_v = 0.0;
    if (CLAMP) {
        clamp_s = (a.clamp.mask >> s) & 1ull;
        clamp_v = a.clamp.values[s];
        lane_face = (i == 0 || i == a.nx - 1 || outer == 0 || outer == a.n_outer - 1);
    }
    double* col = tile + lane;

    // Forward elimination.
    double prev = 0.0;
    for (int c = 0; c < nch; ++c) {
        if (BULK) ptx::mbar_wait(&bars[c], 0);
        const int m0 = c * kChunk;
        const int m1 = min(a.n, m0 + kChunk);
        if (active) {
            int m = m0;
            if (m == 0) {
                prev = fwd_first(col[0], __ldg(dinv));
                col[0] = prev;
                m = 1;
            }
            for (; m + 8 <= m1; m += 8) {
                double v[8], d[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    v[u] = col[(m + u) * kLanes];
                    d[u] = __ldg(dinv + (m + u) * S);
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    prev = fwd(v[u], prev, qs, d[u]);
                    col[(m + u) * kLanes] = prev;
                }
            }
            for (; m < m1; ++m) {
                prev = fwd(col[m * kLanes], prev, qs, __ldg(dinv + m * S));
                col[m * kLanes] = prev;
            }
        }
    }

    // Back substitution, chunk by chunk from the top; each finished chunk is
    // written back while the next one is computed.
    double next = prev;
    const int last = a.n - 1;
    if (CLAMP && active && clamp_s) col[last * kLanes] = clamp_v; // m = n-1 is always a face
    for (int c = nch - 1; c >= 0; --c) {
        const int m0 = c * kChunk;
        const int mtop = min(a.n, m0 + kChunk) - 1;
        if (active) {
            int m = (c == nch - 1) ? mtop - 1 : mtop;
            for (; m - 7 >= m0; m -= 8) {
                double v[8], b[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    v[u] = col[(m - u) * kLanes];
                    b[u] = __ldg(cb + (m - u) * S);
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    next = bwd(v[u], next, b[u]);
                    double out = next;
                    if (CLAMP && clamp_s && (lane_face || (m - u) == 0)) out = clamp_v;
                    col[(m - u) * kLanes] = out;
                }
            }
            for (; m >= m0; --m) {
                next = bwd(col[m * kLanes], next, __ldg(cb + m * S));
                double out = next;
                if (CLAMP && clamp_s && (lane_face || m == 0)) out = clamp_v;
                col[m * kLanes] = out;
            }
        }
        if (BULK) {
            ptx::fence_proxy_async_smem();
            __syncwarp();
            const int m = m0 + lane;
            if (m <= mtop) {
                ptx::bulk_s2g(base + m * a.stride, tile + m * kLanes, static_cast<uint32_t>(width * 8));
                ptx::bulk_commit();
            }
        }
    }
    if (BULK) {
        ptx::bulk_wait_read_all();
    } else {
        __syncwarp();
        for (int m = 0; m < a.n; ++m)
            if (lane < width) base[m * a.stride + lane] = tile[m * kLanes + lane];
    }
}

// ---------------------------------------------------------------------------
// x sweep, shared-memory resident tile of L whole x-lines (contiguous in
// HBM: one bulk copy per line and chunk). Lane -> (line l, substrate s);
// line l lives at tile[l*pitch + i*S + s], pitch padded so that the lanes of
// a half-warp hit distinct banks.
// ---------------------------------------------------------------------------
struct XSweep {
    double* rho;
    const double* q;
    const double* dinv;
    const double* cb;
    long long lines; // ny*nz
    int nx, ny, nz, S;
    int rowlen;      // nx*S
    int pitch;       // smem doubles per line
    int L;           // lines per tile (L*S <= 32)
    Clamp clamp;
};

template <bool CLAMP, bool BULK>
__global__ void __launch_bounds__(kLanes) sweep_x_smem(XSweep a)
{
    extern __shared__ __align__(128) unsigned char smem[];
    const int nch = (a.nx + kChunk - 1) / kChunk;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
    double* tile = reinterpret_cast<double*>(smem + bar_bytes(nch));
    const int lane = threadIdx.x;
    const long long line0 = static_cast<long long>(blockIdx.x) * a.L;
    const int nl = static_cast<int>(min(static_cast<long long>(a.L), a.lines - line0));
    const int S = a.S;
    double* base = a.rho + line0 * a.rowlen;

    if (BULK) {
        if (lane == 0) {
            for (int c = 0; c < nch; ++c) ptx::mbar_init(&bars[c], 1);
            ptx::fence_mbar_init();
            for (int c = 0; c < nch; ++c) {
                const int cnt = min(kChunk, a.nx - c * kChunk);
                ptx::mbar_arrive_expect_tx(&bars[c], static_cast<uint32_t>(nl * cnt * S * 8));
            }
        }
        __syncwarp();
        for (int idx = lane; idx < nl * nch; idx += kLanes) {
            const int c = idx / nl, l = idx % nl;
            const int cnt = min(kChunk, a.nx - c * kChunk);
            const int off = c * kChunk * S;
            ptx::bulk_g2s(tile + l * a.pitch + off, base + static_cast<long long>(l) * a.rowlen + off,
                          static_cast<uint32_t>(cnt * S * 8), &bars[c]);
        }
    } else {
        for (int idx = lane; idx < nl * a.rowlen; idx += kLanes) {
            const int l = idx / a.rowlen, o = idx % a.rowlen;
            tile[l * a.pitch + o] = base[idx];
        }
        __syncwarp();
    }

    const bool active = lane < nl * S;
    const int l = active ? lane / S : 0;
    const int s = active ? lane % S : 0;
    const double qs = a.q[s];
    const double* dinv = a.dinv + s;
    const double* cb = a.cb + s;
    double* v = tile + l * a.pitch + s;
    bool clamp_s = false, lane_face = false;
    double clamp_v = 0.0;
    if (CLAMP) {
        const long long line = line0 + l;
        const int j = static_cast<int>(line % a.ny), k = static_cast<int>(line / a.ny);
        clamp_s = (a.clamp.mask >> s) & 1ull;
        clamp_v = a.clamp.values[s];
        lane_face = (j == 0 || j == a.ny - 1 || k == 0 || k == a.nz - 1);
    }

    double prev = 0.0;
    for (int c = 0; c < nch; ++c) {
        if (BULK) ptx::mbar_wait(&bars[c], 0);
        const int i0 = c * kChunk;
        const int i1 = min(a.nx, i0 + kChunk);
        if (active) {
            int i = i0;
            if (i == 0) {
                prev = fwd_first(v[0], __ldg(dinv));
                v[0] = prev;
                i = 1;
            }
            for (; i + 8 <= i1; i += 8) {
                double x[8], d[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    x[u] = v[(i + u) * S];
                    d[u] = __ldg(dinv + (i + u) * S);
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    prev = fwd(x[u], prev, qs, d[u]);
                    v[(i + u) * S] = prev;
                }
            }
            for (; i < i1; ++i) {
                prev = fwd(v[i * S], prev, qs, __ldg(dinv + i * S));
                v[i * S] = prev;
            }
        }
    }

    double next = prev;
    const int last = a.nx - 1;
    if (CLAMP && active && clamp_s) v[last * S] = clamp_v; // i = nx-1 is a face
    for (int c = nch - 1; c >= 0; --c) {
        const int i0 = c * kChunk;
        const int itop = min(a.nx, i0 + kChunk) - 1;
        if (active) {
            int i = (c == nch - 1) ? itop - 1 : itop;
            for (; i - 7 >= i0; i -= 8) {
                double x[8], b[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    x[u] = v[(i - u) * S];
                    b[u] = __ldg(cb + (i - u) * S);
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    next = bwd(x[u], next, b[u]);
                    double out = next;
                    if (CLAMP && clamp_s && (lane_face || (i - u) == 0)) out = clamp_v;
                    v[(i - u) * S] = out;
                }
            }
            for (; i >= i0; --i) {
                next = bwd(v[i * S], next, __ldg(cb + i * S));
                double out = next;
                if (CLAMP && clamp_s && (lane_face || i == 0)) out = clamp_v;
                v[i * S] = out;
            }
        }
        if (BULK) {
            ptx::fence_proxy_async_smem();
            __syncwarp();
            if (lane < nl) {
                const int cnt = itop - i0 + 1;
                const int off = i0 * S;
                ptx::bulk_s2g(base + static_cast<long long>(lane) * a.rowlen + off, tile + lane * a.pitch + off,
                              static_cast<uint32_t>(cnt * S * 8));
                ptx::bulk_commit();
            }
        }
    }
    if (BULK) {
        ptx::bulk_wait_read_all();
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
