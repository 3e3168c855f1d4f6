// Design-probe microbenchmarks for the LOD sweep kernels (not product code).
// Measures: FP64 dependent-op latency, L2 vs HBM read+write bandwidth, and
// prototype z/x sweep variants on a 256^3 x 4 FP64 field.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench tools/microbench.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__global__ void lat_kernel(double* out, double a, double b, int n, long long* cyc)
{
    double x = out[0];
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        x = __dmul_rn(x, a);
        x = __dadd_rn(x, b);
    }
    long long t1 = clock64();
    out[0] = x;
    cyc[0] = t1 - t0;
}

__global__ void rw_kernel(double* p, long n, int reps)
{
    long stride = (long)gridDim.x * blockDim.x;
    for (int r = 0; r < reps; ++r)
        for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
            p[i] = p[i] * 1.0000001;
}

// z sweep, global two-pass, thread per (row element), persistent over tiles.
template <int PF>
__global__ void __launch_bounds__(256) zsweep_global(double* __restrict__ rho, int rowlen, int ny, int nz, int S,
                                                     const double* __restrict__ q, const double* __restrict__ dinv,
                                                     const double* __restrict__ cb)
{
    const long plane = (long)rowlen * ny;
    const int ntx = (rowlen + blockDim.x - 1) / blockDim.x;
    for (long t = blockIdx.x; t < (long)ntx * ny; t += gridDim.x) {
        const int j = (int)(t / ntx);
        const int e = (int)(t % ntx) * blockDim.x + threadIdx.x;
        if (e >= rowlen) continue;
        const int s = e % S;
        double* p = rho + (long)j * rowlen + e;
        const double qs = q[s];
        double prev = __dmul_rn(p[0], dinv[s]);
        p[0] = prev;
        for (int k0 = 1; k0 < nz; k0 += PF) {
            double buf[PF];
#pragma unroll
            for (int u = 0; u < PF; ++u)
                if (k0 + u < nz) buf[u] = p[(long)(k0 + u) * plane];
#pragma unroll
            for (int u = 0; u < PF; ++u)
                if (k0 + u < nz) {
                    prev = __dmul_rn(__dadd_rn(buf[u], __dmul_rn(qs, prev)), __ldg(dinv + (k0 + u) * S + s));
                    p[(long)(k0 + u) * plane] = prev;
                }
        }
        for (int k0 = nz - 2; k0 >= 0; k0 -= PF) {
            double buf[PF];
#pragma unroll
            for (int u = 0; u < PF; ++u)
                if (k0 - u >= 0) buf[u] = p[(long)(k0 - u) * plane];
#pragma unroll
            for (int u = 0; u < PF; ++u)
                if (k0 - u >= 0) {
                    prev = __dadd_rn(buf[u], __dmul_rn(__ldg(cb + (k0 - u) * S + s), prev));
                    p[(long)(k0 - u) * plane] = prev;
                }
        }
    }
}

// z sweep, smem tile: W columns x nz planes resident in smem, 1 compute warp
// (each lane owns CPL columns), all warps load/store.
template <int CPL>
__global__ void zsweep_smem(double* __restrict__ rho, int rowlen, int ny, int nz, int S,
                            const double* __restrict__ q, const double* __restrict__ dinv,
                            const double* __restrict__ cb)
{
    extern __shared__ double sm[];
    constexpr int W = 32 * CPL;
    const long plane = (long)rowlen * ny;
    const int ntx = rowlen / W;
    const int j = blockIdx.x / ntx;
    const int e0 = (blockIdx.x % ntx) * W;
    double* base = rho + (long)j * rowlen + e0;
    const int nthr = blockDim.x;
    for (int idx = threadIdx.x; idx < W * nz; idx += nthr) {
        int k = idx / W, c = idx % W;
        sm[idx] = base[(long)k * plane + c];
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        double prev[CPL], qs[CPL];
        int sidx[CPL];
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
            int col = lane + 32 * c;
            sidx[c] = (e0 + col) % S;
            qs[c] = q[sidx[c]];
            prev[c] = __dmul_rn(sm[col], dinv[sidx[c]]);
            sm[col] = prev[c];
        }
        for (int k = 1; k < nz; ++k) {
#pragma unroll
            for (int c = 0; c < CPL; ++c) {
                int col = lane + 32 * c;
                double v = sm[k * W + col];
                prev[c] = __dmul_rn(__dadd_rn(v, __dmul_rn(qs[c], prev[c])), __ldg(dinv + k * S + sidx[c]));
                sm[k * W + col] = prev[c];
            }
        }
        for (int k = nz - 2; k >= 0; --k) {
#pragma unroll
            for (int c = 0; c < CPL; ++c) {
                int col = lane + 32 * c;
                double v = sm[k * W + col];
                prev[c] = __dadd_rn(v, __dmul_rn(__ldg(cb + k * S + sidx[c]), prev[c]));
                sm[k * W + col] = prev[c];
            }
        }
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < W * nz; idx += nthr) {
        int k = idx / W, c = idx % W;
        base[(long)k * plane + c] = sm[idx];
    }
}

// x sweep, whole lines in smem: L lines per CTA, thread per (line, s) chain.
__global__ void xsweep_smem(double* __restrict__ rho, int nx, int S, int L, long lines,
                            const double* __restrict__ q, const double* __restrict__ dinv,
                            const double* __restrict__ cb)
{
    extern __shared__ double sm[];
    const int len = nx * S;
    const int pitch = len + 4;
    const long l0 = (long)blockIdx.x * L;
    double* base = rho + l0 * len;
    for (int idx = threadIdx.x; idx < L * len; idx += blockDim.x) {
        int l = idx / len, o = idx % len;
        sm[l * pitch + o] = base[idx];
    }
    __syncthreads();
    if (threadIdx.x < L * S) {
        const int l = threadIdx.x / S, s = threadIdx.x % S;
        double* v = sm + l * pitch + s;
        const double qs = q[s];
        double prev = __dmul_rn(v[0], dinv[s]);
        v[0] = prev;
        for (int i = 1; i < nx; ++i) {
            prev = __dmul_rn(__dadd_rn(v[i * S], __dmul_rn(qs, prev)), __ldg(dinv + i * S + s));
            v[i * S] = prev;
        }
        for (int i = nx - 2; i >= 0; --i) {
            prev = __dadd_rn(v[i * S], __dmul_rn(__ldg(cb + i * S + s), prev));
            v[i * S] = prev;
        }
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < L * len; idx += blockDim.x) {
        int l = idx / len, o = idx % len;
        base[idx] = sm[l * pitch + o];
    }
}

static float time_ms(cudaEvent_t a, cudaEvent_t b) { float ms; cudaEventElapsedTime(&ms, a, b); return ms; }

int main()
{
    int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    printf("SMs=%d\n", sms);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    // 1. latency
    {
        double* d; long long* c; CK(cudaMalloc(&d, 8)); CK(cudaMalloc(&c, 8));
        double one = 1.0; cudaMemcpy(d, &one, 8, cudaMemcpyHostToDevice);
        lat_kernel<<<1, 1>>>(d, 0.999999, 1e-7, 1000, c);
        lat_kernel<<<1, 1>>>(d, 0.999999, 1e-7, 100000, c);
        long long cyc; CK(cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost));
        printf("fp64 dmul+dadd dependent pair: %.2f cycles\n", cyc / 100000.0);
    }
    // 2. bandwidth vs working-set size
    for (long mb : {8L, 16L, 32L, 48L, 64L, 96L, 128L, 1024L, 4096L}) {
        long n = mb * 1024 * 1024 / 8;
        double* d; CK(cudaMalloc(&d, n * 8)); CK(cudaMemset(d, 0, n * 8));
        int reps = mb >= 1024 ? 2 : 20;
        rw_kernel<<<sms * 8, 256>>>(d, n, 1);
        cudaEventRecord(e0);
        rw_kernel<<<sms * 8, 256>>>(d, n, reps);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        double ms = time_ms(e0, e1);
        printf("rw %5ld MB: %.1f GB/s (R+W)\n", mb, 2.0 * n * 8 * reps / ms / 1e6);
        cudaFree(d);
    }
    // 3. sweeps on 256^3 x 4
    const int N = 256, S = 4;
    const long nvox = (long)N * N * N, total = nvox * S;
    double *rho, *q, *dinv, *cb;
    CK(cudaMalloc(&rho, total * 8)); CK(cudaMalloc(&q, S * 8)); CK(cudaMalloc(&dinv, N * S * 8)); CK(cudaMalloc(&cb, N * S * 8));
    std::vector<double> hq(S, 2.5), hd(N * S, 0.2), hc(N * S, 0.5);
    cudaMemcpy(q, hq.data(), S * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dinv, hd.data(), N * S * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(cb, hc.data(), N * S * 8, cudaMemcpyHostToDevice);
    CK(cudaMemset(rho, 0, total * 8));
    const double bytes = 16.0 * total;
    auto report = [&](const char* name, auto&& launch) {
        launch(); CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        for (int r = 0; r < 5; ++r) launch();
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        double ms = time_ms(e0, e1) / 5;
        printf("%-40s %8.1f us  %7.1f GB/s (alg 16B/elem)\n", name, ms * 1e3, bytes / ms / 1e6);
    };
    {
        double* tmp; CK(cudaMalloc(&tmp, total * 8));
        report("memcpy D2D", [&] { cudaMemcpyAsync(tmp, rho, total * 8, cudaMemcpyDeviceToDevice); });
        cudaFree(tmp);
    }
    const int rowlen = N * S;
    for (int blocks_per_sm : {1, 2, 4, 8}) {
        char name[64];
        snprintf(name, 64, "z global PF8 grid=%d*SM", blocks_per_sm);
        report(name, [&] { zsweep_global<8><<<sms * blocks_per_sm, 256>>>(rho, rowlen, N, N, S, q, dinv, cb); });
        snprintf(name, 64, "z global PF16 grid=%d*SM", blocks_per_sm);
        report(name, [&] { zsweep_global<16><<<sms * blocks_per_sm, 256>>>(rho, rowlen, N, N, S, q, dinv, cb); });
    }
    report("z global PF8 full grid", [&] { zsweep_global<8><<<(rowlen / 256) * N, 256>>>(rho, rowlen, N, N, S, q, dinv, cb); });
    {
        CK(cudaFuncSetAttribute(zsweep_smem<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32 * N * 8));
        CK(cudaFuncSetAttribute(zsweep_smem<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * N * 8));
        report("z smem W=32 128thr", [&] { zsweep_smem<1><<<(rowlen / 32) * N, 128, 32 * N * 8>>>(rho, rowlen, N, N, S, q, dinv, cb); });
        report("z smem W=32 256thr", [&] { zsweep_smem<1><<<(rowlen / 32) * N, 256, 32 * N * 8>>>(rho, rowlen, N, N, S, q, dinv, cb); });
        report("z smem W=64 256thr", [&] { zsweep_smem<2><<<(rowlen / 64) * N, 256, 64 * N * 8>>>(rho, rowlen, N, N, S, q, dinv, cb); });
    }
    for (int L : {4, 8, 16}) {
        size_t smem = (size_t)L * (N * S + 4) * 8;
        CK(cudaFuncSetAttribute(xsweep_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        char name[64]; snprintf(name, 64, "x smem L=%d", L);
        long lines = (long)N * N;
        report(name, [&] { xsweep_smem<<<lines / L, 256, smem>>>(rho, N, S, L, lines, q, dinv, cb); });
    }
    return 0;
}
