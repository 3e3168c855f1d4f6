// Design probe: the DRAM ceiling of the sweeps' access pattern without the
// recurrences. A warp streams "columns" of a 256^3 x 4 field through a ring of
// NS shared-memory slots with 3-D TMA boxes (W doubles x 32 positions along y
// or z) and writes them back in place — the sweep kernels' traffic minus the
// compute and the reloads. Compares box widths W = 32 / 64 / 128 doubles.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lcuda tools/tma_copy_probe.cu -o tma_copy_probe
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "../paper_2110_13368_b200/csrc/ptx.cuh"

using namespace biodiff_b200;

constexpr int NX = 256, NY = 256, NZ = 256, S = 4, ROW = NX * S;

template <int W, int NS>
__global__ void __launch_bounds__(32) copy_columns(const __grid_constant__ CUtensorMap tm, int axis, int tiles)
{
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
    double* slots = reinterpret_cast<double*>(smem + 128);
    constexpr int kSlot = W * 32;
    const int lane = threadIdx.x;
    const int tpr = ROW / W;
    const int nch = (axis == 1 ? NY : NZ) / 32;
    if (lane == 0) {
        for (int s = 0; s < NS; ++s) ptx::mbar_init(&bars[s], 1);
        ptx::fence_mbar_init();
    }
    __syncwarp();
    uint32_t parity = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int e0 = (t % tpr) * W, outer = t / tpr;
        auto box = [&](int k, int& c1, int& c2) {
            c1 = axis == 2 ? outer : k * 32;
            c2 = axis == 2 ? k * 32 : outer;
        };
        if (lane == 0)
            for (int k = 0; k < NS && k < nch; ++k) {
                int c1, c2;
                box(k, c1, c2);
                ptx::mbar_arrive_expect_tx(&bars[k], kSlot * 8);
                ptx::tma_load_4d(slots + k * kSlot, &tm, e0, c1, c2, 0, &bars[k]);
            }
        for (int k = 0; k < nch; ++k) {
            const int s = k % NS;
            ptx::mbar_wait(&bars[s], (parity >> s) & 1u);
            parity ^= 1u << s;
            __syncwarp();
            if (lane == 0) {
                int c1, c2;
                box(k, c1, c2);
                ptx::tma_store_4d(&tm, e0, c1, c2, 0, slots + s * kSlot);
                ptx::bulk_commit();
                if (k + NS < nch) {
                    ptx::bulk_wait_read<0>();
                    box(k + NS, c1, c2);
                    ptx::mbar_arrive_expect_tx(&bars[s], kSlot * 8);
                    ptx::tma_load_4d(slots + s * kSlot, &tm, e0, c1, c2, 0, &bars[s]);
                }
            }
            __syncwarp();
        }
        if (lane == 0) ptx::bulk_wait_read<0>();
        __syncwarp();
    }
}

using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                            const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                            CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int W, int NS>
void run(Encode enc, double* d, int axis)
{
    CUtensorMap tm;
    const cuuint64_t dims[4] = {ROW, NY, NZ, 1};
    const cuuint64_t str[3] = {ROW * 8ull, ROW * 8ull * NY, ROW * 8ull * NY * NZ};
    const cuuint32_t box[4] = {W, axis == 1 ? 32u : 1u, axis == 2 ? 32u : 1u, 1};
    const cuuint32_t es[4] = {1, 1, 1, 1};
    if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
        CUDA_SUCCESS) {
        std::printf("encode failed W=%d\n", W);
        return;
    }
    const int smem = 128 + NS * W * 32 * 8;
    auto k = copy_columns<W, NS>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 32, smem);
    const int tiles = (ROW / W) * (axis == 1 ? NZ : NY);
    const int grid = std::min(tiles, per_sm * 148);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int it = 0; it < 3; ++it) k<<<grid, 32, smem>>>(tm, axis, tiles);
    cudaEventRecord(a);
    const int reps = 20;
    for (int it = 0; it < reps; ++it) k<<<grid, 32, smem>>>(tm, axis, tiles);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double bytes = 2.0 * 8.0 * ROW * NY * NZ;
    std::printf("axis %c W=%3d NS=%d ctas/SM=%2d: %7.1f us  %6.0f GB/s  (%s)\n", axis == 1 ? 'y' : 'z', W, NS, per_sm,
                1e3 * ms / reps, bytes / (ms / reps * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main()
{
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<Encode>(fn);
    double* d = nullptr;
    cudaMalloc(&d, sizeof(double) * ROW * NY * NZ);
    cudaMemset(d, 0, sizeof(double) * ROW * NY * NZ);
    for (int axis = 1; axis <= 2; ++axis) {
        run<32, 3>(enc, d, axis);
        run<32, 6>(enc, d, axis);
        run<64, 3>(enc, d, axis);
        run<128, 3>(enc, d, axis);
        run<128, 2>(enc, d, axis);
    }
    // plain cudaMemcpy D2D of the same bytes for reference
    double* e = nullptr;
    cudaMalloc(&e, sizeof(double) * ROW * NY * NZ);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaMemcpy(e, d, sizeof(double) * ROW * NY * NZ, cudaMemcpyDeviceToDevice);
    cudaEventRecord(a);
    for (int it = 0; it < 10; ++it) cudaMemcpy(e, d, sizeof(double) * ROW * NY * NZ, cudaMemcpyDeviceToDevice);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    std::printf("memcpy D2D: %7.1f us  %6.0f GB/s\n", 1e3 * ms / 10, 2.0 * 8.0 * ROW * NY * NZ / (ms / 10 * 1e-3) / 1e9);
    return 0;
}
