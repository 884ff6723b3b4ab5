// tma_copy_probe.cu -- ceiling for zwave's Tb=1 data movement: each CTA streams a tile column
// with TMA box loads (BX x BY, 4-deep ring) and writes the (BX-2h) x (BY-2h) interior back with a
// TMA box store (double-buffered staging), like a const7pt pass without arithmetic.
// usage: tma_copy_probe BX BY H CTAS_PER_SM_HINT
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include "../paper_1510_04995_b200/csrc/zwave.cuh"
using namespace girih_gpu;

__global__ void copyk(const __grid_constant__ CUtensorMap lmap, const __grid_constant__ CUtensorMap smap,
                      int tiles_x, int ntiles, int OX, int OY, int BX, int BY, int Z, int* work) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int plane = BX * BY;
    double* ring = reinterpret_cast<double*>(sm);
    double* stg = ring + 4 * plane;
    uint64_t* bar = reinterpret_cast<uint64_t*>(stg + 2 * OX * OY);
    if (threadIdx.x == 0) {
        for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    uint32_t g = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int tx = t % tiles_x, ty = t / tiles_x;
        auto issue = [&](int z, uint32_t gg) {
            const int s = gg & 3;
            mbar_arrive_expect_tx(&bar[s], plane * 8);
            tma_load_plane(ring + s * plane, &lmap, tx * OX, ty * OY, z, &bar[s]);
        };
        if (threadIdx.x == 0)
            for (int z = 0; z < 3 && z < Z; ++z) issue(z, g + z);
        for (int z = 0; z < Z; ++z, ++g) {
            __syncthreads();
            if (threadIdx.x == 0 && z + 3 < Z) issue(z + 3, g + 3);
            mbar_wait(&bar[g & 3], (g >> 2) & 1);
            const double* src = ring + (g & 3) * plane;
            double* dst = stg + (g & 1) * OX * OY;
            const int h = (BX - OX) / 2, hy = (BY - OY) / 2;
            for (int i = threadIdx.x; i < OX * OY; i += blockDim.x)
                dst[i] = src[(i / OX + hy) * BX + (i % OX) + h];
            fence_proxy_async_smem();
            __syncthreads();
            if (threadIdx.x == 0) {
                tma_store_plane(&smap, dst, tx * OX, ty * OY, z);
                bulk_commit();
                asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) bulk_wait_all();
}

int main(int argc, char** argv) {
    const int BX = atoi(argv[1]), BY = atoi(argv[2]), H = atoi(argv[3]);
    const int NX = 512 + 64, NY = 512 + 64, Z = 512;
    const int OX = BX - 2 * H, OY = BY - 2 * H;
    double *a, *b;
    const size_t n = size_t(NX) * NY * Z;
    cudaMalloc(&a, n * 8);
    cudaMalloc(&b, n * 8);
    cudaMemset(a, 0, n * 8);
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fp, 12000, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp);
    CUtensorMap lm, smp;
    cuuint64_t dims[3] = {NX, NY, Z};
    cuuint64_t str[2] = {cuuint64_t(NX) * 8, cuuint64_t(NX) * NY * 8};
    cuuint32_t box[3] = {cuuint32_t(BX), cuuint32_t(BY), 1}, es[3] = {1, 1, 1};
    enc(&lm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, a, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cuuint32_t sbox[3] = {cuuint32_t(OX), cuuint32_t(OY), 1};
    enc(&smp, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, b, dims, str, sbox, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int tiles_x = 512 / OX, tiles_y = 512 / OY, ntiles = tiles_x * tiles_y;
    const int smem = (4 * BX * BY + 2 * OX * OY) * 8 + 64;
    cudaFuncSetAttribute(copyk, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, copyk, 256, smem);
    const int grid = std::min(ntiles, 148 * occ);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        copyk<<<grid, 256, smem>>>(lm, smp, tiles_x, ntiles, OX, OY, BX, BY, Z, nullptr);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double useful = double(ntiles) * OX * OY * Z * 8 * 2;  // read + write of outputs
        if (rep == 2)
            printf("box %dx%d h %d: tiles %d grid %d (occ %d): %.3f ms, useful r+w %.0f GB/s (%s)\n", BX, BY, H,
                   ntiles, grid, occ, ms, useful / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
