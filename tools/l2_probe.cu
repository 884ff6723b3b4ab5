// l2_probe.cu -- does L2 catch overlapping TMA plane reads from neighbouring CTAs?
// Each CTA streams Z planes of a (BX x BY) box at tile origin (tx*SX, ty*SY) through a 4-deep
// TMA ring and sums it. Overlap = B - S. Optional per-CTA start skew in planes.
// usage: l2_probe BX BY SX SY SKEW
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include "../paper_1510_04995_b200/csrc/zwave.cuh"
using namespace girih_gpu;

__global__ void probe(const __grid_constant__ CUtensorMap map, double* out, int tiles_x, int SX,
                      int SY, int BX, int BY, int Z, int skew, int x0, double* wbuf, int spin) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int plane = BX * BY;
    double* ring = reinterpret_cast<double*>(sm);
    uint64_t* bar = reinterpret_cast<uint64_t*>(ring + 4 * plane);
    const int tx = blockIdx.x % tiles_x, ty = blockIdx.x / tiles_x;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int z0 = (skew * (tx + ty)) % Z;
    auto issue = [&](int z) {
        const int s = z & 3;
        mbar_arrive_expect_tx(&bar[s], plane * 8);
        tma_load_plane(ring + s * plane, &map, x0 + tx * SX, ty * SY, (z0 + z) % Z, &bar[s]);
    };
    if (threadIdx.x == 0)
        for (int z = 0; z < 3; ++z) issue(z);
    double acc = 0;
    for (int z = 0; z < Z; ++z) {
        __syncthreads();
        if (threadIdx.x == 0 && z + 3 < Z) issue(z + 3);
        mbar_wait(&bar[z & 3], (z >> 2) & 1);
        for (int i = threadIdx.x; i < plane; i += blockDim.x) acc += ring[(z & 3) * plane + i];
        if (wbuf) {  // write the tile's interior (stride box) back to a second array
            for (int i = threadIdx.x; i < SX * SY; i += blockDim.x) {
                const int xx = i % SX, yy = i / SX;
                wbuf[((size_t)((z0 + z) % Z) * 512 + ty * SY + yy) * 512 + x0 + tx * SX + xx] = acc;
            }
        }
        for (int w = 0; w < spin; ++w) acc = acc * 0.999 + 1e-9;
    }
    if (acc == 1234.5) out[blockIdx.x] = acc;
}

int main(int argc, char** argv) {
    const int BX = atoi(argv[1]), BY = atoi(argv[2]), SX = atoi(argv[3]), SY = atoi(argv[4]);
    const int skew = atoi(argv[5]);
    const int x0 = argc > 6 ? atoi(argv[6]) : 0;
    const int wr = argc > 7 ? atoi(argv[7]) : 0;
    const int spin = argc > 8 ? atoi(argv[8]) : 0;
    const int NX = 512, NY = 512, Z = 256;
    double* d;
    cudaMalloc(&d, size_t(NX) * NY * Z * 8);
    cudaMemset(d, 0, size_t(NX) * NY * Z * 8);
    double* o;
    cudaMalloc(&o, 1 << 20);
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fp, 12000, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp);
    CUtensorMap map;
    cuuint64_t dims[3] = {NX, NY, Z};
    cuuint64_t str[2] = {cuuint64_t(NX) * 8, cuuint64_t(NX) * NY * 8};
    cuuint32_t box[3] = {cuuint32_t(BX), cuuint32_t(BY), 1}, es[3] = {1, 1, 1};
    enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int tiles_x = (NX - BX - x0) / SX + 1, tiles_y = (NY - BY) / SY + 1;
    double* wbuf = nullptr;
    if (wr) cudaMalloc(&wbuf, size_t(NX) * NY * Z * 8);
    const int smem = 4 * BX * BY * 8 + 64;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a);
        probe<<<tiles_x * tiles_y, 256, smem>>>(map, o, tiles_x, SX, SY, BX, BY, Z, skew, x0, wbuf, spin);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double unique = double(NX) * NY * Z * 8;
        const double loaded = double(tiles_x) * tiles_y * BX * BY * Z * 8;
        if (rep == 2)
            printf("x0 %d wr %d spin %d box %dx%d stride %dx%d skew %d: tiles %d, %.3f ms, loaded/unique %.3f, "
                   "unique GB/s %.0f, loaded GB/s %.0f (%s)\n",
                   x0, wr, spin, BX, BY, SX, SY, skew, tiles_x * tiles_y, ms, loaded / unique, unique / ms / 1e6,
                   loaded / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
