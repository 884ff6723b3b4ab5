// tma_probe.cu -- standalone check of the TMA plane-load + mbarrier path used by zwave.cuh.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_1510_04995_b200/csrc/zwave.cuh"
using namespace girih_gpu;

__global__ void probe(const __grid_constant__ CUtensorMap map, double* out, int x, int y, int z) {
    extern __shared__ __align__(128) unsigned char sm[];
    double* buf = reinterpret_cast<double*>(sm);
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 64 * 32 * 8);
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(bar, 64 * 32 * 8);
        tma_load_plane(buf, &map, x, y, z, bar);
    }
    mbar_wait(bar, 0);
    for (int i = threadIdx.x; i < 64 * 32; i += blockDim.x) out[i] = buf[i];
}

int main(int argc, char** argv) {
    const int only = argc > 1 ? atoi(argv[1]) : -1;
    const int P = 48, Y = 26, Z = 26;
    std::vector<double> h(size_t(P) * Y * Z);
    for (size_t i = 0; i < h.size(); ++i) h[i] = double(i);
    double *d, *o;
    cudaMalloc(&d, h.size() * 8);
    cudaMalloc(&o, 64 * 32 * 8);
    cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fp, 12000, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp);
    CUtensorMap map;
    cuuint64_t dims[3] = {P, Y, Z};
    cuuint64_t str[2] = {cuuint64_t(P) * 8, cuuint64_t(P) * Y * 8};
    cuuint32_t box[3] = {64, 32, 1}, es[3] = {1, 1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, str, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode rc=%d q=%d\n", int(r), int(q));
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 32 * 8 + 64);
    int coords[][3] = {{0, 0, 0}, {2, 0, 0}, {0, 0, -2}, {0, -3, 0}, {0, 3, 0}, {-2, 0, 0}, {-4, 0, 0}, {1, 0, 0}, {40, 20, 25}};
    int ci = -1;
    for (auto& c : coords) {
        ++ci;
        if (only >= 0 && ci != only) continue;
        probe<<<1, 128, 64 * 32 * 8 + 64>>>(map, o, c[0], c[1], c[2]);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<double> ho(64 * 32);
        cudaMemcpy(ho.data(), o, ho.size() * 8, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int yy = 0; yy < 32; ++yy)
            for (int xx = 0; xx < 64; ++xx) {
                int gx = c[0] + xx, gy = c[1] + yy, gz = c[2];
                double want = (gx >= 0 && gx < P && gy >= 0 && gy < Y && gz >= 0 && gz < Z)
                                  ? h[(size_t(gz) * Y + gy) * P + gx] : 0.0;
                bad += ho[yy * 64 + xx] != want;
            }
        printf("coords (%d,%d,%d): err=%s bad=%d\n", c[0], c[1], c[2], cudaGetErrorString(e), bad);
        if (e != cudaSuccess) return 1;
        fflush(stdout);
    }
    return 0;
}
