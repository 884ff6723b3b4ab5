// variants.h -- compiled zwave kernel instantiations (host-visible registry).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include "zwave.cuh"

namespace girih_gpu {

using LaunchFn = cudaError_t (*)(const CUtensorMap& map, const PassParams& p, int grid,
                                 cudaStream_t stream);
using OccFn = cudaError_t (*)(int* blocks_per_sm);

struct Variant {
    int kind, tb, lx, ly, threads, prefetch;
    int smem_bytes;
    LaunchFn launch;
    OccFn occupancy;
};

// one table per kind, defined in variants_<kind>.cu
extern const Variant kVariantsConst7[];
extern const int kNumVariantsConst7;
extern const Variant kVariantsVar7[];
extern const int kNumVariantsVar7;
extern const Variant kVariantsConst25[];
extern const int kNumVariantsConst25;
extern const Variant kVariantsVar25[];
extern const int kNumVariantsVar25;

template <int KIND, int TB, int LX, int LY, int NT, int P>
cudaError_t launch_zwave(const CUtensorMap& map, const PassParams& p, int grid,
                         cudaStream_t stream) {
    using CFG = ZwaveConfig<KIND, TB, LX, LY, NT, P>;
    auto* fn = zwave_kernel<KIND, TB, LX, LY, NT, P>;
    static bool attr_done = false;
    if (!attr_done) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             int(CFG::SMEM));
        if (e != cudaSuccess) return e;
        attr_done = true;
    }
    fn<<<grid, NT, CFG::SMEM, stream>>>(map, p);
    return cudaGetLastError();
}

template <int KIND, int TB, int LX, int LY, int NT, int P>
cudaError_t occupancy_zwave(int* blocks) {
    using CFG = ZwaveConfig<KIND, TB, LX, LY, NT, P>;
    auto* fn = zwave_kernel<KIND, TB, LX, LY, NT, P>;
    cudaError_t e =
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(CFG::SMEM));
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, fn, NT, CFG::SMEM);
}

#define GIRIH_VARIANT(KIND, TB, LX, LY, NT, P)                                              \
    Variant {                                                                                \
        KIND, TB, LX, LY, NT, P, int(ZwaveConfig<KIND, TB, LX, LY, NT, P>::SMEM),          \
            &launch_zwave<KIND, TB, LX, LY, NT, P>, &occupancy_zwave<KIND, TB, LX, LY, NT, P> \
    }

}  // namespace girih_gpu
