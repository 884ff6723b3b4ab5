// variants.h -- compiled zwave kernel instantiations (host-visible registry).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include "zwave.cuh"

namespace girih_gpu {

using LaunchFn = cudaError_t (*)(const CUtensorMap& vmap, const CUtensorMap& cmap,
                                 const CUtensorMap& umap, const CUtensorMap& omap,
                                 const PassParams& p, int grid, cudaStream_t stream);
using LaunchChainFn = cudaError_t (*)(const CUtensorMap& cmap, const ChainDescs& cd,
                                      const PassParams& p, int grid, cudaStream_t stream);
using OccFn = cudaError_t (*)(int* blocks_per_sm);

struct Variant {
    int kind, tb, lx, ly, threads, prefetch, aux_prefetch, min_blocks;
    int smem_bytes;
    int aux_x0, aux_y0, aux_x, aux_y;  // coefficient (aux) box inside the tile
    LaunchFn launch;             // one pass
    LaunchChainFn launch_chain;  // cd.npass chained passes over the same tile grid
    OccFn occupancy;             // resident CTAs per SM, single-pass kernel
    OccFn occupancy_chain;       // the same for the chained kernel
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

template <int KIND, int TB, int LX, int LY, int NT, int P, int PA, int MINB, bool CHAIN>
cudaError_t launch_zwave_impl(const CUtensorMap& cmap, const ChainDescs& cd, const PassParams& p,
                              int grid, cudaStream_t stream) {
    using CFG = ZwaveConfig<KIND, TB, LX, LY, NT, P, PA, MINB>;
    auto* fn = zwave_kernel<KIND, TB, LX, LY, NT, P, PA, MINB, CHAIN>;
    // once per instantiation (thread-safe static initialisation)
    static const cudaError_t attr =
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(CFG::SMEM));
    if (attr != cudaSuccess) return attr;
    fn<<<grid, NT, CFG::SMEM, stream>>>(cmap, cd, p);
    return cudaGetLastError();
}

template <int KIND, int TB, int LX, int LY, int NT, int P, int PA, int MINB>
cudaError_t launch_zwave_chain(const CUtensorMap& cmap, const ChainDescs& cd, const PassParams& p,
                               int grid, cudaStream_t stream) {
    return launch_zwave_impl<KIND, TB, LX, LY, NT, P, PA, MINB, true>(cmap, cd, p, grid, stream);
}

// one pass = a chain of length 1 (no dependency flags)
template <int KIND, int TB, int LX, int LY, int NT, int P, int PA, int MINB>
cudaError_t launch_zwave(const CUtensorMap& vmap, const CUtensorMap& cmap, const CUtensorMap& umap,
                         const CUtensorMap& omap, const PassParams& p, int grid,
                         cudaStream_t stream) {
    ChainDescs cd{};
    cd.d[0].vmap = vmap;
    cd.d[0].umap = umap;
    cd.d[0].omap = omap;
    cd.d[0].dst_final = p.dst_final;
    cd.d[0].dst_penult = p.dst_penult;
    cd.d[0].parity0 = p.parity0;
    cd.pidx[0] = 0;
    cd.npass = 1;
    cd.done = nullptr;
    return launch_zwave_impl<KIND, TB, LX, LY, NT, P, PA, MINB, false>(cmap, cd, p, grid, stream);
}

template <int KIND, int TB, int LX, int LY, int NT, int P, int PA, int MINB, bool CHAIN = false>
cudaError_t occupancy_zwave(int* blocks) {
    using CFG = ZwaveConfig<KIND, TB, LX, LY, NT, P, PA, MINB>;
    auto* fn = zwave_kernel<KIND, TB, LX, LY, NT, P, PA, MINB, CHAIN>;
    cudaError_t e =
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(CFG::SMEM));
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, fn, NT, CFG::SMEM);
}

#define GIRIH_VARIANT(KIND, TB, LX, LY, NT, P, PA, MINB)                                        \
    Variant {                                                                                 \
        KIND, TB, LX, LY, NT, P, PA, MINB, int(ZwaveConfig<KIND, TB, LX, LY, NT, P, PA, MINB>::SMEM),     \
            ZwaveConfig<KIND, TB, LX, LY, NT, P, PA, MINB>::AXO,                                    \
            ZwaveConfig<KIND, TB, LX, LY, NT, P, PA, MINB>::AYO,                                    \
            ZwaveConfig<KIND, TB, LX, LY, NT, P, PA, MINB>::AX,                                     \
            ZwaveConfig<KIND, TB, LX, LY, NT, P, PA, MINB>::AY,                                     \
            &launch_zwave<KIND, TB, LX, LY, NT, P, PA, MINB>,                                       \
            &launch_zwave_chain<KIND, TB, LX, LY, NT, P, PA, MINB>,                                 \
            &occupancy_zwave<KIND, TB, LX, LY, NT, P, PA, MINB>,                                    \
            &occupancy_zwave<KIND, TB, LX, LY, NT, P, PA, MINB, true>                               \
    }

}  // namespace girih_gpu
