// variants.h -- compiled zwave kernel instantiations (host-visible registry).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include "zwave.cuh"

namespace girih_gpu {

using LaunchFn = cudaError_t (*)(const CUtensorMap& cmap, const PassDesc& d, const PassParams& p,
                                 int grid, cudaStream_t stream);
using LaunchChainFn = cudaError_t (*)(const CUtensorMap& cmap, const ChainDescs& cd,
                                      const PassParams& p, int grid, cudaStream_t stream);
using OccFn = cudaError_t (*)(int* max_ctas);  // resident CTAs on the whole current device

struct Variant {
    int kind, tb, lx, ly, threads, prefetch, aux_prefetch, min_blocks;
    int cy;                      // CTAs per thread-block cluster along y (1 = no cluster)
    int smem_bytes;
    int aux_x0, aux_y0, aux_x, aux_y;  // coefficient (aux) box inside the tile
    LaunchFn launch;             // one pass
    LaunchFn launch_instr;       // one pass with the trace / ledger instrumentation compiled in
    LaunchChainFn launch_chain;  // cd.npass chained passes over the same tile grid (cy == 1)
    OccFn occupancy;             // resident CTAs, single-pass kernel (a multiple of cy)
    OccFn occupancy_chain;       // the same for the chained kernel
    int direct_out;              // 1: output level stored straight from registers (no staging)
    int pace;                    // 1: the cluster only paces independent tiles (no shared rows)
    int narrow;                  // > 0: the threads cover only the inner columns of the lx-wide
                                 // box (ZwaveConfig::NARROW) and this is the x halo of the output
                                 // tile, XO + (TB-1) R; 0 = threads on all lx columns
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

template <int KIND, int TB, int LX, int LY, int NT, int P, int PA, int MINB, bool CHAIN, int CF,
          bool INSTR = false>
cudaError_t launch_zwave_impl(const CUtensorMap& cmap, const ChainDescs& cd, const PassParams& p,
                              int grid, cudaStream_t stream) {
    using CFG = ZwaveConfig<KIND, TB, LX, LY, NT, P, PA, MINB, CF>;
    constexpr int CY = CFG::CY;
    auto* fn = zwave_kernel<KIND, TB, LX, LY, NT, P, PA, MINB, CHAIN, CF, INSTR>;
    // once per instantiation (thread-safe static initialisation)
    static const cudaError_t attr =
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(CFG::SMEM));
    if (attr != cudaSuccess) return attr;
    if constexpr (CY == 1) {
        fn<<<grid, NT, CFG::SMEM, stream>>>(cmap, cd, p);
    } else {
        if constexpr (CY > 8) {
            static const cudaError_t np =
                cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            if (np != cudaSuccess) return np;
        }
        cudaLaunchConfig_t lc{};
        lc.gridDim = dim3(unsigned(grid / CY * CY));
        lc.blockDim = dim3(NT);
        lc.dynamicSmemBytes = CFG::SMEM;
        lc.stream = stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = CY;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        const cudaError_t e = cudaLaunchKernelEx(&lc, fn, cmap, cd, p);
        if (e != cudaSuccess) return e;
    }
    return cudaGetLastError();
}

template <int KIND, int TB, int LX, int LY, int NT, int P, int PA, int MINB, int CF>
cudaError_t launch_zwave_chain(const CUtensorMap& cmap, const ChainDescs& cd, const PassParams& p,
                               int grid, cudaStream_t stream) {
    if constexpr ((CF & 255) > 1) {
        return cudaErrorNotSupported;  // cluster kernels run single passes
    } else {
        return launch_zwave_impl<KIND, TB, LX, LY, NT, P, PA, MINB, true, CF>(cmap, cd, p, grid, stream);
    }
}

// one pass = a chain of length 1 (no dependency flags)
template <int KIND, int TB, int LX, int LY, int NT, int P, int PA, int MINB, int CF, bool INSTR = false>
cudaError_t launch_zwave(const CUtensorMap& cmap, const PassDesc& d, const PassParams& p, int grid,
                         cudaStream_t stream) {
    ChainDescs cd{};
    cd.d[0] = d;
    cd.pidx[0] = 0;
    cd.npass = 1;
    cd.done = nullptr;
    return launch_zwave_impl<KIND, TB, LX, LY, NT, P, PA, MINB, false, CF, INSTR>(cmap, cd, p, grid,
                                                                                   stream);
}

template <int KIND, int TB, int LX, int LY, int NT, int P, int PA, int MINB, int CF, bool CHAIN = false>
cudaError_t occupancy_zwave(int* max_ctas) {
    using CFG = ZwaveConfig<KIND, TB, LX, LY, NT, P, PA, MINB, CF>;
    constexpr int CY = CFG::CY;
    *max_ctas = 0;
    if constexpr (CHAIN && CY > 1) {
        return cudaSuccess;  // not launchable chained
    } else {
        auto* fn = zwave_kernel<KIND, TB, LX, LY, NT, P, PA, MINB, CHAIN, CF>;
        cudaError_t e =
            cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(CFG::SMEM));
        if (e != cudaSuccess) return e;
        int dev = 0, sms = 0;
        if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
        if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess)
            return e;
        if constexpr (CY == 1) {
            int per_sm = 0;
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, NT, CFG::SMEM);
            *max_ctas = per_sm * sms;
            return e;
        } else {
            if constexpr (CY > 8) {
                e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
                if (e != cudaSuccess) return e;
            }
            cudaLaunchConfig_t lc{};
            lc.gridDim = dim3(unsigned(CY * sms));
            lc.blockDim = dim3(NT);
            lc.dynamicSmemBytes = CFG::SMEM;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = CY;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            lc.attrs = at;
            lc.numAttrs = 1;
            int clusters = 0;
            e = cudaOccupancyMaxActiveClusters(&clusters, fn, &lc);
            *max_ctas = clusters * CY;
            return e;
        }
    }
}

#define GIRIH_VARIANT_F(KIND, TB, LX, LY, NT, P, PA, MINB, CF)                                \
    Variant {                                                                                 \
        KIND, TB, LX, LY, NT, P, PA, MINB, (CF) & 255,                                        \
            int(ZwaveConfig<KIND, TB, LX, LY, NT, P, PA, MINB, CF>::SMEM),                    \
            ZwaveConfig<KIND, TB, LX, LY, NT, P, PA, MINB, CF>::AXO,                          \
            ZwaveConfig<KIND, TB, LX, LY, NT, P, PA, MINB, CF>::AYO,                          \
            ZwaveConfig<KIND, TB, LX, LY, NT, P, PA, MINB, CF>::AX,                           \
            ZwaveConfig<KIND, TB, LX, LY, NT, P, PA, MINB, CF>::AY,                           \
            &launch_zwave<KIND, TB, LX, LY, NT, P, PA, MINB, CF>,                             \
            &launch_zwave<KIND, TB, LX, LY, NT, P, PA, MINB, CF, true>,                       \
            &launch_zwave_chain<KIND, TB, LX, LY, NT, P, PA, MINB, CF>,                       \
            &occupancy_zwave<KIND, TB, LX, LY, NT, P, PA, MINB, CF>,                          \
            &occupancy_zwave<KIND, TB, LX, LY, NT, P, PA, MINB, CF, true>,                    \
            ((CF) >> 8) & 1, ((CF) >> 9) & 1,                                                 \
            (ZwaveConfig<KIND, TB, LX, LY, NT, P, PA, MINB, CF>::NARROW                       \
                 ? ZwaveConfig<KIND, TB, LX, LY, NT, P, PA, MINB, CF>::XO +                    \
                       ((TB)-1) * ZwaveConfig<KIND, TB, LX, LY, NT, P, PA, MINB, CF>::R        \
                 : 0)                                                                          \
    }
// CY CTAs per y cluster
#define GIRIH_VARIANT_C(KIND, TB, LX, LY, NT, P, PA, MINB, CY) \
    GIRIH_VARIANT_F(KIND, TB, LX, LY, NT, P, PA, MINB, CY)
// direct output stores (no staging planes)
#define GIRIH_VARIANT_D(KIND, TB, LX, LY, NT, P, PA, MINB) \
    GIRIH_VARIANT_F(KIND, TB, LX, LY, NT, P, PA, MINB, 1 | (1 << 8))
// clusters of CY y-neighbour tiles paced in lockstep (ZwaveConfig::PACE), direct output
#define GIRIH_VARIANT_PD(KIND, TB, LX, LY, NT, P, PA, MINB, CY) \
    GIRIH_VARIANT_F(KIND, TB, LX, LY, NT, P, PA, MINB, (CY) | (1 << 8) | (1 << 9))
// output-columns-only thread mapping (single-step kernels; LX = computed columns + 2 XO)
#define GIRIH_VARIANT_N(KIND, TB, LX, LY, NT, P, PA, MINB) \
    GIRIH_VARIANT_F(KIND, TB, LX, LY, NT, P, PA, MINB, 1 | (1 << 10))
#define GIRIH_VARIANT_ND(KIND, TB, LX, LY, NT, P, PA, MINB) \
    GIRIH_VARIANT_F(KIND, TB, LX, LY, NT, P, PA, MINB, 1 | (1 << 8) | (1 << 10))
#define GIRIH_VARIANT(KIND, TB, LX, LY, NT, P, PA, MINB) \
    GIRIH_VARIANT_C(KIND, TB, LX, LY, NT, P, PA, MINB, 1)

}  // namespace girih_gpu
