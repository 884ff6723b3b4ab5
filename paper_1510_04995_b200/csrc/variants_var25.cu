// Best-first within each fused depth: select_variant() takes the first match.
// variants_var25.cu -- zwave instantiations for var25 (kept in its own TU so nvcc builds kinds in parallel).
#include "variants.h"

namespace girih_gpu {

const Variant kVariantsVar25[] = {
    GIRIH_VARIANT(K_VAR25, 1, 32, 16, 64, 1, 1, 2),
    GIRIH_VARIANT(K_VAR25, 1, 32, 32, 128, 2, 1, 1),
    GIRIH_VARIANT_D(K_VAR25, 1, 32, 16, 64, 1, 1, 2),
    // output-columns-only tile (32 output columns from a 40-column box): no gain where the pass
    // already streams at the copy peak (512^3 50.2 K vs 50.8 K); kept for the tuner
    GIRIH_VARIANT_ND(K_VAR25, 1, 40, 16, 64, 2, 1, 2),
    // two fused steps: what the SMEM working set allows at radius 4 (13 coefficient planes
    // reused R iterations later, no coefficient prefetch, 16x4 output per 32x20 box); measured
    // to show why var25pt stays single-step
    GIRIH_VARIANT(K_VAR25, 2, 32, 20, 192, 1, 0, 1),
};
const int kNumVariantsVar25 = sizeof(kVariantsVar25) / sizeof(kVariantsVar25[0]);

}  // namespace girih_gpu
