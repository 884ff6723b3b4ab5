// Best-first within each fused depth: select_variant() takes the first match.
// variants_const25.cu -- zwave instantiations for const25 (kept in its own TU so nvcc builds kinds in parallel).
#include "variants.h"

namespace girih_gpu {

const Variant kVariantsConst25[] = {
    // output-columns-only tile (64 output columns from a 72-column box, direct output): 512^3
    // 162-167 K vs 143 K MLUP/s for the 64x40 staged tile, 256^3 chained 150 K vs 128 K (same box)
    GIRIH_VARIANT_ND(K_CONST25, 1, 72, 40, 256, 1, 1, 1),
    GIRIH_VARIANT(K_CONST25, 1, 64, 40, 256, 1, 1, 1),
    GIRIH_VARIANT(K_CONST25, 1, 64, 32, 384, 1, 1, 1),
    GIRIH_VARIANT(K_CONST25, 1, 64, 32, 256, 1, 1, 1),
    GIRIH_VARIANT(K_CONST25, 1, 64, 16, 128, 1, 1, 2),
    GIRIH_VARIANT(K_CONST25, 1, 64, 20, 128, 1, 1, 2),
    GIRIH_VARIANT(K_CONST25, 1, 64, 20, 128, 2, 1, 2),
    GIRIH_VARIANT(K_CONST25, 2, 32, 32, 192, 2, 1, 1),
    GIRIH_VARIANT_C(K_CONST25, 2, 64, 20, 192, 1, 1, 1, 4),
    GIRIH_VARIANT_C(K_CONST25, 2, 64, 16, 128, 1, 1, 1, 8),
    GIRIH_VARIANT_D(K_CONST25, 1, 64, 40, 256, 1, 1, 1),
    GIRIH_VARIANT_ND(K_CONST25, 1, 72, 40, 256, 2, 1, 1),
};
const int kNumVariantsConst25 = sizeof(kVariantsConst25) / sizeof(kVariantsConst25[0]);

}  // namespace girih_gpu
