// Best-first within each fused depth: select_variant() takes the first match.
// variants_var7.cu -- zwave instantiations for var7 (kept in its own TU so nvcc builds kinds in parallel).
#include "variants.h"

namespace girih_gpu {

const Variant kVariantsVar7[] = {
    GIRIH_VARIANT(K_VAR7, 1, 64, 8, 64, 3, 1, 3),
    GIRIH_VARIANT(K_VAR7, 1, 64, 8, 96, 3, 1, 3),
    GIRIH_VARIANT(K_VAR7, 1, 64, 10, 128, 3, 1, 2),
    GIRIH_VARIANT(K_VAR7, 1, 64, 16, 224, 4, 1, 1),
    GIRIH_VARIANT(K_VAR7, 2, 64, 18, 512, 2, 1, 1),
    GIRIH_VARIANT(K_VAR7, 2, 64, 16, 448, 2, 2, 1),
    GIRIH_VARIANT(K_VAR7, 2, 64, 16, 448, 3, 2, 1),
    GIRIH_VARIANT(K_VAR7, 2, 64, 18, 512, 3, 1, 1),
    GIRIH_VARIANT(K_VAR7, 2, 64, 16, 224, 2, 2, 1),
    GIRIH_VARIANT(K_VAR7, 2, 32, 32, 480, 2, 2, 1),
    GIRIH_VARIANT(K_VAR7, 2, 32, 16, 224, 2, 2, 2),
    GIRIH_VARIANT(K_VAR7, 3, 32, 16, 224, 3, 1, 1),
    GIRIH_VARIANT(K_VAR7, 4, 32, 16, 224, 2, 1, 1),
    GIRIH_VARIANT_C(K_VAR7, 2, 64, 18, 512, 2, 1, 1, 2),
    GIRIH_VARIANT_C(K_VAR7, 2, 64, 18, 512, 2, 1, 1, 4),
    GIRIH_VARIANT_C(K_VAR7, 3, 64, 12, 320, 2, 1, 1, 4),
    GIRIH_VARIANT_C(K_VAR7, 3, 64, 12, 160, 2, 1, 1, 4),
    GIRIH_VARIANT_C(K_VAR7, 4, 64, 10, 256, 2, 1, 1, 4),
    GIRIH_VARIANT_C(K_VAR7, 4, 64, 10, 256, 2, 1, 1, 8),
    GIRIH_VARIANT_C(K_VAR7, 4, 64, 10, 128, 2, 1, 1, 4),
    GIRIH_VARIANT_D(K_VAR7, 2, 64, 18, 512, 2, 1, 1),
    GIRIH_VARIANT_D(K_VAR7, 2, 64, 18, 512, 2, 2, 1),
    GIRIH_VARIANT_D(K_VAR7, 2, 64, 17, 480, 2, 2, 1),
    GIRIH_VARIANT_PD(K_VAR7, 2, 64, 18, 512, 2, 2, 1, 2),
    // inner-columns-only tiles: level 1 on all 64 thread columns of a 68-column box, 62 output
    // columns (1024 = 16.5 x 62: 17 tile columns instead of 18, coefficient boxes 64 wide per
    // 62 outputs instead of per 60)
    GIRIH_VARIANT_ND(K_VAR7, 2, 68, 18, 512, 2, 2, 1),
    GIRIH_VARIANT_ND(K_VAR7, 2, 68, 18, 512, 2, 1, 1),
};
const int kNumVariantsVar7 = sizeof(kVariantsVar7) / sizeof(kVariantsVar7[0]);

}  // namespace girih_gpu
