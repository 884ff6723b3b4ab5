// Best-first within each fused depth: select_variant() takes the first match.
// variants_const7.cu -- zwave instantiations for const7 (kept in its own TU so nvcc builds kinds in parallel).
#include "variants.h"

namespace girih_gpu {

const Variant kVariantsConst7[] = {
    // output-columns-only tiles (64 output columns from a 68-column box, direct output): the
    // chained default (256^3 330-348 K vs 280 K MLUP/s for the 64x10 staged tile, 384^3 368 K vs
    // 313 K, 128^3 144 K vs 106 K, same box)
    GIRIH_VARIANT_ND(K_CONST7, 1, 68, 18, 128, 3, 0, 4),
    GIRIH_VARIANT(K_CONST7, 1, 64, 10, 128, 4, 0, 5),
    GIRIH_VARIANT(K_CONST7, 1, 64, 18, 256, 4, 0, 2),
    GIRIH_VARIANT(K_CONST7, 1, 64, 34, 512, 6, 0, 1),
    GIRIH_VARIANT(K_CONST7, 2, 64, 18, 256, 3, 0, 2),
    GIRIH_VARIANT(K_CONST7, 2, 64, 34, 512, 4, 0, 1),
    GIRIH_VARIANT(K_CONST7, 3, 64, 32, 480, 3, 0, 1),
    GIRIH_VARIANT(K_CONST7, 4, 64, 32, 480, 2, 0, 1),
    GIRIH_VARIANT_C(K_CONST7, 2, 64, 18, 256, 3, 0, 2, 4),
    GIRIH_VARIANT_C(K_CONST7, 3, 64, 32, 480, 3, 0, 1, 4),
    GIRIH_VARIANT_C(K_CONST7, 4, 64, 32, 480, 2, 0, 1, 4),
    GIRIH_VARIANT_D(K_CONST7, 1, 64, 10, 128, 4, 0, 5),
    GIRIH_VARIANT_ND(K_CONST7, 1, 68, 10, 128, 4, 0, 5),
    GIRIH_VARIANT_ND(K_CONST7, 1, 68, 34, 256, 3, 0, 2),
};
const int kNumVariantsConst7 = sizeof(kVariantsConst7) / sizeof(kVariantsConst7[0]);

}  // namespace girih_gpu
