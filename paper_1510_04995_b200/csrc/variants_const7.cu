// variants_const7.cu -- zwave instantiations for const7 (kept in its own TU so nvcc builds kinds in parallel).
#include "variants.h"

namespace girih_gpu {

const Variant kVariantsConst7[] = {
    GIRIH_VARIANT(K_CONST7, 1, 64, 32, 512, 2),
    GIRIH_VARIANT(K_CONST7, 2, 64, 32, 512, 2),
    GIRIH_VARIANT(K_CONST7, 3, 64, 32, 512, 2),
    GIRIH_VARIANT(K_CONST7, 4, 64, 32, 512, 2),
};
const int kNumVariantsConst7 = sizeof(kVariantsConst7) / sizeof(kVariantsConst7[0]);

}  // namespace girih_gpu
