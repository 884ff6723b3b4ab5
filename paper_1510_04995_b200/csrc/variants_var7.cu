// variants_var7.cu -- zwave instantiations for var7 (kept in its own TU so nvcc builds kinds in parallel).
#include "variants.h"

namespace girih_gpu {

const Variant kVariantsVar7[] = {
    GIRIH_VARIANT(K_VAR7, 1, 64, 32, 512, 2),
    GIRIH_VARIANT(K_VAR7, 2, 64, 32, 512, 2),
    GIRIH_VARIANT(K_VAR7, 3, 64, 32, 512, 2),
    GIRIH_VARIANT(K_VAR7, 4, 64, 32, 512, 2),
};
const int kNumVariantsVar7 = sizeof(kVariantsVar7) / sizeof(kVariantsVar7[0]);

}  // namespace girih_gpu
