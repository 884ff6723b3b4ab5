// variants_var25.cu -- zwave instantiations for var25 (kept in its own TU so nvcc builds kinds in parallel).
#include "variants.h"

namespace girih_gpu {

const Variant kVariantsVar25[] = {
    GIRIH_VARIANT(K_VAR25, 1, 64, 32, 512, 2),
    GIRIH_VARIANT(K_VAR25, 2, 32, 32, 256, 2),
};
const int kNumVariantsVar25 = sizeof(kVariantsVar25) / sizeof(kVariantsVar25[0]);

}  // namespace girih_gpu
