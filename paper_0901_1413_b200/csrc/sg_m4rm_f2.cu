// sg_m4rm_f2.cu -- M4RM kernel instantiations for F2 (one translation unit per field so
// the library builds in parallel).
#include "sg_m4rm_kernel.cuh"

namespace sg {

static KernelInfo g_table[] = {
    SG_KTM(F2, 16),  // 8192 rows per table: 16 row-slots in registers + 16 in tensor memory
    SG_KTM(F2, 32),  // 16384 rows per table: 32 + 32 (one-plane slots: 4 words each)
    SG_K(F2, 8, 16, 2, 256),
    SG_KSET8(F2),
    SG_KFUSED(F2),
    SG_KSET8_2PLANE(F2),
    SG_KLOW(F2),
};

int kernels_f2(KernelInfo** out) {
  *out = g_table;
  return (int)(sizeof(g_table) / sizeof(g_table[0]));
}

}  // namespace sg
