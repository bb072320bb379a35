// sg_m4rm_z4.cu -- M4RM kernel instantiations for Z4 (one translation unit per field so
// the library builds in parallel).
#include "sg_m4rm_kernel.cuh"

namespace sg {

static KernelInfo g_table[] = {
    SG_KTM(Z4, 16),  // 8192 rows per table: 16 row-slots in registers + 16 in tensor memory
    SG_K(Z4, 8, 16, 2, 256),
    SG_K(Z4, 8, 8, 2, 256),
    SG_KSET8(Z4),
    SG_KFUSED(Z4),
    SG_KSET8_2PLANE(Z4),
    SG_KLOW(Z4),
};

int kernels_z4(KernelInfo** out) {
  *out = g_table;
  return (int)(sizeof(g_table) / sizeof(g_table[0]));
}

}  // namespace sg
