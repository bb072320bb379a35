// sg_m4rm_z8.cu -- M4RM kernel instantiations for Z8 (one translation unit per field so
// the library builds in parallel).
#include "sg_m4rm_kernel.cuh"

namespace sg {

static KernelInfo g_table[] = {
    SG_KTM(Z8, 8),  // 4096 rows per table: 8 row-slots in registers + 8 in tensor memory
    SG_K(Z8, 8, 8, 2, 256),
    SG_K(Z8, 8, 4, 2, 256),
    SG_KSET8(Z8),
    SG_KFUSED(Z8),
    SG_K(Z8, 8, 8, 1, 256),
    SG_KLOW(Z8),
};

int kernels_z8(KernelInfo** out) {
  *out = g_table;
  return (int)(sizeof(g_table) / sizeof(g_table[0]));
}

}  // namespace sg
