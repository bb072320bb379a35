// sg_m4rm_f5.cu -- M4RM kernel instantiations for F5 (one translation unit per field so
// the library builds in parallel).
#include "sg_m4rm_kernel.cuh"

namespace sg {

static KernelInfo g_table[] = {
    SG_K(F5, 8, 8, 2, 256),
    SG_K(F5, 8, 4, 2, 256),
    SG_KTM(F5, 8),  // 4096 rows per table: 8 row-slots in registers + 8 rotating through TMEM
    SG_KSET8(F5),
    SG_KFUSED(F5),
    SG_K(F5, 8, 8, 1, 256),
    SG_K(F5, 8, 4, 1, 512),
    SG_KLOW(F5),
};

int kernels_f5(KernelInfo** out) {
  *out = g_table;
  return (int)(sizeof(g_table) / sizeof(g_table[0]));
}

}  // namespace sg
