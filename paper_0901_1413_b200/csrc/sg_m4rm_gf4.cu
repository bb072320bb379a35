// sg_m4rm_gf4.cu -- M4RM kernel instantiations for GF4 (one translation unit per field so
// the library builds in parallel).
#include "sg_m4rm_kernel.cuh"

namespace sg {

static KernelInfo g_table[] = {
    SG_K(GF4, 8, 16, 2, 256),
    SG_K(GF4, 8, 16, 5, 256),  // 8 builder warps: the three replicated Karatsuba planes
    SG_KTM(GF4, 16),           // 8192 rows per table: 16 row-slots in registers + 16 in TMEM
    SG_K(GF4, 8, 8, 2, 256),
    SG_KSET8(GF4),
    SG_KFUSED(GF4),
    SG_KSET8_2PLANE(GF4),
    SG_KLOW(GF4),
};

int kernels_gf4(KernelInfo** out) {
  *out = g_table;
  return (int)(sizeof(g_table) / sizeof(g_table[0]));
}

}  // namespace sg
