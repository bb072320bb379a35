// sg_m4rm_f3.cu -- M4RM kernel instantiations for F3 (one translation unit per field so
// the library builds in parallel).
#include "sg_m4rm_kernel.cuh"

namespace sg {

static KernelInfo g_table[] = {
    SG_K(F3, 8, 16, 2, 256),
    SG_KTM(F3, 16),  // 8192 rows per table: 16 row-slots in registers + 16 in tensor memory
    SG_K(F3, 8, 8, 2, 256),
    SG_KSET8(F3),
    SG_KFUSED(F3),
    SG_KSET8_2PLANE(F3),
    SG_KLOW(F3),
#ifdef SG_EXPERIMENTS  // ablation variants (tools/ablate.py): results are wrong by design
    SG_KA(F3, 8, 16, 0, 256, 1),
    SG_KA(F3, 8, 16, 0, 256, 2),
    SG_KA(F3, 8, 16, 0, 256, 4),
    SG_KA(F3, 8, 16, 0, 256, 3),
    SG_KA(F3, 8, 16, 1, 256, 1),
    SG_KA(F3, 8, 16, 1, 256, 2),
    SG_KA(F3, 8, 16, 1, 256, 4),
    SG_KA(F3, 8, 16, 2, 256, 1),
    SG_KA(F3, 8, 16, 2, 256, 2),
    SG_KA(F3, 8, 16, 2, 256, 4),
#endif
};

int kernels_f3(KernelInfo** out) {
  *out = g_table;
  return (int)(sizeof(g_table) / sizeof(g_table[0]));
}

}  // namespace sg
