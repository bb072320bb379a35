// sg_m4rm_f7.cu -- M4RM kernel instantiations for F7 (one translation unit per field so
// the library builds in parallel).
#include "sg_m4rm_kernel.cuh"

namespace sg {

static KernelInfo g_table[] = {
    SG_K(F7, 8, 8, 2, 256),
    SG_K(F7, 8, 4, 2, 256),
    SG_KTM(F7, 8),  // 4096 rows per table: 8 row-slots in registers + 8 in tensor memory
    SG_KSET8(F7),
    SG_KFUSED(F7),
    SG_K(F7, 8, 8, 1, 256),
    SG_K(F7, 8, 4, 1, 512),
    SG_KLOW(F7),
#ifdef SG_EXPERIMENTS  // ablation variants (tools/ablate.py): results are wrong by design
    SG_KA(F7, 8, 8, 1, 256, 1),
    SG_KA(F7, 8, 8, 1, 256, 2),
    SG_KA(F7, 8, 8, 1, 256, 4),
    SG_KA(F7, 8, 8, 2, 256, 2),
    SG_KA(F7, 8, 8, 2, 256, 4),
#endif
};

int kernels_f7(KernelInfo** out) {
  *out = g_table;
  return (int)(sizeof(g_table) / sizeof(g_table[0]));
}

}  // namespace sg
