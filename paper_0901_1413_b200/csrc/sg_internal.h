// sg_internal.h -- launch-level interfaces shared by the .cu translation units.
#pragma once
#include <cstdint>
#include <utility>
#include <cuda.h>
#include <cuda_runtime.h>

namespace sg {

// Programmatic dependent launch: a kernel launched with launch_pdl may start (prologue, smem
// carve-out, launch latency) while its predecessor on the stream drains; it must call pdl_wait()
// before touching memory the predecessor writes.  Predecessors call pdl_trigger() to let it in.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
// SG_PDL (experiments): 0 plain launches, 1 PDL (default)
int pdl_mode();
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_mode() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// X(F) for every supported field (F2, F3, F5, F7, GF4, GF8, Z4, Z8), used to dispatch runtime
// field codes to template instantiations.
#define SG_FOR_EACH_FIELD_CASE(field, X) \
  switch (field) {                       \
    case 0: X(F2); break;                \
    case 1: X(F3); break;                \
    case 2: X(F5); break;                \
    case 3: X(F7); break;                \
    case 4: X(GF4); break;               \
    case 5: X(GF8); break;               \
    case 6: X(Z4); break;                \
    default: X(Z8); break;               \
  }

// the production warp-specialized schedules (TMA staging, setmaxnreg register split): 2 = four
// builder warps, 5 = eight
__host__ __device__ constexpr bool ws_tma(int sched) { return sched == 2 || sched == 5 || sched == 6; }
// schedule 6: warp-specialized (4 builder warps) with a second set of RT row accumulators per
// lookup thread in tensor memory -- each table serves 2 RT NT rows (half the replica-store share)
__host__ __device__ constexpr int rows_of(int rt, int nt, int sched) { return rt * nt * (sched == 6 ? 2 : 1); }

// Column slab per CTA (32-bit words); each lane owns one uint4 (4 words = 128 lanes) of a row.
constexpr int SLAB_WORDS = 4;
// Table replicas: the 8 lanes of one LDS.128 phase read 8 different C rows, so entry g is
// stored 8 times, replica j at bank offset 4j; lane (tid & 7) always reads replica (tid & 7).
constexpr int COPIES = 8;
constexpr int ENTRY_BYTES = COPIES * 16;
constexpr int THREADS = 256;

struct M4rmArgs {
  const uint32_t* B;   // [R][l][wc32]   32-bit view of B's planes (row = 2*W64 words)
  const uint32_t* AT;  // k = 8: index words [wa32 := nwords][mpad]; else A^T planes [R][wa32][mpad]
  uint32_t* C;         // final [R][m][wc32] or partial [splits][R][mpad][wc32]
  int64_t m, l, mpad;
  int wa32, wc32;      // 32-bit words per row of A and of B/C
  int nblocks, bps;    // k-blocks in total, k-blocks per split
  int partial;         // 1: write raw partial sums (split-K), 0: canonical C
  // stream-K (partial = 0): CTA c covers work units [c U / G, (c+1) U / G) of U = tiles x nblocks
  int streamk;
  int64_t units;
  int64_t dp_tiles;    // stream-K hybrid: tiles [0, dp_tiles) go whole, CTA c takes c, c + G, ...; the
                       // units cover tiles [dp_tiles, tiles) only
  int slabs;           // tiles = slabs x row groups, tile t -> slab t % slabs, row group t / slabs
  uint32_t* P2;        // compact stream-K partials [G * SK_SLOTS][R][ROWS][4]
  int early_trigger;   // experiments (SG_PDL=2): release the dependent reduction at kernel start
  int tma_b;           // stage B's k-blocks with one TMA tensor copy each (k = 8, wc32 % 4 == 0,
                       // B 16-B aligned)
  int tma_a;           // ... and A's index words with 1-D bulk copies (with tma_b only)
};
// Streamed B (sg_m4rm_host; stream-K warp-specialized TMA plans, the STRM kernel instantiations):
// B's chunk c -- 4-block groups [chunk_lo(c), chunk_lo(c + 1)): chunks double in size from
// g0 = first_groups up to g0 2^cap_log, then stay at that size -- may be read once ready[c] - epoch >= 0 (written by the upload stream behind
// chunk c's copy).  perm: per tile, the order of its 4-block groups (virtual group
// -> real group) that lets each segment start on blocks that arrive first.  err: set (to the
// chunk + 1) when a wait times out; the product is then garbage and reported failed.
// First 4-block group of B chunk c (g0 = first groups, chunks double up to g0 2^q, then equal);
// chunk_of(g) inverts it.
__host__ __device__ inline int64_t chunk_lo(int c, int g0, int q) {
  return c <= q ? (int64_t)g0 * ((1LL << c) - 1) : (int64_t)g0 * (((1LL << q) - 1) + (int64_t)(c - q) * (1LL << q));
}
__host__ __device__ inline int chunk_of(int g, int g0, int q) {
  const int64_t lq = (int64_t)g0 * ((1LL << q) - 1);
  if (g < lq) {
    const unsigned x = (unsigned)(g / g0 + 1);
    int c = 0;
    while ((2u << c) <= x) ++c;  // floor(log2(x))
    return c;
  }
  return q + (int)((g - lq) / ((int64_t)g0 << q));
}
struct M4rmStreamArgs : M4rmArgs {
  const unsigned* ready;
  unsigned epoch;
  int first_groups;
  int cap_log;
  int nchunks;
  unsigned poll_ns;  // sleep between two polls of a flag that has not landed
  const int* perm;
  int ngroups;
  unsigned* err;
};
constexpr int SK_SLOTS = 2;  // compact partial slots per stream-K CTA: its first and last segment
// Fused small products (one launch, the *_fused instantiations of the serial / pipelined k = 8
// variants): the CTAs stage A's own plane words (no index pre-pass; the bytes are extracted from
// them, F3's "+1" index as A0 ^ A1), write split-K partials to C (= the partial planes), then the
// splits of every tile meet at an arrival counter (a cooperative launch: all CTAs co-resident)
// and each sums its 1/splits of the tile's rows into Cout.  cnt: 2 x tiles arrival / departure
// counters, zero between launches (the last CTA to leave a tile resets them).
struct M4rmFusedArgs : M4rmArgs {
  const uint32_t* A;  // [R][m][wa32]  32-bit view of A's planes
  uint32_t* Cout;     // final [R][m][wc32]
  unsigned* cnt;
  int ntiles;
};

typedef void (*KernelFn)(M4rmArgs, CUtensorMap);  // (args, B as a 3-D u32 tensor map for TMA staging)
typedef void (*StreamKernelFn)(M4rmStreamArgs, CUtensorMap);
typedef void (*FusedKernelFn)(M4rmFusedArgs, CUtensorMap);
// schedule codes seen through the ABI (sg_kernel_info, sg_plan, sg_set_plan_override): a fused
// variant reports its serial / pipelined schedule + SCHED_FUSED
constexpr int SCHED_FUSED = 10;
struct KernelInfo {
  KernelFn fn;
  int field, k, rt, threads;  // threads = lookup threads (rows = rt * threads)
  int launch_threads;  // threads + 32 for the warp-specialized schedule
  int sched;           // 0 serial, 1 pipelined (double-buffered table), 2 warp-specialized
  int smem_bytes;
  int regs;            // filled in lazily from cudaFuncGetAttributes
  int occupancy;       // CTAs per SM, filled lazily
  int ablation;        // experiments only: never planned unless sg_set_ablation selects it
  StreamKernelFn fn_stream;  // the same variant reading streamed B (M4rmStreamArgs), or nullptr
  int smem_stream;           // ... and its dynamic shared memory (+ the staged group order)
  FusedKernelFn fn_fused;    // a fused small-product variant (fn == nullptr then), see M4rmFusedArgs
  int pair_nt;               // k = 8 index records two rows per word (rows r, r + pair_nt), or 0
};
// streamed products stage their tile's group order in shared memory: at most this many groups
constexpr int STRM_MAX_GROUPS = 2048;

// Registry of compiled M4RM instantiations (sg_m4rm.cu).
int m4rm_kernel_count();
KernelInfo* m4rm_kernel_at(int i);

// k = 8: packed index words [nwords][mpad]; k < 8: A^T bit planes [R][wa32][mpad]
cudaError_t launch_transpose_a(int field, int k, const uint32_t* A, uint32_t* AT, int64_t m, int64_t mpad,
                               int wa32, int nwords, int pair_nt, cudaStream_t st);
cudaError_t launch_m4rm(const KernelInfo& ki, const M4rmArgs& a, const CUtensorMap& tmB, dim3 grid,
                        cudaStream_t st);
cudaError_t launch_m4rm_streamed(const KernelInfo& ki, const M4rmStreamArgs& a, const CUtensorMap& tmB, dim3 grid,
                                 cudaStream_t st);
// cooperative launch (every CTA co-resident: the split-K arrival counters spin)
cudaError_t launch_m4rm_fused(const KernelInfo& ki, const M4rmFusedArgs& a, const CUtensorMap& tmB, dim3 grid,
                              cudaStream_t st);
// up to SLICES_MAX equally shaped R-plane row slices with their own plane strides (u32 words)
constexpr int SLICES_MAX = 8;
struct SliceSet {
  const uint32_t* base[SLICES_MAX];
  int64_t pstride[SLICES_MAX];
  int n;
};
cudaError_t launch_sum_slices(int field, const SliceSet& s, uint32_t* out, int64_t out_pstride, int64_t rows,
                              int wc32, cudaStream_t st);
cudaError_t launch_reduce_splits(int field, const uint32_t* P, uint32_t* C, int64_t m, int64_t mpad,
                                 int wc32, int splits, cudaStream_t st);
cudaError_t launch_reduce_streamk(int field, const uint32_t* P2, uint32_t* C, int64_t m, int wc32, int rows_cta,
                                  int slabs, int64_t tiles, int64_t tile0, int nblocks, int64_t units, int ctas,
                                  cudaStream_t st);

// load every auxiliary kernel of `field` (index pre-pass, reductions) ahead of a streamed product
cudaError_t preload_aux_kernels(int field);

// sg_pack.cu
cudaError_t launch_pack(int field, const uint8_t* dense, int64_t m, int64_t n, int64_t ld,
                        uint64_t* planes, int* err_flag, cudaStream_t st);
cudaError_t launch_unpack(int field, const uint64_t* planes, int64_t m, int64_t n, uint8_t* dense,
                          int64_t ld, int* err_flag, cudaStream_t st);
cudaError_t launch_canonicalize(int field, uint64_t* planes, int64_t rows, int64_t w64,
                                cudaStream_t st);
struct Planes {
  uint64_t* p[3];
};
cudaError_t launch_plane_op(int op, Planes dst, Planes src, int64_t rows, int64_t w64, uint64_t tail,
                            int scalar, cudaStream_t st);
cudaError_t launch_block_driver(int field, Planes C, int64_t wc64, Planes A, int64_t wa64, int64_t col0,
                                int kp, Planes T, int64_t row0, int64_t row1, cudaStream_t st);
cudaError_t launch_build_table(int field, Planes B, int64_t b_rows, int64_t row_base, int kp, int64_t wc64,
                               Planes T, cudaStream_t st);
cudaError_t launch_classical(int field, Planes A, int64_t wa64, Planes B, int64_t wb64, Planes C, int64_t m,
                             int64_t l, cudaStream_t st);
cudaError_t launch_classical_block(int field, Planes C, int64_t wc64, Planes A, int64_t wa64, Planes B, int64_t m,
                                   int64_t l, cudaStream_t st);

// sg_peaks.cu
int probe_peaks(int device, double* lop3_per_clk_sm, double* lds_bytes_per_clk_sm, double* sm_mhz);

}  // namespace sg
