// sg_m4rm_kernel.cuh -- the bitsliced Method-of-Four-Russians kernel C = A*B on sm_100a
// (instantiated per field in sg_m4rm_<field>.cu; launched by sg_m4rm.cu).
//
// Reference path (what this replaces): m4rm_multiply = for each k-block s,
// build_table then _core.active().m4rm_block_<f> (_core_py.py:205-281),
// whose per-row loop does  C_i += sum_d alpha_d * T[phi_d(a_i, block s)].
//
// B200 design:
//  * A tile is a 128-column slab of C (4 x 32-bit words per plane) x ROWS = RT*NT rows.  A CTA
//    walks a range of k-blocks of a tile with C in registers: lane (t, tid) holds rows t*NT+tid,
//    one uint4 per accumulator plane.  Work assignment (m4rm_kernel / run_segments): one tile
//    and a split of k per CTA, or stream-K (one wave of CTAs over tiles x k-blocks; whole tiles
//    straight to C, partial ones to compact slots for reduce_streamk_kernel).
//  * Per k-block the CTA builds the 2^K-entry table of its slab in shared memory:
//    phase 1: two half tables (rows 0..3 and 4..7 of the block, 16 entries each) from B rows
//    staged ahead of time; phase 2: T[g] = Thi[g>>4] + Tlo[g&15], one bitsliced field add per
//    word, written as 8 replicas (see COPIES).
//  * Lookups: the 8 lanes of each LDS.128 phase hold 8 different rows, i.e. 8 random table
//    entries.  Replica j of every entry sits at bank offset 4j and lane (tid&7) reads replica
//    tid&7, so each phase touches all 32 banks exactly once: conflict-free for any indices.
//  * Index bytes come from the index pre-pass (A's per-block basis bytes packed into 32-bit
//    records [word][row], F3's first byte pre-XORed to A0^A1): one conflict-free LDS.32 per
//    (row, record word), a PRMT and a LEA per lookup.
//  * Schedules: SCHED 0 serial, 1 pipelined (double-buffered table), 2 warp-specialized
//    (4 builder warps build block s+1 while 8 lookup warps consume block s; FULL / EMPTY named
//    barriers; B's rows staged by one TMA tensor copy per block and A's index words by 1-D bulk
//    copies, both completing on mbarriers; setmaxnreg moves registers from the builder
//    warpgroup to the lookup warpgroups, whose code is compiled separately (ROLE)).
//  * Epilogue: canonical reduce (F5 mod 15 -> mod 5, F7 fold) and store, or canonical partial
//    sums for split-K / stream-K.
#pragma once
#include <cstdio>
#include <type_traits>

#include "sg_field.cuh"
#include "sg_internal.h"

namespace sg {

// Per-CTA phase timestamps (tools/small_timeline.cu builds with SG_TIMELINE; compiled out otherwise)
#ifdef SG_TIMELINE
__device__ unsigned long long g_tl[8192][8];
#define SG_TL(i)                                                                                   \
  do {                                                                                             \
    if (threadIdx.x == 0) {                                                                        \
      unsigned long long t_;                                                                       \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                       \
      g_tl[(blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x][i] = t_;               \
    }                                                                                              \
  } while (0)
#else
#define SG_TL(i) \
  do {           \
  } while (0)
#endif

__device__ __forceinline__ void cp_async16(void* dst, const void* src, int bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(src), "r"(bytes));
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src, int bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(src), "r"(bytes));
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src, int bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(src), "r"(bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N> __device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// ---- TMA bulk copies (cp.async.bulk) completing on shared-memory mbarriers
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_inval(uint64_t* bar) {
  asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred P1;\n LAB_WAIT:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @P1 bra DONE;\n bra LAB_WAIT;\n DONE:\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

// Streamed B: wait until the upload stream has published chunk c (ready[c] - epoch >= 0, a
// cyclic compare; relaxed polls with __nanosleep), and return the last chunk of the run c, c+1, ...
// that has landed (the flags are written in chunk order, so one acquire of that flag orders the
// reads of every chunk up to it); then order the TMA (async proxy) reads after it.  A wait longer
// than 10 s flags an error and gives up instead of hanging the GPU.  (A fence.acq_rel per chunk
// cost ~1.4 us each: 17 us per 2048-row F5 product even with every flag already set.)
__device__ __forceinline__ int wait_chunk(const unsigned* ready, int c, int nchunks, unsigned epoch, unsigned* err,
                                          unsigned poll_ns) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ready + c) : "memory");
  if ((int)(v - epoch) < 0) {
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    do {
      __nanosleep(poll_ns);
      asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ready + c) : "memory");
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 10000000000ull) {
        atomicExch(err, (unsigned)c + 1u);  // the chunk it gave up on, + 1
        return c;
      }
    } while ((int)(v - epoch) < 0);
  }
  // the run of landed chunks after c, 4 flags per round with the loads in flight together (one
  // dependent round trip per flag cost ~0.7 us each, ~5 us per segment start)
  int last = c;
  for (int j0 = c + 1; j0 < nchunks; j0 += 4) {
    unsigned f[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      f[i] = epoch - 1u;  // past nchunks: not landed
      if (j0 + i < nchunks)
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(f[i]) : "l"(ready + j0 + i) : "memory");
    }
    int run = 0;
#pragma unroll
    for (int i = 3; i >= 0; --i) run = (int)(f[i] - epoch) >= 0 ? run + 1 : 0;
    last = j0 + run - 1;
    if (run < 4) break;
  }
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ready + last) : "memory");
  asm volatile("fence.proxy.async.global;" ::: "memory");  // ... for the TMA (async proxy) reads too
  return last;
}

template <int F> __device__ __forceinline__ V<F> vzero() {
  V<F> v;
#pragma unroll
  for (int d = 0; d < Traits<F>::R; ++d) v.p[d] = 0u;
  return v;
}

// GF(4), k = 8: Karatsuba tables.  Besides T0 (over B's plane 0) and T1 (plane 1) the table
// holds T2 = T0 ^ T1 (over B0 ^ B1), and a row's update is C0 += T0[g0] + T1[g1],
// C1 += T2[g0 ^ g1] + T0[g0]  ((a0 + a1 x)(b0 + b1 x) = (a0 b0 + a1 b1) + ((a0 + a1)(b0 + b1) + a0 b0) x
// mod x^2 + x + 1): three one-plane lookups per (row, k-block) instead of two two-plane ones.
template <int F, int K> __host__ __device__ constexpr bool karatsuba() { return F == GF4 && K == 8; }
// table planes in shared memory
template <int F, int K> __host__ __device__ constexpr int table_planes() { return karatsuba<F, K>() ? 3 : Traits<F>::R; }
// staging slots of A's index words: Karatsuba GF(4) needs the room of the third table plane, and
// with two k-blocks per index word two slots are enough (see issue_a)
// half-table buffers: the serial / pipelined schedules build block s+1's (or s+2's) while block
// s's are read; the warp-specialized builders finish with one before the next
__host__ __device__ constexpr int half_bufs(int sched) { return sched >= 2 ? 1 : 2; }

// staged index source: k = 8 packed records from the pre-pass (one plane), else R planes of A
// words (A^T from the transpose pre-pass, or A itself in the fused small-product kernels)
template <int F, int K, bool FUSED = false> __host__ __device__ constexpr bool packed_index() { return K == 8 && !FUSED; }
// k = 8 records of two-index fields (F3, GF(4), Z4: 2 bytes per row and k-block) are packed two
// ROWS per 32-bit word -- rows r and r + NT of each 2 NT-row group, one k-block -- when the
// variant's row-slots come in pairs (RT even): a lane's LDS.32 then serves two of its rows, half
// the index wavefronts of one row per word (the pre-pass writes [k-block][mpad / 2] words).
template <int F, int K, int RT, bool FUSED = false> __host__ __device__ constexpr bool paired_index() {
  return packed_index<F, K, FUSED>() && Traits<F>::NI == 2 && RT % 2 == 0;
}
// (schedule 6 with Karatsuba GF(4): two slots -- the third table plane and the doubled rows leave
// no room for a third; its builders then stage block s's index words just in time, see JIT_A)
template <int F, int K, int RT, bool FUSED = false, int SCHED = 0> __host__ __device__ constexpr int index_slots() {
  return paired_index<F, K, RT, FUSED>() ? (SCHED == 6 && karatsuba<F, K>() ? 2 : 3)
                                         : K == 8 && !FUSED ? (karatsuba<F, K>() || SCHED == 6 ? 2 : 3) : 2;
}
// u32 of shared memory staging A's index words / planes (NSLOT slots)
template <int F, int K, int RT, int NT, bool FUSED = false, int SCHED = 0>
__host__ __device__ constexpr int index_stage_words() {
  return index_slots<F, K, RT, FUSED, SCHED>() * (packed_index<F, K, FUSED>() ? 1 : Traits<F>::R) *
         (paired_index<F, K, RT, FUSED>() ? rows_of(RT, NT, SCHED) / 2 : rows_of(RT, NT, SCHED));
}

// ---- tensor memory (schedule 6): a lookup thread's second set of row accumulators
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const u32 (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, u32 (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr)
               : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const u32 (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, u32 (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_st4(uint32_t taddr, const u32* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr), "r"(r[0]), "r"(r[1]),
               "r"(r[2]), "r"(r[3])
               : "memory");
}
__device__ __forceinline__ void tmem_ld4(uint32_t taddr, u32* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(taddr)
               : "memory");
}
// one row-slot's accumulator words (4 x RS: 4, 8, 12, 16 or 20) to / from tensor memory
template <int N> __device__ __forceinline__ void tmem_st(uint32_t taddr, u32 (&r)[N]) {
  static_assert(N == 4 || N == 8 || N == 12 || N == 16 || N == 20, "4, 8, 12, 16 or 20 accumulator words per row-slot");
  if constexpr (N == 4) {
    tmem_st4(taddr, &r[0]);
  } else if constexpr (N == 8) {
    tmem_st8(taddr, r);
  } else if constexpr (N == 12) {
    tmem_st8(taddr, *reinterpret_cast<u32(*)[8]>(&r[0]));
    tmem_st4(taddr + 8, &r[8]);
  } else if constexpr (N == 16) {
    tmem_st16(taddr, r);
  } else {
    tmem_st16(taddr, *reinterpret_cast<u32(*)[16]>(&r[0]));
    tmem_st4(taddr + 16, &r[16]);
  }
}
template <int N> __device__ __forceinline__ void tmem_ld(uint32_t taddr, u32 (&r)[N]) {
  if constexpr (N == 4) {
    tmem_ld4(taddr, &r[0]);
  } else if constexpr (N == 8) {
    tmem_ld8(taddr, r);
  } else if constexpr (N == 12) {
    tmem_ld8(taddr, *reinterpret_cast<u32(*)[8]>(&r[0]));
    tmem_ld4(taddr + 8, &r[8]);
  } else if constexpr (N == 16) {
    tmem_ld16(taddr, r);
  } else {
    tmem_ld16(taddr, *reinterpret_cast<u32(*)[16]>(&r[0]));
    tmem_ld4(taddr + 16, &r[16]);
  }
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// Row accumulator of one lane: 4 words x RS planes.
template <int F> struct Acc { u32 w[4][Traits<F>::RS]; };

// Table rows of one (row, k-block): NI lookups x R planes, one uint4 (4 words) each.
template <int F> struct Rows { uint4 v[Traits<F>::NI][Traits<F>::R]; };

// Load the table rows at byte offsets e[] (entry * ENTRY_BYTES) from this lane's replica base.
template <int F, int TPL, bool KAR = false>
__device__ __forceinline__ void load_rows(Rows<F>& r, const unsigned char* __restrict__ tl, const u32 (&e)[3]) {
  if constexpr (KAR) {  // T0[g0], T1[g1], T2[g0 ^ g1] (entry offsets are g * ENTRY_BYTES: XOR them)
    r.v[0][0] = *reinterpret_cast<const uint4*>(tl + e[0]);
    r.v[1][0] = *reinterpret_cast<const uint4*>(tl + e[1] + TPL * 16);
    r.v[0][1] = *reinterpret_cast<const uint4*>(tl + (e[0] ^ e[1]) + 2 * TPL * 16);
    return;
  }
#pragma unroll
  for (int i = 0; i < Traits<F>::NI; ++i)
#pragma unroll
    for (int d = 0; d < Traits<F>::R; ++d)
      r.v[i][d] = *reinterpret_cast<const uint4*>(tl + e[i] + d * TPL * 16);
}

__device__ __forceinline__ u32 comp(const uint4& v, int w) { return w == 0 ? v.x : w == 1 ? v.y : w == 2 ? v.z : v.w; }

// One (row, k-block) update of the 4 C words a lane owns from its loaded table rows.
template <int F, bool KAR = false>
__device__ __forceinline__ void accumulate(Acc<F>& c, const Rows<F>& r) {
  if constexpr (KAR) {  // C0 += T0[g0] + T1[g1];  C1 += T2[g0 ^ g1] + T0[g0]   (2 LOP3 per word)
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const u32 t0 = comp(r.v[0][0], w);
      c.w[w][0] ^= t0 ^ comp(r.v[1][0], w);
      c.w[w][1] ^= comp(r.v[0][1], w) ^ t0;
    }
    return;
  }
  if constexpr (F == F5 || F == F7) {
    // carry-save networks issued adder by adder across the four words (ILP 4 per step)
    u32 in[4][9];
#pragma unroll
    for (int w = 0; w < 4; ++w)
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int d = 0; d < 3; ++d) in[w][3 * i + d] = comp(r.v[i][d], w);
    if constexpr (F == F7) f7_acc4(c.w, in); else f5_acc4(c.w, in);
    return;
  }
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    u32* q = c.w[w];
    if constexpr (F == F2) {
      q[0] ^= comp(r.v[0][0], w);
    } else if constexpr (F == F3) {
      // basis {1, -1}: C += T[pos]; C -= T[neg]   (_core_py.py:213-222), 6 LOP3 per word
      f3_add(q[0], q[1], comp(r.v[0][0], w), comp(r.v[0][1], w));
      f3_sub(q[0], q[1], comp(r.v[1][0], w), comp(r.v[1][1], w));
    } else if constexpr (F == GF4) {
      // power basis {1, x}: C += T[g0] + x*T[g1],  x*(t0, t1) = (t1, t0 ^ t1)
      const u32 q1 = comp(r.v[1][1], w);
      q[0] ^= comp(r.v[0][0], w) ^ q1;
      q[1] ^= comp(r.v[0][1], w) ^ comp(r.v[1][0], w) ^ q1;
    } else if constexpr (F == GF8) {
      // power basis {1, x, x^2} mod x^3+x+1: C += a + x*b + x^2*d with
      // x*b = (b2, b0^b2, b1) and x^2*d = (d1, d1^d2, d0^d2); 7 LOP3 per word
      const u32 a0 = comp(r.v[0][0], w), a1 = comp(r.v[0][1], w), a2 = comp(r.v[0][2], w);
      const u32 b0 = comp(r.v[1][0], w), b1 = comp(r.v[1][1], w), b2 = comp(r.v[1][2], w);
      const u32 d0 = comp(r.v[2][0], w), d1 = comp(r.v[2][1], w), d2 = comp(r.v[2][2], w);
      q[0] = q[0] ^ a0 ^ b2 ^ d1;
      q[1] = (q[1] ^ a1 ^ b0) ^ (b2 ^ d1 ^ d2);
      q[2] = q[2] ^ a2 ^ b1 ^ d0 ^ d2;
    } else if constexpr (F == Z4) {
      // basis {1, 2} (_core_py.py:225-238): C += x + 2y mod 4, 3 LOP3 per word
      const u32 x0 = comp(r.v[0][0], w), x1 = comp(r.v[0][1], w), y0 = comp(r.v[1][0], w);
      q[1] = q[1] ^ x1 ^ y0 ^ (q[0] & x0);
      q[0] ^= x0;
    } else if constexpr (F == Z8) {
      // basis {1, 2, 4} (_core_py.py:284-286): C += x + 2y + 4z mod 8 as one carry-save sum
      const u32 x0 = comp(r.v[0][0], w), x1 = comp(r.v[0][1], w), x2 = comp(r.v[0][2], w);
      const u32 y0 = comp(r.v[1][0], w), y1 = comp(r.v[1][1], w), z0 = comp(r.v[2][0], w);
      const u32 k1 = q[0] & x0;
      const u32 a = q[1] ^ x1 ^ y0;
      const u32 ma = lop3<LOP_MAJ>(q[1], x1, y0);
      q[2] = (q[2] ^ x2 ^ y1) ^ (z0 ^ ma ^ (a & k1));
      q[1] = a ^ k1;
      q[0] ^= x0;
    } else {
      // F5 / F7, basis {1, 2, 4}: C += T[g0] + 2*T[g1] + 4*T[g2] (the reference's Horner form,
      // _core_py.py:241-255, reassociated); doubling is a plane rotation in both accumulators.
      const u32 x0 = comp(r.v[0][0], w), x1 = comp(r.v[0][1], w), x2 = comp(r.v[0][2], w);
      const u32 y0 = comp(r.v[1][0], w), y1 = comp(r.v[1][1], w), y2 = comp(r.v[1][2], w);
      const u32 z0 = comp(r.v[2][0], w), z1 = comp(r.v[2][1], w), z2 = comp(r.v[2][2], w);
      if constexpr (F == F7) {
        f7_acc(q[0], q[1], q[2], q[3], x0, x1, x2, y0, y1, y2, z0, z1, z2);
      } else {
        f5_acc(q[0], q[1], q[2], q[3], q[4], x0, x1, x2, y0, y1, y2, z0, z1, z2);
      }
    }
  }
}

// Accumulator -> output planes (canonical for the final C and for split-K partials of F5).
// F7 accumulator (q0, k0, q1, q2): value = (q0,q1,q2) + k0 mod 7.  F5 (q0, q1, q2, k2, q3):
// value = (q0,q1,q2,q3) + 4 k2 mod 15, then mod 5.
template <int F> __device__ __forceinline__ void finish(const u32 (&q)[Traits<F>::RS], u32 (&o)[Traits<F>::R],
                                                        bool canonical) {
  if constexpr (F == F5) {
    u32 v0 = q[0], v1 = q[1], v2 = q[2], v3 = q[4];
    add15(v0, v1, v2, v3, 0u, 0u, q[3], 0u);
    mod15_to_f5(v0, v1, v2, v3, o[0], o[1], o[2]);
  } else if constexpr (F == F7) {
    o[0] = q[0]; o[1] = q[2]; o[2] = q[3];
    f7_add(o[0], o[1], o[2], q[1], 0u, 0u);
    if (canonical) f7_reduce(o[0], o[1], o[2]);
  } else {
#pragma unroll
    for (int d = 0; d < Traits<F>::R; ++d) o[d] = q[d];
  }
}

// Named barriers (id 0 is __syncthreads) for the warp-specialized schedule.
__device__ __forceinline__ void nbar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void nbar_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// SCHED 0: per k-block  phase1 | sync | phase2 | sync | lookups   (one table buffer)
// SCHED 1: per k-block  lookups(s) + phase2(s+1) + phase1(s+2) | sync  (two table buffers)
// SCHED 2/3/4: warp-specialized (k = 8): NT lookup threads + 4/1/2 builder warps that stage B and A
//          with cp.async and builds block s+1's table into the other buffer while the lookup warps
//          consume block s; FULL/EMPTY named barriers hand the two buffers back and forth.
// ABL (experiments only, 0 in production): bit 0 skips the table-replica stores, bit 1 replaces
// the field update by a plain XOR of the looked-up rows, bit 2 skips the lookups.
// builder threads of the warp-specialized schedules: SCHED 2 -> 4 warps, 3 -> 1 warp, 4 -> 2 warps
// SCHED 5: warp-specialized with 8 builder warps (512-thread CTAs: the lookup warps keep 192
// registers, the builders 64) for kernels whose table build is their critical path (GF(4)'s three
// replicated Karatsuba planes)
__host__ __device__ constexpr int ws_builders(int sched) {
  return sched == 2 || sched == 6 ? 128 : sched == 3 ? 32 : sched == 4 ? 64 : sched == 5 ? 256 : 0;
}


// One segment: the CTA's slab (word0) x row group (row0) x k-blocks [s_begin, s_end), written to
// C (mode 0), to split-K partial plane `slot` (mode 1) or to compact stream-K slot `slot` (mode 2).
// ROLE (warp-specialized schedule only): 1 = the builder warps' part, 2 = the lookup warps' part;
// 0 = everything (the other schedules).  The two roles run separately compiled code so that each
// can live with its own register budget (setmaxnreg in m4rm_kernel).
template <int F, int K, int RT, int SCHED, int NT, int ABL, int ROLE, bool STRM, typename AT>
__device__ __forceinline__ void m4rm_segment(const AT& a, const CUtensorMap* tmB, unsigned char* smem,
                                             const int word0,
                                             const int64_t row0, const int s_begin, const int s_end,
                                             const int mode, const int slot) {
  constexpr bool PIPE = SCHED == 1;
  constexpr bool WS = SCHED >= 2;
  constexpr bool TM = SCHED == 6;  // second accumulator set in tensor memory (see rows_of)
  constexpr bool FUSED = std::is_same_v<AT, M4rmFusedArgs>;
  static_assert(!WS || K == 8, "the warp-specialized schedules are k = 8 only");
  constexpr int R = Traits<F>::R;
  constexpr int E = 1 << K;
  constexpr int KLO = K < 4 ? K : 4;
  constexpr int KHI = K - KLO;
  constexpr int ROWS = rows_of(RT, NT, SCHED);
  constexpr bool KAR = karatsuba<F, K>();
  constexpr int TR = table_planes<F, K>();  // table planes (R, or 3 for Karatsuba GF(4))
  constexpr int TPLANE = E * ENTRY_BYTES;  // bytes per table plane
  constexpr int TPL = TPLANE / 16;         // uint4 per table plane
  constexpr int HALF = 16 * R * 4;         // u32 per half table
  constexpr int NTAB = SCHED >= 1 ? 2 : 1;
  constexpr int PD = PIPE ? 3 : 2;         // cp.async prefetch distance of B rows in k-blocks
  constexpr int PDA = 2;                   // ... and of A's index words
  // k = 8: A's index bytes arrive pre-packed as one record of NIP bytes per k-block (the
  // index_words pre-pass), RPW records per 32-bit word, NSLOT staging slots of ROWS words.
  // k < 8: A^T bit planes, R planes x 2 slots.
  constexpr bool IW = packed_index<F, K, FUSED>();
  constexpr int NI = Traits<F>::NI;
  constexpr int NIP = NI == 3 ? 4 : NI;
  constexpr int RPW = 4 / NIP;
  constexpr bool PAIR = paired_index<F, K, RT, FUSED>();  // two rows per record word (see there)
  constexpr int BPU = PAIR ? 1 : RPW;      // (IW) k-blocks per staged unit of index words
  constexpr int ASZ = PAIR ? ROWS / 2 : ROWS;  // u32 per staged unit and plane
  constexpr int NSLOT = index_slots<F, K, RT, FUSED, SCHED>();  // A words in use + blocks in flight
  // two one-block slots (schedule 6, GF(4)): block s's records go up at the builders' iteration
  // s (its slot held block s-2, whose lookups EMPTY(s) has seen end) and are waited for just
  // before FULL(s)
  constexpr bool JIT_A = TM && IW && NSLOT == 2;
  constexpr int NAP = IW ? 1 : R;          // staged A planes per slot
  constexpr int TPE_RAW = NT / E;
  constexpr int TPE = TPE_RAW < 1 ? 1 : (TPE_RAW > COPIES ? COPIES : TPE_RAW);  // threads per entry
  constexpr int CPT = COPIES / TPE;        // replicas written per thread

  uint4* tab = reinterpret_cast<uint4*>(smem);                     // [NTAB][TR][E][COPIES] uint4
  u32* thalf = reinterpret_cast<u32*>(smem + NTAB * TR * TPLANE);  // [bufs][2 half][R][16][4]
  u32* bst = thalf + half_bufs(SCHED) * 2 * HALF;                  // [3 slot][K][R][4]
  u32* ast = bst + 3 * K * R * 4;                                  // [NSLOT][NAP][ASZ]
  uint64_t* mbar_b = reinterpret_cast<uint64_t*>(ast + NSLOT * NAP * ASZ);  // [3] B-slot barriers
  uint64_t* mbar_a = mbar_b + 3;                                               // [3] A-slot barriers
  // STRM only: this segment's tile's group order, staged by the builder warps ([ngroups] u16)
  // warp-specialized schedules: FULL(s) = mbar_full[s & 1], every builder thread arrives, each
  // lookup warp waits on its own (no barrier among the lookup warps: they may drift apart by up
  // to the double-buffered table's one block)
  uint64_t* mbar_full = mbar_a + 3;                                            // [2]
  unsigned short* perm_s = reinterpret_cast<unsigned short*>(mbar_a + 5);

  const int tid = threadIdx.x;
  if (s_begin >= s_end) return;
  // TMA staging of B is compiled into the warp-specialized schedule only (measured: no gain for
  // the others); there it is used when the host found B aligned for it (a.tma_b).
  constexpr bool TMA_OK = WS && K == 8 && !FUSED;
  const bool tma_b = TMA_OK && a.tma_b;
  const bool tma_a = tma_b && a.tma_a;

  int next_word = IW ? s_begin / BPU : (s_begin * K) >> 5;
  // Streamed products (a.perm, k = 8 only): virtual k-block s of this tile is real block
  // real_block(s); the 4-block groups are permuted, blocks inside a group keep their order, so
  // an index record word (RPW blocks) maps to one real record word.  Staging slots, barrier
  // phases and the F5 offset count virtual blocks.
  // (compiled into the STRM instantiations only: the resident-B kernels are unchanged)
  static_assert(!STRM || (WS && K == 8), "streamed B needs the warp-specialized TMA schedule");
  auto real_block = [&](int s) -> int {
    if constexpr (!STRM) return s;
    return (int)perm_s[s >> 2] * 4 + (s & 3);
  };
  // STRM: groups [0, ready_groups) are known to have landed (the upload stream publishes the
  // chunks in order), so only a block past them reads a flag
  int ready_groups = 0;
  auto real_word = [&](int w) -> int {
    if constexpr (!STRM || !IW) return w;
    return real_block(w * BPU) / BPU;
  };
  // Stage block s's B rows (K x R x 16 B) into bst[s % 3].
  auto issue_b = [&](int s, int t0 = -1, int nthr = NT) {
    if (t0 < 0) t0 = tid;
    if (TMA_OK && tma_b) {
      // TMA: one thread sends the block's [R planes][K rows][4 words] box of B as ONE tensor
      // copy (rows past l arrive zero-filled) completing on mbar_b[s % 3]
      if constexpr (K == 8) {
        if (s < s_end && t0 == 0) {
          const int rs = real_block(s);
          if constexpr (STRM) {
            if ((rs >> 2) >= ready_groups) {  // chunk c = groups [chunk_lo(c), chunk_lo(c + 1))
              const int c = wait_chunk(a.ready, chunk_of(rs >> 2, a.first_groups, a.cap_log), a.nchunks, a.epoch,
                                       a.err, a.poll_ns);
              ready_groups = (int)chunk_lo(c + 1, a.first_groups, a.cap_log);
            }
          }
          mbar_expect_tx(&mbar_b[s % 3], (unsigned)(K * R * 16));
          tma_load_3d(bst + (s % 3) * K * R * 4, tmB, word0, rs * K, 0, &mbar_b[s % 3]);
        }
      }
      return;
    }
    if (s < s_end) {
      u32* bdst = bst + (s % 3) * K * R * 4;
      for (int q = t0; q < K * R * 2; q += nthr) {
        const int i = q / (R * 2), d = (q >> 1) % R, half = q & 1;
        const int64_t row = (int64_t)real_block(s) * K + i;
        const int w = word0 + 2 * half;
        const bool ok = row < a.l && w < a.wc32;
        const u32* src = ok ? a.B + ((int64_t)d * a.l + row) * a.wc32 + w : a.B;
        cp_async8(bdst + (i * R + d) * 4 + 2 * half, src, ok ? 8 : 0);
      }
    }
  };
  // Stage the index words block s needs that are not yet staged.
  auto issue_a = [&](int s, int t0 = -1, int nthr = NT) {
    if (t0 < 0) t0 = tid;
    if constexpr (TMA_OK) {
      if (tma_a) {
        // TMA: the CTA's ROWS index records of each new word as ONE 1-D bulk copy
        if (s < s_end) {
          for (const int whi = s / BPU; next_word <= whi; ++next_word) {
            if (t0 == 0) {
              const int sl = next_word % NSLOT;
              mbar_expect_tx(&mbar_a[sl], ASZ * 4);
              tma_load_1d(ast + sl * ASZ, a.AT + (int64_t)real_word(next_word) * (PAIR ? a.mpad / 2 : a.mpad) +
                                             (PAIR ? row0 / 2 : row0),
                          ASZ * 4, &mbar_a[sl]);
            }
          }
        }
        return;
      }
    }
    if (s < s_end) {
      const int whi = IW ? s / BPU : (s * K + K - 1) >> 5;
      for (; next_word <= whi; ++next_word) {
        u32* adst = ast + (next_word % NSLOT) * NAP * ASZ;
        const bool ok = next_word < (PAIR ? a.nblocks : a.wa32);
        const int rw = real_word(next_word);
        if constexpr (FUSED) {
          // A's own plane words, one per (plane, row): [slot][plane][row] like A^T
          for (int q = t0; q < NAP * ROWS; q += nthr) {
            const int d = q / ROWS, r = q % ROWS;
            const bool ok2 = ok && row0 + r < a.m;
            const u32* src = ok2 ? a.A + ((int64_t)d * a.m + row0 + r) * a.wa32 + rw : a.A;
            cp_async4(adst + d * ROWS + r, src, ok2 ? 4 : 0);
          }
          continue;
        }
        if constexpr (PAIR) {
          for (int q = t0; q < ASZ / 4; q += nthr) {
            const u32* src = ok ? a.AT + (int64_t)rw * (a.mpad / 2) + row0 / 2 + 4 * q : a.AT;
            cp_async16(adst + 4 * q, src, ok ? 16 : 0);
          }
          continue;
        }
        for (int q = t0; q < NAP * ROWS / 4; q += nthr) {
          const int d = q / (ROWS / 4), r4 = q % (ROWS / 4);
          const u32* src = ok ? a.AT + ((int64_t)d * a.wa32 + rw) * a.mpad + row0 + 4 * r4 : a.AT;
          cp_async16(adst + d * ROWS + 4 * r4, src, ok ? 16 : 0);
        }
      }
    }
  };

  // staged B piece (row i of the block, plane d): TMA boxes land plane-major [d][i], cp.async
  // writes row-major [i][d] (consecutive threads -> consecutive 8-byte halves, no bank conflicts)
  auto bpos = [&](int i, int d) { return (TMA_OK && tma_b) ? d * K + i : i * R + d; };
  // TMA path: block s's B rows have landed (slot s % 3 is used once per 3 blocks of the segment)
  auto wait_b = [&](int s) {
    if (TMA_OK && tma_b) mbar_wait(&mbar_b[s % 3], (unsigned)(((s - s_begin) / 3) & 1));
  };
  // ... and block s's index word (slot w % NSLOT, used once per NSLOT words of the segment)
  auto wait_a = [&](int s) {
    if (TMA_OK && tma_a) {
      const int w = s / BPU, w0 = s_begin / BPU;
      mbar_wait(&mbar_a[w % NSLOT], (unsigned)(((w - w0) / NSLOT) & 1));
    }
  };

  // phase 1: the two 16-entry half tables of block s (rows 0..KLO-1 and KLO..K-1)
  auto phase1 = [&](int s) {
    const u32* bs = bst + (s % 3) * K * R * 4;
    u32* th = thalf + (s & 1) * 2 * HALF;
    if (tid < 128) {
      wait_b(s);
      const int h = tid >> 6, e = (tid >> 2) & 15, w = tid & 3;
      const int nrows = h ? KHI : KLO;
      if (e < (1 << nrows)) {
        V<F> acc = vzero<F>();
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (i < nrows && ((e >> i) & 1)) {
            V<F> b;
#pragma unroll
            for (int d = 0; d < R; ++d) b.p[d] = bs[bpos(h * KLO + i, d) * 4 + w];
            vadd<F>(acc, b);
          }
        }
#pragma unroll
        for (int d = 0; d < R; ++d) th[((h * R + d) * 16 + e) * 4 + w] = acc.p[d];
      }
    }
  };

  // phase 2a: this thread's table entry g = Thi[g >> KLO] + Tlo[g & (2^KLO - 1)] (4 words x R)
  const int g_own = tid / TPE, part = tid % TPE;
  auto phase2_compute = [&](int s, V<F> (&v)[4]) {
    const u32* th = thalf + (s & 1) * 2 * HALF;
    if (g_own < E) {
      // half tables are [half][plane][16 entries][4 words]: plane d of entry e at (half R + d) 16 + e
      const uint4* lo = reinterpret_cast<const uint4*>(th) + (g_own & ((1 << KLO) - 1));
      const uint4* hi = reinterpret_cast<const uint4*>(th + HALF) + (g_own >> KLO);
      V<F> hv[4];
#pragma unroll
      for (int d = 0; d < R; ++d) {
        const uint4 L = lo[d * 16], H = hi[d * 16];
        v[0].p[d] = L.x; v[1].p[d] = L.y; v[2].p[d] = L.z; v[3].p[d] = L.w;
        hv[0].p[d] = H.x; hv[1].p[d] = H.y; hv[2].p[d] = H.z; hv[3].p[d] = H.w;
      }
      if constexpr (KHI > 0) {
#pragma unroll
        for (int w = 0; w < 4; ++w) vadd<F>(v[w], hv[w]);
      }
    }
  };
  // phase 2b: write replica number cc (of this thread's CPT) of entry g_own into table buffer tb.
  // The replica order is rotated by g so the 8 lanes of a store phase hit 8 different banks.
  auto phase2_store = [&](uint4* tb, const V<F> (&v)[4], int cc) {
    if (!(ABL & 1) && g_own < E) {
      const int copy = (part * CPT + cc + g_own) & (COPIES - 1);
#pragma unroll
      for (int d = 0; d < R; ++d)
        tb[d * TPL + g_own * (ENTRY_BYTES / 16) + copy] = make_uint4(v[0].p[d], v[1].p[d], v[2].p[d], v[3].p[d]);
      if constexpr (KAR)
        tb[2 * TPL + g_own * (ENTRY_BYTES / 16) + copy] = make_uint4(v[0].p[0] ^ v[0].p[1], v[1].p[0] ^ v[1].p[1],
                                                                     v[2].p[0] ^ v[2].p[1], v[3].p[0] ^ v[3].p[1]);
    }
  };

  Acc<F> c[RT];
  // F5: every k-block adds x + 2y + 4z + 2 (mod 5) (see f5_acc); start from -2 * blocks mod 5.
  u32 init[5] = {0u, 0u, 0u, 0u, 0u};
  if constexpr (F == F5) {
    const int v = (5 - (2 * (s_end - s_begin)) % 5) % 5;
    init[0] = (v & 1) ? ~0u : 0u;
    init[1] = (v & 2) ? ~0u : 0u;
    init[2] = (v & 4) ? ~0u : 0u;
  }
#pragma unroll
  for (int t = 0; t < RT; ++t)
#pragma unroll
    for (int w = 0; w < 4; ++w)
#pragma unroll
      for (int d = 0; d < Traits<F>::RS; ++d) c[t].w[w][d] = init[d];

  const unsigned char* tl0 = reinterpret_cast<const unsigned char*>(tab + (tid & (COPIES - 1)));

  // TM: tensor-memory home of row-slot t of accumulator set `region` for this lane: warp w uses
  // lane quarter w & 3 and columns (w >> 2) 256 + region 128 + t 8 (8 words = one slot of a
  // 2-plane field); tm_cur = the set currently in registers
  int tm_cur = 0;
  constexpr int SW = 4 * Traits<F>::RS;  // accumulator words (TMEM columns) per row-slot
  // Two sets of RT slots (registers + one TMEM region each way) when two warps' two regions fit
  // the 512 columns; otherwise (F5: 20-word slots) the rotation: row-slots in 4 groups of RT / 2,
  // two groups in registers, two parked in 3 TMEM regions of RT / 2 slots (one free).
#ifndef SG_X_MBAR_FULL
#define SG_X_MBAR_FULL 1
#endif
#ifndef SG_X_ROT_ALL
#define SG_X_ROT_ALL 0
#endif
  constexpr bool TM_ROT = TM && (4 * RT * SW > 512 || SG_X_ROT_ALL);
  constexpr int TG = TM_ROT ? RT / 2 : RT;  // slots per TMEM region
  auto tm_addr = [&](int region, int t) -> uint32_t {
    const uint32_t base = *reinterpret_cast<const uint32_t*>(mbar_a + 5);
    const int w = tid >> 5;
    return base + ((uint32_t)(32 * (w & 3)) << 16) +
           (uint32_t)(((w >> 2) * (TM_ROT ? 3 : 2) + region) * TG * SW + t * SW);
  };
  static_assert(!TM || 2 * (TM_ROT ? 3 : 2) * TG * SW <= 512, "schedule 6: two warps' regions per lane quarter");
  static_assert(!TM_ROT || RT % 2 == 0, "schedule 6 rotation: two register groups");
  // TM_ROT state after k blocks: register groups A (c[0, TG)) and B (c[TG, RT)) hold logical
  // groups gA, gB = 2 (k & 1) + 0, 1; groups gZ, gW = the other two are parked in TMEM regions
  // rZ = -k mod 3, rW = rZ + 1 mod 3; region rF = rZ + 2 mod 3 is free (warp-uniform, from k)
  struct Rot {
    int gA, gB, gZ, gW, rZ, rW, rF;
  };
  auto rot = [](int k) {
    const int par = k & 1, rz = (3 - k % 3) % 3;
    return Rot{2 * par, 2 * par + 1, 2 - 2 * par, 3 - 2 * par, rz, (rz + 1) % 3, (rz + 2) % 3};
  };
  auto acc8 = [](Acc<F>& x) -> u32(&)[SW] { return *reinterpret_cast<u32(*)[SW]>(&x.w[0][0]); };

  // Byte offsets of row-slot t's table entries for block s.  PAIR: row-slots 2j and 2j+1 share
  // one record word -- it is loaded for the even slot and kept in xw (the callers go through the
  // slots in order, each slot right after the one before it).
  u32 xw = 0u;
  auto entries = [&](int s, int t, u32 (&e)[3]) {
    const int lr = t * NT + tid;
    e[0] = e[1] = e[2] = 0u;
    if constexpr (PAIR) {
      if ((t & 1) == 0) xw = ast[(s % NSLOT) * ASZ + (t >> 1) * NT + tid];
      const int b0 = (t & 1) * NIP;
#pragma unroll
      for (int i = 0; i < NI; ++i) e[i] = __byte_perm(xw, 0u, 0x4440u | (u32)(b0 + i)) * ENTRY_BYTES;
    } else if constexpr (IW) {
      const u32 x = ast[((s / RPW) % NSLOT) * ROWS + lr];
      const int b0 = (s % RPW) * NIP;
#pragma unroll
      for (int i = 0; i < NI; ++i) e[i] = __byte_perm(x, 0u, 0x4440u | (u32)(b0 + i)) * ENTRY_BYTES;
    } else {
      const int col0 = s * K;
      const int w0 = col0 >> 5, sh = col0 & 31;
      const u32* aw0 = ast + (w0 & 1) * R * ROWS;
      const u32* aw1 = ast + ((w0 + 1) & 1) * R * ROWS;
      if constexpr (FUSED && K == 8) {
        // A's plane words: byte s & 3 of each (F3: the "+1" index is A0 ^ A1, fields.py:98)
        u32 x[R];
#pragma unroll
        for (int d = 0; d < R; ++d) x[d] = aw0[d * ROWS + lr];
        if constexpr (F == F3) x[0] ^= x[1];
#pragma unroll
        for (int d = 0; d < R; ++d) e[d] = ((x[d] >> sh) & 255u) * ENTRY_BYTES;
        return;
      }
#pragma unroll
      for (int d = 0; d < R; ++d) {
        u32 x = aw0[d * ROWS + lr];
        if constexpr (32 % K == 0) {
          x = (x >> sh) & (E - 1);
        } else {
          x = ((sh + K > 32) ? __funnelshift_r(x, aw1[d * ROWS + lr], sh) : (x >> sh)) & (E - 1);
        }
        e[d] = x * ENTRY_BYTES;
      }
    }
  };

  // lookups for block s from table buffer tb, software-pipelined LA row-slots ahead (entries
  // and table rows of t+1..t+LA in flight while t accumulates); `between(t)` runs after t.
  constexpr int LA = (RT >= 4 && Traits<F>::R * Traits<F>::NI <= 4 && !(TM_ROT && F == F5)) ? 2 : 1;
  // (general form: registers c[CB .. CB + N) hold row-slots so .. so + N; TM: `set` selects the
  // accumulator set in registers -- row-slots set * RT + t)
  // `pre` runs after the first LA row-slots' table rows are on their way, before any accumulate
  auto lookups_part = [&](int s, int tb, auto&& between, int so, auto cb_ic, auto n_ic, auto&& pre) {
    constexpr int CB = decltype(cb_ic)::value, N = decltype(n_ic)::value;
    if constexpr (ABL & 4) {
#pragma unroll
      for (int t = 0; t < N; ++t) between(t);
      return;
    }
    const unsigned char* tl = tl0 + tb * TR * TPLANE;
    Rows<F> ring[LA + 1];
#pragma unroll
    for (int t = 0; t < LA && t < N; ++t) {
      u32 e[3];
      entries(s, so + t, e);
      load_rows<F, TPL, KAR>(ring[t], tl, e);
    }
    pre();
#pragma unroll
    for (int t = 0; t < N; ++t) {
      if (t + LA < N) {
        u32 e[3];
        entries(s, so + t + LA, e);
        load_rows<F, TPL, KAR>(ring[(t + LA) % (LA + 1)], tl, e);
      }
      if constexpr (ABL & 2) {
#pragma unroll
        for (int w = 0; w < 4; ++w)
#pragma unroll
          for (int d = 0; d < Traits<F>::R; ++d) c[CB + t].w[w][d] ^= comp(ring[t % (LA + 1)].v[0][d], w) ^ comp(ring[t % (LA + 1)].v[Traits<F>::NI - 1][d], w);
      } else {
        accumulate<F, KAR>(c[CB + t], ring[t % (LA + 1)]);
      }
      between(t);
    }
  };
  auto nop = [] {};
  auto lookups = [&](int s, int tb, auto&& between, int set = 0) {
    lookups_part(s, tb, between, set * RT, std::integral_constant<int, 0>{}, std::integral_constant<int, RT>{}, nop);
  };

  if constexpr (WS) {
    constexpr int NBT = ws_builders(SCHED);
    constexpr int NB = NT + NBT;  // all threads take part in every FULL / EMPTY barrier
    constexpr bool MBF = SG_X_MBAR_FULL && ws_tma(SCHED);
    auto FULL = [](int s) { return 1 + (s & 1); };
    auto EMPTY = [](int s) { return 3 + (s & 1); };
    if constexpr (ROLE == 1) {
      // ------------------------------------------------ builder warps
      const int bt = tid - NT;
      auto bsync = [] { nbar_sync(5, NBT); };
      if constexpr (STRM) {
        const int* pt = a.perm + ((row0 / ROWS) * a.slabs + word0 / SLAB_WORDS) * a.ngroups;
        for (int g = bt; g < a.ngroups; g += NBT) perm_s[g] = (unsigned short)__ldg(pt + g);
        bsync();
      }
      issue_b(s_begin, bt, NBT);
      pdl_wait();  // A's index words come from the pre-pass (B's first rows are already on the way)
      issue_a(s_begin, bt, NBT);
      cp_async_commit();
      issue_b(s_begin + 1, bt, NBT);
      cp_async_commit();
      for (int s = s_begin; s < s_end; ++s) {
        if (s >= s_begin + 2) nbar_sync(EMPTY(s), NB);  // lookups of block s-2 left tab[s & 1]
        issue_b(s + 2, bt, NBT);
        issue_a(JIT_A ? s : s + 1, bt, NBT);
        cp_async_commit();
        cp_async_wait<1>();  // B rows of s and A words of s have landed (this thread's copies)
        wait_b(s);           // TMA path: the block's B rows ...
        if constexpr (!JIT_A) wait_a(s);  // ... and index word (published to the lookup warps by FULL)
        bsync();
        // phase 1: 2 halves x 16 entries x 4 words = 128 items
        {
          const u32* bs = bst + (s % 3) * K * R * 4;
          for (int item = bt; item < 128; item += NBT) {
            const int h = item >> 6, e = (item >> 2) & 15, w = item & 3;
            const int nrows = h ? KHI : KLO;
            if (e < (1 << nrows)) {
              V<F> acc = vzero<F>();
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                if (i < nrows && ((e >> i) & 1)) {
                  V<F> b;
#pragma unroll
                  for (int d = 0; d < R; ++d) b.p[d] = bs[bpos(h * KLO + i, d) * 4 + w];
                  vadd<F>(acc, b);
                }
              }
              if constexpr (F == F5) vcanon<F>(acc);  // canonical halves for the lazy phase-2 add
#pragma unroll
              for (int d = 0; d < R; ++d) thalf[((h * R + d) * 16 + e) * 4 + w] = acc.p[d];
            }
          }
        }
        bsync();
        // phase 2: 256 entries x 8 replicas.  A thread's entries g = bt + NBT it share the low
        // half-table entry (NBT is a multiple of 16): it is read once.
        uint4* tb = tab + (s & 1) * TR * TPL;
        static_assert(NBT % 16 == 0, "phase 2 shares the low half entry across a thread's entries");
        const u32* th2 = thalf;
        uint4 Lh[R];
#pragma unroll
        for (int d = 0; d < R; ++d) Lh[d] = reinterpret_cast<const uint4*>(th2)[(bt & ((1 << KLO) - 1)) + d * 16];
#pragma unroll
        for (int it = 0; it < E / NBT; ++it) {
          const int g = bt + NBT * it;
          const uint4* hi = reinterpret_cast<const uint4*>(th2 + HALF) + (g >> KLO);
          V<F> v[4], hv[4];
#pragma unroll
          for (int d = 0; d < R; ++d) {
            const uint4 L = Lh[d], H = hi[d * 16];
            v[0].p[d] = L.x; v[1].p[d] = L.y; v[2].p[d] = L.z; v[3].p[d] = L.w;
            hv[0].p[d] = H.x; hv[1].p[d] = H.y; hv[2].p[d] = H.z; hv[3].p[d] = H.w;
          }
#pragma unroll
          for (int w = 0; w < 4; ++w) {
            if constexpr (F == F5)  // canonical halves: a redundant 3-bit sum is enough
              f5_add_lazy(v[w].p[0], v[w].p[1], v[w].p[2], hv[w].p[0], hv[w].p[1], hv[w].p[2]);
            else
              vadd<F>(v[w], hv[w]);
          }
          if constexpr (!(ABL & 1)) {
#pragma unroll
            for (int cc = 0; cc < COPIES; ++cc) {
              const int copy = (cc + g) & (COPIES - 1);
#pragma unroll
              for (int d = 0; d < R; ++d)
                tb[d * TPL + g * (ENTRY_BYTES / 16) + copy] = make_uint4(v[0].p[d], v[1].p[d], v[2].p[d], v[3].p[d]);
              if constexpr (KAR)
                tb[2 * TPL + g * (ENTRY_BYTES / 16) + copy] =
                    make_uint4(v[0].p[0] ^ v[0].p[1], v[1].p[0] ^ v[1].p[1], v[2].p[0] ^ v[2].p[1], v[3].p[0] ^ v[3].p[1]);
            }
          }
        }
        if constexpr (JIT_A) {  // block s's records, staged at this iteration
          if (tma_a) wait_a(s);
          else cp_async_wait<0>();
        }
        // table of block s (and A words of s) ready
        if constexpr (MBF) mbar_arrive(&mbar_full[s & 1]);
        else nbar_arrive(FULL(s), NB);
      }
      cp_async_wait<0>();
      return;
    }
    // ------------------------------------------------ lookup warps (ROLE 2)
    using IC0 = std::integral_constant<int, 0>;
    using ICG = std::integral_constant<int, TG>;
    if constexpr (TM_ROT) {
#pragma unroll
      for (int t = 0; t < TG; ++t) {
        tmem_st(tm_addr(0, t), acc8(c[t]));
        tmem_st(tm_addr(1, t), acc8(c[t]));
      }
      tmem_wait_st();
    } else if constexpr (TM) {
      // set 1 starts from the initial values (set 0, in registers, holds them too)
#pragma unroll
      for (int t = 0; t < RT; ++t) tmem_st(tm_addr(1, t), acc8(c[t]));
      tmem_wait_st();
    }
    for (int s = s_begin; s < s_end; ++s) {
      if constexpr (MBF) mbar_wait(&mbar_full[s & 1], (unsigned)((s - s_begin) >> 1) & 1u);
      else nbar_sync(FULL(s), NB);
      if constexpr (TM_ROT) {
        const Rot r = rot(s - s_begin);
        const int gA = r.gA, gB = r.gB, gZ = r.gZ, gW = r.gW, rZ = r.rZ, rW = r.rW, rF = r.rF;
        // group A: park each slot in the free region, load Z's slot in its place; group B: park
        // in Z's (now read) region, load W's; then Z and W from registers.  Z's region's loads
        // were waited for before B's stores reuse it.
        // The waits sit one row-slot late so that the last load's latency hides behind work that
        // does not touch the loaded registers: Z's loads are waited for after B's first slot
        // has accumulated (before its store reuses Z's region), W's after Z's lookups.
        lookups_part(s, s & 1, [&](int t) {
          if (t == 0) tmem_wait_st();  // this block's loads read what the last block's stores wrote
          tmem_st(tm_addr(rF, t), acc8(c[t]));
          tmem_ld(tm_addr(rZ, t), acc8(c[t]));
        }, gA * TG, IC0{}, ICG{}, nop);
        lookups_part(s, s & 1, [&](int t) {
          if (t == 0) tmem_wait_ld();
          tmem_st(tm_addr(rZ, t), acc8(c[TG + t]));
          tmem_ld(tm_addr(rW, t), acc8(c[TG + t]));
        }, gB * TG, ICG{}, ICG{}, nop);
        lookups_part(s, s & 1, [](int) {}, gZ * TG, IC0{}, ICG{}, nop);
        lookups_part(s, s & 1, [](int) {}, gW * TG, ICG{}, ICG{}, [] { tmem_wait_ld(); });
        // (now A, B hold gZ, gW; gA sits in rF, gB in rZ; rW is free: rot(k + 1))
      } else if constexpr (TM) {
        // the set in registers; after each of its row-slots: park it in its TMEM region and
        // start loading the same slot of the other set (those loads land behind the remaining
        // slots' lookups), then the other set's lookups from the same table
        lookups(s, s & 1, [&](int t) {
          tmem_st(tm_addr(tm_cur, t), acc8(c[t]));
          tmem_ld(tm_addr(tm_cur ^ 1, t), acc8(c[t]));
        }, tm_cur);
        tm_cur ^= 1;
        // (the wait sits behind the other set's first table-row loads)
        lookups_part(s, s & 1, [](int) {}, tm_cur * RT, std::integral_constant<int, 0>{},
                     std::integral_constant<int, RT>{}, [] { tmem_wait_ld(); });
      } else {
        lookups(s, s & 1, [](int) {});
      }
      if (s + 2 < s_end) nbar_arrive(EMPTY(s), NB);
    }
  } else if constexpr (!PIPE) {
    for (int i = 0; i < PD; ++i) issue_b(s_begin + i);
    pdl_wait();  // A's index words come from the pre-pass
    for (int i = 0; i < PD; ++i) {
      issue_a(s_begin + i);
      cp_async_commit();
    }
    cp_async_wait<PD - 1>();
    __syncthreads();
    SG_TL(1);
    for (int s = s_begin; s < s_end; ++s) {
      phase1(s);
      __syncthreads();
      issue_b(s + PD);
      issue_a(s + PDA);
      cp_async_commit();
      {
        V<F> v[4];
        phase2_compute(s, v);
#pragma unroll
        for (int cc = 0; cc < CPT; ++cc) phase2_store(tab, v, cc);
      }
      cp_async_wait<PD - 1>();
      __syncthreads();
      lookups(s, 0, [](int) {});
    }
  } else {
    for (int i = 0; i < PD; ++i) issue_b(s_begin + i);
    pdl_wait();  // A's index words come from the pre-pass
    for (int i = 0; i < PDA; ++i) issue_a(s_begin + i);
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    phase1(s_begin);
    __syncthreads();
    {
      V<F> v[4];
      phase2_compute(s_begin, v);
#pragma unroll
      for (int cc = 0; cc < CPT; ++cc) phase2_store(tab + (s_begin & 1) * TR * TPL, v, cc);
    }
    if (s_begin + 1 < s_end) phase1(s_begin + 1);
    __syncthreads();
    SG_TL(1);
    for (int s = s_begin; s < s_end; ++s) {
      issue_b(s + PD);
      issue_a(s + PDA);
      cp_async_commit();
      const bool nxt = s + 1 < s_end;
      V<F> v[4];
      if (nxt) phase2_compute(s + 1, v);
      uint4* tnext = tab + ((s + 1) & 1) * TR * TPL;
      // spread the next table's replica stores over the row-slot loop
      lookups(s, s & 1, [&](int t) {
        if (nxt) {
          // replica cc goes out after row-slot floor(cc * RT / CPT): all CPT, spread evenly
#pragma unroll
          for (int cc = 0; cc < CPT; ++cc)
            if ((cc * RT) / CPT == t) phase2_store(tnext, v, cc);
        }
      });
      if (s + 2 < s_end) phase1(s + 2);
      cp_async_wait<0>();
      __syncthreads();
    }
  }

  // ---- epilogue (row-slots set * RT + t from the registers; TM: both sets, the parked one
  // loaded back from tensor memory)
  SG_TL(2);
  // registers c[CB .. CB + N) hold row-slots so .. so + N
  auto write_part = [&](int so, auto cb_ic, auto n_ic) {
    constexpr int CB = decltype(cb_ic)::value, N = decltype(n_ic)::value;
    if (mode == 2) {  // stream-K: compact slot [R][ROWS][4 words], canonical (summed by the reduce)
      u32* out = a.P2 + (int64_t)slot * R * ROWS * 4;
#pragma unroll
      for (int t = 0; t < N; ++t) {
        const int lr = (so + t) * NT + tid;
        u32 o[4][R];
#pragma unroll
        for (int w = 0; w < 4; ++w) finish<F>(c[CB + t].w[w], o[w], true);
#pragma unroll
        for (int d = 0; d < R; ++d)
          *reinterpret_cast<uint4*>(out + ((int64_t)d * ROWS + lr) * 4) = make_uint4(o[0][d], o[1][d], o[2][d], o[3][d]);
      }
      return;
    }
    u32* out = a.C;
    int64_t rows_out = a.m;
    if (mode == 1) {
      out += (int64_t)slot * R * a.mpad * a.wc32;
      rows_out = a.mpad;
    }
#pragma unroll
    for (int t = 0; t < N; ++t) {
      const int64_t row = row0 + (so + t) * NT + tid;
      if (row < a.m) {
        u32 o[4][R];
#pragma unroll
        for (int w = 0; w < 4; ++w) finish<F>(c[CB + t].w[w], o[w], mode == 0);
#pragma unroll
        for (int d = 0; d < R; ++d) {
          u32* dst = out + ((int64_t)d * rows_out + row) * a.wc32 + word0;
          if (word0 < a.wc32) *reinterpret_cast<uint2*>(dst) = make_uint2(o[0][d], o[1][d]);
          if (word0 + 2 < a.wc32) *reinterpret_cast<uint2*>(dst + 2) = make_uint2(o[2][d], o[3][d]);
        }
      }
    }
  };
  auto write_set = [&](int set) {
    write_part(set * RT, std::integral_constant<int, 0>{}, std::integral_constant<int, RT>{});
  };
  if constexpr (TM_ROT) {
    // (only the lookup warps get here in a WS kernel; the rotation state is theirs)
    using IC0 = std::integral_constant<int, 0>;
    using ICG = std::integral_constant<int, TG>;
    const Rot r = rot(s_end - s_begin);
    const int gA = r.gA, gB = r.gB, gZ = r.gZ, gW = r.gW, rZ = r.rZ, rW = r.rW;
    write_part(gA * TG, IC0{}, ICG{});
    write_part(gB * TG, ICG{}, ICG{});
    tmem_wait_st();  // the last block's stores
#pragma unroll
    for (int t = 0; t < TG; ++t) {
      tmem_ld(tm_addr(rZ, t), acc8(c[t]));
      tmem_ld(tm_addr(rW, t), acc8(c[TG + t]));
    }
    tmem_wait_ld();
    write_part(gZ * TG, IC0{}, ICG{});
    write_part(gW * TG, ICG{}, ICG{});
  } else if constexpr (TM) {
    write_set(tm_cur);
#pragma unroll
    for (int t = 0; t < RT; ++t) tmem_ld(tm_addr(tm_cur ^ 1, t), acc8(c[t]));
    tmem_wait_ld();
    write_set(tm_cur ^ 1);
  } else {
    write_set(0);
  }
}

// All of this CTA's segments.  Stream-K: CTA c owns work units [c U / G, (c+1) U / G) of
// U = (tiles - dp_tiles) x k-blocks (after its whole tiles c, c + G, ... < dp_tiles): a partial tail of one tile, whole tiles, a partial head of another; the
// partial segments land in compact slots and reduce_streamk sums the slots of every tile.  Otherwise one segment
// per CTA: (slab, row group, k-split) = blockIdx.
template <int F, int K, int RT, int SCHED, int NT, int ABL, int ROLE, bool STRM, typename AT>
__device__ __forceinline__ void run_segments(const AT& a, const CUtensorMap* tmB, unsigned char* smem,
                                             uint64_t* mbar) {
  constexpr int ROWS = rows_of(RT, NT, SCHED);
  constexpr bool FUSED = std::is_same_v<AT, M4rmFusedArgs>;
  constexpr bool TMA_OK = ws_tma(SCHED) && K == 8;
  if (!a.streamk) {
    const int s_begin = blockIdx.z * a.bps;
    m4rm_segment<F, K, RT, SCHED, NT, ABL, ROLE, STRM>(a, tmB, smem, blockIdx.x * SLAB_WORDS, (int64_t)blockIdx.y * ROWS,
                                                 s_begin, min(a.nblocks, s_begin + a.bps),
                                                 // fused split-K: compact canonical slots [split][tile] (mode 2)
                                                 a.partial ? (FUSED ? 2 : 1) : 0,
                                                 FUSED ? (int)((blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x)
                                                       : (int)blockIdx.z);
    return;
  }
  // shared memory and the barriers are reused by the next segment
  auto next_segment = [&] {
    cp_async_wait<0>();
    __syncthreads();
    if constexpr (ws_tma(SCHED)) {  // fresh barriers: the next segment counts its phases from zero
      if (threadIdx.x == 0) {
        if (TMA_OK && a.tma_b) {
          for (int i = 0; i < 6; ++i) {
            mbar_inval(&mbar[i]);
            mbar_init(&mbar[i], 1);
          }
        }
        for (int i = 6; i < 8; ++i) {
          mbar_inval(&mbar[i]);
          mbar_init(&mbar[i], ws_builders(SCHED));
        }
        fence_mbar_init();
      }
      __syncthreads();
    }
  };
  const int64_t U = a.units, G = gridDim.x;
  // Hybrid: with at least one tile per CTA, tiles [0, dp_tiles) (a multiple of G) go whole, CTA c
  // taking c, c + G, ...: every CTA then walks the k-blocks of neighbouring tiles at the same
  // time, so B's rows and A's index words of a k-block are fetched once into L2 for the whole
  // wave (pure stream-K scatters the CTAs over all of k: F3 32768^3 read 72 GB from HBM per
  // launch against 2 GB).  Only the last, partial wave -- tiles [dp_tiles, tiles) -- is cut
  // into unit ranges.
  // (one call site for both kinds of segment: the segment code is inlined once)
  const int64_t u0 = blockIdx.x * U / G;
  const int64_t u1 = (blockIdx.x + 1) * U / G;
  int64_t dpt = blockIdx.x, u = u0;
  for (;;) {
    int64_t tile;
    int s0, s1, mode, slot;
    if (dpt < a.dp_tiles) {  // a whole tile of the leading waves
      tile = dpt;
      dpt += G;
      s0 = 0, s1 = a.nblocks, mode = 0, slot = 0;
    } else if (u < u1) {
      const int64_t tl = u / a.nblocks;  // among the stream-K tiles
      tile = a.dp_tiles + tl;
      s0 = (int)(u - tl * a.nblocks);
      const int64_t room = u1 - u;
      s1 = (int)(s0 + room < a.nblocks ? s0 + room : (int64_t)a.nblocks);
      // a whole tile goes straight to C; a partial one (only the range's first or last segment
      // can be partial) to compact slot 2c (first) or 2c + 1 (last), summed by reduce_streamk_kernel
      mode = s0 == 0 && s1 == a.nblocks ? 0 : 2;
      slot = (int)(blockIdx.x * SK_SLOTS + (u == u0 ? 0 : 1));
      u += s1 - s0;
    } else {
      break;
    }
    m4rm_segment<F, K, RT, SCHED, NT, ABL, ROLE, STRM>(a, tmB, smem, (int)(tile % a.slabs) * SLAB_WORDS,
                                                 (tile / a.slabs) * ROWS, s0, s1, mode, slot);
    next_segment();
  }
}

// Fused small products: the split-K reduction inside the product kernel.  Every CTA of the tile
// (blockIdx.x, blockIdx.y) has written its partial plane blockIdx.z; they meet at the tile's
// arrival counter (all co-resident: cooperative launch), then CTA z sums rows
// [z ROWS / S, (z+1) ROWS / S) of the tile over the S partials (L2 loads), canonicalizes them
// into Cout, and the last CTA to leave resets the tile's counters for the next launch.
template <int F, int ROWS>
__device__ __forceinline__ void fused_reduce(const M4rmFusedArgs& a) {
  constexpr int R = Traits<F>::R;
  const unsigned S = gridDim.z;
  const int ntiles = gridDim.x * gridDim.y;
  const int tile = blockIdx.y * gridDim.x + blockIdx.x;
  unsigned* arrive = a.cnt + tile;
  unsigned* depart = a.cnt + a.ntiles + tile;
  __threadfence();  // this thread's partial stores, before the CTA's arrival
  __syncthreads();
  SG_TL(3);
  if (threadIdx.x == 0) {
    atomicAdd(arrive, 1u);
    unsigned v;
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(arrive) : "memory");
      if (v >= S) break;
      __nanosleep(32);
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 4000000000ull) __trap();  // 4 s: a split never arrived (cannot happen co-resident)
    }
  }
  __syncthreads();
  SG_TL(4);
  // slots [split][tile][plane][ROWS][4 words]: thread = (row, word) of rows [r_lo, r_hi)
  const int64_t row0 = (int64_t)blockIdx.y * ROWS;
  const int word0 = blockIdx.x * SLAB_WORDS;
  const int r_lo = (int)(blockIdx.z * ROWS / S), r_hi = (int)((blockIdx.z + 1) * ROWS / S);
  const int64_t sstride = (int64_t)ntiles * R * ROWS * 4;  // one split's slots
  const u32* base = a.P2 + (int64_t)tile * R * ROWS * 4;
  for (int it = threadIdx.x; it < (r_hi - r_lo) * SLAB_WORDS; it += blockDim.x) {
    const int lr = r_lo + it / SLAB_WORDS, w = it % SLAB_WORDS;
    const int64_t row = row0 + lr;
    const u32* p = base + lr * 4 + w;
    V<F> acc = vzero<F>();
    // eight splits' loads in flight before their adds (L2 latency, not bandwidth, bound)
    for (unsigned s0 = 0; s0 < S; s0 += 8) {
      V<F> x[8];
#pragma unroll
      for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int d = 0; d < R; ++d) x[j].p[d] = s0 + j < S ? __ldcg(p + (s0 + j) * sstride + d * ROWS * 4) : 0u;
#pragma unroll
      for (int j = 0; j < 8; ++j) vadd<F>(acc, x[j]);  // zero is the additive identity of every encoding
    }
    vcanon<F>(acc);
    if (row < a.m && word0 + w < a.wc32) {
#pragma unroll
      for (int d = 0; d < R; ++d) a.Cout[((int64_t)d * a.m + row) * a.wc32 + word0 + w] = acc.p[d];
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && atomicAdd(depart, 1u) == S - 1) {  // every split has read its rows
    *arrive = 0u;
    *depart = 0u;
  }
  SG_TL(5);
}

// fused small-product kernels with few accumulator registers run two CTAs per SM (more warps to
// hide the per-k-block latency of a short split)
template <int F, int RT, bool FUSED> __host__ __device__ constexpr int min_ctas_per_sm() {
  return FUSED && RT * Traits<F>::RS * 4 <= 32 ? 2 : 1;
}

template <int F, int K, int RT, int SCHED, int NT, int ABL = 0, bool STRM = false, bool FUSED = false>
__global__ void __launch_bounds__(NT + ws_builders(SCHED), (min_ctas_per_sm<F, RT, FUSED>()))
    m4rm_kernel(const std::conditional_t<STRM, M4rmStreamArgs, std::conditional_t<FUSED, M4rmFusedArgs, M4rmArgs>> a,
                const __grid_constant__ CUtensorMap tmB) {
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int ROWS = rows_of(RT, NT, SCHED);
  SG_TL(0);
  if (a.early_trigger) pdl_trigger();
  // launched with PDL behind the index pre-pass: each schedule waits for it (pdl_wait) just
  // before its first read of A's index words, so the B staging overlaps the pre-pass's tail
  constexpr int R = Traits<F>::R;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + (SCHED >= 1 ? 2 : 1) * table_planes<F, K>() * (1 << K) * ENTRY_BYTES +
                                               (half_bufs(SCHED) * 2 * 16 * R * 4 + 3 * K * R * 4 +
                                                index_stage_words<F, K, RT, NT, FUSED, SCHED>()) * 4);
  constexpr bool TMA_OK = ws_tma(SCHED) && K == 8;
  if constexpr (ws_tma(SCHED)) {
    if (threadIdx.x == 0) {
      if (TMA_OK && a.tma_b)
        for (int i = 0; i < 6; ++i) mbar_init(&mbar[i], 1);  // 3 B slots, 3 A slots
      for (int i = 6; i < 8; ++i) mbar_init(&mbar[i], ws_builders(SCHED));  // FULL of the two table buffers
      fence_mbar_init();
    }
    __syncthreads();
  }
  if constexpr (ws_tma(SCHED)) {
    // warp-specialized: the builder warpgroup hands registers to the two lookup warpgroups,
    // whose row accumulators need them (384 x 168 = 128 x BREGS + 256 x LREGS; SCHED 5:
    // 512 x 128 = 256 x 64 + 256 x 192)
    // (F5: 72 / 216 measured ~1 % faster than 56 / 224 -- its builders' carry-save table adds
    // need the registers, its lookups fit in 216; F7 and GF(4) lost 1-2 % with the same split.
    // The streamed-B variant's builders also check chunk flags: at least 64 for them.)
    constexpr int NBT = ws_builders(SCHED), PER = 65536 / (NT + NBT) / 8 * 8;
#ifndef SG_X_F5_BREGS6
#define SG_X_F5_BREGS6 64
#endif
    constexpr int BREGS = SCHED == 5 ? 64 : F == F5 ? (SCHED == 6 ? SG_X_F5_BREGS6 : 72) : STRM ? 64 : 56;
    constexpr int LREGS = (PER * (NT + NBT) - BREGS * NBT) / NT / 8 * 8;
    // schedule 6: warp 0 allocates all 512 TMEM columns (one CTA per SM) for the lookup warps'
    // second accumulator sets; its address goes to the word after the mbarriers
    uint32_t* tslot = reinterpret_cast<uint32_t*>(mbar + 8);
    if constexpr (SCHED == 6) {
      if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncthreads();
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    if (threadIdx.x >= NT) {
      asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(BREGS));
      run_segments<F, K, RT, SCHED, NT, ABL, 1, STRM>(a, &tmB, smem, mbar);
    } else {
      asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(LREGS));
      run_segments<F, K, RT, SCHED, NT, ABL, 2, STRM>(a, &tmB, smem, mbar);
    }
    if constexpr (SCHED == 6) {
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncthreads();
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (threadIdx.x < 32)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(*tslot));
    }
  } else {
    run_segments<F, K, RT, SCHED, NT, ABL, 0, STRM>(a, &tmB, smem, mbar);
    if constexpr (FUSED) {
      if (a.partial) fused_reduce<F, ROWS>(a);
    }
  }
}

// ------------------------------------------------------------------ registry helpers
template <int F, int K, int RT, int SCHED, int NT, bool FUSED = false>
constexpr int smem_bytes_for() {
  constexpr int R = Traits<F>::R;
  return (SCHED >= 1 ? 2 : 1) * table_planes<F, K>() * (1 << K) * ENTRY_BYTES + half_bufs(SCHED) * 2 * 16 * R * 4 * 4 +
         3 * K * R * 4 * 4 +
         index_stage_words<F, K, RT, NT, FUSED, SCHED>() * 4 + 8 * 8 +  // + the B- / A-slot and FULL mbarriers
         (SCHED == 6 ? 16 : 0);                                         // + the TMEM address (schedule 6)
}

// the streamed-B instantiation of a warp-specialized k = 8 variant (nullptr for the others)
template <int F, int K, int RT, int P, int NT>
constexpr StreamKernelFn stream_variant() {
  if constexpr (ws_tma(P) && K == 8) return m4rm_kernel<F, K, RT, P, NT, 0, true>;
  else return nullptr;
}

#define SG_K(F, K, RT, P, NT) {m4rm_kernel<F, K, RT, P, NT>, F, K, RT, NT, (NT) + ws_builders(P), P, \
                               smem_bytes_for<F, K, RT, P, NT>(), 0, 0, 0, stream_variant<F, K, RT, P, NT>(), \
                               smem_bytes_for<F, K, RT, P, NT>() + 2 * STRM_MAX_GROUPS, nullptr, \
                               paired_index<F, K, RT>() ? (NT) : 0}
#define SG_KA(F, K, RT, P, NT, A) {m4rm_kernel<F, K, RT, P, NT, A>, F, K, RT, NT, (NT) + ws_builders(P), P, \
                                   smem_bytes_for<F, K, RT, P, NT>(), 0, 0, A, nullptr, 0, nullptr, \
                                   paired_index<F, K, RT>() ? (NT) : 0}
// schedule 6 (second accumulator set in TMEM): KernelInfo.rt counts both sets' row-slots
#define SG_KTM(F, RT) {m4rm_kernel<F, 8, RT, 6, 256>, F, 8, 2 * (RT), 256, 256 + ws_builders(6), 6, \
                       smem_bytes_for<F, 8, RT, 6, 256>(), 0, 0, 0, nullptr, 0, nullptr, \
                       paired_index<F, 8, RT>() ? 256 : 0}
// fused small-product variants (k = 8, serial / pipelined; see M4rmFusedArgs)
#define SG_KF(F, RT, P) {nullptr, F, 8, RT, 256, 256, P, smem_bytes_for<F, 8, RT, P, 256, true>(), 0, 0, 0, nullptr, 0, \
                         m4rm_kernel<F, 8, RT, P, 256, 0, false, true>, 0}
#define SG_KFUSED(F) SG_KF(F, 1, 0), SG_KF(F, 2, 0), SG_KF(F, 4, 0), SG_KF(F, 2, 1), SG_KF(F, 4, 1)
// k = 8: 256-thread CTAs (RT 1..8, both schedules) and 512-thread CTAs (16 warps per SM)
#define SG_KSET8(F)                                                                                 \
  SG_K(F, 8, 1, 0, 256), SG_K(F, 8, 2, 0, 256), SG_K(F, 8, 4, 0, 256), SG_K(F, 8, 8, 0, 256), \
  SG_K(F, 8, 1, 1, 256), SG_K(F, 8, 2, 1, 256), SG_K(F, 8, 4, 1, 256),                      \
  SG_K(F, 8, 2, 0, 512), SG_K(F, 8, 4, 0, 512), SG_K(F, 8, 2, 1, 512)
#define SG_KSET8_2PLANE(F)                                                                          \
  SG_K(F, 8, 16, 0, 256), SG_K(F, 8, 8, 1, 256), SG_K(F, 8, 16, 1, 256),                  \
  SG_K(F, 8, 8, 0, 512), SG_K(F, 8, 4, 1, 512), SG_K(F, 8, 8, 1, 512)
// k < 8: parity and generality (k-invariance), one variant each + a pipelined k=5
#define SG_KLOW(F)                                                                                  \
  SG_K(F, 1, 1, 0, 256), SG_K(F, 2, 1, 0, 256), SG_K(F, 3, 1, 0, 256), SG_K(F, 4, 1, 0, 256), \
  SG_K(F, 5, 1, 0, 256), SG_K(F, 6, 1, 0, 256), SG_K(F, 7, 1, 0, 256), SG_K(F, 5, 1, 1, 256)

}  // namespace sg
