// sg_pack.cu -- HBM-bound kernels around the M4RM product:
//   pack / unpack        dense uint8 residues <-> bit planes   (BitslicedMatrix.from_dense /
//                        to_dense; layout implied by _core_py.py:186-192)
//   canonicalize         f5_reduce / f7_reduce over whole planes (_core_py.py:143-148, 171-175)
//   plane ops            the reference backend's in-place plane kernels on device arrays
//                        (_core_py.py:24-175; argument order dst planes then src planes)
//   block driver / table the plugin-granularity mirror of m4rm_block_<f> (_core_py.py:205-281)
//                        and build_table for callers of the _core API.
// Layout everywhere: planes [R][rows][W64] uint64, column c -> word c>>6, bit c&63;
// viewed as 32-bit words, column c -> word c>>5, bit c&31 (little endian).
#include <algorithm>

#include "sg_field.cuh"
#include "sg_internal.h"

namespace sg {

__host__ __device__ inline int planes_of(int field) {
  return field == F2 ? 1 : (field == F5 || field == F7 || field == GF8 || field == Z8) ? 3 : 2;
}
__host__ __device__ inline int order_of(int field) {
  switch (field) {
    case F2: return 2;
    case F3: return 3;
    case F5: return 5;
    case F7: return 7;
    case GF4: case Z4: return 4;
    default: return 8;  // GF8, Z8
  }
}

// 4 bytes of a word -> bit d of each byte gathered into a nibble (byte i -> bit i)
__device__ __forceinline__ u32 gather_bit(u32 x, int d) {
  return ((((x >> d) & 0x01010101u) * 0x01020408u) >> 24) & 0xFu;
}
// nibble -> one 0/1 byte per bit (bit i -> byte i)
__device__ __forceinline__ u32 spread_nibble(u32 nib) { return (nib * 0x00204081u) & 0x01010101u; }

// Pack / unpack: thread (blockIdx.x * 256 + threadIdx.x) owns 32-bit plane word w of every
// row blockIdx.y, blockIdx.y + gridDim.y, ... (2-D grid: no 64-bit index division), two rows per
// iteration with both rows' loads issued first.  Field-templated (constant plane count).
// 256-bit streaming global accesses (sm_100: ld / st .v8.b32): a lane's 32 dense bytes in one
// request, so a warp's load covers 1024 contiguous bytes with every 32-byte sector asked for once
// (two LDG.128 per lane ask for each sector twice).  The address must be 32-byte aligned.
__device__ __forceinline__ void ldcs256(const void* p, u32 (&x)[8]) {
  asm volatile("ld.global.cs.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(x[0]), "=r"(x[1]), "=r"(x[2]), "=r"(x[3]), "=r"(x[4]), "=r"(x[5]), "=r"(x[6]), "=r"(x[7])
               : "l"(p));
}
__device__ __forceinline__ void stcs256(void* p, const u32 (&x)[8]) {
  asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(x[0]), "r"(x[1]), "r"(x[2]),
               "r"(x[3]), "r"(x[4]), "r"(x[5]), "r"(x[6]), "r"(x[7])
               : "memory");
}

template <int F>
__device__ __forceinline__ void pack_word(const uint8_t* __restrict__ src, bool full, int64_t c0, int64_t n,
                                          u32 (&p)[3], bool& bad) {
  constexpr int R = F == F2 ? 1 : (F == F5 || F == F7 || F == GF8 || F == Z8) ? 3 : 2;
  constexpr u32 order = F == F2 ? 2 : F == F3 ? 3 : F == F5 ? 5 : F == F7 ? 7 : (F == GF4 || F == Z4) ? 4 : 8;
  u32 x[8];
  // a full word's 32 bytes by the widest accesses the row's alignment allows (rows of a ragged
  // matrix start at any byte), a partial last word byte by byte
  const uintptr_t al = reinterpret_cast<uintptr_t>(src);
  if (full && (al & 31) == 0) {
    ldcs256(src, x);
  } else if (full && (al & 15) == 0) {
    const uint4 a = __ldcs(reinterpret_cast<const uint4*>(src)), b = __ldcs(reinterpret_cast<const uint4*>(src) + 1);
    x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w; x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
  } else if (full && (al & 7) == 0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint2 a = __ldcs(reinterpret_cast<const uint2*>(src) + q);
      x[2 * q] = a.x; x[2 * q + 1] = a.y;
    }
  } else if (full && (al & 3) == 0) {
#pragma unroll
    for (int q = 0; q < 8; ++q) x[q] = __ldcs(reinterpret_cast<const u32*>(src) + q);
  } else if (full) {
    // an odd row start: the seven aligned words inside the 32 bytes, the 4 - a head and a tail
    // bytes one by one (nothing outside this thread's columns is read), funnel-shifted into place
    const int a = (int)(al & 3);  // 1..3
    const u32* base = reinterpret_cast<const u32*>(al - a);
    u32 y[9];
    y[0] = 0u;
    for (int c = 0; c < 4 - a; ++c) y[0] |= (u32)src[c] << (8 * (a + c));
#pragma unroll
    for (int j = 1; j < 8; ++j) y[j] = __ldcs(base + j);
    y[8] = 0u;
    for (int c = 0; c < a; ++c) y[8] |= (u32)src[32 - a + c] << (8 * c);
#pragma unroll
    for (int q = 0; q < 8; ++q) x[q] = __funnelshift_r(y[q], y[q + 1], 8 * a);
  } else {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      u32 v = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int64_t c = c0 + 4 * q + b;
        if (c < n) v |= (u32)src[4 * q + b] << (8 * b);
      }
      x[q] = v;
    }
  }
  // Gather bit b of the 32 bytes into raw plane I[b]: (x & 0x01010101 << b) * 0x01020408 puts byte
  // i's bit at 24 + b + i (the 16 partial products fall on distinct positions, the rest below
  // 20 + b or past bit 31), one shift moves the nibble to 4q.  The range check and F3's value ->
  // pattern map work on whole plane words afterwards (32 columns per instruction).
  constexpr int NB = F == F2 ? 1 : (F == F3 || F == GF4 || F == Z4) ? 2 : 3;  // input bits per residue
  u32 I[3] = {0u, 0u, 0u};
  u32 any = 0u;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    any |= x[q];
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const u32 t = (x[q] & (0x01010101u << b)) * 0x01020408u;
      const int sh = 24 + b - 4 * q;
      I[b] |= (sh >= 0 ? t >> sh : t << -sh) & (0xFu << (4 * q));
    }
  }
  bad |= (any & ~(((1u << NB) - 1u) * 0x01010101u)) != 0u;  // a byte >= 2^NB
  if constexpr (F == F3) {
    bad |= (I[0] & I[1]) != 0u;  // the residue 3
    p[0] = I[0] | I[1];          // 1 -> 01, 2 -> 11 (fields.py:88-101)
    p[1] = I[1];
    p[2] = 0u;
  } else {
    if constexpr (order == 5) bad |= (I[2] & (I[1] | I[0])) != 0u;  // 5, 6, 7
    if constexpr (order == 7) bad |= (I[0] & I[1] & I[2]) != 0u;    // 7
    p[0] = I[0]; p[1] = I[1]; p[2] = I[2];
  }
}

// Bad input: OR `bit` into the caller's status word (mapped page-locked host memory, read by
// sg_stream_check).  Every writer of one kernel sets the same bit and the kernels of one stream
// run in order, so a plain read-or-write suffices (no system-scope atomics over PCIe).
__device__ __forceinline__ void flag_error(int* err, int bit) {
  volatile int* v = err;
  *v = *v | bit;
  __threadfence_system();
}

template <int F>
__global__ void __launch_bounds__(256) pack_kernel(const uint8_t* __restrict__ dense, int64_t m, int64_t n,
                                                   int64_t ld, u32* __restrict__ planes, int wc32, int* err) {
  constexpr int R = F == F2 ? 1 : (F == F5 || F == F7 || F == GF8 || F == Z8) ? 3 : 2;
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= wc32) return;
  const int64_t c0 = (int64_t)w * 32;
  bool bad = false;
  const int64_t step = gridDim.y;
  for (int64_t row = blockIdx.y; row < m; row += 2 * step) {
    const int64_t row2 = row + step;
    const uint8_t* s1 = dense + row * ld + c0;
    const uint8_t* s2 = dense + row2 * ld + c0;
    const bool full = c0 + 32 <= n;
    u32 p1[3], p2[3];
    pack_word<F>(s1, full, c0, n, p1, bad);
    if (row2 < m) pack_word<F>(s2, full, c0, n, p2, bad);
#pragma unroll
    for (int d = 0; d < R; ++d) {
      __stcs(planes + ((int64_t)d * m + row) * wc32 + w, p1[d]);
      if (row2 < m) __stcs(planes + ((int64_t)d * m + row2) * wc32 + w, p2[d]);
    }
  }
  if (bad) flag_error(err, 1);
}

template <int F>
__device__ __forceinline__ void unpack_word(const u32 (&pin)[3], u32 (&x)[8], bool& bad) {
  // canonical patterns first, on whole plane words (32 columns per instruction): F5's 5, 6, 7 and
  // F7's 7 are redundant encodings of 0, 1, 2 and 0 (_core_py.py:143-148, 171-175)
  u32 p[3] = {pin[0], pin[1], pin[2]};
  if constexpr (F == F5) f5_reduce(p[0], p[1], p[2]);
  if constexpr (F == F7) f7_reduce(p[0], p[1], p[2]);
  if constexpr (F == F3) bad |= (p[1] & ~p[0]) != 0u;  // sign without unit: illegal (fields.py:88-101)
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const u32 b0 = spread_nibble((p[0] >> (4 * q)) & 0xFu);
    const u32 b1 = spread_nibble((p[1] >> (4 * q)) & 0xFu);
    const u32 b2 = spread_nibble((p[2] >> (4 * q)) & 0xFu);
    if constexpr (F == F3) x[q] = b0 + b1;
    else x[q] = b0 | (b1 << 1) | (b2 << 2);
  }
}

template <int F>
__global__ void __launch_bounds__(256) unpack_kernel(const u32* __restrict__ planes, int64_t m, int64_t n,
                                                     uint8_t* __restrict__ dense, int64_t ld, int wc32, int* err) {
  constexpr int R = F == F2 ? 1 : (F == F5 || F == F7 || F == GF8 || F == Z8) ? 3 : 2;
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t c0 = (int64_t)w * 32;
  if (w >= wc32 || c0 >= n) return;
  bool bad = false;
  const int64_t step = gridDim.y;
  for (int64_t row = blockIdx.y; row < m; row += 2 * step) {
    const int64_t row2 = row + step;
    u32 p1[3] = {0u, 0u, 0u}, p2[3] = {0u, 0u, 0u};
#pragma unroll
    for (int d = 0; d < R; ++d) {
      p1[d] = __ldcs(planes + ((int64_t)d * m + row) * wc32 + w);
      if (row2 < m) p2[d] = __ldcs(planes + ((int64_t)d * m + row2) * wc32 + w);
    }
    for (int h = 0; h < 2; ++h) {
      const int64_t r = h ? row2 : row;
      if (r >= m) break;
      u32 x[8];
      unpack_word<F>(h ? p2 : p1, x, bad);
      uint8_t* dst = dense + r * ld + c0;
      if (c0 + 32 <= n && ((reinterpret_cast<uintptr_t>(dst) & 31) == 0)) {
        stcs256(dst, x);
      } else if (c0 + 32 <= n && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
        __stcs(reinterpret_cast<uint4*>(dst), make_uint4(x[0], x[1], x[2], x[3]));
        __stcs(reinterpret_cast<uint4*>(dst) + 1, make_uint4(x[4], x[5], x[6], x[7]));
      } else if (c0 + 32 <= n && ((reinterpret_cast<uintptr_t>(dst) & 7) == 0)) {
#pragma unroll
        for (int q = 0; q < 4; ++q) __stcs(reinterpret_cast<uint2*>(dst) + q, make_uint2(x[2 * q], x[2 * q + 1]));
      } else if (c0 + 32 <= n && ((reinterpret_cast<uintptr_t>(dst) & 3) == 0)) {
#pragma unroll
        for (int q = 0; q < 8; ++q) __stcs(reinterpret_cast<u32*>(dst) + q, x[q]);
      } else if (c0 + 32 <= n) {
        // an odd row start: a head bytes up to the next 4-byte boundary, seven aligned words
        // assembled by funnel shifts, then the 4 - a tail bytes
        const int a = (int)((4 - (reinterpret_cast<uintptr_t>(dst) & 3)) & 3);  // 1..3 here
        for (int c = 0; c < a; ++c) dst[c] = (uint8_t)(x[0] >> (8 * c));
#pragma unroll
        for (int j = 0; j < 7; ++j)
          __stcs(reinterpret_cast<u32*>(dst + a) + j, __funnelshift_r(x[j], x[j + 1], 8 * a));
        for (int c = a + 28; c < 32; ++c) dst[c] = (uint8_t)(x[7] >> (8 * (c & 3)));
      } else {
        for (int c = 0; c < 32 && c0 + c < n; ++c) dst[c] = (uint8_t)(x[c >> 2] >> (8 * (c & 3)));
      }
    }
  }
  if (bad) flag_error(err, 2);
}

__global__ void canonicalize_kernel(int field, uint64_t* __restrict__ p, int64_t n_words) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_words;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t a = p[i], b = p[n_words + i], c = p[2 * n_words + i];
    u32 lo[3] = {(u32)a, (u32)b, (u32)c}, hi[3] = {(u32)(a >> 32), (u32)(b >> 32), (u32)(c >> 32)};
    if (field == F5) { f5_reduce(lo[0], lo[1], lo[2]); f5_reduce(hi[0], hi[1], hi[2]); }
    else { f7_reduce(lo[0], lo[1], lo[2]); f7_reduce(hi[0], hi[1], hi[2]); }
    p[i] = lo[0] | ((uint64_t)hi[0] << 32);
    p[n_words + i] = lo[1] | ((uint64_t)hi[1] << 32);
    p[2 * n_words + i] = lo[2] | ((uint64_t)hi[2] << 32);
  }
}

// ------------------------------------------------------------------ plane ops (plugin kernels)
// op codes mirror include/slicegemm_b200.h SG_OP_*
enum {
  OP_F2_ADD = 0, OP_F3_ADD, OP_F3_SUB, OP_F3_NEG, OP_F5_ADD, OP_F5_SUB, OP_F5_NEG, OP_F5_DOUBLE,
  OP_F5_REDUCE, OP_F7_ADD, OP_F7_SUB, OP_F7_NEG, OP_F7_DOUBLE, OP_F7_REDUCE, OP_GF4_ADD,
  OP_GF4_MULX, OP_F5_FOLD5, OP_SCALAR_MUL_F3, OP_SCALAR_MUL_F5, OP_SCALAR_MUL_F7,
  OP_SCALAR_MUL_GF4, OP_Z4_ADD, OP_Z4_SUB, OP_Z4_NEG, OP_Z8_ADD, OP_Z8_SUB, OP_Z8_NEG, OP_GF8_ADD,
  OP_GF8_MULX, OP_SCALAR_MUL_Z4, OP_SCALAR_MUL_Z8, OP_SCALAR_MUL_GF8, OP_COUNT
};

__device__ __forceinline__ void apply_op(int op, u32* d, const u32* s, u32 tail, int scalar) {
  switch (op) {
    case OP_F2_ADD: d[0] ^= s[0]; break;
    case OP_GF4_ADD: d[0] ^= s[0]; d[1] ^= s[1]; break;
    case OP_GF4_MULX: { u32 t = d[1]; d[1] ^= d[0]; d[0] = t; } break;
    case OP_F3_ADD: f3_add(d[0], d[1], s[0], s[1]); break;
    case OP_F3_SUB: f3_sub(d[0], d[1], s[0], s[1]); break;
    case OP_F3_NEG: d[1] ^= d[0]; break;
    case OP_F5_ADD: f5_add(d[0], d[1], d[2], s[0], s[1], s[2]); break;
    case OP_F5_SUB: { u32 a = s[0], b = s[1], c = s[2]; f5_neg(a, b, c); f5_add(d[0], d[1], d[2], a, b, c); } break;
    case OP_F5_NEG: f5_neg(d[0], d[1], d[2]); break;
    case OP_F5_DOUBLE: f5_double(d[0], d[1], d[2]); break;
    case OP_F5_REDUCE: f5_reduce(d[0], d[1], d[2]); break;
    case OP_F5_FOLD5: { u32 r0, r1, r2; fold5(d[0], d[1], d[2], s[0], r0, r1, r2); d[0] = r0; d[1] = r1; d[2] = r2; } break;
    case OP_F7_ADD: f7_add(d[0], d[1], d[2], s[0], s[1], s[2]); break;
    case OP_F7_SUB: { u32 a = s[0], b = s[1], c = s[2]; f7_neg(a, b, c, tail); f7_add(d[0], d[1], d[2], a, b, c); } break;
    case OP_F7_NEG: f7_neg(d[0], d[1], d[2], tail); break;
    case OP_F7_DOUBLE: f7_double(d[0], d[1], d[2]); break;
    case OP_F7_REDUCE: f7_reduce(d[0], d[1], d[2]); break;
    case OP_SCALAR_MUL_F3: {  // c in {0, 1, 2}: 0 clears, 2 = -1 negates
      if (scalar == 0) { d[0] = 0; d[1] = 0; } else if (scalar == 2) d[1] ^= d[0];
    } break;
    case OP_SCALAR_MUL_F5:
    case OP_SCALAR_MUL_F7: {  // Horner over the bits of c with double and add
      const bool five = op == OP_SCALAR_MUL_F5;
      u32 x0 = d[0], x1 = d[1], x2 = d[2], a0 = 0, a1 = 0, a2 = 0;
      for (int b = 2; b >= 0; --b) {
        if (five) f5_double(a0, a1, a2); else f7_double(a0, a1, a2);
        if ((scalar >> b) & 1) { if (five) f5_add(a0, a1, a2, x0, x1, x2); else f7_add(a0, a1, a2, x0, x1, x2); }
      }
      d[0] = a0; d[1] = a1; d[2] = a2;
    } break;
    case OP_Z4_ADD: z4_add(d[0], d[1], s[0], s[1]); break;
    case OP_Z4_SUB: { u32 a = s[0], b = s[1]; z4_neg(a, b); z4_add(d[0], d[1], a, b); } break;
    case OP_Z4_NEG: z4_neg(d[0], d[1]); break;
    case OP_Z8_ADD: z8_add(d[0], d[1], d[2], s[0], s[1], s[2]); break;
    case OP_Z8_SUB: { u32 a = s[0], b = s[1], c = s[2]; z8_neg(a, b, c); z8_add(d[0], d[1], d[2], a, b, c); } break;
    case OP_Z8_NEG: z8_neg(d[0], d[1], d[2]); break;
    case OP_GF8_ADD: d[0] ^= s[0]; d[1] ^= s[1]; d[2] ^= s[2]; break;
    case OP_GF8_MULX: gf8_mulx(d[0], d[1], d[2]); break;
    case OP_SCALAR_MUL_Z4: {  // Horner over the bits of c
      u32 a0 = 0, a1 = 0;
      for (int b = 1; b >= 0; --b) {
        a1 = a0; a0 = 0;
        if ((scalar >> b) & 1) z4_add(a0, a1, d[0], d[1]);
      }
      d[0] = a0; d[1] = a1;
    } break;
    case OP_SCALAR_MUL_Z8: {
      u32 a0 = 0, a1 = 0, a2 = 0;
      for (int b = 2; b >= 0; --b) {
        a2 = a1; a1 = a0; a0 = 0;
        if ((scalar >> b) & 1) z8_add(a0, a1, a2, d[0], d[1], d[2]);
      }
      d[0] = a0; d[1] = a1; d[2] = a2;
    } break;
    case OP_SCALAR_MUL_GF8: {  // c = c0 + c1 x + c2 x^2
      u32 x0 = d[0], x1 = d[1], x2 = d[2], r0 = 0, r1 = 0, r2 = 0;
      for (int b = 0; b < 3; ++b) {
        if ((scalar >> b) & 1) { r0 ^= x0; r1 ^= x1; r2 ^= x2; }
        gf8_mulx(x0, x1, x2);
      }
      d[0] = r0; d[1] = r1; d[2] = r2;
    } break;
    case OP_SCALAR_MUL_GF4: {  // c = c0 + c1 x
      const u32 x0 = d[0], x1 = d[1];
      u32 r0 = 0, r1 = 0;
      if (scalar & 1) { r0 ^= x0; r1 ^= x1; }
      if (scalar & 2) { r0 ^= x1; r1 ^= x0 ^ x1; }
      d[0] = r0; d[1] = r1;
    } break;
  }
}

__device__ __forceinline__ int op_planes(int op) {
  switch (op) {
    case OP_F2_ADD: return 1;
    case OP_F3_ADD: case OP_F3_SUB: case OP_F3_NEG: case OP_GF4_ADD: case OP_GF4_MULX:
    case OP_SCALAR_MUL_F3: case OP_SCALAR_MUL_GF4: case OP_Z4_ADD: case OP_Z4_SUB: case OP_Z4_NEG:
    case OP_SCALAR_MUL_Z4: return 2;
    default: return 3;
  }
}

// dst/src: R planes (one device pointer each) of rows * w64 words; the tail mask applies to
// the last word of every row (padding lanes, _core_py.py:155-168).
__global__ void plane_op_kernel(int op, Planes dst, Planes src, int64_t rows, int64_t w64, uint64_t tail,
                                int scalar, int has_src) {
  const int R = op_planes(op);
  const int RS = has_src ? (op == OP_F5_FOLD5 ? 1 : R) : 0;  // fold5's 4th input bit is src plane 0
  const int64_t total = rows * w64;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t tm = (i % w64 == w64 - 1) ? tail : ~0ull;
    u32 dl[3] = {0, 0, 0}, dh[3] = {0, 0, 0}, sl[3] = {0, 0, 0}, shh[3] = {0, 0, 0};
    for (int d = 0; d < R; ++d) {
      const uint64_t x = dst.p[d][i];
      dl[d] = (u32)x; dh[d] = (u32)(x >> 32);
    }
    for (int d = 0; d < RS; ++d) {
      const uint64_t y = src.p[d][i];
      sl[d] = (u32)y; shh[d] = (u32)(y >> 32);
    }
    apply_op(op, dl, sl, (u32)tm, scalar);
    apply_op(op, dh, shh, (u32)(tm >> 32), scalar);
    for (int d = 0; d < R; ++d) dst.p[d][i] = dl[d] | ((uint64_t)dh[d] << 32);
  }
}

// ------------------------------------------------------------------ block-level plugin mirror
// C_i += sum_d alpha_d T[phi_d(A_i, col0..col0+kp)] for rows row0..row1 (_core_py.py:205-281).
// One thread per (row, 64-bit word of C); the table uses the reference layout, one plane array
// of 2^kp rows x wc64 words each.
template <int F>
__global__ void block_driver_kernel(Planes C, int64_t wc64, Planes A, int64_t wa64, int64_t col0, int kp,
                                    Planes T, int64_t row0, int64_t row1) {
  constexpr int R = Traits<F>::R;
  const int64_t total = (row1 - row0) * wc64;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = row0 + i / wc64, w = i % wc64;
    u32 g[3] = {0, 0, 0};
    for (int d = 0; d < R; ++d) {
      u32 x = 0;
      for (int t = 0; t < kp; ++t) {
        const int64_t c = col0 + t;
        x |= (u32)((A.p[d][row * wa64 + (c >> 6)] >> (c & 63)) & 1ull) << t;
      }
      g[d] = x;
    }
    if (F == F3) g[0] ^= g[1];  // pos = A0 ^ A1, neg = A1
    // the reference skips a row whose indices are all zero without touching C or T[0]
    // (_core_py.py:208-209, 218-222, 230-231, 247-248); F3 skips its add and its sub separately
    if ((g[0] | g[1] | g[2]) == 0u) continue;
    uint64_t out[3] = {0, 0, 0};
    for (int half = 0; half < 2; ++half) {
      const int sh = 32 * half;
      V<F> c;
      for (int d = 0; d < R; ++d) c.p[d] = (u32)(C.p[d][row * wc64 + w] >> sh);
      auto T_ = [&](int d, u32 gg) { return (u32)(T.p[d][(int64_t)gg * wc64 + w] >> sh); };
      if constexpr (F == F2) {
        c.p[0] ^= T_(0, g[0]);
      } else if constexpr (F == F3) {
        if (g[0]) f3_add(c.p[0], c.p[1], T_(0, g[0]), T_(1, g[0]));
        if (g[1]) f3_sub(c.p[0], c.p[1], T_(0, g[1]), T_(1, g[1]));
      } else if constexpr (F == GF4) {
        const u32 q1 = T_(1, g[1]);
        c.p[0] ^= T_(0, g[0]) ^ q1;
        c.p[1] ^= T_(1, g[0]) ^ T_(0, g[1]) ^ q1;
      } else if constexpr (F == Z4) {  // acc = 2 T[g1] + T[g0]; C += acc  (_core_py.py:225-238)
        u32 a0 = 0u, a1 = T_(0, g[1]);
        if (g[0]) z4_add(a0, a1, T_(0, g[0]), T_(1, g[0]));
        z4_add(c.p[0], c.p[1], a0, a1);
      } else if constexpr (F == GF8) {  // power basis: C += T[g0] + x T[g1] + x^2 T[g2]
        u32 x0 = T_(0, g[2]), x1 = T_(1, g[2]), x2 = T_(2, g[2]);
        gf8_mulx(x0, x1, x2);
        x0 ^= T_(0, g[1]); x1 ^= T_(1, g[1]); x2 ^= T_(2, g[1]);
        gf8_mulx(x0, x1, x2);
        c.p[0] ^= x0 ^ T_(0, g[0]); c.p[1] ^= x1 ^ T_(1, g[0]); c.p[2] ^= x2 ^ T_(2, g[0]);
      } else if constexpr (F == Z8) {  // Horner over {1, 2, 4} with doubling = shift (_core_py.py:262-286)
        u32 x0 = 0u, x1 = T_(0, g[2]), x2 = T_(1, g[2]);
        z8_add(x0, x1, x2, T_(0, g[1]), T_(1, g[1]), T_(2, g[1]));
        x2 = x1; x1 = x0; x0 = 0u;
        z8_add(x0, x1, x2, T_(0, g[0]), T_(1, g[0]), T_(2, g[0]));
        z8_add(c.p[0], c.p[1], c.p[2], x0, x1, x2);
      } else {
        u32 x0 = T_(0, g[2]), x1 = T_(1, g[2]), x2 = T_(2, g[2]);
        if constexpr (F == F5) {
          f5_double(x0, x1, x2); f5_add(x0, x1, x2, T_(0, g[1]), T_(1, g[1]), T_(2, g[1]));
          f5_double(x0, x1, x2); f5_add(x0, x1, x2, T_(0, g[0]), T_(1, g[0]), T_(2, g[0]));
          f5_add(c.p[0], c.p[1], c.p[2], x0, x1, x2);
        } else {
          f7_double(x0, x1, x2); f7_add(x0, x1, x2, T_(0, g[1]), T_(1, g[1]), T_(2, g[1]));
          f7_double(x0, x1, x2); f7_add(x0, x1, x2, T_(0, g[0]), T_(1, g[0]), T_(2, g[0]));
          f7_add(c.p[0], c.p[1], c.p[2], x0, x1, x2);
        }
      }
      for (int d = 0; d < R; ++d) out[d] |= (uint64_t)c.p[d] << sh;
    }
    for (int d = 0; d < R; ++d) C.p[d][row * wc64 + w] = out[d];
  }
}

// T[g] = sum over set bits t of g of B[row_base + t]  (mask-indexed); rows past
// b_rows are zero.  One thread per (entry, 64-bit word).
template <int F>
__global__ void build_table_kernel(Planes B, int64_t b_rows, int64_t row_base, int kp, int64_t wc64, Planes T) {
  constexpr int R = Traits<F>::R;
  const int64_t total = ((int64_t)1 << kp) * wc64;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = i / wc64, w = i % wc64;
    uint64_t out[3] = {0, 0, 0};
    for (int half = 0; half < 2; ++half) {
      const int sh = 32 * half;
      V<F> acc;
      for (int d = 0; d < R; ++d) acc.p[d] = 0;
      for (int t = 0; t < kp; ++t) {
        if (((g >> t) & 1) && row_base + t < b_rows) {
          V<F> b;
          for (int d = 0; d < R; ++d) b.p[d] = (u32)(B.p[d][(row_base + t) * wc64 + w] >> sh);
          vadd<F>(acc, b);
        }
      }
      for (int d = 0; d < R; ++d) out[d] |= (uint64_t)acc.p[d] << sh;
    }
    for (int d = 0; d < R; ++d) T.p[d][g * wc64 + w] = out[d];
  }
}

// ------------------------------------------------------------------ classical product
// C_i = sum_j a_ij B_j row by row (_core_py.py:289-366): no tables, one thread
// per (row, 32-bit word of C), every coefficient expanded over the field's basis.  O(m l n / 32)
// word operations: the independent mid-level cross-check of the M4RM kernel, not a fast path.
template <int F>
__global__ void classical_kernel(Planes A, int64_t wa64, Planes B, int64_t wb64, Planes C, int64_t m, int64_t l) {
  constexpr int R = Traits<F>::R;
  const int64_t wc32 = 2 * wb64;
  const int64_t total = m * wc32;
  const u32* Bp[3];
  for (int d = 0; d < R; ++d) Bp[d] = reinterpret_cast<const u32*>(B.p[d]);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / wc32, w = i % wc32;
    V<F> acc;
    for (int d = 0; d < R; ++d) acc.p[d] = 0u;
    for (int64_t j = 0; j < l; ++j) {
      unsigned pat = 0;
      for (int d = 0; d < R; ++d) pat |= (unsigned)((A.p[d][row * wa64 + (j >> 6)] >> (j & 63)) & 1ull) << d;
      if (!pat) continue;
      V<F> b;
      for (int d = 0; d < R; ++d) b.p[d] = Bp[d][j * wc32 + w];
      if constexpr (F == F3) {  // pattern 01 = 1, 11 = -1
        if (pat == 1) f3_add(acc.p[0], acc.p[1], b.p[0], b.p[1]);
        else f3_sub(acc.p[0], acc.p[1], b.p[0], b.p[1]);
      } else if constexpr (F == GF4 || F == GF8) {  // a = sum_d bit_d x^d
        for (int d = 0; d < R; ++d) {
          if ((pat >> d) & 1)
            for (int e = 0; e < R; ++e) acc.p[e] ^= b.p[e];
          if (F == GF4) { const u32 t = b.p[1]; b.p[1] ^= b.p[0]; b.p[0] = t; }
          else gf8_mulx(b.p[0], b.p[1], b.p[2]);
        }
      } else {  // binary digits with doubling: F2, F5, F7, Z4, Z8
        for (int d = 0; d < R; ++d) {
          if ((pat >> d) & 1) vadd<F>(acc, b);
          if constexpr (F == F5) f5_double(b.p[0], b.p[1], b.p[2]);
          if constexpr (F == F7) f7_double(b.p[0], b.p[1], b.p[2]);
          if constexpr (F == Z4) { b.p[1] = b.p[0]; b.p[0] = 0u; }
          if constexpr (F == Z8) { b.p[2] = b.p[1]; b.p[1] = b.p[0]; b.p[0] = 0u; }
        }
      }
    }
    vcanon<F>(acc);
    for (int d = 0; d < R; ++d) reinterpret_cast<u32*>(C.p[d])[row * wc32 + w] = acc.p[d];
  }
}

// The reference backend's classical drivers, raw and in place (_core_py.py:292-366): for every
// row j of B in order, C_i += a_ij B_j with the reference's per-field expansion -- F2 XOR; F3 sub
// for -1 (sign bit), else add for 1; Z/4 acc = 2 B_j [a1] + B_j [a0]; F5 / F7 / Z/8 Horner over
// the bits of a_ij (acc = B_j [a2]; 2 acc (+ B_j [a1]); 2 acc (+ B_j [a0])).  A row whose
// coefficient is 0 is skipped.  C keeps its raw patterns (no canonical reduction), so the
// output bits equal the pure backend's for any legal input C.  One thread per (row, 32-bit word).
template <int F>
__global__ void classical_block_kernel(Planes C, int64_t wc64, Planes A, int64_t wa64, Planes B, int64_t m,
                                       int64_t l) {
  constexpr int R = Traits<F>::R;
  const int64_t wc32 = 2 * wc64;
  const int64_t total = m * wc32;
  const u32* Bp[3];
  u32* Cp[3];
  for (int d = 0; d < R; ++d) {
    Bp[d] = reinterpret_cast<const u32*>(B.p[d]);
    Cp[d] = reinterpret_cast<u32*>(C.p[d]);
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / wc32, w = i % wc32;
    V<F> c;
    for (int d = 0; d < R; ++d) c.p[d] = Cp[d][row * wc32 + w];
    for (int64_t j = 0; j < l; ++j) {
      unsigned v = 0;
      for (int d = 0; d < R; ++d) v |= (unsigned)((A.p[d][row * wa64 + (j >> 6)] >> (j & 63)) & 1ull) << d;
      if (!v) continue;
      V<F> b;
      for (int d = 0; d < R; ++d) b.p[d] = Bp[d][j * wc32 + w];
      if constexpr (F == F2 || F == GF4 || F == GF8) {
        // (GF4 / GF8 have no reference driver: power basis, C += sum_d bit_d x^d B_j)
        V<F> x = b;
        for (int d = 0; d < R; ++d) {
          if ((v >> d) & 1)
            for (int e = 0; e < R; ++e) c.p[e] ^= x.p[e];
          if constexpr (F == GF4) { const u32 t = x.p[1]; x.p[1] ^= x.p[0]; x.p[0] = t; }
          if constexpr (F == GF8) gf8_mulx(x.p[0], x.p[1], x.p[2]);
        }
      } else if constexpr (F == F3) {
        if (v & 2) f3_sub(c.p[0], c.p[1], b.p[0], b.p[1]);
        else f3_add(c.p[0], c.p[1], b.p[0], b.p[1]);
      } else if constexpr (F == Z4) {
        u32 a0 = 0u, a1 = (v & 2) ? b.p[0] : 0u;
        if (v & 1) z4_add(a0, a1, b.p[0], b.p[1]);
        z4_add(c.p[0], c.p[1], a0, a1);
      } else {  // F5, F7, Z8
        V<F> acc;
        for (int d = 0; d < R; ++d) acc.p[d] = (v & 4) ? b.p[d] : 0u;
        for (int bit = 1; bit >= 0; --bit) {
          if constexpr (F == F5) f5_double(acc.p[0], acc.p[1], acc.p[2]);
          if constexpr (F == F7) f7_double(acc.p[0], acc.p[1], acc.p[2]);
          if constexpr (F == Z8) { acc.p[2] = acc.p[1]; acc.p[1] = acc.p[0]; acc.p[0] = 0u; }
          if ((v >> bit) & 1) vadd<F>(acc, b);
        }
        vadd<F>(c, acc);
      }
    }
    for (int d = 0; d < R; ++d) Cp[d][row * wc32 + w] = c.p[d];
  }
}

static unsigned grid_for(int64_t work, int threads) {
  int64_t b = (work + threads - 1) / threads;
  if (b > 148 * 32) b = 148 * 32;
  return (unsigned)(b < 1 ? 1 : b);
}

// 2-D grid for pack / unpack: x covers the words of a row, y strides over rows (~16 CTAs per SM)
static dim3 grid_2d(int64_t m, int wc32) {
  const unsigned gx = (unsigned)((wc32 + 255) / 256);
  int64_t gy = (148 * 16 + gx - 1) / gx;
  gy = std::min<int64_t>(std::max<int64_t>(gy, 1), std::min<int64_t>(m, 65535));
  return dim3(gx, (unsigned)std::max<int64_t>(gy, 1));
}

cudaError_t launch_pack(int field, const uint8_t* dense, int64_t m, int64_t n, int64_t ld,
                        uint64_t* planes, int* err, cudaStream_t st) {
  const int wc32 = (int)(2 * ((n + 63) / 64));
  if (m == 0 || wc32 == 0) return cudaSuccess;
#define SG_PK(FF) pack_kernel<FF><<<grid_2d(m, wc32), 256, 0, st>>>(dense, m, n, ld, reinterpret_cast<u32*>(planes), \
                                                                   wc32, err)
  SG_FOR_EACH_FIELD_CASE(field, SG_PK)
#undef SG_PK
  return cudaGetLastError();
}

cudaError_t launch_unpack(int field, const uint64_t* planes, int64_t m, int64_t n, uint8_t* dense,
                          int64_t ld, int* err, cudaStream_t st) {
  const int wc32 = (int)(2 * ((n + 63) / 64));
  if (m == 0 || wc32 == 0) return cudaSuccess;
#define SG_UPK(FF) unpack_kernel<FF><<<grid_2d(m, wc32), 256, 0, st>>>(reinterpret_cast<const u32*>(planes), m, n, \
                                                                      dense, ld, wc32, err)
  SG_FOR_EACH_FIELD_CASE(field, SG_UPK)
#undef SG_UPK
  return cudaGetLastError();
}

cudaError_t launch_canonicalize(int field, uint64_t* planes, int64_t rows, int64_t w64, cudaStream_t st) {
  if (field != F5 && field != F7) return cudaSuccess;
  const int64_t nw = rows * w64;
  if (nw == 0) return cudaSuccess;
  canonicalize_kernel<<<grid_for(nw, 256), 256, 0, st>>>(field, planes, nw);
  return cudaGetLastError();
}

cudaError_t launch_plane_op(int op, Planes dst, Planes src, int64_t rows, int64_t w64, uint64_t tail,
                            int scalar, cudaStream_t st) {
  if (op < 0 || op >= OP_COUNT) return cudaErrorInvalidValue;
  const int64_t nw = rows * w64;
  if (nw == 0) return cudaSuccess;
  plane_op_kernel<<<grid_for(nw, 256), 256, 0, st>>>(op, dst, src, rows, w64, tail, scalar, src.p[0] != nullptr);
  return cudaGetLastError();
}

#define SG_FIELD_SWITCH(field, KERNEL, ...)                                   \
  switch (field) {                                                            \
    case F2: KERNEL<F2><<<g, 256, 0, st>>>(__VA_ARGS__); break;               \
    case F3: KERNEL<F3><<<g, 256, 0, st>>>(__VA_ARGS__); break;               \
    case F5: KERNEL<F5><<<g, 256, 0, st>>>(__VA_ARGS__); break;               \
    case F7: KERNEL<F7><<<g, 256, 0, st>>>(__VA_ARGS__); break;               \
    case GF4: KERNEL<GF4><<<g, 256, 0, st>>>(__VA_ARGS__); break;             \
    case GF8: KERNEL<GF8><<<g, 256, 0, st>>>(__VA_ARGS__); break;             \
    case Z4: KERNEL<Z4><<<g, 256, 0, st>>>(__VA_ARGS__); break;               \
    default: KERNEL<Z8><<<g, 256, 0, st>>>(__VA_ARGS__); break;               \
  }

cudaError_t launch_block_driver(int field, Planes C, int64_t wc64, Planes A, int64_t wa64, int64_t col0, int kp,
                                Planes T, int64_t row0, int64_t row1, cudaStream_t st) {
  const int64_t work = (row1 - row0) * wc64;
  if (work <= 0) return cudaSuccess;
  const unsigned g = grid_for(work, 256);
  SG_FIELD_SWITCH(field, block_driver_kernel, C, wc64, A, wa64, col0, kp, T, row0, row1);
  return cudaGetLastError();
}

cudaError_t launch_build_table(int field, Planes B, int64_t b_rows, int64_t row_base, int kp, int64_t wc64,
                               Planes T, cudaStream_t st) {
  const int64_t work = ((int64_t)1 << kp) * wc64;
  if (work <= 0) return cudaSuccess;
  const unsigned g = grid_for(work, 256);
  SG_FIELD_SWITCH(field, build_table_kernel, B, b_rows, row_base, kp, wc64, T);
  return cudaGetLastError();
}

}  // namespace sg

namespace sg {
cudaError_t launch_classical(int field, Planes A, int64_t wa64, Planes B, int64_t wb64, Planes C, int64_t m,
                             int64_t l, cudaStream_t st) {
  const int64_t work = m * 2 * wb64;
  if (work <= 0) return cudaSuccess;
  const unsigned g = grid_for(work, 256);
  SG_FIELD_SWITCH(field, classical_kernel, A, wa64, B, wb64, C, m, l);
  return cudaGetLastError();
}

cudaError_t launch_classical_block(int field, Planes C, int64_t wc64, Planes A, int64_t wa64, Planes B, int64_t m,
                                   int64_t l, cudaStream_t st) {
  const int64_t work = m * 2 * wc64;
  if (work <= 0) return cudaSuccess;
  const unsigned g = grid_for(work, 256);
  SG_FIELD_SWITCH(field, classical_block_kernel, C, wc64, A, wa64, B, m, l);
  return cudaGetLastError();
}
}  // namespace sg
