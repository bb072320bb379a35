// sg_field.cuh -- bitsliced field arithmetic on 32-bit plane words (32 lanes per word).
//
// Every function is lanewise boolean logic; nvcc folds the two-input networks into LOP3.
// The networks compute the same lane functions as the reference kernels:
//   F3  (plane0 = unit, plane1 = sign; 0=00, 1=01, -1=11)   _core_py.py:28-43, kernels.py:151-199
//   F5  (3-bit value, residue = value mod 5; redundant)     _core_py.py:65-75, 91-97, 116-148
//   F7  (3-bit value, residue = value mod 7; 7 == 0)         _core_py.py:65-75, 84-88, 151-175
//   F2  (1 plane, xor)                                        _core_py.py:24-25
//   GF4 (F2[x]/(x^2+x+1), plane0 = coeff of 1, plane1 = coeff of x)   fields.py:215
//   GF8 (F2[x]/(x^3+x+1), planes = coefficients of 1, x, x^2)           fields.py:216
//   Z4 / Z8 (2 / 3-bit binary, unique)                _core_py.py:46-62, 100-113, kernels.py:121-136, 399-415
// Exhaustive lane tables for each formula (kernels.py:466-509, 550-590) are replayed on the
// device through sg_plane_op by tests/test_gpu_parity.py.
#pragma once
#include <cstdint>

namespace sg {

enum Field : int { F2 = 0, F3 = 1, F5 = 2, F7 = 3, GF4 = 4, GF8 = 5, Z4 = 6, Z8 = 7 };

typedef uint32_t u32;

// One LOP3 (any 3-input boolean function; IMM = F(0xF0, 0xCC, 0xAA)).  Not volatile: the
// compiler schedules it freely.
template <int IMM> __device__ __forceinline__ u32 lop3(u32 a, u32 b, u32 c) {
  u32 d;
  asm("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(d) : "r"(a), "r"(b), "r"(c), "n"(IMM));
  return d;
}
constexpr int LOP_XOR3 = 0x96, LOP_MAJ = 0xE8, LOP_AND2 = 0xC0;

template <int F> struct Traits;
// R = bit planes per element; NI = table lookups per (row, k-block) = basis size;
// RS = planes of the M4RM kernel's row accumulator (carry-save: F5 5 planes mod 15, F7 4).
template <> struct Traits<F2>  { static constexpr int R = 1, NI = 1, RS = 1; };
template <> struct Traits<F3>  { static constexpr int R = 2, NI = 2, RS = 2; };
template <> struct Traits<F5>  { static constexpr int R = 3, NI = 3, RS = 5; };
template <> struct Traits<F7>  { static constexpr int R = 3, NI = 3, RS = 4; };
template <> struct Traits<GF4> { static constexpr int R = 2, NI = 2, RS = 2; };
template <> struct Traits<GF8> { static constexpr int R = 3, NI = 3, RS = 3; };
template <> struct Traits<Z4>  { static constexpr int R = 2, NI = 2, RS = 2; };
template <> struct Traits<Z8>  { static constexpr int R = 3, NI = 3, RS = 3; };

// ---------------------------------------------------------------- F3
// x += y and x -= y in three LOP3 each (a minimum found by exhaustive search over LOP3
// networks, tools/lop3/search.c; the reference spends six 2-input ops on each,
// kernels.py:151-168).  Both share w = F(xu, xs, ys).  Valid on the three legal patterns;
// the illegal pattern 10 is a don't-care (SPEC.md design decisions).
__device__ __forceinline__ void f3_add(u32& xu, u32& xs, u32 yu, u32 ys) {
  const u32 w = lop3<0x61>(xu, xs, ys);
  const u32 ru = lop3<0x7c>(xu, yu, w);
  xs = lop3<0x24>(xs, yu, w);
  xu = ru;
}
__device__ __forceinline__ void f3_sub(u32& xu, u32& xs, u32 yu, u32 ys) {
  const u32 w = lop3<0x61>(xu, xs, ys);
  const u32 ru = lop3<0xbc>(xu, yu, w);
  xs = lop3<0x28>(xs, yu, w);
  xu = ru;
}
__device__ __forceinline__ void f3_neg(u32& /*xu*/, u32& xs, u32 xu_in) { xs ^= xu_in; }

// ---------------------------------------------------------------- 3-bit adder + folds
// s = x + y as a 4-bit lane integer (grade-school chain, 12 2-input ops)
__device__ __forceinline__ void add3(u32 x0, u32 x1, u32 x2, u32 y0, u32 y1, u32 y2,
                                     u32& s0, u32& s1, u32& s2, u32& s3) {
  u32 c0 = x0 & y0;
  u32 t1 = x1 ^ y1;
  u32 c1 = (x1 & y1) | (t1 & c0);
  u32 t2 = x2 ^ y2;
  s0 = x0 ^ y0;
  s1 = t1 ^ c0;
  s2 = t2 ^ c1;
  s3 = (x2 & y2) | (t2 & c1);
}
// 8 == 3 (mod 5): fold bit 3 into bits 0..2, residue preserved, result in 0..7
__device__ __forceinline__ void fold5(u32 s0, u32 s1, u32 s2, u32 s3, u32& r0, u32& r1, u32& r2) {
  u32 t = s2 | s1;
  r2 = s0 ^ t;
  r1 = (r2 & s0) ^ (s3 ^ s1);
  r0 = (t ^ s2) | (r1 & s3);
}
__device__ __forceinline__ void f5_add(u32& x0, u32& x1, u32& x2, u32 y0, u32 y1, u32 y2) {
  u32 s0, s1, s2, s3;
  add3(x0, x1, x2, y0, y1, y2, s0, s1, s2, s3);
  fold5(s0, s1, s2, s3, x0, x1, x2);
}
// x + y for canonical F5 lanes (x, y <= 4): a 3-bit representative of the residue (0..7, not
// canonical): the only carry out is x = y = 4, sum 8 == 3 (mod 5) -- OR it into bits 0 and 1.
// 7 LOP3 against f5_add's ~13; the M4RM table entries may be redundant (the lookup networks are
// exact mod 15 for every 3-bit input, tools/lop3/csa_gen.py), their half-table inputs canonical.
__device__ __forceinline__ void f5_add_lazy(u32& x0, u32& x1, u32& x2, u32 y0, u32 y1, u32 y2) {
  const u32 c0 = x0 & y0;
  const u32 c1 = lop3<LOP_MAJ>(x1, y1, c0);
  const u32 s3 = lop3<LOP_MAJ>(x2, y2, c1);
  x2 = lop3<LOP_XOR3>(x2, y2, c1);
  const u32 s1 = lop3<LOP_XOR3>(x1, y1, c0);
  x0 = (x0 ^ y0) | s3;
  x1 = s1 | s3;
}
// x += y mod 7 as a 3-bit one's-complement (end-around-carry) adder: 8 LOP3.  co = [x+y >= 8]
// re-enters at bit 0 (8 == 1 mod 7); x + y + co never carries out again (<= 15 - 8).  Same
// residues as the reference's 17-op adder chain + fold (_core_py.py:65-88), any of 0/7 for zero.
__device__ __forceinline__ void f7_add(u32& x0, u32& x1, u32& x2, u32 y0, u32 y1, u32 y2) {
  const u32 c0 = lop3<LOP_AND2>(x0, y0, 0u);
  const u32 c1 = lop3<LOP_MAJ>(x1, y1, c0);
  const u32 co = lop3<LOP_MAJ>(x2, y2, c1);
  const u32 k1 = lop3<LOP_MAJ>(x0, y0, co);
  const u32 k2 = lop3<LOP_MAJ>(x1, y1, k1);
  x0 = lop3<LOP_XOR3>(x0, y0, co);
  x2 = lop3<LOP_XOR3>(x2, y2, k2);
  x1 = lop3<LOP_XOR3>(x1, y1, k1);
}
// -x mod 5 on 3-bit lanes (4 ops)
__device__ __forceinline__ void f5_neg(u32& p0, u32& p1, u32& p2) {
  u32 r2 = p2 ^ p0;
  u32 r1 = (r2 & p2) ^ p1;
  p0 = r1 & p1;
  p1 = r1;
  p2 = r2;
}
// 2x mod 5 (5 ops): fold5 of the shifted lane with the constant zero propagated
__device__ __forceinline__ void f5_double(u32& p0, u32& p1, u32& p2) {
  u32 t = p1 | p0;
  u32 r1 = p2 ^ p0;
  p0 = (t ^ p1) | (r1 & p2);
  p1 = r1;
  p2 = t;
}
// 2x mod 7: plane rotation, zero ops
__device__ __forceinline__ void f7_double(u32& p0, u32& p1, u32& p2) {
  u32 t = p2; p2 = p1; p1 = p0; p0 = t;
}
// -x mod 7 on 3-bit lanes: complement (7 - v); `tail` re-zeroes padding lanes
__device__ __forceinline__ void f7_neg(u32& p0, u32& p1, u32& p2, u32 tail) {
  p0 = ~p0 & tail; p1 = ~p1 & tail; p2 = ~p2 & tail;
}
// canonical residue 0..4: lanes >= 5 get 3 added and bit 2 cleared
__device__ __forceinline__ void f5_reduce(u32& p0, u32& p1, u32& p2) {
  u32 c = p2 & (p1 | p0);
  u32 w = c & ~p0;
  p0 ^= c;
  p2 ^= c;
  p1 &= ~w;
}
// canonical residue 0..6: the pattern 7 becomes 0
__device__ __forceinline__ void f7_reduce(u32& p0, u32& p1, u32& p2) {
  u32 t = p0 & p1 & p2;
  p0 ^= t; p1 ^= t; p2 ^= t;
}

// ---------------------------------------------------------------- F5 accumulator (mod 15)
// The M4RM kernel accumulates F5 rows as 4-bit lanes modulo 15 (a multiple of 5): doubling is
// a free 4-bit rotation (16 == 1 mod 15) and the add is an 11-LOP3 one's-complement adder,
// against the reference's 5-op double + 20-op add per Horner step (_core_py.py:116-140).
// Table entries stay 3-bit F5 values (any representative mod 5 is a valid mod-15 input).
__device__ __forceinline__ void add15(u32& a0, u32& a1, u32& a2, u32& a3, u32 b0, u32 b1, u32 b2, u32 b3) {
  const u32 c0 = a0 & b0;
  const u32 c1 = lop3<LOP_MAJ>(a1, b1, c0);
  const u32 c2 = lop3<LOP_MAJ>(a2, b2, c1);
  const u32 co = lop3<LOP_MAJ>(a3, b3, c2);
  const u32 k1 = lop3<LOP_MAJ>(a0, b0, co);
  const u32 k2 = lop3<LOP_MAJ>(a1, b1, k1);
  const u32 k3 = lop3<LOP_MAJ>(a2, b2, k2);
  a0 = a0 ^ b0 ^ co;
  a1 = a1 ^ b1 ^ k1;
  a2 = a2 ^ b2 ^ k2;
  a3 = a3 ^ b3 ^ k3;
}
// 4-bit lane value 0..15 -> canonical F5 residue 0..4 in 3 planes (6 LOP3, searched)
__device__ __forceinline__ void mod15_to_f5(u32 v0, u32 v1, u32 v2, u32 v3, u32& r0, u32& r1, u32& r2) {
  const u32 w4 = lop3<0x07>(v0, v1, v2);
  const u32 w5 = lop3<0x18>(v0, v1, v2);
  const u32 w6 = lop3<0x2c>(v1, v3, w5);
  r0 = lop3<0x29>(v2, w4, w6);
  r1 = lop3<0x14>(v1, v3, w5);
  r2 = lop3<0x24>(v0, v2, w6);
}

// ---------------------------------------------------------------- carry-save row accumulators
// C += x + 2y + 4z as ONE multi-operand carry-save addition (full adder = xor3 + majority, a
// carry out of the top column re-enters column 0), generated and verified lane-exactly by
// tools/lop3/csa_gen.py from the adder schedule found by tools/lop3/csa_plan.py.
// F7: 18 LOP3 per (row, k-block, word) against 3 x 8 for three sequential mod-7 adds; the
//     accumulator keeps two bits in column 0: value = q0 + k0 + 2 q1 + 4 q2 (mod 7).
__device__ __forceinline__ void f7_acc(u32& q_0, u32& k_0, u32& q_1, u32& q_2, u32 x0, u32 x1, u32 x2,
                                       u32 y0, u32 y1, u32 y2, u32 z0, u32 z1, u32 z2) {
  const u32 t1 = lop3<0x96>(q_0, k_0, x0);
  const u32 t2 = lop3<0xe8>(q_0, k_0, x0);
  const u32 t3 = lop3<0x96>(y2, z1, t1);
  const u32 t4 = lop3<0xe8>(y2, z1, t1);
  const u32 t5 = lop3<0x96>(q_1, x1, y0);
  const u32 t6 = lop3<0xe8>(q_1, x1, y0);
  const u32 t7 = lop3<0x96>(q_2, x2, y1);
  const u32 t8 = lop3<0xe8>(q_2, x2, y1);
  const u32 t9 = lop3<0x96>(z0, t6, t7);
  const u32 t10 = lop3<0xe8>(z0, t6, t7);
  const u32 t11 = lop3<0x96>(t8, t3, t10);
  const u32 t12 = lop3<0xe8>(t8, t3, t10);
  const u32 t13 = lop3<0x96>(z2, t2, t5);
  const u32 t14 = lop3<0xe8>(z2, t2, t5);
  const u32 t15 = lop3<0x96>(t4, t13, t12);
  const u32 t16 = lop3<0xe8>(t4, t13, t12);
  const u32 t17 = lop3<0x96>(t9, t14, t16);
  const u32 t18 = lop3<0xe8>(t9, t14, t16);
  q_0 = t11; k_0 = t18; q_1 = t15; q_2 = t17;
}
// F5, accumulated mod 15 (5 | 15): 4z is replaced by -z (4 == -1 mod 5) and -z = ~z - 8 in
// 4-bit one's complement, so the complemented z bits are free LOP3 input inversions and each
// k-block adds x + 2y + (7 - z) == x + 2y + 4z + 2 (mod 5); the kernel pre-pays -2 per k-block
// in the accumulator's initial value.  20 LOP3 against 32 for three one's-complement adds.
// value = q0 + 2 q1 + 4 q2 + 4 k2 + 8 q3 (mod 15).
__device__ __forceinline__ void f5_acc(u32& q_0, u32& q_1, u32& q_2, u32& k_2, u32& q_3, u32 x0, u32 x1,
                                       u32 x2, u32 y0, u32 y1, u32 y2, u32 z0, u32 z1, u32 z2) {
  const u32 t1 = lop3<0x69>(q_0, x0, z0);
  const u32 t2 = lop3<0xd4>(q_0, x0, z0);
  const u32 t3 = lop3<0x96>(q_1, x1, y0);
  const u32 t4 = lop3<0xe8>(q_1, x1, y0);
  const u32 t5 = lop3<0x69>(z1, t2, t3);
  const u32 t6 = lop3<0x8e>(z1, t2, t3);
  const u32 t7 = lop3<0x96>(q_2, k_2, x2);
  const u32 t8 = lop3<0xe8>(q_2, k_2, x2);
  const u32 t9 = lop3<0x69>(y1, z2, t4);
  const u32 t10 = lop3<0xb2>(y1, z2, t4);
  const u32 t11 = lop3<0x96>(t7, t6, t9);
  const u32 t12 = lop3<0xe8>(t7, t6, t9);
  const u32 t13 = lop3<0x96>(q_3, y2, t8);
  const u32 t14 = lop3<0xe8>(q_3, y2, t8);
  const u32 t15 = lop3<0x96>(t10, t13, t12);
  const u32 t16 = lop3<0xe8>(t10, t13, t12);
  const u32 t17 = lop3<0x96>(t1, t14, t16);
  const u32 t18 = lop3<0xe8>(t1, t14, t16);
  const u32 t19 = lop3<0x96>(t5, t18, 0u);
  const u32 t20 = lop3<0xe8>(t5, t18, 0u);
  q_0 = t17; q_1 = t19; q_2 = t11; k_2 = t20; q_3 = t15;
}

// 4-word interleaved form of f7_acc: each adder is issued for all four words in turn
__device__ __forceinline__ void f7_acc4(u32 (&q)[4][4], const u32 (&in)[4][9]) {
  u32 t1[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) t1[w] = lop3<0x96>(q[w][0], q[w][1], in[w][0]);
  u32 t2[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) t2[w] = lop3<0xe8>(q[w][0], q[w][1], in[w][0]);
  u32 t3[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) t3[w] = lop3<0x96>(in[w][5], in[w][7], t1[w]);
  u32 t4[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) t4[w] = lop3<0xe8>(in[w][5], in[w][7], t1[w]);
  u32 t5[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) t5[w] = lop3<0x96>(q[w][2], in[w][1], in[w][3]);
  u32 t6[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) t6[w] = lop3<0xe8>(q[w][2], in[w][1], in[w][3]);
  u32 t7[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) t7[w] = lop3<0x96>(q[w][3], in[w][2], in[w][4]);
  u32 t8[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) t8[w] = lop3<0xe8>(q[w][3], in[w][2], in[w][4]);
  u32 t9[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) t9[w] = lop3<0x96>(in[w][6], t6[w], t7[w]);
  u32 t10[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) t10[w] = lop3<0xe8>(in[w][6], t6[w], t7[w]);
  u32 t11[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) t11[w] = lop3<0x96>(t8[w], t3[w], t10[w]);
  u32 t12[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) t12[w] = lop3<0xe8>(t8[w], t3[w], t10[w]);
  u32 t13[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) t13[w] = lop3<0x96>(in[w][8], t2[w], t5[w]);
  u32 t14[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) t14[w] = lop3<0xe8>(in[w][8], t2[w], t5[w]);
  u32 t15[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) t15[w] = lop3<0x96>(t4[w], t13[w], t12[w]);
  u32 t16[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) t16[w] = lop3<0xe8>(t4[w], t13[w], t12[w]);
  u32 t17[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) t17[w] = lop3<0x96>(t9[w], t14[w], t16[w]);
  u32 t18[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) t18[w] = lop3<0xe8>(t9[w], t14[w], t16[w]);
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    q[w][0] = t11[w];
    q[w][1] = t18[w];
    q[w][2] = t15[w];
    q[w][3] = t17[w];
  }
}

// 4-word interleaved form of f5_acc: each adder is issued for all four words in turn
__device__ __forceinline__ void f5_acc4(u32 (&q)[4][5], const u32 (&in)[4][9]) {
  u32 t1[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) t1[w] = lop3<0x69>(q[w][0], in[w][0], in[w][6]);
  u32 t2[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) t2[w] = lop3<0xd4>(q[w][0], in[w][0], in[w][6]);
  u32 t3[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) t3[w] = lop3<0x96>(q[w][1], in[w][1], in[w][3]);
  u32 t4[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) t4[w] = lop3<0xe8>(q[w][1], in[w][1], in[w][3]);
  u32 t5[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) t5[w] = lop3<0x69>(in[w][7], t2[w], t3[w]);
  u32 t6[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) t6[w] = lop3<0x8e>(in[w][7], t2[w], t3[w]);
  u32 t7[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) t7[w] = lop3<0x96>(q[w][2], q[w][3], in[w][2]);
  u32 t8[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) t8[w] = lop3<0xe8>(q[w][2], q[w][3], in[w][2]);
  u32 t9[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) t9[w] = lop3<0x69>(in[w][4], in[w][8], t4[w]);
  u32 t10[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) t10[w] = lop3<0xb2>(in[w][4], in[w][8], t4[w]);
  u32 t11[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) t11[w] = lop3<0x96>(t7[w], t6[w], t9[w]);
  u32 t12[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) t12[w] = lop3<0xe8>(t7[w], t6[w], t9[w]);
  u32 t13[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) t13[w] = lop3<0x96>(q[w][4], in[w][5], t8[w]);
  u32 t14[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) t14[w] = lop3<0xe8>(q[w][4], in[w][5], t8[w]);
  u32 t15[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) t15[w] = lop3<0x96>(t10[w], t13[w], t12[w]);
  u32 t16[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) t16[w] = lop3<0xe8>(t10[w], t13[w], t12[w]);
  u32 t17[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) t17[w] = lop3<0x96>(t1[w], t14[w], t16[w]);
  u32 t18[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) t18[w] = lop3<0xe8>(t1[w], t14[w], t16[w]);
  u32 t19[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) t19[w] = lop3<0x96>(t5[w], t18[w], 0u);
  u32 t20[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) t20[w] = lop3<0xe8>(t5[w], t18[w], 0u);
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    q[w][0] = t17[w];
    q[w][1] = t19[w];
    q[w][2] = t11[w];
    q[w][3] = t20[w];
    q[w][4] = t15[w];
  }
}

// ---------------------------------------------------------------- Z/4, Z/8, GF(8)
// x += y mod 4 (3 LOP3: r1 = x1 ^ y1 ^ (x0 & y0))
__device__ __forceinline__ void z4_add(u32& x0, u32& x1, u32 y0, u32 y1) {
  x1 = x1 ^ y1 ^ (x0 & y0);
  x0 ^= y0;
}
// -x mod 4 (two's complement: (x0, x0 ^ x1)), kernels.py:125-126
__device__ __forceinline__ void z4_neg(u32& x0, u32& x1) { x1 ^= x0; }
// x += y mod 8: grade-school chain without the final carry (kernels.py:399-401)
__device__ __forceinline__ void z8_add(u32& x0, u32& x1, u32& x2, u32 y0, u32 y1, u32 y2) {
  const u32 c1 = x0 & y0;
  const u32 c2 = lop3<LOP_MAJ>(x1, y1, c1);
  x2 = x2 ^ y2 ^ c2;
  x1 = x1 ^ y1 ^ c1;
  x0 ^= y0;
}
// -x mod 8 (two's complement: flip above the lowest set bit), kernels.py:404-406
__device__ __forceinline__ void z8_neg(u32& x0, u32& x1, u32& x2) {
  x2 ^= x0 | x1;
  x1 ^= x0;
}
// multiply by x in GF(8) = F2[x]/(x^3+x+1): (c0, c1, c2) -> (c2, c0 ^ c2, c1)
__device__ __forceinline__ void gf8_mulx(u32& c0, u32& c1, u32& c2) {
  const u32 t = c2;
  c2 = c1;
  c1 = c0 ^ t;
  c0 = t;
}

// ---------------------------------------------------------------- generic row helpers
// Plane-vector types: V<F> holds the R plane words of one 32-lane group.
template <int F> struct V { u32 p[Traits<F>::R]; };

template <int F> __device__ __forceinline__ void vadd(V<F>& x, const V<F>& y) {
  if constexpr (F == F2) {
    x.p[0] ^= y.p[0];
  } else if constexpr (F == GF4) {
    x.p[0] ^= y.p[0]; x.p[1] ^= y.p[1];
  } else if constexpr (F == GF8) {
    x.p[0] ^= y.p[0]; x.p[1] ^= y.p[1]; x.p[2] ^= y.p[2];
  } else if constexpr (F == Z4) {
    z4_add(x.p[0], x.p[1], y.p[0], y.p[1]);
  } else if constexpr (F == Z8) {
    z8_add(x.p[0], x.p[1], x.p[2], y.p[0], y.p[1], y.p[2]);
  } else if constexpr (F == F3) {
    f3_add(x.p[0], x.p[1], y.p[0], y.p[1]);
  } else if constexpr (F == F5) {
    f5_add(x.p[0], x.p[1], x.p[2], y.p[0], y.p[1], y.p[2]);
  } else {
    f7_add(x.p[0], x.p[1], x.p[2], y.p[0], y.p[1], y.p[2]);
  }
}

template <int F> __device__ __forceinline__ void vcanon(V<F>& x) {
  if constexpr (F == F5) f5_reduce(x.p[0], x.p[1], x.p[2]);
  if constexpr (F == F7) f7_reduce(x.p[0], x.p[1], x.p[2]);
}

}  // namespace sg
