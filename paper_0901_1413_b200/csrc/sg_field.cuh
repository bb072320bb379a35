// sg_field.cuh -- bitsliced field arithmetic on 32-bit plane words (32 lanes per word).
//
// Every function is lanewise boolean logic; nvcc folds the two-input networks into LOP3.
// The networks compute the same lane functions as the reference kernels:
//   F3  (plane0 = unit, plane1 = sign; 0=00, 1=01, -1=11)   _core_py.py:28-43, kernels.py:151-199
//   F5  (3-bit value, residue = value mod 5; redundant)     _core_py.py:65-75, 91-97, 116-148
//   F7  (3-bit value, residue = value mod 7; 7 == 0)         _core_py.py:65-75, 84-88, 151-175
//   F2  (1 plane, xor)                                        _core_py.py:24-25
//   GF4 (F2[x]/(x^2+x+1), plane0 = coeff of 1, plane1 = coeff of x)   fields.py:215
// Exhaustive lane tables for each formula (kernels.py:466-509, 550-590) are replayed on the
// device through sg_plane_op by tests/test_gpu_parity.py.
#pragma once
#include <cstdint>

namespace sg {

enum Field : int { F2 = 0, F3 = 1, F5 = 2, F7 = 3, GF4 = 4 };

typedef uint32_t u32;

template <int F> struct Traits;
// R = bit planes per element; NI = table lookups per (row, k-block) = basis size;
template <> struct Traits<F2>  { static constexpr int R = 1, NI = 1; };
template <> struct Traits<F3>  { static constexpr int R = 2, NI = 2; };
template <> struct Traits<F5>  { static constexpr int R = 3, NI = 3; };
template <> struct Traits<F7>  { static constexpr int R = 3, NI = 3; };
template <> struct Traits<GF4> { static constexpr int R = 2, NI = 2; };

// ---------------------------------------------------------------- F3
// x += y : the two shared subexpressions u = xu^ys, v = xs^yu make this six 2-input ops.
__device__ __forceinline__ void f3_add(u32& xu, u32& xs, u32 yu, u32 ys) {
  u32 u = xu ^ ys, v = xs ^ yu;
  u32 ru = (u ^ xs) | (v ^ ys);
  xs = u & v;
  xu = ru;
}
// x -= y : six 2-input ops (one fewer than neg-then-add).
__device__ __forceinline__ void f3_sub(u32& xu, u32& xs, u32 yu, u32 ys) {
  u32 t = xu ^ yu;
  u32 rs = (t ^ ys) & (yu ^ xs);
  xu = t | (xs ^ ys);
  xs = rs;
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
// 8 == 1 (mod 7): end-around carry; the sum of two lanes <= 14 never carries out again
__device__ __forceinline__ void fold7(u32 s0, u32 s1, u32 s2, u32 s3, u32& r0, u32& r1, u32& r2) {
  u32 c0 = s0 & s3;
  r0 = s0 ^ s3;
  r1 = s1 ^ c0;
  r2 = s2 ^ (s1 & c0);
}

__device__ __forceinline__ void f5_add(u32& x0, u32& x1, u32& x2, u32 y0, u32 y1, u32 y2) {
  u32 s0, s1, s2, s3;
  add3(x0, x1, x2, y0, y1, y2, s0, s1, s2, s3);
  fold5(s0, s1, s2, s3, x0, x1, x2);
}
__device__ __forceinline__ void f7_add(u32& x0, u32& x1, u32& x2, u32 y0, u32 y1, u32 y2) {
  u32 s0, s1, s2, s3;
  add3(x0, x1, x2, y0, y1, y2, s0, s1, s2, s3);
  fold7(s0, s1, s2, s3, x0, x1, x2);
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

// ---------------------------------------------------------------- generic row helpers
// Plane-vector types: V<F> holds the R plane words of one 32-lane group.
template <int F> struct V { u32 p[Traits<F>::R]; };

template <int F> __device__ __forceinline__ void vadd(V<F>& x, const V<F>& y) {
  if constexpr (F == F2) {
    x.p[0] ^= y.p[0];
  } else if constexpr (F == GF4) {
    x.p[0] ^= y.p[0]; x.p[1] ^= y.p[1];
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
