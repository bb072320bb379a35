/*
 * sg_oracle.c -- CPU restatement of the reference's bitsliced M4RM path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker and the CPU baseline
 * ("port") for the B200 kernels; it is never linked into, loaded by, or called from the
 * product path (paper_0901_1413_b200/), which fails loudly without its CUDA library.
 *
 * It restates, in plain C on 64-bit words (64 lanes per word, column c -> word c>>6,
 * bit c&63, padding lanes zero), what the reference computes:
 *   encodings        fields.py:78-129 (F2, F3 unit/sign, F5/F7 plain 3-bit, redundant)
 *   GF(4) encoding   fields.py:215 (F2[x]/(x^2+x+1)); plane0 = coeff of 1, plane1 = coeff of x
 *   plane kernels    _core_py.py:24-39 (f2_add, f3_add, f3_sub), :65-97 (3-bit adder
 *                    chain + F5/F7 folds), :116-148 (f5_add/neg/sub/double/reduce),
 *                    :151-175 (f7_add/neg/sub/reduce)
 *   block drivers    _core_py.py:186-222 (index extraction, f2/f3 drivers),
 *                    :241-281 (Horner over the basis {1,2,4} for f5/f7)
 *   table build      SPEC.md:313-325 (Gray order, T[0] = 0, one add/sub per entry)
 *   multiply loop    SPEC.md:326-332, 354-360 (ascending k-blocks, narrow final block,
 *                    row partition gives bit-identical output)
 *   GF(4) direct     power basis {1, x}: acc = x*T[g1] + T[g0], x*(c0,c1) = (c1, c0^c1)
 *                    (SURVEY.md 8a a8); decode-equal to oracle.py:192-215
 *   GF(8) direct     power basis {1, x, x^2} mod x^3+x+1 (fields.py:216), Horner with x*c =
 *                    (c2, c0^c2, c1); decode-equal to oracle_ext_multiply(F8)
 *   Z/4, Z/8         _core_py.py:46-62, 100-113 (ring kernels), :225-238, 262-266, 284-286
 *                    (block drivers: Horner over {1, 2[, 4]}, doubling = plane shift)
 * Parity pins: tests/golden/m4rm_<field>.npz, gf4.npz and kernel_cases.json, generated from the reference
 * itself by tests/golden/make_golden.py ("Oracle").
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "sg_oracle.h"

typedef uint64_t w64;

int sgo_planes(int field) {
  switch (field) {
    case SGO_F2: return 1;
    case SGO_F3: case SGO_GF4: case SGO_Z4: return 2;
    case SGO_F5: case SGO_F7: case SGO_GF8: case SGO_Z8: return 3;
    default: return -1;
  }
}

int sgo_order(int field) {
  switch (field) {
    case SGO_F2: return 2;
    case SGO_F3: return 3;
    case SGO_F5: return 5;
    case SGO_F7: return 7;
    case SGO_GF4: case SGO_Z4: return 4;
    case SGO_GF8: case SGO_Z8: return 8;
    default: return -1;
  }
}

/* residue -> canonical pattern (fields.py canonical_table); GF(4) element bits are the
 * coefficient planes directly. */
static unsigned pattern_of(int field, unsigned v) {
  if (field == SGO_F3) return v == 0 ? 0u : (v == 1 ? 1u : 3u);
  return v;
}

/* pattern -> residue (fields.py decode_table); returns 255 for an illegal pattern. */
static unsigned residue_of(int field, unsigned p) {
  switch (field) {
    case SGO_F3: return p == 0 ? 0 : p == 1 ? 1 : p == 3 ? 2 : 255;
    case SGO_F5: return p % 5;
    case SGO_F7: return p % 7;
    default: return p;
  }
}

int sgo_pack(int field, const uint8_t* dense, int64_t m, int64_t n, w64* planes) {
  int r = sgo_planes(field), order = sgo_order(field);
  int64_t W = (n + 63) / 64;
  memset(planes, 0, sizeof(w64) * (size_t)(r * m * W));
  for (int64_t i = 0; i < m; ++i)
    for (int64_t c = 0; c < n; ++c) {
      unsigned v = dense[i * n + c];
      if ((int)v >= order) return -1;
      unsigned p = pattern_of(field, v);
      for (int d = 0; d < r; ++d)
        if ((p >> d) & 1u) planes[(d * m + i) * W + (c >> 6)] |= (w64)1 << (c & 63);
    }
  return 0;
}

int sgo_unpack(int field, const w64* planes, int64_t m, int64_t n, uint8_t* dense) {
  int r = sgo_planes(field);
  int64_t W = (n + 63) / 64;
  for (int64_t i = 0; i < m; ++i)
    for (int64_t c = 0; c < n; ++c) {
      unsigned p = 0;
      for (int d = 0; d < r; ++d) p |= (unsigned)((planes[(d * m + i) * W + (c >> 6)] >> (c & 63)) & 1u) << d;
      unsigned v = residue_of(field, p);
      if (v == 255) return -1;
      dense[i * n + c] = (uint8_t)v;
    }
  return 0;
}

/* ---------------------------------------------------------------- word kernels
 * x[] holds the destination planes (updated in place), y[] the source planes. */
static inline void f3_add(w64* x, const w64* y) {
  w64 u = x[0] ^ y[1], v = x[1] ^ y[0];
  w64 lo = (u ^ x[1]) | (v ^ y[1]);
  x[1] = u & v;
  x[0] = lo;
}

static inline void f3_sub(w64* x, const w64* y) {
  w64 t = x[0] ^ y[0];
  w64 hi = (t ^ y[1]) & (y[0] ^ x[1]);
  x[0] = t | (x[1] ^ y[1]);
  x[1] = hi;
}

/* lanewise s = x + y as a 4-bit integer (s[0..3]) by the grade-school chain */
static inline void add3(const w64* x, const w64* y, w64* s) {
  w64 c0 = x[0] & y[0];
  w64 t1 = x[1] ^ y[1];
  w64 c1 = (x[1] & y[1]) | (t1 & c0);
  w64 t2 = x[2] ^ y[2];
  s[0] = x[0] ^ y[0];
  s[1] = t1 ^ c0;
  s[2] = t2 ^ c1;
  s[3] = (x[2] & y[2]) | (t2 & c1);
}

/* fold the 8s bit (8 = 3 mod 5) into three bits, residue preserved (_core_py.py:91-97) */
static inline void fold5(const w64* s, w64* r) {
  w64 t = s[2] | s[1];
  w64 r2 = s[0] ^ t;
  w64 r1 = (r2 & s[0]) ^ (s[3] ^ s[1]);
  r[0] = (t ^ s[2]) | (r1 & s[3]);
  r[1] = r1;
  r[2] = r2;
}

/* fold the 8s bit (8 = 1 mod 7) back into bit 0 (_core_py.py:84-88) */
static inline void fold7(const w64* s, w64* r) {
  w64 c0 = s[0] & s[3];
  r[0] = s[0] ^ s[3];
  r[1] = s[1] ^ c0;
  r[2] = s[2] ^ (s[1] & c0);
}

static inline void f5_add(w64* x, const w64* y) { w64 s[4]; add3(x, y, s); fold5(s, x); }
static inline void f7_add(w64* x, const w64* y) { w64 s[4]; add3(x, y, s); fold7(s, x); }

static inline void f5_neg(const w64* p, w64* o) {
  w64 r2 = p[2] ^ p[0];
  w64 r1 = (r2 & p[2]) ^ p[1];
  o[0] = r1 & p[1];
  o[1] = r1;
  o[2] = r2;
}

static inline void f5_sub(w64* x, const w64* y) { w64 n[3]; f5_neg(y, n); f5_add(x, n); }

static inline void f7_sub(w64* x, const w64* y, w64 tail) {
  w64 n[3] = {~y[0] & tail, ~y[1] & tail, ~y[2] & tail};
  f7_add(x, n);
}

static inline void f5_double(w64* p) {
  w64 t = p[1] | p[0];
  w64 r1 = p[2] ^ p[0];
  p[0] = (t ^ p[1]) | (r1 & p[2]);
  p[1] = r1;
  p[2] = t;
}

static inline void f7_double(w64* p) { w64 t = p[2]; p[2] = p[1]; p[1] = p[0]; p[0] = t; }

static inline void f5_reduce(w64* p) {
  w64 c = p[2] & (p[1] | p[0]);
  w64 w = c & ~p[0];
  p[0] ^= c;
  p[2] ^= c;
  p[1] &= ~w;
}

static inline void f7_reduce(w64* p) {
  w64 t = p[0] & p[1] & p[2];
  p[0] ^= t; p[1] ^= t; p[2] ^= t;
}

static inline void z4_add(w64* x, const w64* y) {
  w64 c = x[0] & y[0];
  x[0] ^= y[0];
  x[1] ^= y[1] ^ c;
}
static inline void z4_sub(w64* x, const w64* y) {
  w64 n[2] = {y[0], y[0] ^ y[1]};
  z4_add(x, n);
}
static inline void z8_add(w64* x, const w64* y) {
  w64 s[4];
  add3(x, y, s);
  x[0] = s[0]; x[1] = s[1]; x[2] = s[2];
}
static inline void z8_sub(w64* x, const w64* y) {
  w64 n[3] = {y[0], y[0] ^ y[1], (y[0] | y[1]) ^ y[2]};
  z8_add(x, n);
}
static inline void gf8_mulx(w64* c) {
  w64 t = c[2];
  c[2] = c[1];
  c[1] = c[0] ^ t;
  c[0] = t;
}

void sgo_canonicalize(int field, w64* planes, int64_t rows, int64_t W) {
  int64_t N = rows * W;
  if (field != SGO_F5 && field != SGO_F7) return;
  for (int64_t i = 0; i < N; ++i) {
    w64 p[3] = {planes[i], planes[N + i], planes[2 * N + i]};
    if (field == SGO_F5) f5_reduce(p); else f7_reduce(p);
    planes[i] = p[0]; planes[N + i] = p[1]; planes[2 * N + i] = p[2];
  }
}

/* Lanewise evaluation of one named kernel, for the exhaustive-case tests.
 * in/out are plane words, destination planes first then source planes. */
int sgo_word_op(const char* name, const w64* in, w64* out) {
  w64 x[3] = {in[0], in[1], in[2]}, y[3] = {0, 0, 0};
#define IS(s) (strcmp(name, s) == 0)
  if (IS("f3_add") || IS("f3_sub")) {
    y[0] = in[2]; y[1] = in[3];
    if (IS("f3_add")) f3_add(x, y); else f3_sub(x, y);
    out[0] = x[0]; out[1] = x[1];
    return 2;
  }
  if (IS("f3_neg")) { out[0] = in[0]; out[1] = in[0] ^ in[1]; return 2; }
  if (IS("f5_add") || IS("f7_add")) {
    y[0] = in[3]; y[1] = in[4]; y[2] = in[5];
    if (IS("f5_add")) f5_add(x, y); else f7_add(x, y);
    memcpy(out, x, sizeof x);
    return 3;
  }
  if (IS("f5_fold5")) { fold5(in, out); return 3; }
  if (IS("f5_double")) { f5_double(x); memcpy(out, x, sizeof x); return 3; }
  if (IS("f5_neg")) { f5_neg(in, out); return 3; }
  if (IS("f5_reduce")) { f5_reduce(x); memcpy(out, x, sizeof x); return 3; }
  if (IS("f7_double")) { f7_double(x); memcpy(out, x, sizeof x); return 3; }
  if (IS("f7_neg")) { out[0] = ~in[0]; out[1] = ~in[1]; out[2] = ~in[2]; return 3; }
  if (IS("f7_reduce")) { f7_reduce(x); memcpy(out, x, sizeof x); return 3; }
#undef IS
  return -1;
}

/* ---------------------------------------------------------------- M4RM */
typedef struct {
  int field, k, r;
  const w64 *A, *B;
  w64* C;
  int64_t m, l, n, W, WA, row0, row1;
} job_t;

/* bit t of the k-bit index = column col0+t of the given A plane row (_core_py.py:186-192) */
static inline unsigned extract(const w64* row, int64_t col0, int kp) {
  unsigned g = 0;
  for (int t = 0; t < kp; ++t) {
    int64_t c = col0 + t;
    g |= (unsigned)((row[c >> 6] >> (c & 63)) & 1u) << t;
  }
  return g;
}

static void table_add(int field, w64* T, int64_t stride, int64_t dst, int64_t src_row_idx,
                      const w64* B, int64_t l, int64_t W, int r, int sub, w64 tail) {
  for (int64_t w = 0; w < W; ++w) {
    w64 x[3], y[3];
    for (int d = 0; d < r; ++d) {
      x[d] = T[d * stride + dst * W + w];
      y[d] = B[(d * l + src_row_idx) * W + w];
    }
    switch (field) {
      case SGO_F2: case SGO_GF4: case SGO_GF8:
        for (int d = 0; d < r; ++d) x[d] ^= y[d];
        break;
      case SGO_Z4: if (sub) z4_sub(x, y); else z4_add(x, y); break;
      case SGO_Z8: if (sub) z8_sub(x, y); else z8_add(x, y); break;
      case SGO_F3: if (sub) f3_sub(x, y); else f3_add(x, y); break;
      case SGO_F5: if (sub) f5_sub(x, y); else f5_add(x, y); break;
      case SGO_F7: if (sub) f7_sub(x, y, w == W - 1 ? tail : ~(w64)0); else f7_add(x, y); break;
    }
    for (int d = 0; d < r; ++d) T[d * stride + dst * W + w] = x[d];
  }
}

static void* run_job(void* arg) {
  job_t* j = (job_t*)arg;
  int field = j->field, k = j->k, r = j->r;
  int64_t W = j->W, WA = j->WA, m = j->m, l = j->l;
  int64_t stride = ((int64_t)1 << k) * W;  /* words per table plane */
  w64* T = (w64*)calloc((size_t)(r * stride), sizeof(w64));
  w64 tail = (j->n % 64) ? (((w64)1 << (j->n % 64)) - 1) : ~(w64)0;
  for (int64_t s = 0; s * k < l; ++s) {
    int64_t col0 = s * k;
    int kp = (int)((l - col0) < k ? (l - col0) : k);
    /* Gray-order build: entry g from its predecessor with one row add or sub */
    memset(T, 0, sizeof(w64) * (size_t)(r * stride));
    unsigned prev = 0;
    for (unsigned i = 1; i < (1u << kp); ++i) {
      unsigned g = i ^ (i >> 1);
      int t = __builtin_ctz(g ^ prev);
      for (int d = 0; d < r; ++d)
        memcpy(T + d * stride + (int64_t)g * W, T + d * stride + (int64_t)prev * W, sizeof(w64) * W);
      table_add(field, T, stride, g, col0 + t, j->B, l, W, r, !((g >> t) & 1u), tail);
      prev = g;
    }
    for (int64_t i = j->row0; i < j->row1; ++i) {
      unsigned gi[3] = {0, 0, 0};
      if (field == SGO_F3) {
        /* pos = bits of A0^A1 (the element 1), neg = bits of A1 (the element -1) */
        unsigned a0 = extract(j->A + i * WA, col0, kp), a1 = extract(j->A + (m + i) * WA, col0, kp);
        gi[0] = a0 ^ a1; gi[1] = a1;
      } else {
        for (int d = 0; d < r; ++d) gi[d] = extract(j->A + (d * m + i) * WA, col0, kp);
      }
      if (!(gi[0] | gi[1] | gi[2])) continue;
      for (int64_t w = 0; w < W; ++w) {
        w64 c[3], acc[3], t0[3];
        for (int d = 0; d < r; ++d) c[d] = j->C[(d * m + i) * W + w];
#define TE(d, g) T[(d) * stride + (int64_t)(g) * W + w]
        switch (field) {
          case SGO_F2:
            c[0] ^= TE(0, gi[0]);
            break;
          case SGO_F3:
            t0[0] = TE(0, gi[0]); t0[1] = TE(1, gi[0]); f3_add(c, t0);
            t0[0] = TE(0, gi[1]); t0[1] = TE(1, gi[1]); f3_sub(c, t0);
            break;
          case SGO_GF4: {
            w64 p0 = TE(0, gi[0]), p1 = TE(1, gi[0]), q0 = TE(0, gi[1]), q1 = TE(1, gi[1]);
            c[0] ^= p0 ^ q1;
            c[1] ^= p1 ^ q0 ^ q1;
            break;
          }
          case SGO_GF8: /* Horner: acc = x*(x*T[g2] + T[g1]) + T[g0] */
            for (int d = 0; d < 3; ++d) acc[d] = TE(d, gi[2]);
            gf8_mulx(acc);
            for (int d = 0; d < 3; ++d) acc[d] ^= TE(d, gi[1]);
            gf8_mulx(acc);
            for (int d = 0; d < 3; ++d) c[d] ^= acc[d] ^ TE(d, gi[0]);
            break;
          case SGO_Z4: /* acc = 2 T[g1] + T[g0] */
            acc[0] = 0; acc[1] = TE(0, gi[1]);
            t0[0] = TE(0, gi[0]); t0[1] = TE(1, gi[0]);
            z4_add(acc, t0);
            z4_add(c, acc);
            break;
          case SGO_Z8: /* Horner over {1, 2, 4}, doubling = plane shift */
            acc[0] = 0; acc[1] = TE(0, gi[2]); acc[2] = TE(1, gi[2]);
            for (int d = 0; d < 3; ++d) t0[d] = TE(d, gi[1]);
            z8_add(acc, t0);
            acc[2] = acc[1]; acc[1] = acc[0]; acc[0] = 0;
            for (int d = 0; d < 3; ++d) t0[d] = TE(d, gi[0]);
            z8_add(acc, t0);
            z8_add(c, acc);
            break;
          default: /* F5, F7: Horner over {1, 2, 4} */
            for (int d = 0; d < 3; ++d) acc[d] = TE(d, gi[2]);
            if (field == SGO_F5) f5_double(acc); else f7_double(acc);
            for (int d = 0; d < 3; ++d) t0[d] = TE(d, gi[1]);
            if (field == SGO_F5) f5_add(acc, t0); else f7_add(acc, t0);
            if (field == SGO_F5) f5_double(acc); else f7_double(acc);
            for (int d = 0; d < 3; ++d) t0[d] = TE(d, gi[0]);
            if (field == SGO_F5) { f5_add(acc, t0); f5_add(c, acc); }
            else { f7_add(acc, t0); f7_add(c, acc); }
        }
#undef TE
        for (int d = 0; d < r; ++d) j->C[(d * m + i) * W + w] = c[d];
      }
    }
  }
  free(T);
  return NULL;
}

int sgo_m4rm(int field, const w64* A, const w64* B, w64* C, int64_t m, int64_t l, int64_t n,
             int k, int threads, int64_t row0, int64_t row1) {
  int r = sgo_planes(field);
  if (r < 0 || k < 1 || k > 16 || m < 0 || l < 0 || n < 0) return -1;
  if (row1 < 0) row1 = m;
  if (row0 < 0 || row0 > row1 || row1 > m) return -1;
  if (threads < 1) threads = 1;
  int64_t W = (n + 63) / 64, WA = (l + 63) / 64;
  for (int d = 0; d < r; ++d)
    for (int64_t i = row0; i < row1; ++i) memset(C + (d * m + i) * W, 0, sizeof(w64) * W);
  if (l == 0 || W == 0 || row0 == row1) return 0;
  int64_t rows = row1 - row0;
  if (threads > rows) threads = (int)rows;
  pthread_t* tid = (pthread_t*)malloc(sizeof(pthread_t) * threads);
  job_t* jobs = (job_t*)malloc(sizeof(job_t) * threads);
  for (int t = 0; t < threads; ++t) {
    job_t* j = &jobs[t];
    j->field = field; j->k = k; j->r = r; j->A = A; j->B = B; j->C = C;
    j->m = m; j->l = l; j->n = n; j->W = W; j->WA = WA;
    j->row0 = row0 + rows * t / threads;
    j->row1 = row0 + rows * (t + 1) / threads;
    if (threads > 1) pthread_create(&tid[t], NULL, run_job, j); else run_job(j);
  }
  if (threads > 1)
    for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
  free(tid);
  free(jobs);
  return 0;
}
