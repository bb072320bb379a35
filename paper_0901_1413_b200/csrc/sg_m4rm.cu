// sg_m4rm.cu -- the bitsliced Method-of-Four-Russians product C = A*B on sm_100a.
//
// Reference path (what this replaces): m4rm_multiply = for each k-block s,
// build_table then _core.active().m4rm_block_<f> (_core_py.py:205-281),
// whose per-row loop does  C_i += sum_d alpha_d * T[phi_d(a_i, block s)].
//
// B200 design:
//  * One CTA owns a 128-column slab of C (4 x 32-bit words per plane) and ROWS = RT*256 rows,
//    and walks the k-blocks of its split of the inner dimension.  C lives in registers for
//    the whole walk: lane (t, tid) holds rows t*256+tid, one uint4 per plane.
//  * Per k-block the CTA builds the 2^K-entry table of its slab in shared memory:
//    phase 1: two half tables (rows 0..3 and 4..7 of the block, 16 entries each) from the B
//    rows that cp.async staged two blocks ahead; phase 2: T[g] = Thi[g>>4] + Tlo[g&15],
//    one bitsliced field add per word, written as 8 replicas (see COPIES).
//  * Lookups: the 8 lanes of each LDS.128 phase hold 8 different rows, i.e. 8 random table
//    entries.  Replica j of every entry sits at bank offset 4j and lane (tid&7) reads replica
//    tid&7, so each phase touches all 32 banks exactly once: conflict-free for any indices.
//  * Index bytes come from A^T (A's planes transposed to [plane][word][row] by a pre-pass, F3's
//    plane 0 pre-XORed to A0^A1), staged per 32-bit word into shared memory by cp.async: one
//    conflict-free LDS.32 per (row, block, plane).
//  * Epilogue: canonical reduce (F5/F7) and store, or raw partial sums for split-K.
#include <cstdio>

#include "sg_field.cuh"
#include "sg_internal.h"

namespace sg {

__device__ __forceinline__ void cp_async16(void* dst, const void* src, int bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(src), "r"(bytes));
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src, int bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(src), "r"(bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N> __device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

template <int F> __device__ __forceinline__ V<F> vzero() {
  V<F> v;
#pragma unroll
  for (int d = 0; d < Traits<F>::R; ++d) v.p[d] = 0u;
  return v;
}

// Row accumulator of one lane: 4 words x RS planes.
template <int F> struct Acc { u32 w[4][Traits<F>::RS]; };

// One (row, k-block) update of the 4 C words a lane owns.  tl = this lane's replica base,
// TPL = uint4 stride between table planes, e = the byte offsets of the basis entries.
template <int F, int TPL>
__device__ __forceinline__ void accumulate(Acc<F>& c, const unsigned char* __restrict__ tl, const u32 (&e)[3]) {
  auto T = [&](int d, int i) { return *reinterpret_cast<const uint4*>(tl + e[i] + d * TPL * 16); };
  if constexpr (F == F2) {
    const uint4 p = T(0, 0);
    c.w[0][0] ^= p.x; c.w[1][0] ^= p.y; c.w[2][0] ^= p.z; c.w[3][0] ^= p.w;
  } else if constexpr (F == F3) {
    // basis {1, -1}: C += T[pos]; C -= T[neg]   (_core_py.py:213-222), 6 LOP3 per word
    const uint4 pu = T(0, 0), ps = T(1, 0), nu = T(0, 1), ns = T(1, 1);
    const u32 PU[4] = {pu.x, pu.y, pu.z, pu.w}, PS[4] = {ps.x, ps.y, ps.z, ps.w};
    const u32 NU[4] = {nu.x, nu.y, nu.z, nu.w}, NS[4] = {ns.x, ns.y, ns.z, ns.w};
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      f3_add(c.w[w][0], c.w[w][1], PU[w], PS[w]);
      f3_sub(c.w[w][0], c.w[w][1], NU[w], NS[w]);
    }
  } else if constexpr (F == GF4) {
    // power basis {1, x}: C += T[g0] + x*T[g1],  x*(t0, t1) = (t1, t0 ^ t1)
    const uint4 p0 = T(0, 0), p1 = T(1, 0), q0 = T(0, 1), q1 = T(1, 1);
    c.w[0][0] ^= p0.x ^ q1.x; c.w[0][1] ^= p1.x ^ q0.x ^ q1.x;
    c.w[1][0] ^= p0.y ^ q1.y; c.w[1][1] ^= p1.y ^ q0.y ^ q1.y;
    c.w[2][0] ^= p0.z ^ q1.z; c.w[2][1] ^= p1.z ^ q0.z ^ q1.z;
    c.w[3][0] ^= p0.w ^ q1.w; c.w[3][1] ^= p1.w ^ q0.w ^ q1.w;
  } else {
    // F5 / F7, basis {1, 2, 4}: C += T[g0] + 2*T[g1] + 4*T[g2] (the reference's Horner form,
    // _core_py.py:241-255, reassociated); doubling is a plane rotation in both accumulators.
    const uint4 a0 = T(0, 0), a1 = T(1, 0), a2 = T(2, 0);
    const uint4 b0 = T(0, 1), b1 = T(1, 1), b2 = T(2, 1);
    const uint4 d0 = T(0, 2), d1 = T(1, 2), d2 = T(2, 2);
    const u32 X0[4] = {a0.x, a0.y, a0.z, a0.w}, X1[4] = {a1.x, a1.y, a1.z, a1.w}, X2[4] = {a2.x, a2.y, a2.z, a2.w};
    const u32 Y0[4] = {b0.x, b0.y, b0.z, b0.w}, Y1[4] = {b1.x, b1.y, b1.z, b1.w}, Y2[4] = {b2.x, b2.y, b2.z, b2.w};
    const u32 Z0[4] = {d0.x, d0.y, d0.z, d0.w}, Z1[4] = {d1.x, d1.y, d1.z, d1.w}, Z2[4] = {d2.x, d2.y, d2.z, d2.w};
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      u32* q = c.w[w];
      if constexpr (F == F7) {  // 2y = (y2, y0, y1), 4z = (z1, z2, z0) mod 7; 3 x 8 LOP3
        f7_add(q[0], q[1], q[2], X0[w], X1[w], X2[w]);
        f7_add(q[0], q[1], q[2], Y2[w], Y0[w], Y1[w]);
        f7_add(q[0], q[1], q[2], Z1[w], Z2[w], Z0[w]);
      } else {  // mod 15: x = (x0,x1,x2,0), 2y = (0,y0,y1,y2), 4z = (z2,0,z0,z1)
        add15(q[0], q[1], q[2], q[3], X0[w], X1[w], X2[w], 0u);
        add15(q[0], q[1], q[2], q[3], 0u, Y0[w], Y1[w], Y2[w]);
        add15(q[0], q[1], q[2], q[3], Z2[w], 0u, Z0[w], Z1[w]);
      }
    }
  }
}

// Accumulator -> output planes (canonical for the final C; F5 always leaves mod 15 here).
template <int F> __device__ __forceinline__ void finish(const u32 (&q)[Traits<F>::RS], u32 (&o)[Traits<F>::R],
                                                        bool canonical) {
  if constexpr (F == F5) {
    mod15_to_f5(q[0], q[1], q[2], q[3], o[0], o[1], o[2]);
  } else {
#pragma unroll
    for (int d = 0; d < Traits<F>::R; ++d) o[d] = q[d];
    if constexpr (F == F7) {
      if (canonical) f7_reduce(o[0], o[1], o[2]);
    }
  }
}

template <int F, int K, int RT>
__global__ void __launch_bounds__(THREADS, 1) m4rm_kernel(const M4rmArgs a) {
  constexpr int NT = THREADS;
  constexpr int R = Traits<F>::R;
  constexpr int E = 1 << K;
  constexpr int KLO = K < 4 ? K : 4;
  constexpr int KHI = K - KLO;
  constexpr int ROWS = RT * NT;
  constexpr int TPLANE = E * ENTRY_BYTES;  // bytes per table plane
  constexpr int TPL = TPLANE / 16;         // uint4 per table plane
  constexpr int HALF = 16 * R * 4;         // u32 per half table

  extern __shared__ __align__(128) unsigned char smem[];
  uint4* tab = reinterpret_cast<uint4*>(smem);
  u32* thalf = reinterpret_cast<u32*>(smem + R * TPLANE);  // [2 buf][2 half][16][R][4]
  u32* bst = thalf + 2 * 2 * HALF;                          // [2 buf][K][R][4]
  u32* ast = bst + 2 * K * R * 4;                           // [2 slot][R][ROWS]

  const int tid = threadIdx.x;
  const int word0 = blockIdx.x * SLAB_WORDS;
  const int64_t row0 = (int64_t)blockIdx.y * ROWS;
  const int s_begin = blockIdx.z * a.bps;
  const int s_end = min(a.nblocks, s_begin + a.bps);
  if (s_begin >= s_end) return;

  int next_word = (s_begin * K) >> 5;
  // Stage block s's B rows (K x R x 16 B) and any A^T words it needs that are not yet staged.
  auto issue = [&](int s) {
    if (s < s_end) {
      u32* bdst = bst + (s & 1) * K * R * 4;
      for (int q = tid; q < K * R * 2; q += NT) {
        const int i = q / (R * 2), d = (q >> 1) % R, half = q & 1;
        const int64_t row = (int64_t)s * K + i;
        const int w = word0 + 2 * half;
        const bool ok = row < a.l && w < a.wc32;
        const u32* src = ok ? a.B + ((int64_t)d * a.l + row) * a.wc32 + w : a.B;
        cp_async8(bdst + (i * R + d) * 4 + 2 * half, src, ok ? 8 : 0);
      }
      const int whi = (s * K + K - 1) >> 5;
      for (; next_word <= whi; ++next_word) {
        u32* adst = ast + (next_word & 1) * R * ROWS;
        const bool ok = next_word < a.wa32;
        for (int q = tid; q < R * ROWS / 4; q += NT) {
          const int d = q / (ROWS / 4), r4 = q % (ROWS / 4);
          const u32* src = ok ? a.AT + ((int64_t)d * a.wa32 + next_word) * a.mpad + row0 + 4 * r4 : a.AT;
          cp_async16(adst + d * ROWS + 4 * r4, src, ok ? 16 : 0);
        }
      }
    }
    cp_async_commit();
  };

  issue(s_begin);
  issue(s_begin + 1);
  cp_async_wait<1>();
  __syncthreads();

  Acc<F> c[RT];
#pragma unroll
  for (int t = 0; t < RT; ++t)
#pragma unroll
    for (int w = 0; w < 4; ++w)
#pragma unroll
      for (int d = 0; d < Traits<F>::RS; ++d) c[t].w[w][d] = 0u;

  const unsigned char* tl = reinterpret_cast<const unsigned char*>(tab + (tid & (COPIES - 1)));

  for (int s = s_begin; s < s_end; ++s) {
    // ---- phase 1: half tables from the staged B rows
    {
      const u32* bs = bst + (s & 1) * K * R * 4;
      u32* th = thalf + (s & 1) * 2 * HALF;
      if (tid < 128) {
        const int h = tid >> 6, e = (tid >> 2) & 15, w = tid & 3;
        const int nrows = h ? KHI : KLO;
        if (e < (1 << nrows)) {
          V<F> acc = vzero<F>();
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            if (i < nrows && ((e >> i) & 1)) {
              V<F> b;
#pragma unroll
              for (int d = 0; d < R; ++d) b.p[d] = bs[((h * KLO + i) * R + d) * 4 + w];
              vadd<F>(acc, b);
            }
          }
#pragma unroll
          for (int d = 0; d < R; ++d) th[((h * 16 + e) * R + d) * 4 + w] = acc.p[d];
        }
      }
    }
    __syncthreads();
    issue(s + 2);
    // ---- phase 2: full table, 8 replicas
    {
      constexpr int TPE_RAW = NT / E;
      constexpr int TPE = TPE_RAW < 1 ? 1 : (TPE_RAW > COPIES ? COPIES : TPE_RAW);
      constexpr int CPT = COPIES / TPE;  // replicas written per thread
      const u32* th = thalf + (s & 1) * 2 * HALF;
      const int g = tid / TPE, part = tid % TPE;
      if (g < E) {
        const uint4* lo = reinterpret_cast<const uint4*>(th + (g & ((1 << KLO) - 1)) * R * 4);
        const uint4* hi = reinterpret_cast<const uint4*>(th + HALF + (g >> KLO) * R * 4);
        V<F> v[4], hv[4];
#pragma unroll
        for (int d = 0; d < R; ++d) {
          const uint4 L = lo[d], H = hi[d];
          v[0].p[d] = L.x; v[1].p[d] = L.y; v[2].p[d] = L.z; v[3].p[d] = L.w;
          hv[0].p[d] = H.x; hv[1].p[d] = H.y; hv[2].p[d] = H.z; hv[3].p[d] = H.w;
        }
        if constexpr (KHI > 0) {
#pragma unroll
          for (int w = 0; w < 4; ++w) vadd<F>(v[w], hv[w]);
        }
#pragma unroll
        for (int cc = 0; cc < CPT; ++cc) {
          // rotate the replica order by g so the 8 lanes of a store phase hit 8 different banks
          const int copy = (part * CPT + cc + g) & (COPIES - 1);
#pragma unroll
          for (int d = 0; d < R; ++d)
            tab[d * TPL + g * (ENTRY_BYTES / 16) + copy] = make_uint4(v[0].p[d], v[1].p[d], v[2].p[d], v[3].p[d]);
        }
      }
    }
    cp_async_wait<1>();
    __syncthreads();
    // ---- phase 3: lookups and accumulation for this k-block
    {
      const int col0 = s * K;
      const int w0 = col0 >> 5, sh = col0 & 31;
      const u32* aw0 = ast + (w0 & 1) * R * ROWS;
      const u32* aw1 = ast + ((w0 + 1) & 1) * R * ROWS;
      const u32 sel = 0x4440u | (u32)(sh >> 3);  // PRMT: byte sh/8 of x, zero-extended
#pragma unroll
      for (int t = 0; t < RT; ++t) {
        const int lr = t * NT + tid;
        u32 e[3] = {0u, 0u, 0u};
#pragma unroll
        for (int d = 0; d < R; ++d) {
          u32 x = aw0[d * ROWS + lr];
          if constexpr (K == 8) {
            x = __byte_perm(x, 0u, sel);
          } else if constexpr (32 % K == 0) {
            x = (x >> sh) & (E - 1);
          } else {
            x = ((sh + K > 32) ? __funnelshift_r(x, aw1[d * ROWS + lr], sh) : (x >> sh)) & (E - 1);
          }
          e[d] = x * ENTRY_BYTES;
        }
        accumulate<F, TPL>(c[t], tl, e);
      }
    }
  }

  // ---- epilogue
  u32* out = a.C;
  int64_t rows_out = a.m;
  if (a.partial) {
    out += (int64_t)blockIdx.z * R * a.mpad * a.wc32;
    rows_out = a.mpad;
  }
#pragma unroll
  for (int t = 0; t < RT; ++t) {
    const int64_t row = row0 + t * NT + tid;
    if (row < a.m) {
      u32 o[4][R];
#pragma unroll
      for (int w = 0; w < 4; ++w) finish<F>(c[t].w[w], o[w], !a.partial);
#pragma unroll
      for (int d = 0; d < R; ++d) {
        u32* dst = out + ((int64_t)d * rows_out + row) * a.wc32 + word0;
        if (word0 < a.wc32) *reinterpret_cast<uint2*>(dst) = make_uint2(o[0][d], o[1][d]);
        if (word0 + 2 < a.wc32) *reinterpret_cast<uint2*>(dst + 2) = make_uint2(o[2][d], o[3][d]);
      }
    }
  }
}

// ------------------------------------------------------------------ A transpose pre-pass
// A planes [R][m][wa32] -> A^T [R][wa32][mpad]; F3's plane 0 becomes A0 ^ A1 (the "+1" basis
// coefficient, fields.py:98), plane 1 stays A1 (the "-1" coefficient, fields.py:99).
__global__ void transpose_a_kernel(const u32* __restrict__ A, u32* __restrict__ AT, int64_t m,
                                   int64_t mpad, int wa32, int f3) {
  __shared__ u32 tile[32][33];
  const int d = blockIdx.z;
  const int64_t rbase = (int64_t)blockIdx.y * 32;
  const int wbase = blockIdx.x * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t row = rbase + ty + 8 * i;
    const int w = wbase + tx;
    u32 v = 0;
    if (row < m && w < wa32) {
      v = A[((int64_t)d * m + row) * wa32 + w];
      if (f3 && d == 0) v ^= A[(m + row) * wa32 + w];
    }
    tile[ty + 8 * i][tx] = v;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int w = wbase + ty + 8 * i;
    const int64_t row = rbase + tx;
    if (w < wa32 && row < mpad) AT[((int64_t)d * wa32 + w) * mpad + row] = tile[tx][ty + 8 * i];
  }
}

// ------------------------------------------------------------------ split-K reduction
template <int F>
__global__ void reduce_splits_kernel(const u32* __restrict__ P, u32* __restrict__ C, int64_t m,
                                     int64_t mpad, int wc32, int splits) {
  constexpr int R = Traits<F>::R;
  const int64_t total = m * wc32;
  const int64_t plane = mpad * (int64_t)wc32;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / wc32, w = i % wc32;
    const int64_t off = row * wc32 + w;
    V<F> acc;
#pragma unroll
    for (int d = 0; d < R; ++d) acc.p[d] = P[d * plane + off];
    for (int sp = 1; sp < splits; ++sp) {
      V<F> x;
#pragma unroll
      for (int d = 0; d < R; ++d) x.p[d] = P[((int64_t)sp * R + d) * plane + off];
      vadd<F>(acc, x);
    }
    vcanon<F>(acc);
#pragma unroll
    for (int d = 0; d < R; ++d) C[(d * m + row) * wc32 + w] = acc.p[d];
  }
}

// ------------------------------------------------------------------ registry
template <int F, int K, int RT>
constexpr int smem_bytes_for() {
  constexpr int R = Traits<F>::R;
  return R * (1 << K) * ENTRY_BYTES + 2 * 2 * 16 * R * 4 * 4 + 2 * K * R * 4 * 4 + 2 * R * RT * THREADS * 4;
}

#define SG_K(F, K, RT) {m4rm_kernel<F, K, RT>, F, K, RT, THREADS, smem_bytes_for<F, K, RT>(), 0, 0}
#define SG_KSET8(F) SG_K(F, 8, 1), SG_K(F, 8, 2), SG_K(F, 8, 4), SG_K(F, 8, 8)
#define SG_KLOW(F) SG_K(F, 1, 1), SG_K(F, 2, 1), SG_K(F, 3, 1), SG_K(F, 4, 1), SG_K(F, 5, 1), SG_K(F, 6, 1), SG_K(F, 7, 1)

static KernelInfo g_kernels[] = {
    SG_KSET8(F2), SG_K(F2, 8, 16), SG_KLOW(F2),
    SG_KSET8(F3), SG_K(F3, 8, 16), SG_KLOW(F3),
    SG_KSET8(GF4), SG_K(GF4, 8, 16), SG_KLOW(GF4),
    SG_KSET8(F5), SG_KLOW(F5),
    SG_KSET8(F7), SG_KLOW(F7),
};

int m4rm_kernel_count() { return (int)(sizeof(g_kernels) / sizeof(g_kernels[0])); }
KernelInfo* m4rm_kernel_at(int i) { return &g_kernels[i]; }

cudaError_t launch_m4rm(const KernelInfo& ki, const M4rmArgs& a, dim3 grid, cudaStream_t st) {
  ki.fn<<<grid, ki.threads, ki.smem_bytes, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_transpose_a(int field, const uint32_t* A, uint32_t* AT, int64_t m, int64_t mpad,
                               int wa32, cudaStream_t st) {
  const int R = field == F2 ? 1 : (field == F5 || field == F7) ? 3 : 2;
  dim3 grid((wa32 + 31) / 32, (unsigned)((mpad + 31) / 32), R);
  transpose_a_kernel<<<grid, dim3(32, 8), 0, st>>>(A, AT, m, mpad, wa32, field == F3);
  return cudaGetLastError();
}

cudaError_t launch_reduce_splits(int field, const uint32_t* P, uint32_t* C, int64_t m, int64_t mpad,
                                 int wc32, int splits, cudaStream_t st) {
  const int64_t total = m * wc32;
  const int threads = 256;
  int64_t blocks = (total + threads - 1) / threads;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  switch (field) {
    case F2: reduce_splits_kernel<F2><<<(unsigned)blocks, threads, 0, st>>>(P, C, m, mpad, wc32, splits); break;
    case F3: reduce_splits_kernel<F3><<<(unsigned)blocks, threads, 0, st>>>(P, C, m, mpad, wc32, splits); break;
    case F5: reduce_splits_kernel<F5><<<(unsigned)blocks, threads, 0, st>>>(P, C, m, mpad, wc32, splits); break;
    case F7: reduce_splits_kernel<F7><<<(unsigned)blocks, threads, 0, st>>>(P, C, m, mpad, wc32, splits); break;
    default: reduce_splits_kernel<GF4><<<(unsigned)blocks, threads, 0, st>>>(P, C, m, mpad, wc32, splits); break;
  }
  return cudaGetLastError();
}

}  // namespace sg
