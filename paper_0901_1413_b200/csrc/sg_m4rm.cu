#include <algorithm>
#include <cstdlib>
// sg_m4rm.cu -- pre-pass, split-K reduction and launch glue around the M4RM kernel
// (kernel template: sg_m4rm_kernel.cuh; per-field instantiations: sg_m4rm_<field>.cu).
#include <vector>

#include "sg_m4rm_kernel.cuh"

namespace sg {

// ------------------------------------------------------------------ A transpose pre-pass
// A planes [R][m][wa32] -> A^T [R][wa32][mpad]; F3's plane 0 becomes A0 ^ A1 (the "+1" basis
// coefficient, fields.py:98), plane 1 stays A1 (the "-1" coefficient, fields.py:99).
__global__ void transpose_a_kernel(const u32* __restrict__ A, u32* __restrict__ AT, int64_t m,
                                   int64_t mpad, int wa32, int f3) {
  __shared__ u32 tile[32][33];
  pdl_trigger();
  const int d = blockIdx.z;
  const int wbase = blockIdx.x * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;
  // row tiles blockIdx.y, blockIdx.y + gridDim.y, ... (grid.y is capped at 65535)
  for (int64_t rbase = (int64_t)blockIdx.y * 32; rbase < mpad; rbase += (int64_t)gridDim.y * 32) {
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
    __syncthreads();
  }
}

// ------------------------------------------------------------------ k = 8 index-word pre-pass
// A planes [R][m][wa32] -> IW [nwords][mpad]: for k-block s (column byte s of each plane) the
// NI basis index bytes (F3: A0^A1 then A1; F5/F7: planes 0..2; GF4: planes 0..1; F2: plane 0)
// form one record of NIP bytes; RPW = 4/NIP records per 32-bit word.  A 32-row x 32-word tile
// of each plane is staged through shared memory so both reads and writes are coalesced.
template <int F>
__global__ void index_words_kernel(const u32* __restrict__ A, u32* __restrict__ IW, int64_t m, int64_t mpad,
                                   int wa32, int nwords) {
  constexpr int R = Traits<F>::R, NI = Traits<F>::NI;
  constexpr int NIP = NI == 3 ? 4 : NI, RPW = 4 / NIP;
  __shared__ u32 tile[R][32][33];
  pdl_trigger();  // the product kernel may launch now; it waits for this grid before reading IW
  const int wbase = blockIdx.x * 32;  // A words wbase.. (= k-blocks 4*wbase ..)
  const int tx = threadIdx.x, ty = threadIdx.y;
  // row tiles blockIdx.y, blockIdx.y + gridDim.y, ... (grid.y is capped at 65535)
  for (int64_t rbase = (int64_t)blockIdx.y * 32; rbase < mpad; rbase += (int64_t)gridDim.y * 32) {
#pragma unroll
    for (int d = 0; d < R; ++d)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int64_t row = rbase + ty + 8 * i;
        const int w = wbase + tx;
        tile[d][ty + 8 * i][tx] = (row < m && w < wa32) ? A[((int64_t)d * m + row) * wa32 + w] : 0u;
      }
    __syncthreads();
    // 128 k-blocks per tile -> 128 / RPW output words
    for (int q = ty; q < 128 / RPW; q += 8) {
      const int oq = (wbase * 4) / RPW + q;
      const int64_t row = rbase + tx;
      if (oq >= nwords || row >= mpad) continue;
      u32 v = 0;
#pragma unroll
      for (int b = 0; b < RPW; ++b) {
        const int sl = q * RPW + b;  // k-block within the tile
        const int aw = sl >> 2, sh = 8 * (sl & 3);
#pragma unroll
        for (int i = 0; i < NI; ++i) {
          u32 byte;
          if constexpr (F == F3) {
            byte = i == 0 ? ((tile[0][tx][aw] ^ tile[1][tx][aw]) >> sh) : (tile[1][tx][aw] >> sh);
          } else {
            byte = tile[i][tx][aw] >> sh;
          }
          v |= (byte & 0xFFu) << (8 * (b * NIP + i));
        }
      }
      IW[(int64_t)oq * mpad + row] = v;
    }
    __syncthreads();
  }
}

// Two-row records (paired_index, sg_m4rm_kernel.cuh): IW [nblocks][mpad / 2], word
// (g NT + j) of k-block s = the 2-byte records of rows g 2NT + j (low half) and g 2NT + NT + j
// (high half).  A block stages a 32-word x 32-row tile of each plane for both rows of 32 pairs.
template <int F>
__global__ void index_pairs_kernel(const u32* __restrict__ A, u32* __restrict__ IW, int64_t m, int64_t mpad,
                                   int wa32, int nblocks, int nt) {
  constexpr int R = Traits<F>::R;
  __shared__ u32 tile[2][R][32][33];
  pdl_trigger();  // the product kernel may launch now; it waits for this grid before reading IW
  const int wbase = blockIdx.x * 32;  // A words wbase.. (= k-blocks 4*wbase ..)
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int64_t half = mpad / 2;
  const int per_group = nt / 32;      // 32-pair tiles per 2 NT-row group
  for (int64_t pt = blockIdx.y; pt < half / 32; pt += gridDim.y) {
    const int64_t g = pt / per_group;
    const int64_t lo0 = g * 2 * nt + (pt % per_group) * 32;  // first low row; high rows + nt
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int d = 0; d < R; ++d)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int64_t row = lo0 + h * nt + ty + 8 * i;
          const int w = wbase + tx;
          tile[h][d][ty + 8 * i][tx] = (row < m && w < wa32) ? A[((int64_t)d * m + row) * wa32 + w] : 0u;
        }
    __syncthreads();
    for (int sl = ty; sl < 128; sl += 8) {
      const int s = wbase * 4 + sl;
      if (s >= nblocks) continue;
      const int aw = sl >> 2, sh = 8 * (sl & 3);
      u32 v = 0;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        u32 b0, b1;
        if constexpr (F == F3) {  // "+1" index from A0 ^ A1, "-1" from A1 (fields.py:98-99)
          b0 = (tile[h][0][tx][aw] ^ tile[h][1][tx][aw]) >> sh;
          b1 = tile[h][1][tx][aw] >> sh;
        } else {
          b0 = tile[h][0][tx][aw] >> sh;
          b1 = tile[h][1][tx][aw] >> sh;
        }
        v |= ((b0 & 0xFFu) | (b1 & 0xFFu) << 8) << (16 * h);
      }
      IW[(int64_t)s * half + g * nt + (pt % per_group) * 32 + tx] = v;
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ split-K reduction
__device__ __forceinline__ u32 comp4(const uint4& v, int w) { return w == 0 ? v.x : w == 1 ? v.y : w == 2 ? v.z : v.w; }
__device__ __forceinline__ void set4(uint4& v, int w, u32 x) {
  if (w == 0) v.x = x; else if (w == 1) v.y = x; else if (w == 2) v.z = x; else v.w = x;
}

template <int F>
__global__ void __launch_bounds__(256) reduce_splits_kernel(const u32* __restrict__ P, u32* __restrict__ C, int64_t m,
                                                            int64_t mpad, int wc32, int splits) {
  constexpr int R = Traits<F>::R;
  pdl_wait();  // launched with PDL behind the product kernel
  // thread x: word w of rows blockIdx.y, blockIdx.y + gridDim.y, ... (no index division)
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= wc32) return;
  const int64_t plane = mpad * (int64_t)wc32;
  for (int64_t row = blockIdx.y; row < m; row += gridDim.y) {
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

// ------------------------------------------------------------------ slice sums (host pipeline)
// out rows = sum over the n slices (each canonical or raw field values, R planes of `rows` x wc32
// words at base[i] with plane stride pstride[i] words), canonicalized.
template <int F>
__global__ void sum_slices_kernel(const SliceSet s, u32* __restrict__ out, int64_t out_pstride, int64_t rows,
                                  int wc32) {
  constexpr int R = Traits<F>::R;
  const int64_t total = rows * wc32;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    V<F> acc;
#pragma unroll
    for (int d = 0; d < R; ++d) acc.p[d] = s.base[0][d * s.pstride[0] + i];
    for (int j = 1; j < s.n; ++j) {
      V<F> x;
#pragma unroll
      for (int d = 0; d < R; ++d) x.p[d] = s.base[j][d * s.pstride[j] + i];
      vadd<F>(acc, x);
    }
    vcanon<F>(acc);
#pragma unroll
    for (int d = 0; d < R; ++d) out[d * out_pstride + i] = acc.p[d];
  }
}

cudaError_t launch_sum_slices(int field, const SliceSet& s, uint32_t* out, int64_t out_pstride, int64_t rows,
                              int wc32, cudaStream_t st) {
  const int64_t total = rows * wc32;
  const int threads = 256;
  int64_t blocks = (total + threads - 1) / threads;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
#define SG_SS(FF) sum_slices_kernel<FF><<<(unsigned)blocks, threads, 0, st>>>(s, out, out_pstride, rows, wc32)
  SG_FOR_EACH_FIELD_CASE(field, SG_SS)
#undef SG_SS
  return cudaGetLastError();
}

// ------------------------------------------------------------------ stream-K reduction
// C(tile t) = sum of the compact slots of the CTAs whose unit ranges intersect tile t's
// [t nb, (t+1) nb), canonicalized.  One thread per (tile row, word); slots are summed in CTA
// order (the field sums are exact, so any order gives the same bits).
// Tiles with more than 64 contributors (forced stream-K plans with a few units per CTA).
template <int F>
__device__ __noinline__ void reduce_streamk_tile_slow(const u32* __restrict__ P2, u32* __restrict__ C, int64_t m,
                                                      int wc32, int rows_cta, int slabs, int64_t t, int64_t tile0,
                                                      int nb, int64_t U, int G) {
  constexpr int R = Traits<F>::R;
  const int64_t lo = t * nb, hi = lo + nb;
  int64_t c0 = lo * G / U;
  while (c0 > 0 && c0 * U / G > lo) --c0;
  while ((c0 + 1) * U / G <= lo) ++c0;
  const int64_t row0 = ((tile0 + t) / slabs) * rows_cta;
  const int word0 = (int)((tile0 + t) % slabs) * SLAB_WORDS;
  for (int lr = blockIdx.y * blockDim.x + threadIdx.x; lr < rows_cta; lr += gridDim.y * blockDim.x) {
    const int64_t row = row0 + lr;
    if (row >= m) break;
    V<F> acc[4];
    bool first = true;
    for (int64_t c = c0; c < G && c * U / G < hi; ++c) {
      const int64_t u0 = c * U / G;
      if ((c + 1) * U / G == u0) continue;
      const int64_t slot = c * SK_SLOTS + (u0 / nb == t ? 0 : 1);
      V<F> b[4];
#pragma unroll
      for (int d = 0; d < R; ++d) {
        const uint4 x = *reinterpret_cast<const uint4*>(P2 + ((slot * R + d) * rows_cta + lr) * 4);
        b[0].p[d] = x.x; b[1].p[d] = x.y; b[2].p[d] = x.z; b[3].p[d] = x.w;
      }
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        if (first) acc[w] = b[w];
        else vadd<F>(acc[w], b[w]);
      }
      first = false;
    }
#pragma unroll
    for (int w = 0; w < 4; ++w) vcanon<F>(acc[w]);
#pragma unroll
    for (int d = 0; d < R; ++d)
      for (int w = 0; w < 4 && word0 + w < wc32; ++w) C[((int64_t)d * m + row) * wc32 + word0 + w] = acc[w].p[d];
  }
}

template <int F>
__global__ void __launch_bounds__(256) reduce_streamk_kernel(const u32* __restrict__ P2, u32* __restrict__ C, int64_t m,
                                                             int wc32, int rows_cta, int slabs, int64_t tiles,
                                                             int64_t tile0, int nb, int64_t U, int G) {
  constexpr int R = Traits<F>::R;
  pdl_wait();  // launched with PDL behind the product kernel
  // blockIdx.x = tile among the stream-K tiles (tile0 + blockIdx.x of the product: tiles below tile0
  // were written whole by the product kernel); the slots of the CTAs whose unit ranges touch it are listed once per block
  constexpr int MAXS = 64;
  const int64_t t = blockIdx.x;
  __shared__ int slots[MAXS + 1];  // [0] = count (0: the tile was written by the product kernel)
  if (threadIdx.x == 0) {
    const int64_t lo = t * nb, hi = lo + nb;
    int64_t c = lo * G / U;
    while (c > 0 && c * U / G > lo) --c;
    while ((c + 1) * U / G <= lo) ++c;
    int n = 0;
    // a tile inside one CTA's range was written to C by the product kernel itself
    const bool whole = c * U / G <= lo && (c + 1) * U / G >= hi;
    for (; !whole && c < G && c * U / G < hi; ++c) {
      const int64_t u0 = c * U / G;
      if ((c + 1) * U / G == u0) continue;  // an empty range owns no slot
      // the tile holds c's first segment (slot 2c) or its last (slot 2c + 1)
      if (n < MAXS) slots[1 + n] = (int)(c * SK_SLOTS + (u0 / nb == t ? 0 : 1));
      ++n;
    }
    slots[0] = n;
  }
  __syncthreads();
  const int n = slots[0];
  if (n == 0) return;
  if (n > MAXS) {  // very short CTA ranges (forced plans): enumerate per thread
    reduce_streamk_tile_slow<F>(P2, C, m, wc32, rows_cta, slabs, t, tile0, nb, U, G);
    return;
  }
  const int64_t row0 = ((tile0 + t) / slabs) * rows_cta;
  const int word0 = (int)((tile0 + t) % slabs) * SLAB_WORDS;
  for (int lr = blockIdx.y * blockDim.x + threadIdx.x; lr < rows_cta; lr += gridDim.y * blockDim.x) {
    const int64_t row = row0 + lr;
    if (row >= m) break;
    uint4 acc[R];
    // slots two at a time: both loads in flight before the adds (latency, not bandwidth, bound)
    for (int j = 0; j < n; j += 2) {
      const bool two = j + 1 < n;
      const u32* s0 = P2 + ((int64_t)slots[1 + j] * R * rows_cta + lr) * 4;
      const u32* s1 = P2 + ((int64_t)slots[1 + (two ? j + 1 : j)] * R * rows_cta + lr) * 4;
      uint4 x[R], y[R];
#pragma unroll
      for (int d = 0; d < R; ++d) {
        x[d] = *reinterpret_cast<const uint4*>(s0 + (int64_t)d * rows_cta * 4);
        y[d] = *reinterpret_cast<const uint4*>(s1 + (int64_t)d * rows_cta * 4);
      }
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        V<F> a, b;
#pragma unroll
        for (int d = 0; d < R; ++d) {
          a.p[d] = comp4(x[d], w);
          b.p[d] = comp4(y[d], w);
        }
        if (two) vadd<F>(a, b);
        if (j > 0) {
          V<F> c;
#pragma unroll
          for (int d = 0; d < R; ++d) c.p[d] = comp4(acc[d], w);
          vadd<F>(a, c);
        }
#pragma unroll
        for (int d = 0; d < R; ++d) set4(acc[d], w, a.p[d]);
      }
    }
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      V<F> a;
#pragma unroll
      for (int d = 0; d < R; ++d) a.p[d] = comp4(acc[d], w);
      vcanon<F>(a);
#pragma unroll
      for (int d = 0; d < R; ++d) set4(acc[d], w, a.p[d]);
    }
#pragma unroll
    for (int d = 0; d < R; ++d) {
      u32* dst = C + ((int64_t)d * m + row) * wc32 + word0;
      if (word0 + 4 <= wc32 && (wc32 & 3) == 0) {
        *reinterpret_cast<uint4*>(dst) = acc[d];
      } else {
        for (int w = 0; w < 4 && word0 + w < wc32; ++w) dst[w] = comp4(acc[d], w);
      }
    }
  }
}

cudaError_t launch_reduce_streamk(int field, const uint32_t* P2, uint32_t* C, int64_t m, int wc32, int rows_cta,
                                  int slabs, int64_t tiles, int64_t tile0, int nblocks, int64_t units, int ctas,
                                  cudaStream_t st) {
  if (tiles <= 0) return cudaSuccess;
  const dim3 grid((unsigned)tiles, (unsigned)((rows_cta + 255) / 256));
#define SG_RK(FF) return launch_pdl(reduce_streamk_kernel<FF>, grid, dim3(256), 0, st, P2, C, m, wc32, rows_cta, \
                                 slabs, tiles, tile0, nblocks, units, ctas)
  SG_FOR_EACH_FIELD_CASE(field, SG_RK)
#undef SG_RK
  return cudaGetLastError();
}

// ------------------------------------------------------------------ registry
int kernels_f2(KernelInfo** out);
int kernels_f3(KernelInfo** out);
int kernels_gf4(KernelInfo** out);
int kernels_f5(KernelInfo** out);
int kernels_f7(KernelInfo** out);
int kernels_gf8(KernelInfo** out);
int kernels_z4(KernelInfo** out);
int kernels_z8(KernelInfo** out);

static std::vector<KernelInfo*>& registry() {
  static std::vector<KernelInfo*> all = [] {
    std::vector<KernelInfo*> v;
    for (auto fn : {kernels_f2, kernels_f3, kernels_gf4, kernels_f5, kernels_f7, kernels_gf8, kernels_z4, kernels_z8}) {
      KernelInfo* t = nullptr;
      const int n = fn(&t);
      for (int i = 0; i < n; ++i) v.push_back(&t[i]);
    }
    return v;
  }();
  return all;
}

int pdl_mode() {
  static const int mode = [] {
    const char* e = getenv("SG_PDL");
    return e ? atoi(e) : 1;
  }();
  return mode;
}

int m4rm_kernel_count() { return (int)registry().size(); }
KernelInfo* m4rm_kernel_at(int i) { return registry()[i]; }
cudaError_t launch_m4rm(const KernelInfo& ki, const M4rmArgs& a, const CUtensorMap& tmB, dim3 grid,
                        cudaStream_t st) {
  return launch_pdl(ki.fn, grid, dim3(ki.launch_threads), ki.smem_bytes, st, a, tmB);
}
cudaError_t launch_m4rm_streamed(const KernelInfo& ki, const M4rmStreamArgs& a, const CUtensorMap& tmB, dim3 grid,
                                 cudaStream_t st) {
  if (!ki.fn_stream) return cudaErrorInvalidDeviceFunction;
  return launch_pdl(ki.fn_stream, grid, dim3(ki.launch_threads), ki.smem_stream, st, a, tmB);
}

cudaError_t launch_m4rm_fused(const KernelInfo& ki, const M4rmFusedArgs& a, const CUtensorMap& tmB, dim3 grid,
                              cudaStream_t st) {
  if (!ki.fn_fused) return cudaErrorInvalidDeviceFunction;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(ki.launch_threads);
  cfg.dynamicSmemBytes = ki.smem_bytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  // co-residency matters only for the split-K meeting (SG_FUSED_COOP=0, experiments: a plain
  // launch -- the planner keeps the grid within one wave either way)
  static const bool coop = [] {
    const char* e = getenv("SG_FUSED_COOP");
    return !e || atoi(e) != 0;
  }();
  cfg.numAttrs = a.partial && coop ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, ki.fn_fused, a, tmB);
}

cudaError_t launch_transpose_a(int field, int k, const uint32_t* A, uint32_t* AT, int64_t m, int64_t mpad,
                               int wa32, int nwords, int pair_nt, cudaStream_t st) {
  if (k == 8 && pair_nt) {
    const int nblocks = (int)std::min<int64_t>((int64_t)nwords * 2, ((int64_t)wa32 * 32 + 7) / 8);
    dim3 grid((wa32 + 31) / 32, (unsigned)std::min<int64_t>(std::max<int64_t>(1, mpad / 64), 65535), 1);
    // (two-index fields only: F3, GF(4), Z4)
    if (field == F3) index_pairs_kernel<F3><<<grid, dim3(32, 8), 0, st>>>(A, AT, m, mpad, wa32, nblocks, pair_nt);
    else if (field == GF4) index_pairs_kernel<GF4><<<grid, dim3(32, 8), 0, st>>>(A, AT, m, mpad, wa32, nblocks, pair_nt);
    else if (field == Z4) index_pairs_kernel<Z4><<<grid, dim3(32, 8), 0, st>>>(A, AT, m, mpad, wa32, nblocks, pair_nt);
    else return cudaErrorInvalidValue;
    return cudaGetLastError();
  }
  if (k == 8) {
    dim3 grid((wa32 + 31) / 32, (unsigned)std::min<int64_t>((mpad + 31) / 32, 65535), 1);
#define SG_IW(FF) index_words_kernel<FF><<<grid, dim3(32, 8), 0, st>>>(A, AT, m, mpad, wa32, nwords)
    SG_FOR_EACH_FIELD_CASE(field, SG_IW)
#undef SG_IW
    return cudaGetLastError();
  }
  const int R = field == F2 ? 1 : (field == F5 || field == F7 || field == GF8 || field == Z8) ? 3 : 2;
  dim3 grid((wa32 + 31) / 32, (unsigned)std::min<int64_t>((mpad + 31) / 32, 65535), R);
  transpose_a_kernel<<<grid, dim3(32, 8), 0, st>>>(A, AT, m, mpad, wa32, field == F3);
  return cudaGetLastError();
}

cudaError_t preload_aux_kernels(int field) {
  // Load the pre-pass and reduction kernels of a field now: a lazily loaded kernel may wait for
  // the device to drain, which a streamed product (waiting on its upload) must never meet.
  cudaFuncAttributes fa;
#define SG_PL(FF)                                                  \
  cudaFuncGetAttributes(&fa, index_words_kernel<FF>);             \
  cudaFuncGetAttributes(&fa, reduce_streamk_kernel<FF>);          \
  cudaFuncGetAttributes(&fa, reduce_splits_kernel<FF>);           \
  cudaFuncGetAttributes(&fa, sum_slices_kernel<FF>)
  SG_FOR_EACH_FIELD_CASE(field, SG_PL)
#undef SG_PL
  cudaFuncGetAttributes(&fa, transpose_a_kernel);
  if (field == F3) cudaFuncGetAttributes(&fa, index_pairs_kernel<F3>);
  if (field == GF4) cudaFuncGetAttributes(&fa, index_pairs_kernel<GF4>);
  if (field == Z4) cudaFuncGetAttributes(&fa, index_pairs_kernel<Z4>);
  return cudaGetLastError();
}

cudaError_t launch_reduce_splits(int field, const uint32_t* P, uint32_t* C, int64_t m, int64_t mpad,
                                 int wc32, int splits, cudaStream_t st) {
  if (m <= 0 || wc32 <= 0) return cudaSuccess;
  const unsigned gx = (unsigned)((wc32 + 255) / 256);
  const int64_t gy = std::min<int64_t>(std::min<int64_t>(m, 65535), std::max<int64_t>(1, (148 * 16 + gx - 1) / gx));
  const dim3 grid(gx, (unsigned)gy);
#define SG_RS(FF) return launch_pdl(reduce_splits_kernel<FF>, grid, dim3(256), 0, st, P, C, m, mpad, wc32, splits)
  SG_FOR_EACH_FIELD_CASE(field, SG_RS)
#undef SG_RS
  return cudaGetLastError();
}

}  // namespace sg
