// tmem_probe.cu -- measured TMEM (tcgen05.ld / tcgen05.st 32x32b.x32) throughput and latency on
// one SM, alone and concurrent with conflict-free LDS.128 traffic: could TMEM hold extra row
// accumulators of the M4RM lookup warps (more rows per shared-memory table) without taking
// shared-memory bandwidth?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tmem_probe tools/tmem_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define R32(a) a[0], a[1], a[2], a[3], a[4], a[5], a[6], a[7], a[8], a[9], a[10], a[11], a[12], a[13], a[14], a[15], \
               a[16], a[17], a[18], a[19], a[20], a[21], a[22], a[23], a[24], a[25], a[26], a[27], a[28], a[29],   \
               a[30], a[31]
__device__ __forceinline__ void tld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tst32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]));
}
__device__ __forceinline__ void twait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void twait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// mode bit 0: TMEM loads (2 x x32 then wait::ld), bit 1: TMEM stores (2 x x32), bit 2: LDS.128
// (8-replica conflict-free pattern, 16 per iteration); `warps` warps per CTA take part
__global__ void __launch_bounds__(512, 1) probe(int mode, int iters, int warps, unsigned long long* cycles,
                                                uint32_t* sink) {
  __shared__ uint32_t taddr_s;
  __shared__ __align__(16) uint4 tab[2048];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) tab[i] = make_uint4(i, i * 3, i * 5, i * 7);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (unsigned)__cvta_generic_to_shared(&taddr_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  // warps w and w + 4, w + 8, ... share lane quarter w % 4; each gets its own 64 columns
  const uint32_t base = taddr_s + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(64 * (warp >> 2));
  uint32_t acc = 0;
  uint32_t r[32], q[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) r[k] = q[k] = lane + k;
  unsigned idx = lane * 2654435761u;
  __syncthreads();
  const unsigned long long t0 = clock64();
  if (warp < warps) {
    for (int it = 0; it < iters; ++it) {
      if (mode & 2) {
        tst32(base, r);
        tst32(base + 32, q);
      }
      if (mode & 1) {
        tld32(base, r);
        tld32(base + 32, q);
      }
      if (mode & 4) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          idx = idx * 1664525u + 1013904223u;
          const uint4 v = tab[((idx >> 24) << 3) + (lane & 7)];
          acc ^= v.x ^ v.y ^ v.z ^ v.w;
        }
      }
      if (mode & 1) {
        twait_ld();
#pragma unroll
        for (int k = 0; k < 32; ++k) { r[k] ^= acc; q[k] += r[k]; }
      }
    }
    if (mode & 2) twait_st();
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  uint32_t s = acc;
#pragma unroll
  for (int k = 0; k < 32; ++k) s ^= r[k] ^ q[k];
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(taddr_s));
}

int main() {
  unsigned long long* cyc;
  uint32_t* sink;
  cudaMalloc(&cyc, 148 * 8);
  cudaMalloc(&sink, 148 * 512 * 4);
  const int iters = 4096;
  const char* names[] = {"", "tmem ld", "tmem st", "tmem st+ld", "lds.128", "lds + tmem ld", "lds + tmem st",
                         "lds + tmem st+ld"};
  for (int warps : {1, 4, 8, 16}) {
    for (int mode = 1; mode < 8; ++mode) {
      probe<<<148, 512>>>(mode, iters, warps, cyc, sink);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("mode %d: %s\n", mode, cudaGetErrorString(e)); return 1; }
      unsigned long long h[148];
      cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
      double c = 0;
      for (int i = 0; i < 148; ++i) c += h[i];
      c /= 148;
      // per warp per iteration: 2 x 32 regs x 32 lanes x 4 B = 8 KB each way; 16 LDS.128 x 512 B
      const double tm = 8192.0 * warps * iters, ld = 16.0 * 512 * warps * iters;
      const int dirs = (mode & 1) + ((mode >> 1) & 1);
      printf("warps %2d %-18s %7.1f cyc/iter  tmem %6.1f B/clk/SM  lds %6.1f B/clk/SM\n", warps, names[mode],
             c / iters, dirs ? tm * dirs / c : 0.0, (mode & 4) ? ld / c : 0.0);
    }
  }
  return 0;
}
