// tmem_probe.cu -- measured TMEM (tcgen05.ld / tcgen05.st 32x32b) throughput on one SM, alone
// and concurrent with conflict-free LDS.128 traffic: does TMEM give the M4RM lookup warps
// accumulator storage without taking shared-memory bandwidth?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tmem_probe tools/tmem_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void tld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tst8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]));
}
__device__ __forceinline__ void twait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void twait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// mode bit 0: TMEM loads, bit 1: TMEM stores, bit 2: LDS.128 (8-replica conflict-free pattern)
__global__ void __launch_bounds__(256, 1) probe(int mode, int iters, unsigned long long* cycles, uint32_t* sink) {
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
  const uint32_t base = taddr_s + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(256 * (warp >> 2));
  uint32_t acc = 0;
  uint32_t r[4][8];
  for (int j = 0; j < 4; ++j)
    for (int k = 0; k < 8; ++k) r[j][k] = lane + j + k;
  unsigned idx = lane * 2654435761u;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const uint32_t col = (uint32_t)((it * 32) & 255);
    if (mode & 1) {
      tld8(base + col, r[0]);
      tld8(base + col + 8, r[1]);
      tld8(base + col + 16, r[2]);
      tld8(base + col + 24, r[3]);
      twait_ld();
    }
    if (mode & 2) {
      tst8(base + col, r[0]);
      tst8(base + col + 8, r[1]);
      tst8(base + col + 16, r[2]);
      tst8(base + col + 24, r[3]);
    }
    if (mode & 4) {
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        idx = idx * 1664525u + 1013904223u;
        const uint4 v = tab[((idx >> 24) << 3) + (lane & 7)];
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
      }
    }
    for (int j = 0; j < 4; ++j) acc += r[j][it & 7];
  }
  if (mode & 2) twait_st();
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(taddr_s));
}

int main() {
  unsigned long long* cyc;
  uint32_t* sink;
  cudaMalloc(&cyc, 148 * 8);
  cudaMalloc(&sink, 148 * 256 * 4);
  const int iters = 4096;
  const char* names[] = {"", "tmem ld", "tmem st", "tmem ld+st", "lds.128", "lds + tmem ld", "lds + tmem st",
                         "lds + tmem ld+st"};
  for (int mode = 1; mode < 8; ++mode) {
    probe<<<148, 256>>>(mode, iters, cyc, sink);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("mode %d: %s\n", mode, cudaGetErrorString(e)); return 1; }
    unsigned long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double c = 0;
    for (int i = 0; i < 148; ++i) c += h[i];
    c /= 148;
    // per SM per iteration: 8 warps x (4 x 1 KB TMEM) each way; 8 warps x 16 x 512 B LDS
    const double tm = 8.0 * 4 * 1024 * iters, ld = 8.0 * 16 * 512 * iters;
    printf("%-18s %10.0f cyc  tmem %6.1f B/clk/SM  lds %6.1f B/clk/SM\n", names[mode], c,
           (mode & 3) ? tm * ((mode & 1) + ((mode >> 1) & 1)) / c : 0.0, (mode & 4) ? ld / c : 0.0);
  }
  return 0;
}
