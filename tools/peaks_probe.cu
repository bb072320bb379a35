// Standalone probe of the two M4RM roofline denominators on the box:
// LOP3 issue rate (ALU pipe) and conflict-free LDS.128 bandwidth, per SM per clock.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int CHAINS>
__global__ void lop3_probe(uint32_t* out, int iters, uint32_t seed) {
  uint32_t v[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) v[c] = seed * (threadIdx.x + 1) + c;
  uint32_t a = seed ^ threadIdx.x, b = seed + blockIdx.x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int c = 0; c < CHAINS; ++c)
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(v[c]) : "r"(a), "r"(b));
    }
  }
  uint32_t acc = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc ^= v[c];
  if (acc == 0x12345678u) out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void lds_probe(uint32_t* out, int iters) {
  extern __shared__ uint4 sm[];
  const int n = 4096;  // 64 KiB
  for (int i = threadIdx.x; i < n; i += blockDim.x) sm[i] = make_uint4(i, i * 3, i * 5, i * 7);
  __syncthreads();
  uint4 acc = make_uint4(0, 0, 0, 0);
  unsigned lane = threadIdx.x & 31;
  // 8 lanes per 128-B phase read 8 consecutive uint4: conflict free.
  unsigned off = (lane & 7) + ((threadIdx.x >> 3) & 7) * 8;
  for (int i = 0; i < iters; ++i) {
    const uint4* p = sm + ((i * 64) & (n / 2 - 1)) + off;
#pragma unroll
    for (int u = 0; u < 8; u += 2) {
      uint4 t = p[u * 256], s = p[u * 256 + 128];
      acc.x ^= t.x ^ s.x; acc.y ^= t.y ^ s.y; acc.z ^= t.z ^ s.z; acc.w ^= t.w ^ s.w;
    }
  }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) out[threadIdx.x] = acc.x;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_attr_mhz\": %.0f}\n", p.name, p.multiProcessorCount, clk_khz / 1e3);
  uint32_t* out; CK(cudaMalloc(&out, 1 << 24));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  // LOP3: blocks of 256 threads, 4 per SM -> 32 warps/SM.
  for (int tpb : {256, 512, 1024}) {
    int blocks = sms * (2048 / tpb);
    int iters = 4096;
    lop3_probe<8><<<blocks, tpb>>>(out, 16, 1);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      lop3_probe<8><<<blocks, tpb>>>(out, iters, r + 1);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double ops = (double)blocks * tpb * iters * 16 * 8;
    printf("{\"probe\": \"lop3\", \"tpb\": %d, \"ms\": %.4f, \"Tlop3_per_s\": %.3f, \"lop3_per_clk_per_sm_at_1965\": %.2f}\n",
           tpb, best, ops / best / 1e9, ops / (best * 1e-3) / sms / 1.965e9);
  }
  {
    int tpb = 512, blocks = sms * 3, iters = 4096;
    CK(cudaFuncSetAttribute(lds_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
    lds_probe<<<blocks, tpb, 65536>>>(out, 16);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      lds_probe<<<blocks, tpb, 65536>>>(out, iters);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double bytes = (double)blocks * tpb * iters * 8 * 16;
    printf("{\"probe\": \"lds128\", \"ms\": %.4f, \"TB_per_s\": %.3f, \"B_per_clk_per_sm_at_1965\": %.2f}\n",
           best, bytes / best / 1e9, bytes / (best * 1e-3) / sms / 1.965e9);
  }
  return 0;
}
