// Probe: throughput of the M4RM lookup pattern (LDS.128 of random table entries, 8 replicas,
// lane j reads replica j&7) vs warps per SM and loads in flight per warp.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int INFLIGHT>
__global__ void probe(uint32_t* out, int iters, int tabkb) {
  extern __shared__ uint4 sm[];
  const int n = tabkb * 64;  // uint4 count
  for (int i = threadIdx.x; i < n; i += blockDim.x) sm[i] = make_uint4(i, i * 3, i * 5, i * 7);
  __syncthreads();
  uint32_t x = threadIdx.x * 2654435761u + blockIdx.x;
  uint4 acc = make_uint4(0, 0, 0, 0);
  const int rep = threadIdx.x & 7;
  const int entries = n / 8;
  for (int i = 0; i < iters; ++i) {
    uint4 v[INFLIGHT];
#pragma unroll
    for (int u = 0; u < INFLIGHT; ++u) {
      x = x * 1664525u + 1013904223u;
      const int g = (x >> 8) & (entries - 1);
      v[u] = sm[g * 8 + rep];
    }
#pragma unroll
    for (int u = 0; u < INFLIGHT; ++u) { acc.x ^= v[u].x; acc.y ^= v[u].y; acc.z ^= v[u].z; acc.w ^= v[u].w; }
  }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345u) out[threadIdx.x] = 1;
}

template <int IF>
void run(int warps_per_sm, int sms, uint32_t* out) {
  int tpb = 256, per_sm = warps_per_sm / 8;
  int tabkb = 64;
  cudaFuncSetAttribute(probe<IF>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  int iters = 4096 / IF;
  probe<IF><<<sms * per_sm, tpb, tabkb * 1024>>>(out, 16, tabkb);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe<IF><<<sms * per_sm, tpb, tabkb * 1024>>>(out, iters, tabkb);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double bytes = (double)sms * per_sm * tpb * iters * IF * 16;
  printf("{\"warps_per_sm\": %d, \"inflight\": %d, \"B_per_clk_per_sm_at_1965\": %.1f, \"err\": \"%s\"}\n",
         warps_per_sm, IF, bytes / (ms * 1e-3) / sms / 1.965e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* out; cudaMalloc(&out, 1 << 16);
  for (int w : {8, 16}) { run<1>(w, sms, out); run<2>(w, sms, out); run<4>(w, sms, out); run<8>(w, sms, out); run<16>(w, sms, out); }
  return 0;
}
