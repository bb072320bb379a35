// sg_peaks.cu -- live microbenchmarks of the two denominators of the M4RM roofline:
// the LOP3 issue rate of the ALU pipe and conflict-free LDS.128 bandwidth, per SM per clock.
// Cycle counts come from clock64() inside the probe and wall time from %globaltimer, so
// the per-clock rates do not assume a clock frequency; the effective SM MHz is reported too.
#include <cstdint>
#include <cuda_runtime.h>

#include "sg_internal.h"

namespace sg {

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Whole-launch span from %globaltimer (min start, max end over CTAs) and the SM clock from
// CTA 0's clock64 / globaltimer ratio: rate = total work / (span x clock) / SMs.
__device__ void record_span(unsigned long long* st, long long c0, long long c1, uint64_t t0, uint64_t t1) {
  atomicMin(&st[0], (unsigned long long)t0);
  atomicMax(&st[1], (unsigned long long)t1);
  if (blockIdx.x == 0) {
    st[2] = (unsigned long long)(c1 - c0);
    st[3] = (unsigned long long)(t1 - t0);
  }
}

__global__ void lop3_probe_kernel(uint32_t* out, unsigned long long* stats, int iters, uint32_t seed) {
  uint32_t v[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) v[c] = seed * (threadIdx.x + 1) + c;
  const uint32_t a = seed ^ threadIdx.x, b = seed + blockIdx.x;
  __syncthreads();
  const long long c0 = clock64();
  const uint64_t t0 = gtimer();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int c = 0; c < 8; ++c) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(v[c]) : "r"(a), "r"(b));
  }
  __syncthreads();
  const long long c1 = clock64();
  const uint64_t t1 = gtimer();
  uint32_t acc = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) acc ^= v[c];
  if (acc == 0x12345678u) out[threadIdx.x] = acc;
  if (threadIdx.x == 0) record_span(stats, c0, c1, t0, t1);
}

__global__ void lds_probe_kernel(uint32_t* out, unsigned long long* stats, int iters) {
  extern __shared__ uint4 sm[];
  const int n = 4096;  // 64 KiB
  for (int i = threadIdx.x; i < n; i += blockDim.x) sm[i] = make_uint4(i, i * 3, i * 5, i * 7);
  __syncthreads();
  uint4 acc = make_uint4(0, 0, 0, 0);
  const unsigned lane = threadIdx.x & 31;
  const unsigned off = (lane & 7) + ((threadIdx.x >> 3) & 7) * 8;  // 8 lanes = one 128-B phase
  const long long c0 = clock64();
  const uint64_t t0 = gtimer();
  for (int i = 0; i < iters; ++i) {
    const uint4* p = sm + ((i * 64) & (n / 2 - 1)) + off;
#pragma unroll
    for (int u = 0; u < 8; u += 2) {
      const uint4 t = p[u * 256], s = p[u * 256 + 128];
      acc.x ^= t.x ^ s.x; acc.y ^= t.y ^ s.y; acc.z ^= t.z ^ s.z; acc.w ^= t.w ^ s.w;
    }
  }
  __syncthreads();
  const long long c1 = clock64();
  const uint64_t t1 = gtimer();
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) out[threadIdx.x] = acc.x;
  if (threadIdx.x == 0) record_span(stats, c0, c1, t0, t1);
}

static int run_probe(bool lop3, int sms, uint32_t* out, unsigned long long* stats, int rep, double* rate,
                     double* mhz) {
  const unsigned long long init[4] = {~0ull, 0ull, 0ull, 0ull};
  if (cudaMemcpy(stats, init, sizeof init, cudaMemcpyHostToDevice) != cudaSuccess) return -1;
  double work = 0;
  if (lop3) {
    const int tpb = 256, per_sm = 8, iters = 2048;
    lop3_probe_kernel<<<sms * per_sm, tpb>>>(out, stats, iters, rep + 1);
    work = (double)sms * per_sm * tpb * iters * 16 * 8;
  } else {
    const int tpb = 512, per_sm = 3, iters = 2048;
    lds_probe_kernel<<<sms * per_sm, tpb, 65536>>>(out, stats, iters);
    work = (double)sms * per_sm * tpb * iters * 8 * 16;
  }
  unsigned long long h[4];
  if (cudaMemcpy(h, stats, sizeof h, cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
  const double span_ns = (double)(h[1] - h[0]);
  const double f_ghz = h[3] ? (double)h[2] / (double)h[3] : 0.0;
  if (span_ns <= 0 || f_ghz <= 0) return -1;
  *rate = work / (span_ns * f_ghz) / sms;
  *mhz = f_ghz * 1e3;
  return 0;
}

int probe_peaks(int device, double* lop3_per_clk_sm, double* lds_bytes_per_clk_sm, double* sm_mhz) {
  if (cudaSetDevice(device) != cudaSuccess) return -1;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  uint32_t* out = nullptr;
  unsigned long long* stats = nullptr;
  if (cudaMalloc(&out, 1 << 16) != cudaSuccess) return -1;
  if (cudaMalloc(&stats, 32) != cudaSuccess) { cudaFree(out); return -1; }
  cudaFuncSetAttribute(lds_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  double best_lop3 = 0, best_lds = 0, mhz = 0;
  for (int rep = 0; rep < 3; ++rep) {
    double r, f;
    if (run_probe(true, sms, out, stats, rep, &r, &f) == 0 && r > best_lop3) { best_lop3 = r; mhz = f; }
    if (run_probe(false, sms, out, stats, rep, &r, &f) == 0 && r > best_lds) best_lds = r;
  }
  cudaFree(out);
  cudaFree(stats);
  if (cudaGetLastError() != cudaSuccess || best_lop3 <= 0 || best_lds <= 0) return -1;
  *lop3_per_clk_sm = best_lop3;
  *lds_bytes_per_clk_sm = best_lds;
  *sm_mhz = mhz;
  return 0;
}

}  // namespace sg
