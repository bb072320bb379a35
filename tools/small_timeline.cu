// small_timeline.cu -- per-CTA phase timeline of the fused small-product kernel (F3 1024^3 by
// default): globaltimer stamps at kernel entry (0), first table ready (1), end of the k loop
// (2), partial stored (3), splits met (4), reduction done (5).  Built with SG_TIMELINE.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DSG_TIMELINE -lcuda -o /tmp/small_timeline tools/small_timeline.cu
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <vector>

#include "../paper_0901_1413_b200/csrc/sg_m4rm_kernel.cuh"

using namespace sg;

template <int RT, int SC>
void run(int splits, int coop = 1) {
  const int64_t m = 1024, l = 1024, n = 1024;
  const int R = 2, wa32 = (int)(2 * ((l + 63) / 64)), wc32 = (int)(2 * ((n + 63) / 64));
  const int rows = RT * 256, rgroups = (int)((m + rows - 1) / rows), slabs = (wc32 + 3) / 4;
  const int nblocks = (int)(l / 8), bps = (nblocks + splits - 1) / splits;
  std::vector<uint32_t> ha((size_t)R * m * wa32), hb((size_t)R * l * wc32);
  uint32_t x = 1;
  for (auto& v : ha) v = (x = x * 1664525u + 1013904223u);
  for (auto& v : hb) v = (x = x * 1664525u + 1013904223u);
  for (size_t i = 0; i < ha.size() / 2; ++i) ha[i] |= ha[ha.size() / 2 + i];  // legal F3: sign => unit
  for (size_t i = 0; i < hb.size() / 2; ++i) hb[i] |= hb[hb.size() / 2 + i];
  uint32_t *A, *B, *C, *Pp;
  unsigned* cnt;
  cudaMalloc(&A, ha.size() * 4);
  cudaMalloc(&B, hb.size() * 4);
  cudaMalloc(&C, (size_t)R * m * wc32 * 4);
  cudaMalloc(&Pp, (size_t)splits * R * rgroups * rows * wc32 * 4);
  cudaMalloc(&cnt, 8192 * 4);
  cudaMemset(cnt, 0, 8192 * 4);
  cudaMemcpy(A, ha.data(), ha.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hb.data(), hb.size() * 4, cudaMemcpyHostToDevice);
  M4rmFusedArgs a;
  memset(&a, 0, sizeof(a));
  a.B = B; a.A = A; a.C = C; a.P2 = Pp; a.Cout = C; a.m = m; a.l = l; a.mpad = (int64_t)rgroups * rows;
  a.wa32 = wa32; a.wc32 = wc32; a.nblocks = nblocks; a.bps = bps; a.partial = 1; a.cnt = cnt;
  a.ntiles = slabs * rgroups;
  auto fn = m4rm_kernel<F3, 8, RT, SC, 256, 0, false, true>;
  const int smem = smem_bytes_for<F3, 8, RT, SC, 256, true>();
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  CUtensorMap tm;
  memset(&tm, 0, sizeof(tm));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(slabs, rgroups, splits);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = coop;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e9;
  static unsigned long long tl[8192][8];
  const int nct = slabs * rgroups * splits;
  for (int rep = 0; rep < 6; ++rep) {
    cudaEventRecord(e0);
    cudaError_t err = cudaLaunchKernelEx(&cfg, fn, a, tm);
    cudaEventRecord(e1);
    if (err != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
      printf("launch failed: %s\n", cudaGetErrorString(cudaGetLastError()));
      return;
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best) {
      best = ms;
      cudaMemcpyFromSymbol(tl, g_tl, sizeof(unsigned long long) * 8 * nct);
    }
  }
  unsigned long long t0 = ~0ull;
  for (int c = 0; c < nct; ++c) t0 = std::min(t0, tl[c][0]);
  printf("RT %d sched %d splits %d coop %d: %d CTAs, %d blocks each, event %.1f us\n", RT, SC, splits, coop, nct, bps,
         best * 1e3);
  const char* names[] = {"start", "table0", "loop end", "partial", "met", "done"};
  for (int i = 0; i < 6; ++i) {
    std::vector<double> v;
    for (int c = 0; c < nct; ++c) v.push_back((tl[c][i] - t0) * 1e-3);
    std::sort(v.begin(), v.end());
    printf("  %-9s min %6.2f  med %6.2f  max %6.2f us\n", names[i], v.front(), v[v.size() / 2], v.back());
  }
  cudaFree(A); cudaFree(B); cudaFree(C); cudaFree(Pp); cudaFree(cnt);
}

__global__ void empty_kernel() {}
__global__ void flush_kernel(uint4* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_uint4(i, 0, 0, 0);
}

// event-timed launch overheads: an empty kernel, and an empty kernel after a 256 MB flush
void overheads() {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  uint4* f;
  cudaMalloc(&f, 256 << 20);
  for (int flush = 0; flush < 2; ++flush) {
    float best = 1e9;
    for (int i = 0; i < 10; ++i) {
      if (flush) flush_kernel<<<148 * 4, 256>>>(f, (256 << 20) / 16);
      cudaEventRecord(e0);
      empty_kernel<<<1, 32>>>();
      cudaEventRecord(e1);
      cudaDeviceSynchronize();
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = std::min(best, ms);
    }
    printf("empty kernel%s: event %.1f us\n", flush ? " after flush" : "", best * 1e3);
  }
  cudaFree(f);
}

int main() {
  overheads();
  run<4, 0>(16);
  run<4, 0>(16, 0);
  run<4, 1>(16);
  run<4, 0>(18);
  run<2, 0>(9);
  run<2, 0>(9, 0);
  run<4, 0>(1);
  return 0;
}
