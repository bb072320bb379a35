// dma_probe.cu -- host<->device copy experiments for the streamed host pipeline (sg_m4rm_host):
//  * pinned H2D / D2H throughput of cudaMemcpy2DAsync by row width (column chunks of A are 2-D),
//  * H2D and D2H at once,
//  * stream memory operations: cuStreamWriteValue32 seen by a spinning kernel, cuStreamWaitValue32
//    released by a kernel's atomic (latency of each),
//  * zero-copy reads of pinned host memory by a kernel on a few SMs.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/dma_probe tools/dma_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("ERR %s line %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void spin_until(const volatile unsigned* flag, unsigned v, unsigned long long* t_seen) {
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (true) {
    unsigned x;
    asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(x) : "l"(flag));
    if ((int)(x - v) >= 0) break;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 2000000000ull) { *t_seen = 0; return; }
  }
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *t_seen = t;
}
__global__ void stamp(unsigned long long* t) {
  unsigned long long x;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(x));
  *t = x;
}
__global__ void bump(unsigned* ctr, unsigned long long* t) {
  unsigned long long x;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(x));
  *t = x;
  __threadfence();
  atomicAdd(ctr, 1u);
}
// zero-copy: each thread reads uint4 from host memory, sums (to keep the loads)
__global__ void zc_read(const uint4* __restrict__ h, size_t n16, unsigned* out) {
  unsigned acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = h[i];
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) *out = acc;
}

int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  CK(cudaSetDevice(0));
  const size_t total = 12u << 20;
  void *h, *d, *h2, *d2;
  CK(cudaMallocHost(&h, total));
  CK(cudaMallocHost(&h2, total));
  CK(cudaMalloc(&d, total));
  CK(cudaMalloc(&d2, total));
  cudaStream_t s1, s2;
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  cudaEvent_t e0, e1, e2, e3;
  cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&e2); cudaEventCreate(&e3);
  // 2-D copies: a column chunk of `width` bytes out of rows of pitch 8 * width (like 1/8 of A)
  for (int dir = 0; dir < 2; ++dir) {
    for (size_t width : {64, 128, 256, 512, 1024, 2048, 8192, 0}) {
      const size_t pitch = width ? width * 8 : total;
      const size_t rows = width ? total / pitch : 1;
      const size_t w = width ? width : total;
      float best = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0, s1);
        if (dir == 0) CK(cudaMemcpy2DAsync(d, w, h, pitch, w, rows, cudaMemcpyHostToDevice, s1));
        else CK(cudaMemcpy2DAsync(h, pitch, d, w, w, rows, cudaMemcpyDeviceToHost, s1));
        cudaEventRecord(e1, s1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      printf("%s width %6zu B x %7zu rows (%.2f MB): %.3f ms  %.1f GB/s\n", dir ? "D2H" : "H2D", w, rows,
             w * rows / 1e6, best, w * rows / best / 1e6);
    }
  }
  // the host pipeline's shapes: A's row piece (3 planes x 1 MB, pitch 2 MB) and a B chunk
  // (3 planes x 256 KB, pitch 2 MB), against the same bytes contiguous
  for (int rep2 = 0; rep2 < 2; ++rep2) {
    for (size_t width : {(size_t)1 << 20, (size_t)256 << 10}) {
      float b2d = 1e9, b1d = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0, s1);
        CK(cudaMemcpy2DAsync(d, width, h, 2 * width, width, 3, cudaMemcpyHostToDevice, s1));
        cudaEventRecord(e1, s1);
        CK(cudaMemcpyAsync(d, h, 3 * width, cudaMemcpyHostToDevice, s1));
        cudaEventRecord(e2, s1);
        cudaEventSynchronize(e2);
        float ms, ms1; cudaEventElapsedTime(&ms, e0, e1); cudaEventElapsedTime(&ms1, e1, e2);
        if (ms < b2d) b2d = ms;
        if (ms1 < b1d) b1d = ms1;
      }
      printf("pipeline shape: 3 x %zu B (pitch %zu): 2-D %.4f ms %.1f GB/s | contiguous %.4f ms %.1f GB/s\n", width,
             2 * width, b2d, 3 * width / b2d / 1e6, b1d, 3 * width / b1d / 1e6);
    }
  }
  // contiguous copies of various sizes (latency + bandwidth)
  for (size_t sz : {(size_t)64 << 10, (size_t)256 << 10, (size_t)1 << 20, (size_t)3 << 20, (size_t)12 << 20}) {
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0, s1);
      CK(cudaMemcpyAsync(d, h, sz, cudaMemcpyHostToDevice, s1));
      cudaEventRecord(e1, s1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    printf("H2D contiguous %8zu B: %.4f ms %.1f GB/s\n", sz, best, sz / best / 1e6);
  }
  // 8 back-to-back 1.5 MB H2D copies (one per chunk) vs one 12 MB
  {
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0, s1);
      for (int j = 0; j < 8; ++j)
        CK(cudaMemcpyAsync((char*)d + j * (total / 8), (char*)h + j * (total / 8), total / 8, cudaMemcpyHostToDevice, s1));
      cudaEventRecord(e1, s1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    printf("H2D 8 x 1.5 MB back to back: %.4f ms %.1f GB/s\n", best, total / best / 1e6);
  }
  // simultaneous H2D (s1) and D2H (s2)
  {
    float best = 1e9, b2 = 0;
    for (int rep = 0; rep < 5; ++rep) {
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0, s1);
      cudaStreamWaitEvent(s2, e0, 0);
      CK(cudaMemcpyAsync(d, h, total, cudaMemcpyHostToDevice, s1));
      CK(cudaMemcpyAsync(h2, d2, total / 2, cudaMemcpyDeviceToHost, s2));
      cudaEventRecord(e1, s1);
      cudaEventRecord(e2, s2);
      cudaEventSynchronize(e1); cudaEventSynchronize(e2);
      float ms, ms2; cudaEventElapsedTime(&ms, e0, e1); cudaEventElapsedTime(&ms2, e0, e2);
      if (ms < best) { best = ms; b2 = ms2; }
    }
    printf("concurrent: H2D 12 MB %.3f ms (%.1f GB/s) with D2H 6 MB %.3f ms (%.1f GB/s)\n", best, total / best / 1e6, b2,
           total / 2 / b2 / 1e6);
  }
  // stream memory operations
  {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    PFN_cuStreamWriteValue32_v11070 wv = nullptr;
    PFN_cuStreamWaitValue32_v11070 wt = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &fn, cudaEnableDefault, &q) == cudaSuccess && q == cudaDriverEntryPointSuccess)
      wv = (PFN_cuStreamWriteValue32_v11070)fn;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &fn, cudaEnableDefault, &q) == cudaSuccess && q == cudaDriverEntryPointSuccess)
      wt = (PFN_cuStreamWaitValue32_v11070)fn;
    int a92 = -1, a122 = -1;
    cudaDeviceGetAttribute(&a92, (cudaDeviceAttr)92, 0);
    cudaDeviceGetAttribute(&a122, (cudaDeviceAttr)122, 0);
    printf("stream mem ops: write %p wait %p attr92 %d attr122 %d\n", (void*)wv, (void*)wt, a92, a122);
    unsigned* flag;
    unsigned long long* ts;
    CK(cudaMalloc(&flag, 64));
    CK(cudaMalloc(&ts, 64));
    CK(cudaMemset(flag, 0, 64));
    CK(cudaDeviceSynchronize());
    if (wv && wt) {
      for (unsigned ep = 1; ep <= 3; ++ep) {
        // kernel on s2 spins on the flag; s1: 1.5 MB H2D copy then write the flag; stamp on s1
        spin_until<<<1, 1, 0, s2>>>(flag, ep, ts);
        CK(cudaMemcpyAsync(d, h, total / 8, cudaMemcpyHostToDevice, s1));
        stamp<<<1, 1, 0, s1>>>(ts + 1);  // time just before the write (copy done)
        CUresult r = wv((CUstream)s1, (CUdeviceptr)flag, ep, 0);
        CK(cudaDeviceSynchronize());
        unsigned long long t[2];
        cudaMemcpy(t, ts, 16, cudaMemcpyDeviceToHost);
        printf("write value %u: rc %d, spinning kernel saw it %.2f us after the stamp\n", ep, (int)r,
               t[0] ? (double)(t[0] - t[1]) / 1e3 : -1.0);
      }
      for (unsigned ep = 1; ep <= 3; ++ep) {
        // s2: wait value (counter >= ep) then stamp; s1: bump the counter after a delay
        CUresult r = wt((CUstream)s2, (CUdeviceptr)(flag + 4), ep, CU_STREAM_WAIT_VALUE_GEQ);
        stamp<<<1, 1, 0, s2>>>(ts + 2);
        CK(cudaMemcpyAsync(d, h, total / 8, cudaMemcpyHostToDevice, s1));
        bump<<<1, 1, 0, s1>>>(flag + 4, ts + 3);
        CK(cudaDeviceSynchronize());
        unsigned long long t[4];
        cudaMemcpy(t, ts, 32, cudaMemcpyDeviceToHost);
        printf("wait value %u: rc %d, waiter ran %.2f us after the bump\n", ep, (int)r, (double)(t[2] - t[3]) / 1e3);
      }
    }
  }
  // zero-copy reads from pinned host memory on a few SMs
  {
    unsigned* out;
    CK(cudaMalloc(&out, 4));
    void* hd;
    CK(cudaHostGetDevicePointer(&hd, h, 0));
    for (int blocks : {2, 4, 8, 16, 32, 148}) {
      for (int thr : {256, 1024}) {
        float best = 1e9;
        for (int rep = 0; rep < 3; ++rep) {
          cudaEventRecord(e0, s1);
          zc_read<<<blocks, thr, 0, s1>>>((const uint4*)hd, total / 16, out);
          cudaEventRecord(e1, s1);
          CK(cudaEventSynchronize(e1));
          float ms; cudaEventElapsedTime(&ms, e0, e1);
          if (ms < best) best = ms;
        }
        printf("zero-copy read %d CTAs x %d threads: %.3f ms %.1f GB/s\n", blocks, thr, best, total / best / 1e6);
      }
    }
  }
  printf("done\n");
  return 0;
}
