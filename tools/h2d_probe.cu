// h2d_probe.cu -- host-to-device copy bandwidth of 6.3 MB pinned buffers by allocation kind
// (cudaHostAlloc default / write-combined / cudaHostRegister of malloc'ed memory), best and median of
// 20 copies: is the per-process H2D variance on the shared host tied to how the buffer is pinned?
// nvcc -O3 -o /tmp/h2d_probe tools/h2d_probe.cu
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>

int main() {
  const size_t bytes = 6291456;
  void* d;
  cudaMalloc(&d, bytes);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[] = {"cudaHostAlloc default", "cudaHostAlloc write-combined", "malloc + cudaHostRegister",
                         "cudaHostAlloc default (2nd)"};
  for (int kind = 0; kind < 4; ++kind) {
    void* h = nullptr;
    if (kind == 0 || kind == 3) cudaHostAlloc(&h, bytes, cudaHostAllocDefault);
    if (kind == 1) cudaHostAlloc(&h, bytes, cudaHostAllocWriteCombined);
    if (kind == 2) {
      h = aligned_alloc(4096, bytes);
      memset(h, 1, bytes);
      cudaHostRegister(h, bytes, cudaHostRegisterDefault);
    }
    memset(h, 3, bytes);
    std::vector<float> t;
    for (int i = 0; i < 25; ++i) {
      cudaEventRecord(e0, s);
      cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (i >= 5) t.push_back(ms);
    }
    std::sort(t.begin(), t.end());
    printf("%-30s H2D best %.1f GB/s median %.1f GB/s\n", names[kind], bytes / t[0] / 1e6, bytes / t[t.size() / 2] / 1e6);
  }
  return 0;
}
