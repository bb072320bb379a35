// zc_probe.cu -- small host<->device transfers: copy engine (cudaMemcpyAsync from/to pinned
// memory) against SM-driven zero-copy (a kernel reading / writing mapped pinned host memory),
// for the small-product end-to-end path (F3 1024^3: 2 x 256 KB up, 256 KB down).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/zc_probe tools/zc_probe.cu
#include <chrono>
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void copy_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, int64_t n16) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}
__global__ void copy2_kernel(const uint4* __restrict__ s0, uint4* __restrict__ d0, const uint4* __restrict__ s1,
                             uint4* __restrict__ d1, int64_t n16) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 2 * n16; i += (int64_t)gridDim.x * blockDim.x)
    if (i < n16) d0[i] = s0[i]; else d1[i - n16] = s1[i - n16];
}

static double now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
  for (int64_t bytes : {64 << 10, 256 << 10, 1 << 20, 4 << 20}) {
    const int64_t n16 = bytes / 16;
    uint4 *hA, *hB, *hC, *dA, *dB, *dC;
    cudaHostAlloc(&hA, bytes, cudaHostAllocMapped);
    cudaHostAlloc(&hB, bytes, cudaHostAllocMapped);
    cudaHostAlloc(&hC, bytes, cudaHostAllocMapped);
    cudaMalloc(&dA, bytes);
    cudaMalloc(&dB, bytes);
    cudaMalloc(&dC, bytes);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    const int reps = 50;
    auto run = [&](const char* name, auto&& body) {
      for (int i = 0; i < 5; ++i) body();
      cudaStreamSynchronize(s);
      double best = 1e30, tot = 0;
      for (int i = 0; i < reps; ++i) {
        const double t0 = now_us();
        body();
        cudaStreamSynchronize(s);
        const double t = now_us() - t0;
        tot += t;
        if (t < best) best = t;
      }
      printf("%8lld B  %-44s best %7.1f us  mean %7.1f us\n", (long long)bytes, name, best, tot / reps);
    };
    const int grid = 148 * 4;
    run("CE: A up, B up, C down (3 memcpyAsync)", [&] {
      cudaMemcpyAsync(dA, hA, bytes, cudaMemcpyHostToDevice, s);
      cudaMemcpyAsync(dB, hB, bytes, cudaMemcpyHostToDevice, s);
      cudaMemcpyAsync(hC, dC, bytes, cudaMemcpyDeviceToHost, s);
    });
    run("CE: A up only", [&] { cudaMemcpyAsync(dA, hA, bytes, cudaMemcpyHostToDevice, s); });
    run("CE: C down only", [&] { cudaMemcpyAsync(hC, dC, bytes, cudaMemcpyDeviceToHost, s); });
    run("SM: A+B up (1 kernel), C down (1 kernel)", [&] {
      copy2_kernel<<<grid, 256, 0, s>>>(hA, dA, hB, dB, n16);
      copy_kernel<<<grid, 256, 0, s>>>(dC, hC, n16);
    });
    run("SM: A+B up (1 kernel)", [&] { copy2_kernel<<<grid, 256, 0, s>>>(hA, dA, hB, dB, n16); });
    run("SM: C down (1 kernel)", [&] { copy_kernel<<<grid, 256, 0, s>>>(dC, hC, n16); });
    run("empty kernel", [&] { copy_kernel<<<1, 32, 0, s>>>(dC, dA, 0); });
    cudaFreeHost(hA); cudaFreeHost(hB); cudaFreeHost(hC);
    cudaFree(dA); cudaFree(dB); cudaFree(dC);
    cudaStreamDestroy(s);
  }
  return 0;
}
