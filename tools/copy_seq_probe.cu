// copy_seq_probe.cu -- the upload sequences of the host pipeline on their own (F5 4096^3 sizes:
// A, B = 3 planes x 4096 rows x 512 B), one stream: (1) streamed order with 2-D copies (A's row
// piece 0, B in 6 geometric chunks, A's piece 1), (2) the same bytes as per-plane contiguous
// copies, (3) B-first order (B whole, A's pieces per plane).  Times each sequence.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/copy_seq_probe tools/copy_seq_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  const size_t R = 3, rows = 4096, rowb = 512, plane = rows * rowb;  // bytes
  char *hA, *hB, *dA, *dB;
  cudaMallocHost(&hA, R * plane);
  cudaMallocHost(&hB, R * plane);
  cudaMalloc(&dA, R * plane);
  cudaMalloc(&dB, R * plane);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const size_t half = plane / 2;                 // A's row piece per plane (2048 rows)
  const size_t g0 = 4 * 32 * rowb;               // B chunk j: [g0 (2^j - 1), g0 (2^(j+1) - 1)) per plane
  auto chunk_lo = [&](int j) { size_t x = g0 * ((1ull << j) - 1); return x < plane ? x : plane; };
  for (int rep = 0; rep < 6; ++rep) {
    float t[3];
    for (int v = 0; v < 3; ++v) {
      cudaEventRecord(e0, s);
      if (v == 0) {  // 2-D: A piece 0, B chunks, A piece 1
        cudaMemcpy2DAsync(dA, half, hA, plane, half, R, cudaMemcpyHostToDevice, s);
        for (int j = 0; chunk_lo(j) < plane; ++j)
          cudaMemcpy2DAsync(dB + chunk_lo(j), plane, hB + chunk_lo(j), plane, chunk_lo(j + 1) - chunk_lo(j), R,
                            cudaMemcpyHostToDevice, s);
        cudaMemcpy2DAsync(dA + R * half, half, hA + half, plane, half, R, cudaMemcpyHostToDevice, s);
      } else if (v == 1) {  // the same bytes, per plane contiguous
        for (size_t p = 0; p < R; ++p) cudaMemcpyAsync(dA + p * half, hA + p * plane, half, cudaMemcpyHostToDevice, s);
        for (int j = 0; chunk_lo(j) < plane; ++j)
          for (size_t p = 0; p < R; ++p)
            cudaMemcpyAsync(dB + p * plane + chunk_lo(j), hB + p * plane + chunk_lo(j), chunk_lo(j + 1) - chunk_lo(j),
                            cudaMemcpyHostToDevice, s);
        for (size_t p = 0; p < R; ++p)
          cudaMemcpyAsync(dA + R * half + p * half, hA + p * plane + half, half, cudaMemcpyHostToDevice, s);
      } else {  // B first, whole; then A's pieces per plane
        cudaMemcpyAsync(dB, hB, R * plane, cudaMemcpyHostToDevice, s);
        for (int r = 0; r < 2; ++r)
          for (size_t p = 0; p < R; ++p)
            cudaMemcpyAsync(dA + (r * R + p) * half, hA + p * plane + r * half, half, cudaMemcpyHostToDevice, s);
      }
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&t[v], e0, e1);
    }
    printf("12.6 MB up: 2-D streamed order %.3f ms | per-plane streamed order %.3f ms | B first %.3f ms\n", t[0], t[1],
           t[2]);
  }
  return 0;
}
