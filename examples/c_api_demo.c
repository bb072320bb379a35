/* c_api_demo.c -- the drop-in boundary used from plain C (no Python, no torch): what a non-Python
 * host (a cgo / JNI / N-API binding) would do.  Packs two small F3 matrices, multiplies them with
 * sg_m4rm_host (host buffers, copies included) and with the device entry points
 * (sg_pack -> sg_m4rm -> sg_unpack), and checks both against a schoolbook product mod 3.
 *
 *   gcc -O2 -o examples/c_api_demo examples/c_api_demo.c -Iinclude \
 *       -Lpaper_0901_1413_b200 -lslicegemm_b200 -lcudart -Wl,-rpath,'$ORIGIN/../paper_0901_1413_b200'
 * (build with `make -C examples`; needs a CUDA device to run) */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime.h>

#include "slicegemm_b200.h"

#define M 70
#define L 130
#define N 65

static void pack_f3_host(const uint8_t* d, int64_t rows, int64_t cols, uint64_t* planes) {
  /* F3 patterns: 0 = 00, 1 = 01, 2 = 11 (plane 0 = unit, plane 1 = sign) */
  const int64_t w = (cols + 63) / 64;
  memset(planes, 0, sizeof(uint64_t) * 2 * rows * w);
  for (int64_t i = 0; i < rows; ++i)
    for (int64_t j = 0; j < cols; ++j) {
      const uint8_t v = d[i * cols + j];
      if (v) planes[i * w + (j >> 6)] |= 1ull << (j & 63);
      if (v == 2) planes[(rows + i) * w + (j >> 6)] |= 1ull << (j & 63);
    }
}

static int check(const char* what, int rc) {
  if (rc != SG_OK) {
    fprintf(stderr, "%s failed (%d): %s\n", what, rc, sg_last_error());
    exit(1);
  }
  return rc;
}

int main(void) {
  static uint8_t a[M * L], b[L * N], want[M * N], got[M * N];
  uint32_t s = 12345u;
  for (int i = 0; i < M * L; ++i) a[i] = (uint8_t)((s = s * 1103515245u + 12345u) >> 16) % 3;
  for (int i = 0; i < L * N; ++i) b[i] = (uint8_t)((s = s * 1103515245u + 12345u) >> 16) % 3;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      int acc = 0;
      for (int t = 0; t < L; ++t) acc += a[i * L + t] * b[t * N + j];
      want[i * N + j] = (uint8_t)(acc % 3);
    }
  const int64_t wa = (L + 63) / 64, wc = (N + 63) / 64;

  /* 1. host buffers: sg_m4rm_host */
  uint64_t* ap = malloc(sizeof(uint64_t) * 2 * M * wa);
  uint64_t* bp = malloc(sizeof(uint64_t) * 2 * L * wc);
  uint64_t* cp = calloc(2 * M * wc, sizeof(uint64_t));
  pack_f3_host(a, M, L, ap);
  pack_f3_host(b, L, N, bp);
  check("sg_m4rm_host", sg_m4rm_host(SG_F3, ap, bp, cp, M, L, N, 8, 0));
  int bad = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      const int u = (int)((cp[i * wc + (j >> 6)] >> (j & 63)) & 1);
      const int sg = (int)((cp[(M + i) * wc + (j >> 6)] >> (j & 63)) & 1);
      bad += (u + sg) != want[i * N + j];
    }

  /* 2. device buffers: sg_pack -> sg_m4rm -> sg_unpack on the default stream */
  uint8_t *da, *db, *dd;
  uint64_t *pa, *pb, *pc;
  cudaMalloc((void**)&da, M * L);
  cudaMalloc((void**)&db, L * N);
  cudaMalloc((void**)&dd, M * N);
  cudaMalloc((void**)&pa, sizeof(uint64_t) * 2 * M * wa);
  cudaMalloc((void**)&pb, sizeof(uint64_t) * 2 * L * wc);
  cudaMalloc((void**)&pc, sizeof(uint64_t) * 2 * M * wc);
  cudaMemcpy(da, a, M * L, cudaMemcpyHostToDevice);
  cudaMemcpy(db, b, L * N, cudaMemcpyHostToDevice);
  check("sg_pack A", sg_pack(SG_F3, da, M, L, L, pa, NULL));
  check("sg_pack B", sg_pack(SG_F3, db, L, N, N, pb, NULL));
  check("sg_m4rm", sg_m4rm(SG_F3, pa, pb, pc, M, L, N, 8, NULL, 0, NULL));
  check("sg_unpack", sg_unpack(SG_F3, pc, M, N, dd, N, NULL));
  cudaMemcpy(got, dd, M * N, cudaMemcpyDeviceToHost);
  for (int i = 0; i < M * N; ++i) bad += got[i] != want[i];
  printf("c_api_demo: abi %d, F3 %dx%dx%d, %s\n", sg_abi_version(), M, L, N, bad ? "MISMATCH" : "bit-exact");
  return bad ? 1 : 0;
}
