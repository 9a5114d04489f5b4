/* c_abi_demo.c -- using libsquares.so from plain C through include/squares.h (no Python, no
 * torch): key utility, a key-by-value squares32 fill, a device-keys f32 fill and the fused
 * statistics, all on one CUDA stream.
 *
 * Build: gcc -O2 -I include -I /usr/local/cuda/include examples/c_abi_demo.c \
 *            -L paper_2004_06278_b200 -lsquares -L /usr/local/cuda/lib64 -lcudart \
 *            -Wl,-rpath,$PWD/paper_2004_06278_b200 -o c_abi_demo
 * Run:   ./c_abi_demo            (prints the key, the first outputs and count checks)
 */
#include <cuda_runtime.h>
#include <inttypes.h>
#include <stdio.h>
#include <stdlib.h>

#include "squares.h"

#define CHECK(call)                                                                    \
  do {                                                                                 \
    int rc_ = (call);                                                                  \
    if (rc_ != SQ_OK) {                                                                \
      fprintf(stderr, "%s failed: %s\n", #call, sq_strerror(rc_));                     \
      return 1;                                                                        \
    }                                                                                  \
  } while (0)
#define CUDA(call)                                                                     \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess) {                                                           \
      fprintf(stderr, "%s: %s\n", #call, cudaGetErrorString(e_));                      \
      return 1;                                                                        \
    }                                                                                  \
  } while (0)

int main(void) {
  const uint64_t n = 1 << 20;
  uint64_t keys[4];
  CHECK(sq_keygen(1, 4, keys));                       /* "different digits" keys, seed 1 */
  printf("key %016" PRIx64 " valid=%u\n", keys[0], sq_validate_key(keys[0]) == 0);

  cudaStream_t s;
  CUDA(cudaStreamCreate(&s));
  uint32_t *u32_d;
  float *f32_d;
  uint64_t *keys_d, *hist_d, *ones_d;
  CUDA(cudaMalloc((void **)&u32_d, n * sizeof(uint32_t)));
  CUDA(cudaMalloc((void **)&f32_d, 4 * 1024 * sizeof(float)));
  CUDA(cudaMalloc((void **)&keys_d, sizeof(keys)));
  CUDA(cudaMalloc((void **)&hist_d, 65536 * sizeof(uint64_t)));
  CUDA(cudaMalloc((void **)&ones_d, 32 * sizeof(uint64_t)));
  CUDA(cudaMemcpyAsync(keys_d, keys, sizeof(keys), cudaMemcpyHostToDevice, s));
  CUDA(cudaMemsetAsync(hist_d, 0, 65536 * sizeof(uint64_t), s));
  CUDA(cudaMemsetAsync(ones_d, 0, 32 * sizeof(uint64_t), s));

  CHECK(sq_fill_u32_k(keys[0], 0, n, u32_d, s));                      /* squares32(0..n-1, key) */
  CHECK(sq_fill_f32(keys_d, 4, 0, 1000, f32_d, 1024, s));            /* 4 rows, ld 1024 */
  CHECK(sq_fused_stats(keys[0], 0, n, hist_d, ones_d, s));            /* no output stored */

  uint32_t first[4];
  float f[4];
  uint64_t *hist = (uint64_t *)malloc(65536 * sizeof(uint64_t)), ones[32];
  CUDA(cudaMemcpyAsync(first, u32_d, sizeof(first), cudaMemcpyDeviceToHost, s));
  CUDA(cudaMemcpyAsync(f, f32_d + 1024, sizeof(f), cudaMemcpyDeviceToHost, s));   /* row 1 */
  CUDA(cudaMemcpyAsync(hist, hist_d, 65536 * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
  CUDA(cudaMemcpyAsync(ones, ones_d, sizeof(ones), cudaMemcpyDeviceToHost, s));
  CUDA(cudaStreamSynchronize(s));

  uint64_t total = 0, top = 0;
  for (int b = 0; b < 65536; b++) {
    total += hist[b];
    if (b & 0x8000) top += hist[b];
  }
  printf("u32 %08x %08x %08x %08x\n", first[0], first[1], first[2], first[3]);
  printf("f32 %.9g %.9g %.9g %.9g\n", f[0], f[1], f[2], f[3]);
  printf("hist_total %" PRIu64 " (n %" PRIu64 ") ones31 %" PRIu64 " (top-bin sum %" PRIu64 ")\n",
         total, n, ones[31], top);
  printf("%s\n", (total == n && ones[31] == top) ? "ok" : "MISMATCH");
  free(hist);
  return (total == n && ones[31] == top) ? 0 : 1;
}
