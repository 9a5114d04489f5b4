// mixbench.cu -- issue model of the integer pipes on B200: throughput of clean instruction
// mixes (8 independent in-place accumulator chains per thread, no register moves).
// Prints lane-operations per clock per SM for each mix.  Not part of the product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mixbench tools/mixbench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

// MIX bits: 1 = IMAD.WIDE (in place), 2 = IMAD, 4 = IADD3 (3 regs), 8 = IADD3 (2 regs + imm),
//           16 = IMAD.HI (64-bit addend), 32 = LOP3
template <int MIX>
__global__ void kmix(uint32_t* out, int iters, unsigned long long* cyc) {
  uint64_t w[8];
  uint32_t a[8], b[8], c[8], d[8];
  uint32_t m = 0x9E3779B9u ^ threadIdx.x;
#pragma unroll
  for (int j = 0; j < 8; j++) {
    a[j] = threadIdx.x * 7 + j; b[j] = a[j] * 3 + 1; c[j] = a[j] ^ 0x55; d[j] = a[j] + 9;
    w[j] = ((uint64_t)a[j] << 32) | b[j];
  }
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 8; j++) {
      if (MIX & 1) w[j] = (uint64_t)(uint32_t)(w[j] >> 32) * m + w[j];   // IMAD.WIDE.U32 in place
      if (MIX & 2) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(b[j]) : "r"(m), "r"(a[j]));
      if (MIX & 4) asm volatile("{.reg .u32 t; add.u32 t, %0, %1; add.u32 %0, t, %2;}" : "+r"(c[j]) : "r"(a[j]), "r"(b[j]));
      if (MIX & 8) asm volatile("add.u32 %0, %0, 12345;" : "+r"(d[j]));
      if (MIX & 16) a[j] = (uint32_t)(((uint64_t)a[j] * m + w[j]) >> 32);   // IMAD.HI.U32, 64-bit addend
      if (MIX & 32) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(c[j]) : "r"(m), "r"(d[j]));
    }
  }
  long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int j = 0; j < 8; j++) s += a[j] + b[j] + c[j] + d[j] + (uint32_t)w[j] + (uint32_t)(w[j] >> 32);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = (unsigned long long)(t1 - t0);
}

template <int MIX>
static void run(const char* name, int ops_per_j) {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int threads = 256, bps = 8, blocks = sms * bps, iters = 2048;
  uint32_t* out; unsigned long long* cyc;
  cudaMalloc(&out, (size_t)blocks * threads * 4); cudaMalloc(&cyc, blocks * 8);
  kmix<MIX><<<blocks, threads>>>(out, iters, cyc);
  cudaDeviceSynchronize();
  double best = 0;
  for (int r = 0; r < 3; r++) {
    kmix<MIX><<<blocks, threads>>>(out, iters, cyc);
    unsigned long long h[2048]; cudaMemcpy(h, cyc, blocks * 8, cudaMemcpyDeviceToHost);
    unsigned long long mx = 0; for (int i = 0; i < blocks; i++) if (h[i] > mx) mx = h[i];
    double per = (double)blocks * threads * iters * 8 / sms / (double)mx;  // j-iterations per clk per SM
    if (per > best) best = per;
  }
  printf("{\"mix\": \"%s\", \"iters_per_clk_per_sm\": %.2f, \"lane_ops_per_clk_per_sm\": %.2f}\n", name, best, best * ops_per_j);
  cudaFree(out); cudaFree(cyc);
}

int main() {
  run<1>("WIDE", 1);
  run<2>("IMAD", 1);
  run<16>("HI64", 1);
  run<4>("IADD3_3reg", 1);
  run<8>("IADD_imm", 1);
  run<32>("LOP3", 1);
  run<1 | 2>("WIDE+IMAD", 2);
  run<1 | 4>("WIDE+IADD3", 2);
  run<2 | 4>("IMAD+IADD3", 2);
  run<1 | 2 | 4>("WIDE+IMAD+IADD3", 3);
  run<1 | 2 | 4 | 8>("WIDE+IMAD+IADD3+IADDimm", 4);
  run<1 | 1 | 2 | 4 | 8 | 32>("WIDE+IMAD+IADD3+IADDimm+LOP3", 5);
  run<4 | 8 | 32>("IADD3+IADDimm+LOP3", 3);
  return 0;
}
