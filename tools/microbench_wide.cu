// mb2.cu -- throughput of IMAD.WIDE.U32 / IMAD.HI.U32 / IMAD on B200 (experiment, not product)
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
template <int OP>
__global__ void __launch_bounds__(256) kb(uint32_t* out, int iters, unsigned long long* cyc, uint32_t opq) {
  uint32_t a[8]; uint64_t w[8];
#pragma unroll
  for (int j = 0; j < 8; j++) { a[j] = threadIdx.x * 7 + j + 1; w[j] = ((uint64_t)(a[j] * 3u) << 32) | (a[j] * 5u); }
  const uint32_t m = 0x9E3779B9u ^ blockIdx.x;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 8; j++) {
      if (OP == 0) w[j] = (uint64_t)(uint32_t)(w[j] >> 32) * m + w[j];              // IMAD.WIDE, 64-bit addend
      if (OP == 1) a[j] = (uint32_t)(((uint64_t)a[j] * m + w[j]) >> 32);         // IMAD.HI 64-bit addend
      if (OP == 2) a[j] = a[j] * m + w[j & 3];                                     // IMAD
      if (OP == 3) { // IMAD + IMAD.HI pair forced apart with an opaque xor
        uint32_t x = (uint32_t)(w[j] >> 32), x2 = x ^ opq;
        uint32_t lo = x * m + (uint32_t)w[j];
        uint32_t hi = (uint32_t)(((uint64_t)x2 * m + w[j]) >> 32);
        w[j] = ((uint64_t)hi << 32) | lo;
      }
      if (OP == 4) w[j] = (uint64_t)(uint32_t)(w[j] >> 32) * m;                     // IMAD.WIDE no addend
      if (OP == 5) { // round: WIDE + IMAD (squaring)
        uint32_t xl = (uint32_t)(w[j] >> 32), xh = (uint32_t)w[j];
        uint64_t t = (uint64_t)xl * xl + w[(j + 1) & 7];
        uint32_t hi = (uint32_t)(t >> 32) + xl * (xh << 1);
        w[j] = ((uint64_t)(uint32_t)t << 32) | hi;
      }
    }
  }
  long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int j = 0; j < 8; j++) s += a[j] + (uint32_t)w[j] + (uint32_t)(w[j] >> 32);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = (unsigned long long)(t1 - t0);
}
template <int OP> void run(const char* name, int per_iter) {
  int occ; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kb<OP>, 256, 0);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int blocks = sms * occ, iters = 4096;
  uint32_t* o; unsigned long long* c; cudaMalloc(&o, blocks * 256 * 4); cudaMalloc(&c, blocks * 8);
  kb<OP><<<blocks, 256>>>(o, iters, c, 0); cudaDeviceSynchronize();
  kb<OP><<<blocks, 256>>>(o, iters, c, 0); cudaDeviceSynchronize();
  unsigned long long* hc = new unsigned long long[blocks];
  cudaMemcpy(hc, c, blocks * 8, cudaMemcpyDeviceToHost);
  double mx = 0; for (int b = 0; b < blocks; b++) if (hc[b] > mx) mx = hc[b];
  // lane-ops per clock per SM (for the op of interest, per_iter per chain step)
  double ops = (double)occ * 256 * iters * 8 * per_iter;
  printf("{\"op\": \"%s\", \"occ\": %d, \"lane_ops_per_clk_per_sm\": %.2f}\n", name, occ, ops / mx);
  cudaFree(o); cudaFree(c);
}
int main() {
  run<0>("IMAD.WIDE.U32+c64", 1);
  run<4>("IMAD.WIDE.U32", 1);
  run<1>("IMAD.HI.U32+c64", 1);
  run<2>("IMAD", 1);
  run<3>("pair IMAD+IMAD.HI (+LOP3)", 1);
  run<5>("round WIDE+IMAD(+SHL)", 1);
  return 0;
}
