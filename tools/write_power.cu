// write_power.cu -- board power (NVML) of write-only kernels (4 GiB per launch, ~3 s of steady
// state each): store pattern, cache hints, data entropy.  Not product code.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o write_power write_power.cu -lnvidia-ml
#include <cuda_runtime.h>
#include <nvml.h>
#include <cstdio>
#include <cstdint>
#include <unistd.h>
#include <chrono>
template <int H>
__device__ __forceinline__ void st256(void* p, uint32_t a) {
  if (H == 0) asm volatile("st.global.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(p), "r"(a) : "memory");
  if (H == 1) asm volatile("st.global.cs.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(p), "r"(a) : "memory");
  if (H == 2) asm volatile("st.global.L1::no_allocate.L2::evict_first.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(p), "r"(a) : "memory");
}
// MODE 0: each warp a contiguous segment of 2 KiB chunks; MODE 1: chunks grid-strided over warps
template <int MODE>
__global__ void __launch_bounds__(256) kw(char* out, size_t chunks) {
  const size_t nw = (size_t)gridDim.x * 8, w = (size_t)blockIdx.x * 8 + threadIdx.x / 32;
  const uint32_t lane = threadIdx.x & 31;
  if (MODE != 1) {
    size_t c0 = w * chunks / nw, c1 = (w + 1) * chunks / nw;
    for (size_t c = c0; c < c1; c++) { char* p = out + c * 2048 + lane * 64; st256<MODE == 0 ? 0 : MODE - 1>(p, (uint32_t)c * 0x9E3779B9u); st256<MODE == 0 ? 0 : MODE - 1>(p + 32, lane * 0x85EBCA6Bu ^ (uint32_t)c); }
  } else {
    for (size_t c = w; c < chunks; c += nw) { char* p = out + c * 2048 + lane * 64; st256<0>(p, (uint32_t)c * 0x9E3779B9u); st256<0>(p + 32, lane * 0x85EBCA6Bu ^ (uint32_t)c); }
  }
}
template <int MODE> void run(char* buf, size_t bytes, nvmlDevice_t h, const char* name) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  size_t chunks = bytes / 2048;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 3; i++) kw<MODE><<<sms * 3, 256>>>(buf, chunks);
  cudaDeviceSynchronize();
  auto t0 = std::chrono::steady_clock::now();
  double psum = 0; int pn = 0; float msum = 0; int n = 0;
  while (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() < 6.0) {
    cudaEventRecord(a);
    for (int i = 0; i < 50; i++) kw<MODE><<<sms * 3, 256>>>(buf, chunks);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > 3.0) {
      unsigned int mw; nvmlDeviceGetPowerUsage(h, &mw); psum += mw / 1000.0; pn++; msum += ms; n += 50;
    }
  }
  printf("{\"pattern\": \"%s\", \"GBps\": %.0f, \"power_w\": %.0f}\n", name, (double)bytes * n / (msum * 1e6), psum / pn);
}
int main() {
  nvmlInit(); nvmlDevice_t h; nvmlDeviceGetHandleByIndex(0, &h);
  size_t bytes = 4ull << 30; char* buf; cudaMalloc(&buf, bytes);
  run<0>(buf, bytes, h, "warp segments");
  sleep(3);
  run<2>(buf, bytes, h, "warp segments .cs");
  sleep(3);
  run<3>(buf, bytes, h, "warp segments L1::no_allocate.L2::evict_first");
  sleep(3);
  run<0>(buf, bytes, h, "warp segments");
  return 0;
}
