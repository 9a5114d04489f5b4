// write_power.cu -- board power (NVML) of write-only kernels: per-warp contiguous segments vs
// grid-strided 2 KiB chunks, 4 GiB per launch, ~3 s of steady state each.  Not product code.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o write_power write_power.cu -lnvidia-ml
#include <cuda_runtime.h>
#include <nvml.h>
#include <cstdio>
#include <cstdint>
#include <unistd.h>
#include <chrono>
__device__ __forceinline__ void st256(void* p, uint32_t a) {
  asm volatile("st.global.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(p), "r"(a) : "memory");
}
// MODE 0: each warp a contiguous segment of 2 KiB chunks; MODE 1: chunks grid-strided over warps
template <int MODE>
__global__ void __launch_bounds__(256) kw(char* out, size_t chunks) {
  const size_t nw = (size_t)gridDim.x * 8, w = (size_t)blockIdx.x * 8 + threadIdx.x / 32;
  const uint32_t lane = threadIdx.x & 31;
  if (MODE == 0) {
    size_t c0 = w * chunks / nw, c1 = (w + 1) * chunks / nw;
    for (size_t c = c0; c < c1; c++) { char* p = out + c * 2048 + lane * 64; st256(p, (uint32_t)c); st256(p + 32, lane); }
  } else {
    for (size_t c = w; c < chunks; c += nw) { char* p = out + c * 2048 + lane * 64; st256(p, (uint32_t)c); st256(p + 32, lane); }
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
  run<1>(buf, bytes, h, "grid-stride chunks");
  sleep(3);
  run<0>(buf, bytes, h, "warp segments");
  return 0;
}
