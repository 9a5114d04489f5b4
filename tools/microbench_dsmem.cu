// dsmem.cu -- throughput of red.shared::cluster.add.u32 (local vs peer CTA of a 2-CTA cluster)
#include <cuda_runtime.h>
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
namespace cg = cooperative_groups;
template <int MODE>   // 0: local atom.shared (ret), 1: local red.shared::cluster, 2: 50% peer red, 3: 100% peer red
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(1024, 1) kb(uint32_t* out, int iters, unsigned long long* cyc) {
  extern __shared__ uint32_t tab[];
  cg::cluster_group cl = cg::this_cluster();
  for (int i = threadIdx.x; i < 32768; i += blockDim.x) tab[i] = 0;
  cl.sync();
  const uint32_t me = cl.block_rank();
  uint32_t local = (uint32_t)__cvta_generic_to_shared(tab), b0, b1;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(b0) : "r"(local), "r"(0u));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(b1) : "r"(local), "r"(1u));
  uint32_t st = 0x12345u * (threadIdx.x + 1) + blockIdx.x * 977u, acc = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 8; j++) {
      st = st * 1664525u + 1013904223u;
      const uint32_t off = (st >> 15) & 0x1FFFCu;
      if (MODE == 0) {
        uint32_t old;
        asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(local + off), "r"(1u) : "memory");
        acc |= old;
      } else {
        uint32_t base = (MODE == 1) ? (me ? b1 : b0) : (MODE == 3) ? (me ? b0 : b1) : ((st >> 31) ? b1 : b0);
        asm volatile("red.shared::cluster.add.u32 [%0], %1;" :: "r"(base + off), "r"(1u) : "memory");
      }
    }
  }
  long long t1 = clock64();
  cl.sync();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc + tab[threadIdx.x];
  if (threadIdx.x == 0) cyc[blockIdx.x] = (unsigned long long)(t1 - t0);
}
template <int MODE> void run(const char* name) {
  auto k = kb<MODE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int blocks = sms, iters = 2048;
  uint32_t* o; unsigned long long* c; cudaMalloc(&o, blocks * 1024 * 4); cudaMalloc(&c, blocks * 8);
  k<<<blocks, 1024, 131072>>>(o, iters, c); 
  cudaError_t e = cudaDeviceSynchronize(); if (e) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a); k<<<blocks, 1024, 131072>>>(o, iters, c); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  unsigned long long* hc = new unsigned long long[blocks];
  cudaMemcpy(hc, c, blocks * 8, cudaMemcpyDeviceToHost);
  double mx = 0; for (int i = 0; i < blocks; i++) if (hc[i] > mx) mx = hc[i];
  double ops = 1024.0 * iters * 8;
  printf("{\"mode\": \"%s\", \"ops_per_clk_per_sm\": %.2f, \"Gops_per_s_total\": %.1f}\n", name, ops / mx, ops * blocks / (ms * 1e6));
}
int main() {
  run<0>("local atom.shared (ret)");
  run<1>("local red.shared::cluster");
  run<2>("50% peer red.shared::cluster");
  run<3>("100% peer red.shared::cluster");
  return 0;
}
