// devapi_kernels.cu -- test kernels for the header-only device API (include/squares_dev.cuh).
// Built into tests/libdevapi_test.so by __graft_entry__.build(); called from
// tests/test_gpu_devapi.py and compared with the CPU oracle.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../include/squares_dev.cuh"

__global__ void k_pairs(const uint64_t* ctr, const uint64_t* key, uint64_t n, uint32_t* o32, uint64_t* o64) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    o32[i] = sq::squares32(ctr[i], key[i]);
    o64[i] = sq::squares64(ctr[i], key[i]);
  }
}

// thread t draws `per` values from Stream(ctr0 + t*per, key), after skip(skip0) and with the
// counter advanced by skip0 accordingly (so out[t*per + i] = G(ctr0 + t*per + skip0 + i)).
__global__ void k_stream(uint64_t key, uint64_t ctr0, uint64_t per, uint64_t skip0, int kind, uint64_t threads,
                         void* out) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (t >= threads) return;
  sq::Stream st(ctr0 + t * per, key);
  if (skip0) st.skip(skip0);
  for (uint64_t i = 0; i < per; i++) {
    const uint64_t j = t * per + i;
    if (kind == 0) ((uint32_t*)out)[j] = st.next_u32();
    else if (kind == 1) ((uint64_t*)out)[j] = st.next_u64();
    else if (kind == 2) ((float*)out)[j] = st.next_f32();
    else ((double*)out)[j] = st.next_f64();
  }
}

extern "C" int devapi_pairs(const uint64_t* ctr, const uint64_t* key, uint64_t n, uint32_t* o32, uint64_t* o64) {
  k_pairs<<<148, 256>>>(ctr, key, n, o32, o64);
  return (int)cudaDeviceSynchronize();
}

extern "C" int devapi_stream(uint64_t key, uint64_t ctr0, uint64_t per, uint64_t skip0, int kind, uint64_t threads,
                             void* out) {
  k_stream<<<(unsigned)((threads + 127) / 128), 128>>>(key, ctr0, per, skip0, kind, threads, out);
  return (int)cudaDeviceSynchronize();
}

// Generate-inside-the-consumer throughput (tools/bench_next.py): thread t draws `per`
// consecutive squares32 values of Stream(ctr0 + t*per, key) and XOR-folds them (nothing
// stored but one word per thread).  Asynchronous on the default stream (timed with events).
__global__ void k_stream_xor(uint64_t key, uint64_t ctr0, uint64_t per, uint32_t* out) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  sq::Stream st(ctr0 + t * per, key);
  uint32_t acc = 0;
  for (uint64_t i = 0; i < per; i++) acc ^= st.next_u32();
  out[t] = acc;
}

extern "C" int devapi_stream_xor(uint64_t key, uint64_t ctr0, uint64_t per, uint64_t blocks, uint32_t* out) {
  k_stream_xor<<<(unsigned)blocks, 256>>>(key, ctr0, per, out);
  return (int)cudaGetLastError();
}
