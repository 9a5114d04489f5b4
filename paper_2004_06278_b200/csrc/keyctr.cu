// keyctr.cu -- "key counter" mode: the counter is fixed and only the key
// changes.  out[j] = G(ctr, keys[j]) for j < nkeys, for every output kind.
//
// Each sample has its own key, so there is no Weyl walk: y = ctr*key is a full 64x64
// multiply and round 1 is a square (15 FMA-pipe slots per squares32 sample instead of 9).
// 8 bytes are read (the key) and 4 or 8 bytes written per sample, so the kernel is HBM-bound.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/squares_dev.cuh"
#include "sq_internal.h"

namespace sq {

// The value of one sample j (raw output bits, 4 or 8 bytes).
template <int KIND>
__device__ __forceinline__ uint64_t keyctr_value(uint64_t ctr, uint64_t key) {
  const uint64_t y = ctr * key;          // y = x = ctr * key; z = y + key
  const uint64_t z = y + key;
  const uint64_t u = y * y + y;          // round 1 sum
  if (KIND == KIND_U32 || KIND == KIND_F32) {
    const uint32_t o = squares32_from(y, z, u);
    return (KIND == KIND_F32) ? __float_as_uint(u32_to_unit_f32(o)) : o;
  }
  const uint64_t o = squares64_from(y, z, u);
  if (KIND == KIND_U64) return o;
  if (KIND == KIND_F64) return (uint64_t)__double_as_longlong(u64_to_unit_f64(o));
  return ((uint64_t)__float_as_uint(u32_to_unit_f32(hi32(o))) << 32) | __float_as_uint(u32_to_unit_f32(lo32(o)));
}

// Each thread handles groups of 4 consecutive keys: two 16-byte key loads are issued before any
// arithmetic (4x the bytes in flight of a one-key loop: the kernel is bound by memory-level
// parallelism, 12 B/sample for u32), then 4 samples and one 16- or 32-byte store.  Groups are
// grid-strided; the ragged tail (nkeys % 4) is done per key by the first threads.
template <int KIND>
__global__ void __launch_bounds__(256) keyctr_kernel(const uint64_t* __restrict__ keys, uint64_t nkeys,
                                                     uint64_t ctr, char* __restrict__ out) {
  constexpr int ES = kind_elem_bytes(KIND);
  const uint64_t T = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t groups = nkeys / 4;
  const bool vec = (((uintptr_t)keys | (uintptr_t)out) & 15) == 0;   // 16-byte aligned arrays
  if (vec) {
    // the next group's keys are loaded before the current group's arithmetic (prefetch)
    ulonglong2 na = make_ulonglong2(0, 0), nb = na;
    if (tid < groups) {
      na = __ldg((const ulonglong2*)(keys + 4 * tid));
      nb = __ldg((const ulonglong2*)(keys + 4 * tid + 2));
    }
    for (uint64_t g = tid; g < groups; g += T) {
      const ulonglong2 a = na, b = nb;
      if (g + T < groups) {
        na = __ldg((const ulonglong2*)(keys + 4 * (g + T)));
        nb = __ldg((const ulonglong2*)(keys + 4 * (g + T) + 2));
      }
      const uint64_t v0 = keyctr_value<KIND>(ctr, a.x), v1 = keyctr_value<KIND>(ctr, a.y);
      const uint64_t v2 = keyctr_value<KIND>(ctr, b.x), v3 = keyctr_value<KIND>(ctr, b.y);
      if (ES == 4) {
        *(uint4*)(out + 16 * g) = make_uint4((uint32_t)v0, (uint32_t)v1, (uint32_t)v2, (uint32_t)v3);
      } else {
        *(ulonglong2*)(out + 32 * g) = make_ulonglong2(v0, v1);
        *(ulonglong2*)(out + 32 * g + 16) = make_ulonglong2(v2, v3);
      }
    }
  }
  for (uint64_t j = (vec ? 4 * groups : 0) + tid; j < nkeys; j += T) {   // tail, or all if unaligned
    const uint64_t v = keyctr_value<KIND>(ctr, __ldg(keys + j));
    if (ES == 4) ((uint32_t*)out)[j] = (uint32_t)v;
    else ((uint64_t*)out)[j] = v;
  }
}

int launch_keyctr(int kind, const uint64_t* keys, uint64_t nkeys, uint64_t ctr, void* out,
                  cudaStream_t stream) {
  const DeviceInfo* di = device_info();
  if (!di) return SQ_ECUDA;
  uint64_t blocks = (nkeys + 255) / 256;
  const uint64_t cap = (uint64_t)di->sms * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  switch (kind) {
    case KIND_U32: keyctr_kernel<KIND_U32><<<(unsigned)blocks, 256, 0, stream>>>(keys, nkeys, ctr, (char*)out); break;
    case KIND_U64: keyctr_kernel<KIND_U64><<<(unsigned)blocks, 256, 0, stream>>>(keys, nkeys, ctr, (char*)out); break;
    case KIND_F32: keyctr_kernel<KIND_F32><<<(unsigned)blocks, 256, 0, stream>>>(keys, nkeys, ctr, (char*)out); break;
    case KIND_F64: keyctr_kernel<KIND_F64><<<(unsigned)blocks, 256, 0, stream>>>(keys, nkeys, ctr, (char*)out); break;
    case KIND_F32X2: keyctr_kernel<KIND_F32X2><<<(unsigned)blocks, 256, 0, stream>>>(keys, nkeys, ctr, (char*)out); break;
    default: return SQ_EINVAL;
  }
  return set_cuda_error(cudaGetLastError());
}

}  // namespace sq
