// keyctr.cu -- "key counter" mode: the counter is fixed and only the key
// changes.  out[j] = G(ctr, keys[j]) for j < nkeys, for every output kind.
//
// Each sample has its own key, so there is no Weyl walk: y = ctr*key is a full 64x64
// multiply and round 1 is a square (15 FMA-pipe slots per squares32 sample instead of 9).
// 8 bytes are read (the key) and 4 or 8 bytes written per sample, so the kernel is HBM-bound:
// a grid-stride loop with coalesced 8-byte key loads and 4/8-byte stores per lane.
#include <cuda_runtime.h>
#include <stdint.h>

#include "squares_device.cuh"
#include "sq_internal.h"

namespace sq {

template <int KIND>
__global__ void __launch_bounds__(256) keyctr_kernel(const uint64_t* __restrict__ keys, uint64_t nkeys,
                                                     uint64_t ctr, char* __restrict__ out) {
  const uint64_t T = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nkeys; j += T) {
    const uint64_t key = __ldg(keys + j);
    const uint64_t y = ctr * key;          // y = x = ctr * key; z = y + key
    const uint64_t z = y + key;
    const uint64_t u = y * y + y;          // round 1 sum
    if (KIND == KIND_U32 || KIND == KIND_F32) {
      const uint32_t o = squares32_from(y, z, u);
      ((uint32_t*)out)[j] = (KIND == KIND_F32) ? __float_as_uint(u32_to_unit_f32(o)) : o;
    } else {
      const uint64_t o = squares64_from(y, z, u);
      uint64_t w;
      if (KIND == KIND_U64) w = o;
      else if (KIND == KIND_F64) w = (uint64_t)__double_as_longlong(u64_to_unit_f64(o));
      else w = ((uint64_t)__float_as_uint(u32_to_unit_f32(hi32(o))) << 32) |
               __float_as_uint(u32_to_unit_f32(lo32(o)));
      ((uint64_t*)out)[j] = w;
    }
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
