// fill.cu -- bulk fills sq_fill_u32 / sq_fill_u64 / sq_fill_f32 (BASELINE.json configs 1-4).
//
// out[k*ld + i] = G(ctr0 + i mod 2^64, keys[k]) with G = squares32,
// squares64, or the float32 map (u32 >> 8) * 2^-24.
//
// Work decomposition: each row's element range is tiled by WARP CHUNKS of
// 32 lanes x V elements (V*elem = 32 bytes per lane, so a chunk is 1 KiB, contiguous, and
// every lane issues one 256-bit store STG.E.ENL2.256).  Chunks are aligned to 32-byte
// addresses: chunk 0 of a row starts m elements before the row (m = row misalignment), and
// elements outside [0, n) are masked (head, ragged tail).  The flattened (row, chunk) space
// is split into one contiguous range per warp of a persistent grid (#SM x occupancy CTAs),
// balanced to within one chunk.  A lane walks its chunks with the multiply-free jump of
// squares_device.cuh (J = 32*V counters) and its V consecutive counters with the Weyl step.
#include <cuda_runtime.h>
#include <stdint.h>

#include "squares_device.cuh"
#include "sq_internal.h"

namespace sq {

template <int KIND>
struct FillTraits;
template <>
struct FillTraits<KIND_U32> { static constexpr int ES = 4; };
template <>
struct FillTraits<KIND_F32> { static constexpr int ES = 4; };
template <>
struct FillTraits<KIND_U64> { static constexpr int ES = 8; };

__device__ __forceinline__ void st256(void* p, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                      uint32_t a4, uint32_t a5, uint32_t a6, uint32_t a7) {
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(a0), "r"(a1),
               "r"(a2), "r"(a3), "r"(a4), "r"(a5), "r"(a6), "r"(a7)
               : "memory");
}

template <int KIND>
__global__ void __launch_bounds__(kFillThreads) fill_kernel(FillArgs a) {
  constexpr int ES = FillTraits<KIND>::ES;
  constexpr int V = 32 / ES;           // elements per lane per chunk
  constexpr int J = 32 * V;            // counters per warp chunk
  constexpr int LOGJ = (V == 8) ? 8 : 7;
  static_assert((1 << LOGJ) == J, "J must be 2^LOGJ");

  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warps_per_cta = blockDim.x >> 5;
  const uint64_t w = (uint64_t)blockIdx.x * warps_per_cta + (threadIdx.x >> 5);
  // contiguous balanced range of chunks for this warp: [c, c_end)
  uint64_t c = w * a.chunks_q + (w < a.chunks_r ? w : a.chunks_r);
  const uint64_t c_end = c + a.chunks_q + (w < a.chunks_r ? 1 : 0);

  uint64_t row = c / a.chunks_per_row;
  uint64_t cc = c - row * a.chunks_per_row;
  while (c < c_end) {
    const uint64_t key = a.keys ? __ldg(a.keys + row) : a.key_imm;
    char* rowp = a.out + row * a.ld_bytes;
    const uint64_t m = ((uintptr_t)rowp & 31) / ES;      // row misalignment in elements
    const uint64_t k2x2 = 2 * key * key;
    const uint64_t jk = (uint64_t)J * key;
    const uint64_t cj = (uint64_t)J * (uint64_t)(J - 1) * key * key;
    const uint64_t dj = (uint64_t)J * k2x2;
    // element index of this lane's first element in chunk cc (may be "negative": wraps)
    uint64_t i0 = cc * J + lane * V - m;
    State s = state_at(a.ctr0 + i0, key);
    uint64_t run = a.chunks_per_row - cc;
    if (run > c_end - c) run = c_end - c;
    for (uint64_t r = 0; r < run; r++) {
      State t = s;
      uint32_t v[8];
      if (KIND == KIND_U64) {
#pragma unroll
        for (int j = 0; j < 4; j++) {
          uint64_t z = add64(t.y, key);
          uint64_t o = squares64_from(t.y, z, t.u);
          v[2 * j] = lo32(o);
          v[2 * j + 1] = hi32(o);
          if (j < 3) step(t, key, k2x2);
        }
      } else {
#pragma unroll
        for (int j = 0; j < 8; j++) {
          uint64_t z = add64(t.y, key);
          uint32_t o = squares32_from(t.y, z, t.u);
          v[j] = (KIND == KIND_F32) ? __float_as_uint(u32_to_unit_f32(o)) : o;
          if (j < 7) step(t, key, k2x2);
        }
      }
      char* p = rowp + (int64_t)i0 * ES;   // i0 "negative" only in the masked head
      if ((int64_t)i0 >= 0 && i0 + V <= a.n) {
        st256(p, v[0], v[1], v[2], v[3], v[4], v[5], v[6], v[7]);
      } else {
#pragma unroll
        for (int j = 0; j < V; j++) {
          const uint64_t idx = i0 + j;
          if ((int64_t)idx >= 0 && idx < a.n) {
            if (ES == 4) *(uint32_t*)(p + j * 4) = v[j];
            else *(uint64_t*)(p + j * 8) = ((uint64_t)v[2 * j + 1] << 32) | v[2 * j];
          }
        }
      }
      jump<LOGJ>(s, jk, cj, dj);
      i0 += J;
    }
    c += run;
    row += 1;
    cc = 0;
  }
}

template <int KIND>
static int launch_fill(const FillArgs& a0, uint64_t nkeys, uint64_t n, cudaStream_t stream) {
  constexpr int ES = FillTraits<KIND>::ES;
  constexpr int V = 32 / ES;
  constexpr int J = 32 * V;
  FillArgs a = a0;
  // worst-case misalignment over rows: all rows share it when ld*ES is a multiple of 32
  uint64_t m_max;
  if (nkeys == 1 || (a.ld_bytes % 32) == 0) m_max = ((uintptr_t)a.out & 31) / ES;
  else m_max = V - 1;
  a.chunks_per_row = (n + m_max + J - 1) / J;
  const uint64_t total = a.chunks_per_row * nkeys;
  int occ = 0;
  const DeviceInfo* di = device_info();
  if (!di) return SQ_ECUDA;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fill_kernel<KIND>, kFillThreads, 0);
  if (e != cudaSuccess) return set_cuda_error(e);
  if (occ < 1) occ = 1;
  uint64_t blocks = (uint64_t)di->sms * occ;
  const uint64_t wpc = kFillThreads / 32;
  // no more warps than chunks
  uint64_t need = (total + wpc - 1) / wpc;
  if (blocks > need) blocks = need;
  if (blocks < 1) blocks = 1;
  const uint64_t nw = blocks * wpc;
  a.chunks_q = total / nw;
  a.chunks_r = total % nw;
  fill_kernel<KIND><<<(unsigned)blocks, kFillThreads, 0, stream>>>(a);
  return set_cuda_error(cudaGetLastError());
}

int launch_fill_kind(int kind, const FillArgs& a, uint64_t nkeys, uint64_t n, cudaStream_t stream) {
  switch (kind) {
    case KIND_U32: return launch_fill<KIND_U32>(a, nkeys, n, stream);
    case KIND_U64: return launch_fill<KIND_U64>(a, nkeys, n, stream);
    case KIND_F32: return launch_fill<KIND_F32>(a, nkeys, n, stream);
    default: return SQ_EINVAL;
  }
}

}  // namespace sq
