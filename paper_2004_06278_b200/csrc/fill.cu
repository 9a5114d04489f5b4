// fill.cu -- bulk fills sq_fill_u32 / sq_fill_u64 / sq_fill_f32 (BASELINE.json configs 1-4).
//
// out[k*ld + i] = G(ctr0 + i mod 2^64, keys[k]) with G = squares32,
// squares64, or the float32 map (u32 >> 8) * 2^-24.
//
// Work decomposition: each row's element range is tiled by WARP CHUNKS of
// 32 lanes x SPL elements (SPL*elem = 64 bytes per lane: two 256-bit stores STG.E.ENL2.256,
// so a chunk is 2 KiB, contiguous).  Chunks are aligned to 32-byte addresses: chunk 0 of a
// row starts m elements before the row (m = row misalignment), and elements outside [0, n)
// are masked (head, ragged tail).  The flattened (row, chunk) space is split into one
// contiguous range per warp of a persistent grid (#SM x occupancy CTAs), balanced to within
// one chunk.  A lane walks its chunks with the multiply-free jump of include/squares_dev.cuh
// (J = 32*SPL counters) and its SPL consecutive counters with the Weyl step.
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include "../../include/squares_dev.cuh"
#include "sq_internal.h"

namespace sq {

// Unroll factor of the full-chunk loop, per output kind: 2 for the 64-bit kinds (store-bound:
// c3 808.6 -> 827.2 Gsamples/s in burst A/B), 1 for the 32-bit kinds (unrolling by 2 or 4 costs
// them 1-7 %).  SQ_FILL_UNROLL > 0 forces one factor for all kinds.
#ifndef SQ_FILL_UNROLL
#define SQ_FILL_UNROLL 0
#endif
template <int KIND>
__host__ __device__ constexpr int fill_unroll() {
  return SQ_FILL_UNROLL > 0 ? SQ_FILL_UNROLL : (kind_elem_bytes(KIND) == 8 ? 2 : 1);
}
#ifndef SQ_FILL_LANE_BYTES
#define SQ_FILL_LANE_BYTES 64
#endif
template <int KIND>
struct FillTraits {
  // ES = element bytes; SPL = samples per lane per chunk (64 bytes per lane = two 256-bit
  // stores); J = 32 * SPL counters per warp chunk = 2^LOGJ.
  static constexpr int ES = kind_elem_bytes(KIND);
  static constexpr int LB = SQ_FILL_LANE_BYTES;   // bytes per lane per chunk (64: two 256-bit stores)
  static constexpr int W = LB / 4;                 // 32-bit words per lane per chunk
  static constexpr int SPL = LB / ES;
  static constexpr int LOGJ = 5 + (SPL == 32 ? 5 : SPL == 16 ? 4 : SPL == 8 ? 3 : 2);
};

__device__ __forceinline__ void st256(void* p, const uint32_t* v) {
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v[0]), "r"(v[1]),
               "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}

// Per-row constants of the counter walk (include/squares_dev.cuh): the key, the stepping
// increment K = stride*key, the chunk jump (J*K, J(J-1)K^2, 2JK^2) and cst[j] = j*2K^2 for
// the in-chunk 3-input u step.
template <int SPL>
struct RowConst {
  uint64_t key, K, jk, cj, dj, k2x2;
  uint64_t cst[SPL];
};

template <int SPL>
__device__ __forceinline__ RowConst<SPL> row_const(uint64_t key, uint64_t stride) {
  constexpr uint64_t J = 32 * SPL;
  RowConst<SPL> rc;
  const uint64_t K = stride * key;
  const uint64_t k2x2 = 2 * K * K;
  rc.key = key;
  rc.K = K;
  rc.jk = J * K;
  rc.cj = J * (J - 1) * K * K;
  rc.dj = J * k2x2;
  rc.k2x2 = k2x2;
  rc.cst[0] = 0;
#pragma unroll
  for (int j = 1; j < SPL; j++) rc.cst[j] = rc.cst[j - 1] + k2x2;
  return rc;
}

// Output words of one sample j of kind KIND into v (little-endian 64-bit elements).
// Cross-term form (squares_dev.cuh cross_add): the squares64 kinds (store-bound) use the plain
// form 0 in every round (fill_form); the 32-bit kinds use a form per round (SQ_FILL_MIX*,
// below).  SQ_FILL_FORM >= 0 forces one form for every kind and round (experiments).
#ifndef SQ_FILL_FORM
#define SQ_FILL_FORM -1
#endif
#ifndef SQ_FILL64_FORM
#define SQ_FILL64_FORM 0   // cross-term form of the squares64 kinds (all rounds)
#endif
#ifndef SQ_FILL_FMUL2
#define SQ_FILL_FMUL2 1   // f32 scale as a packed FMUL2 over word pairs (gen_lane)
#endif
template <int KIND>
__host__ __device__ constexpr int fill_form() {
  return SQ_FILL_FORM >= 0 ? SQ_FILL_FORM : SQ_FILL64_FORM;
}
// Cross-term forms per round for the 32-bit kinds (include/squares_dev.cuh cross_add): rounds 2
// and 3 as form 11 (= 8 + 3: the square's addend through an explicit carry chain, which drops
// ptxas' VIADD copy after each IMAD.WIDE, and the funnel-shift doubling), round 4 as form 3.
// Burst A/B on B200 (c2 by value / c2 device keys / c4): 11/11/3 1460 / 1379 /
// 1344 vs 3/3/3 1392 / 1353 / 1266; 11/3/3 1461 / 1354 / 1333; 8/8/3 1403 / 1339 / 1298;
// 9/9/3 1357 / 1378 / 1295; 11/11/0 1399 / 1340 / 1302.
#ifndef SQ_FILL_MIX2
#define SQ_FILL_MIX2 11
#define SQ_FILL_MIX3 11
#define SQ_FILL_MIX4 3
#endif
template <int KIND, int FORM, int NW>
__device__ __forceinline__ void put(uint32_t (&v)[NW], int j, uint64_t y, uint64_t z, uint64_t u, uint32_t one) {
  if (KIND == KIND_U32 || KIND == KIND_F32) {
    const uint32_t o = (SQ_FILL_FORM >= 0) ? squares32_from<(SQ_FILL_FORM >= 0 ? SQ_FILL_FORM : 0)>(y, z, u, one)
                                           : squares32_mix<SQ_FILL_MIX2, SQ_FILL_MIX3, SQ_FILL_MIX4>(y, z, u, one);
    // f32: the exact integer float(u >> 8) here; the 2^-24 scale is applied to pairs of lanes'
    // words afterwards with one packed FMUL2 (scale_f32_pairs), exact as before
    v[j] = (KIND == KIND_F32) ? (SQ_FILL_FMUL2 ? __float_as_uint(__uint2float_rn(o >> 8))
                                               : __float_as_uint(u32_to_unit_f32(o)))
                              : o;
  } else {
    const uint64_t o = squares64_from<FORM>(y, z, u, one);
    if (KIND == KIND_U64) {
      v[2 * j] = lo32(o);
      v[2 * j + 1] = hi32(o);
    } else if (KIND == KIND_F64) {
      const uint64_t d = (uint64_t)__double_as_longlong(u64_to_unit_f64(o));
      v[2 * j] = lo32(d);
      v[2 * j + 1] = hi32(d);
    } else {  // KIND_F32X2: low half first, then high half
      v[2 * j] = __float_as_uint(u32_to_unit_f32(lo32(o)));
      v[2 * j + 1] = __float_as_uint(u32_to_unit_f32(hi32(o)));
    }
  }
}

// (float)(u >> 8) * 2^-24 for two words at once: one FMUL2 (packed f32x2 multiply, sm_100) by
// the exact power of two -- same bits as u32_to_unit_f32 (BASELINE.json config 4).
template <int NW>
__device__ __forceinline__ void scale_f32_pairs(uint32_t (&v)[NW]) {
#pragma unroll
  for (int i = 0; i < NW; i += 2) {
    unsigned long long x = ((unsigned long long)v[i + 1] << 32) | v[i], r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(x), "l"(0x3380000033800000ull));
    v[i] = (uint32_t)r;
    v[i + 1] = (uint32_t)(r >> 32);
  }
}

// The SPL outputs of one lane from state s (not modified).  Consecutive counters
// (STRIDED = false): z = y + key is the next counter's y.  Strided: y steps by K and
// z = y + key separately (one more 64-bit add per sample).
#ifndef SQ_FILL_CHAIN2
#define SQ_FILL_CHAIN2 0
#endif
#ifndef SQ_FILL_Y3
#define SQ_FILL_Y3 0
#endif
template <int KIND, int SPL, bool STRIDED, bool CHAIN2 = false>
__device__ __forceinline__ void gen_lane(const State& s, const RowConst<SPL>& rc, uint32_t (&v)[FillTraits<KIND>::W], uint32_t one) {
  uint64_t y = s.y, u = s.u, e = s.e;
#if SQ_FILL_Y3
  // y + key as a 3-input add y + (key - one) + one with the opaque one: IMAD cannot express a
  // 3-input add, so both halves stay on the ALU pipe (IADD3 / IADD3.X with two carries)
  const uint64_t km1 = rc.key - one, one64 = one;
#endif
#pragma unroll
  for (int j = 0; j < SPL; j++) {
#if SQ_FILL_Y3
    const uint64_t z = add64_3(y, km1, one64);
#else
    const uint64_t z = add64(y, rc.key);
#endif
    put<KIND, fill_form<KIND>()>(v, j, y, z, u, one);
    if (j < SPL - 1) {
      y = STRIDED ? add64(y, rc.K) : z;
      if (CHAIN2) {   // u += e; e += 2K^2: no per-row constant table (fewer registers)
        u = add64(u, e);
        e = add64(e, rc.k2x2);
      } else {
        u = j ? add64_3(u, s.e, rc.cst[j]) : add64(u, s.e);
      }
    }
  }
  if (KIND == KIND_F32 && SQ_FILL_FMUL2) scale_f32_pairs(v);
}

// SQ_DEBUG_BOUNDS builds (tests only: SQ_LIB=<debug build> pytest -m gpu) trap any store
// outside row `row`'s written span [row*ld, row*ld + n) elements -- a stronger check than the
// tests' sentinel guards, since compute-sanitizer is unavailable on this pool.
#ifdef SQ_DEBUG_BOUNDS
#define SQ_CHECK_STORE(a, row, ptr, bytes)                                                       \
  do {                                                                                         \
    const char* lo_ = (a).out + (row) * (a).ld_bytes;                                          \
    const char* hi_ = lo_ + (a).n * (uint64_t)(FillTraits<KIND>::ES);                           \
    if ((const char*)(ptr) < lo_ || (const char*)(ptr) + (bytes) > hi_) __trap();             \
  } while (0)
#else
#define SQ_CHECK_STORE(a, row, ptr, bytes) do { } while (0)
#endif

// KEYIMM: a single row whose key is a kernel parameter, so ptxas can keep the key and the
// per-row constants in uniform registers (sq_fill_*_k).  Otherwise keys[row] from memory.
template <int KIND, bool KEYIMM, bool STRIDED>
__global__ void __launch_bounds__(kFillThreads, KEYIMM ? kFillMinBlocksImm : kFillMinBlocks) fill_kernel(FillArgs a) {
  constexpr int ES = FillTraits<KIND>::ES;
  constexpr int SPL = FillTraits<KIND>::SPL;
  constexpr int LOGJ = FillTraits<KIND>::LOGJ;
  constexpr int J = 32 * SPL;            // counters per warp chunk
  static_assert((1 << LOGJ) == J && SPL * ES == FillTraits<KIND>::LB, "chunk geometry");

  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warps_per_cta = blockDim.x >> 5;
  const uint64_t w = (uint64_t)blockIdx.x * warps_per_cta + (threadIdx.x >> 5);
  // contiguous balanced range of chunks for this warp: [c, c_end)
  uint64_t c = w * a.chunks_q + (w < a.chunks_r ? w : a.chunks_r);
  const uint64_t c_end = c + a.chunks_q + (w < a.chunks_r ? 1 : 0);

  uint64_t row = c / a.chunks_per_row;
  uint64_t cc = c - row * a.chunks_per_row;
#ifdef SQ_FILL_NOSTORE
  uint32_t nostore_acc = 0;
#endif
  while (c < c_end) {
    const RowConst<SPL> rc =
        row_const<SPL>(KEYIMM ? a.key_imm : __ldg(a.keys + row), STRIDED ? a.stride : 1);
    char* rowp = a.out + row * a.ld_bytes;
    const uint64_t m = ((uintptr_t)rowp & 31) / ES;      // row misalignment in elements
    uint64_t run = a.chunks_per_row - cc;
    if (run > c_end - c) run = c_end - c;
    const uint64_t cc_stop = cc + run;
    // chunks [full_lo, full_hi) lie entirely inside [0, n): no masking needed there
    const uint64_t full_lo = m ? 1 : 0;
    const uint64_t full_hi = (a.n + m) / J;
    // element index of this lane's first element in chunk cc ("negative" wraps mod 2^64)
    uint64_t i0 = cc * J + lane * SPL - m;
    State s = STRIDED ? state_at_strided(a.ctr0 + i0 * a.stride, rc.key, rc.K)
                      : state_at(a.ctr0 + i0, rc.key);
    while (cc < cc_stop) {
      uint32_t v[FillTraits<KIND>::W];
      if (cc >= full_lo && cc < full_hi) {
        // fast path: a run of full chunks, two 256-bit stores per lane each
        uint64_t nfull = (full_hi < cc_stop ? full_hi : cc_stop) - cc;
        char* p = rowp + (int64_t)i0 * ES;
        i0 += nfull * J;
        cc += nfull;
#pragma unroll fill_unroll<KIND>()
        for (; nfull; nfull--) {
          gen_lane<KIND, SPL, STRIDED, SQ_FILL_CHAIN2 && !KEYIMM>(s, rc, v, a.one);
#ifdef SQ_FILL_NOSTORE   // experiment: generation without the output stream
#pragma unroll
          for (int j = 0; j < FillTraits<KIND>::W; j++) nostore_acc ^= v[j];
#else
#pragma unroll
          for (int q = 0; q < FillTraits<KIND>::W / 8; q++) {
            SQ_CHECK_STORE(a, row, p + 32 * q, 32);
            st256(p + 32 * q, v + 8 * q);
          }
#endif
          jump<LOGJ>(s, rc.jk, rc.cj, rc.dj);
          p += J * ES;
        }
      } else {
        // boundary chunk (row head or ragged tail): per-element masked stores
        gen_lane<KIND, SPL, STRIDED, SQ_FILL_CHAIN2 && !KEYIMM>(s, rc, v, a.one);
        char* p = rowp + (int64_t)i0 * ES;
#pragma unroll
        for (int j = 0; j < SPL; j++) {
          const uint64_t idx = i0 + j;
          if ((int64_t)idx >= 0 && idx < a.n) {
            SQ_CHECK_STORE(a, row, p + j * ES, ES);
            if (ES == 4) *(uint32_t*)(p + j * 4) = v[j];
            else *(uint64_t*)(p + j * 8) = ((uint64_t)v[2 * j + 1] << 32) | v[2 * j];
          }
        }
        jump<LOGJ>(s, rc.jk, rc.cj, rc.dj);
        i0 += J;
        cc++;
      }
    }
    c += run;
    row += 1;
    cc = 0;
  }
#ifdef SQ_FILL_NOSTORE
  if (nostore_acc == 0x9E3779B9u) *(uint32_t*)a.out = nostore_acc;
#endif
}

template <int KIND>
static int launch_fill(const FillArgs& a0, uint64_t nkeys, uint64_t n, cudaStream_t stream) {
  constexpr int ES = FillTraits<KIND>::ES;
  constexpr int SPL = FillTraits<KIND>::SPL;
  constexpr int J = 32 * SPL;
  FillArgs a = a0;
  // worst-case misalignment over rows: all rows share it when ld*ES is a multiple of 32
  uint64_t m_max;
  if (nkeys == 1 || (a.ld_bytes % 32) == 0) m_max = ((uintptr_t)a.out & 31) / ES;
  else m_max = 32 / ES - 1;
  a.chunks_per_row = (n + m_max + J - 1) / J;
  const uint64_t total = a.chunks_per_row * nkeys;
  int occ = 0;
  const DeviceInfo* di = device_info();
  if (!di) return SQ_ECUDA;
  void (*kern)(FillArgs);
  if (a.stride == 1) kern = a.keys ? fill_kernel<KIND, false, false> : fill_kernel<KIND, true, false>;
  else kern = a.keys ? fill_kernel<KIND, false, true> : fill_kernel<KIND, true, true>;
  // occupancy is a property of (device, kernel): queried once, then cached (host overhead per
  // call matters in the launch-bound small-n regime)
  static std::atomic<int> occ_cache[kMaxDevices][2][2];
  std::atomic<int>& oc = occ_cache[di->device][a.keys ? 0 : 1][a.stride == 1 ? 0 : 1];
  occ = oc.load(std::memory_order_relaxed);
  if (occ == 0) {
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kFillThreads, 0);
    if (e != cudaSuccess) return set_cuda_error(e);
    if (occ < 1) occ = 1;
    oc.store(occ, std::memory_order_relaxed);
  }
  uint64_t blocks = (uint64_t)di->sms * occ;
  const uint64_t wpc = kFillThreads / 32;
  // no more warps than chunks
  uint64_t need = (total + wpc - 1) / wpc;
  if (blocks > need) blocks = need;
  if (blocks < 1) blocks = 1;
  const uint64_t nw = blocks * wpc;
  a.chunks_q = total / nw;
  a.chunks_r = total % nw;
  kern<<<(unsigned)blocks, kFillThreads, 0, stream>>>(a);
  return set_cuda_error(cudaGetLastError());
}

int launch_fill_kind(int kind, const FillArgs& a, uint64_t nkeys, uint64_t n, cudaStream_t stream) {
  switch (kind) {
    case KIND_U32: return launch_fill<KIND_U32>(a, nkeys, n, stream);
    case KIND_U64: return launch_fill<KIND_U64>(a, nkeys, n, stream);
    case KIND_F32: return launch_fill<KIND_F32>(a, nkeys, n, stream);
    case KIND_F64: return launch_fill<KIND_F64>(a, nkeys, n, stream);
    case KIND_F32X2: return launch_fill<KIND_F32X2>(a, nkeys, n, stream);
    default: return SQ_EINVAL;
  }
}

}  // namespace sq
