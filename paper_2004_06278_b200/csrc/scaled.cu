// scaled.cu -- exhaustive reduced-width uniformity:
// the W-bit analogue of squares32 (64 -> W and 32 -> W/2 everywhere), evaluated for EVERY
// counter 0 .. 2^W - 1 of each key, histogrammed over its 2^(W/2) outputs.  This scales the
// paper's footnote-1 claim ("The probability of any given output is 1/2^32") from the
// CPU's W <= 24 to W = 32: 2^32 counters per key, a 65536-bin histogram per key.
//
// Arithmetic: W <= 32, so every intermediate fits a 32-bit register and x*x mod 2^W is the
// low W bits of one 32-bit IMAD; the rotation by W/2 is two shifts (a PRMT for W = 32).  The
// counter walk is the Weyl step y(c+1) = y(c) + key.  The histogram is the packed
// 16-bit sweep scheme of hist16.cuh (epochs of 32 samples per thread), as in fused.cu.
#include <cuda_runtime.h>
#include <stdint.h>

#include "hist16.cuh"
#include "sq_internal.h"

namespace sq {

constexpr int kScaledThreads = 1024;
constexpr int kScaledEpoch = 32;
constexpr uint32_t kScaledT = sweep_threshold(kScaledThreads * kScaledEpoch);
constexpr uint32_t kScaledMask = sweep_mask(kScaledT);
static_assert(kScaledT >= 0x100, "sweep-scheme epoch bound");

struct ScaledArgs {
  const uint64_t* keys;
  unsigned long long* hist;   // [nkeys][2^(W/2)]
  uint64_t slice_len;         // counters per CTA slice (last slice takes the rest)
  uint32_t W, h, mask;        // width, half width, 2^W - 1
  uint32_t slices;
  uint32_t one;               // the value 1 (hist16.cuh increment)
};

__device__ __forceinline__ uint32_t rot_h(uint32_t x, uint32_t h, uint32_t mask) {
  return ((x >> h) | (x << h)) & mask;
}

// squares32_scaled for one counter given y = ctr*key and z = y + key (both mod 2^W), returned
// in histogram position: the W/2-bit output v shifted to bits 16.. (v << 16 for W < 32; for
// W = 32 the round-4 sum itself, whose bits 16..31 ARE v: hist16.cuh reads only those).
// W32: mask = all ones (no AND) and the rotation by 16 is one funnel shift.
template <bool W32>
__device__ __forceinline__ uint32_t scaled_from(uint32_t y, uint32_t z, uint32_t h, uint32_t mask) {
  if (W32) {
    uint32_t x = __funnelshift_l(y * y + y, y * y + y, 16);   // round 1 + rotation
    x = x * x + z;                                            // round 2
    x = __funnelshift_l(x, x, 16);
    x = x * x + y;                                            // round 3
    x = __funnelshift_l(x, x, 16);
    return x * x + z;                                         // round 4 (bits 16..31 = output)
  }
  uint32_t x = (y * y + y) & mask;        // round 1
  x = rot_h(x, h, mask);
  x = (x * x + z) & mask;                 // round 2
  x = rot_h(x, h, mask);
  x = (x * x + y) & mask;                 // round 3
  x = rot_h(x, h, mask);
  return (((x * x + z) & mask) >> h) << 16;   // round 4
}

// Histogram update with the increment (v & 0x10000) | one as ONE LOP3 (`one` is the opaque
// kernel argument; with two immediates ptxas needs two instructions).  SQ_SCALED_INC2 keeps
// hist16.cuh's predicate + select form.
__device__ __forceinline__ uint32_t scaled_hist_add(uint32_t* bins, uint32_t v, uint32_t one, bool valid = true) {
#ifdef SQ_SCALED_INC2
  return hist_add_sweep(bins, v, one, valid);
#else
  uint32_t inc;
  asm("lop3.b32 %0, %1, 0x10000, %2, 0xEA;" : "=r"(inc) : "r"(v), "r"(one));   // (a & b) | c
  if (!valid) inc = 0;
  return atomicAdd(&bins[v >> 17], inc);
#endif
}

// All words -> the key's global histogram row, zeroed (A/B packing of hist16.cuh).
__device__ __noinline__ void flush_scaled(uint32_t* bins, uint32_t nwords, uint32_t nbins,
                                          unsigned long long* hrow) {
  for (uint32_t w = threadIdx.x; w < nwords; w += kScaledThreads) {
    const uint32_t v = bins[w];
    if (!v) continue;
    bins[w] = 0;
    uint32_t even, odd;
    sweep_word_counts(v, even, odd);
    if (even) atomicAdd(&hrow[2 * w], (unsigned long long)even);
    if (odd && 2 * w + 1 < nbins) atomicAdd(&hrow[2 * w + 1], (unsigned long long)odd);
  }
}

template <bool W32>
__global__ void __launch_bounds__(kScaledThreads, 1) scaled_hist_kernel(ScaledArgs a) {
  extern __shared__ __align__(16) uint32_t bins[];
  const uint32_t nbins = 1u << a.h, nwords = (nbins + 1) / 2;
  __shared__ uint32_t hot_stamp_[2];
  volatile uint32_t* hot_stamp = hot_stamp_;
  if (threadIdx.x < 2) hot_stamp[threadIdx.x] = 0;
  for (uint32_t i = threadIdx.x; i < nwords; i += kScaledThreads) bins[i] = 0;
  __syncthreads();
  const uint64_t krow = blockIdx.y;
  const uint32_t key = (uint32_t)(a.keys[krow] & a.mask);
  const uint64_t total = 1ull << a.W;
  const uint64_t s0 = (uint64_t)blockIdx.x * a.slice_len;
  const uint64_t slen = (blockIdx.x == a.slices - 1) ? total - s0 : a.slice_len;
  const uint64_t q = slen / kScaledThreads, r = slen % kScaledThreads;
  const uint64_t t = threadIdx.x;
  const uint64_t start = s0 + t * q + (t < r ? t : r);
  const uint64_t cnt = q + (t < r ? 1 : 0);
  const uint64_t epochs = (q + (r ? 1 : 0) + kScaledEpoch - 1) / kScaledEpoch;
  unsigned long long* hrow = a.hist + krow * nbins;
  uint32_t y = (uint32_t)(start * key) & a.mask;       // ctr*key mod 2^W
  uint64_t done = 0;
  for (uint64_t ep = 0; ep < epochs; ep++) {
    uint32_t acc = 0;
    if (done + kScaledEpoch <= cnt) {
#pragma unroll 8
      for (int i = 0; i < kScaledEpoch; i++) {
        const uint32_t z = W32 ? y + key : (y + key) & a.mask;
        acc |= scaled_hist_add(bins, scaled_from<W32>(y, z, a.h, a.mask), a.one);
        y = z;
      }
    } else {
#pragma unroll 4
      for (int i = 0; i < kScaledEpoch; i++) {
        const uint32_t z = W32 ? y + key : (y + key) & a.mask;
        acc |= scaled_hist_add(bins, scaled_from<W32>(y, z, a.h, a.mask), a.one, done + i < cnt);
        y = z;
      }
    }
    done += kScaledEpoch;
    // epoch boundary of the sweep scheme (hist16.cuh): epoch-stamped vote + plain barrier
    // (as fused.cu), sweep if any word got hot
    if (acc & kScaledMask) hot_stamp[ep & 1] = (uint32_t)ep + 1;
    __syncthreads();
    if (hot_stamp[ep & 1] == (uint32_t)ep + 1) {
      flush_scaled(bins, nwords, nbins, hrow);
      __syncthreads();
    }
  }
  flush_scaled(bins, nwords, nbins, hrow);
}

int launch_scaled_hist(int W, const uint64_t* keys, uint64_t nkeys, uint64_t* hist, cudaStream_t stream) {
  const DeviceInfo* di = device_info();
  if (!di) return SQ_ECUDA;
  if (nkeys > 65535) return SQ_ERANGE;   // grid.y limit; callers batch larger key sets
  ScaledArgs a;
  a.keys = keys;
  a.one = 1;
  a.hist = (unsigned long long*)hist;
  a.W = (uint32_t)W;
  a.h = (uint32_t)W / 2;
  a.mask = (W == 32) ? 0xFFFFFFFFu : ((1u << W) - 1);
  const uint64_t total = 1ull << W;
  // slices of >= 2^22 counters, at most one wave of CTAs over all keys
  uint64_t slices = total >> 22;
  const uint64_t cap = (uint64_t)di->sms / (nkeys < (uint64_t)di->sms ? nkeys : di->sms);
  if (slices > cap) slices = cap;
  if (slices < 1) slices = 1;
  a.slices = (uint32_t)slices;
  a.slice_len = total / slices;
  const size_t smem = (size_t)(((1u << a.h) + 1) / 2) * 4;
  auto kern = (W == 32) ? scaled_hist_kernel<true> : scaled_hist_kernel<false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return set_cuda_error(e);
  kern<<<dim3((unsigned)slices, (unsigned)nkeys), kScaledThreads, smem, stream>>>(a);
  return set_cuda_error(cudaGetLastError());
}

}  // namespace sq
