// fused.cu -- sq_fused_stats: generate squares32 and reduce without storing
// (BASELINE.json config 5; the GPU analogue of PAPER.md P:45's "basic uniformity test").
//
//   hist[b] += #{i : u_i >> 16 == b},  ones[j] += #{i : bit j of u_i},  u_i = squares32(ctr0+i, key)
//
// Design:
//  * One CTA of 1024 threads per SM (persistent), each thread owning one contiguous counter
//    range, walked with the multiply-free Weyl/finite-difference step (squares_device.cuh).
//  * hist: a 65536-bin histogram held in shared memory as 16-bit counters packed two per
//    32-bit word (128 KiB; 32-bit bins would need 256 KiB > 227 KiB): word w holds
//    A = count(2w) + count(2w+1) and B = count(2w+1).  Exact by the sweep scheme of
//    hist16.cuh: a CTA barrier follows every 32 samples per thread (<= 0x8000 increments per
//    epoch); each ATOMS's old word is ORed into a per-thread flag word, and the CTA sweeps all
//    bins to global memory at a barrier where some A was seen >= 0x4000, so A stays <= 0xC000.
//    No per-sample branch on an ATOMS result.
//  * ones[16..31] are derived exactly from the histogram (bit j of u is bit j-16 of its bin):
//    from the bins each sweep (and the final flush) moves to global memory.
//  * ones[0..15]: bit-sliced carry-save counting.  Two samples' low halves are packed in one
//    32-bit word (columns j and j+16 both count bit j); a Harley-Seal tree folds 16 words
//    (one epoch) into a weight-16 word, which is ripple-added into 6 vertical counter planes,
//    flushed to shared-memory totals every 63 epochs.  ~1.3 LOP3 per sample.
//  * At exit: residual bins -> global hist (RED.ADD.64), CTA bit totals -> global ones.
//  * Source order: generation runs one 8-sample batch ahead of its reduction (SQ_FUSED_PIPE).
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include "hist16.cuh"
#include "squares_device.cuh"
#include "sq_internal.h"

namespace sq {

// Geometry: kFusedThreads threads per CTA (one CTA per SM), kEpoch samples per thread between
// barriers, so at most kFusedThreads * kEpoch increments per epoch; the sweep threshold is the
// largest power of two T with T + increments <= 0xFFFF (hist16.cuh).
#ifndef SQ_FUSED_EPOCH
#define SQ_FUSED_EPOCH (0x8000 / SQ_FUSED_THREADS)
#endif
constexpr int kEpoch = SQ_FUSED_EPOCH;
constexpr uint32_t kEpochIncs = (uint32_t)kFusedThreads * kEpoch;
constexpr uint32_t kT = sweep_threshold(kEpochIncs);
constexpr uint32_t kMask = sweep_mask(kT);
constexpr int kTrees = kEpoch / 32;               // 16-word Harley-Seal trees per epoch
constexpr int kPlanes = 6;                        // vertical planes for weight-16 words: counts up to 63
constexpr int kFlushEvery = 63 / kTrees;          // epochs between plane flushes
static_assert(kEpoch % 32 == 0 && kTrees >= 1, "fused geometry");
static_assert(kT >= 0x100 && kT + kEpochIncs <= 0xFFFFu, "epoch bound of the sweep scheme");
constexpr size_t kFusedSmem = 32768 * 4 + 16 * 8 + 16 * 8 + 2 * 4;

// carry-save adder: (h, l) = (maj(a,b,c), a^b^c)
__device__ __forceinline__ void csa(uint32_t& h, uint32_t& l, uint32_t a, uint32_t b, uint32_t c) {
  const uint32_t u = a ^ b;
  h = (a & b) | (u & c);
  l = u ^ c;
}

// Adds weight*(count of set bits in columns j and j+16 of `word`) for j = 0..15 into cnt[].
__device__ __forceinline__ void columns_add(uint32_t (&cnt)[16], uint32_t word, uint32_t weight) {
#pragma unroll
  for (int j = 0; j < 16; j++) cnt[j] += (((word >> j) & 1u) + ((word >> (j + 16)) & 1u)) * weight;
}

__device__ __forceinline__ void warp_flush16(uint32_t (&cnt)[16], unsigned long long* dst) {
#pragma unroll
  for (int j = 0; j < 16; j++) {
    const uint32_t s = __reduce_add_sync(0xffffffffu, cnt[j]);
    if ((threadIdx.x & 31) == 0 && s) atomicAdd(&dst[j], (unsigned long long)s);
    cnt[j] = 0;
  }
}

// Per-key constants of the counter walk: K = stride*key (the y step), cst[j] = j*2K^2 (j < 8),
// cst8 = 8*2K^2.
struct WalkConst {
  uint64_t key, K;
  uint64_t cst[8];
  uint64_t cst8;
};

// 8 consecutive samples from state s; s advances by 8 counters.  u uses the 3-input step
// u(c+j+1) = u(c+j) + e(c) + j*2k^2 (squares_device.cuh), e advances once per group.
// STRIDED: counters advance by `stride` (y by K, z = y + key separately); BITREV: each
// output is bit-reversed before it is counted ("bits-reversed tests").
#ifndef SQ_FUSED_PIPE
#define SQ_FUSED_PIPE 1
#endif
#ifndef SQ_FUSED_FORM
#define SQ_FUSED_FORM 0
#endif
template <bool STRIDED, bool BITREV>
__device__ __forceinline__ void gen8(State& s, const WalkConst& wc, uint32_t (&v)[8], uint32_t one) {
  uint64_t y = s.y, u = s.u;
#pragma unroll
  for (int j = 0; j < 8; j++) {
    const uint64_t z = add64(y, wc.key);
    // FORM 0 (plain doubling) measured fastest with the sweep scheme (991 vs 947 Gs/s FORM 1)
#ifdef SQ_FUSED_MIX2
    const uint32_t o = squares32_mix<SQ_FUSED_MIX2, SQ_FUSED_MIX3, SQ_FUSED_MIX4>(y, z, u, one);
#else
    const uint32_t o = squares32_from<SQ_FUSED_FORM>(y, z, u, one);
#endif
    v[j] = BITREV ? __brev(o) : o;
    y = STRIDED ? add64(y, wc.K) : z;
    u = j ? add64_3(u, s.e, wc.cst[j]) : add64(u, s.e);
  }
  s.y = y;
  s.u = u;
  s.e = add64(s.e, wc.cst8);
}

// Histogram updates for 8 samples (masked ones add 0) and their packed low halves:
// w[i] = low half of v[2i] | low half of v[2i+1] << 16 (masked samples contribute 0).
// The ATOMS results only feed the sweep vote (acc), so the 8 updates issue back to back.
template <bool MASKED>
__device__ __forceinline__ void reduce8(const uint32_t (&v)[8], uint32_t (&w)[4], uint32_t* bins, uint32_t& acc,
                                        int64_t base_rem, uint32_t one) {
#pragma unroll
  for (int i = 0; i < 4; i++) {
    uint32_t a = v[2 * i], b = v[2 * i + 1];
    if (MASKED) {
      const bool va = base_rem > 2 * i, vb = base_rem > 2 * i + 1;
      acc |= hist_add_sweep(bins, a, one, va) | hist_add_sweep(bins, b, one, vb);
      if (!va) a = 0;
      if (!vb) b = 0;
    } else {
      acc |= hist_add_sweep(bins, a, one) | hist_add_sweep(bins, b, one);
    }
    w[i] = __byte_perm(a, b, 0x5410);
  }
}

// One epoch (32 samples = 16 packed words) folded by Harley-Seal into a weight-16 word.
template <bool MASKED, bool STRIDED, bool BITREV>
__device__ __forceinline__ uint32_t epoch(State& s, const WalkConst& wc, uint32_t one, uint32_t* bins,
                                          uint32_t& acc, int64_t rem, uint32_t& ones, uint32_t& twos,
                                          uint32_t& fours, uint32_t& eights) {
  uint32_t eightsAB[2], foursAB[2];
#if SQ_FUSED_PIPE
  // generation one 8-sample batch ahead of the reduction (software pipelined source order)
  uint32_t vb[2][8];
  gen8<STRIDED, BITREV>(s, wc, vb[0], one);
#pragma unroll
  for (int k = 0; k < 4; k++) {
    const int blk = k >> 1, h = k & 1;
    if (k < 3) gen8<STRIDED, BITREV>(s, wc, vb[(k + 1) & 1], one);
    uint32_t w[4], twosA, twosB;
    reduce8<MASKED>(vb[k & 1], w, bins, acc, rem - 8 * k, one);
    csa(twosA, ones, ones, w[0], w[1]);
    csa(twosB, ones, ones, w[2], w[3]);
    csa(foursAB[h], twos, twos, twosA, twosB);
    if (h) csa(eightsAB[blk], fours, fours, foursAB[0], foursAB[1]);
  }
#else
#pragma unroll
  for (int blk = 0; blk < 2; blk++) {
#pragma unroll
    for (int h = 0; h < 2; h++) {
      uint32_t v[8], w[4], twosA, twosB;
      gen8<STRIDED, BITREV>(s, wc, v, one);
      reduce8<MASKED>(v, w, bins, acc, rem - 8 * (2 * blk + h), one);
      csa(twosA, ones, ones, w[0], w[1]);
      csa(twosB, ones, ones, w[2], w[3]);
      csa(foursAB[h], twos, twos, twosA, twosB);
    }
    csa(eightsAB[blk], fours, fours, foursAB[0], foursAB[1]);
  }
#endif
  uint32_t sixteens;
  csa(sixteens, eights, eights, eightsAB[0], eightsAB[1]);
  return sixteens;
}

// Moves every bin of the CTA's shared histogram to the global histogram and zeroes it (a
// sweep, or the final flush), adding the moved counts per set bin bit into hi_cnt[0..15]
// (ones[16 + j] counts bit j of the bin: bit 0 is the word's odd bin, bits 1..15 the word
// index).  Thread tid visits words tid, tid + T, ... (conflict-free banks).  Rare (the final
// flush plus about one sweep per 2^29 samples per CTA), so it favours simplicity.  Called by
// all threads between barriers (no concurrent ATOMS).
__device__ __noinline__ void flush_bins(uint32_t* bins, unsigned long long* hist, unsigned long long* hi_cnt) {
  uint32_t colcnt[16];
#pragma unroll
  for (int j = 0; j < 16; j++) colcnt[j] = 0;
  for (uint32_t w = threadIdx.x; w < 32768; w += blockDim.x) {
    const uint32_t wv = bins[w];
    if (!wv) continue;
    bins[w] = 0;
    uint32_t lo, hi;   // counts of bins 2w and 2w + 1 (each <= 0xFFFF)
    sweep_word_counts(wv, lo, hi);
    if (lo) atomicAdd(&hist[2 * w], (unsigned long long)lo);
    if (hi) atomicAdd(&hist[2 * w + 1], (unsigned long long)hi);
    colcnt[0] += hi;
#pragma unroll
    for (int j = 1; j < 16; j++) colcnt[j] += ((w >> (j - 1)) & 1u) ? (lo + hi) : 0u;
  }
  // per thread <= 43 words x 0x1FFFE per flush: no 32-bit overflow before warp_flush16
  warp_flush16(colcnt, hi_cnt);
}

template <bool STRIDED, bool BITREV>
__global__ void __launch_bounds__(kFusedThreads, 1)
fused_kernel(uint64_t key, uint64_t ctr0, uint64_t stride, uint64_t q, uint64_t r, uint32_t epochs,
             unsigned long long* __restrict__ hist, unsigned long long* __restrict__ ones_out, uint32_t one) {
  extern __shared__ __align__(16) uint32_t smem[];
  uint32_t* bins = smem;
  unsigned long long* lo_cnt = (unsigned long long*)(smem + 32768);
  unsigned long long* hi_cnt = lo_cnt + 16;
  volatile uint32_t* hot_stamp = (volatile uint32_t*)(hi_cnt + 16);   // [2], epoch-stamped vote
  const uint32_t tid = threadIdx.x;
  for (uint32_t i = tid; i < 32768; i += kFusedThreads) bins[i] = 0;
  if (tid < 16) { lo_cnt[tid] = 0; hi_cnt[tid] = 0; }
  if (tid < 2) hot_stamp[tid] = 0;
  __syncthreads();

  const uint64_t t = (uint64_t)blockIdx.x * kFusedThreads + tid;
  const uint64_t start = t * q + (t < r ? t : r);
  const uint64_t cnt = q + (t < r ? 1 : 0);
  const uint64_t K = STRIDED ? stride * key : key;
  State s = STRIDED ? state_at_strided(ctr0 + start * stride, key, K) : state_at(ctr0 + start, key);
  WalkConst wc;
  {
    const uint64_t k2x2 = 2 * K * K;
    wc.key = key;
    wc.K = K;
    wc.cst[0] = 0;
#pragma unroll
    for (int j = 1; j < 8; j++) wc.cst[j] = wc.cst[j - 1] + k2x2;
    wc.cst8 = wc.cst[7] + k2x2;
  }

  uint32_t ones = 0, twos = 0, fours = 0, eights = 0;
  uint32_t pl[kPlanes];
#pragma unroll
  for (int p = 0; p < kPlanes; p++) pl[p] = 0;
  uint64_t done = 0;
  int since_flush = 0;
  for (uint32_t ep = 0; ep < epochs; ep++) {
    uint32_t acc = 0;
#pragma unroll
    for (int tr = 0; tr < kTrees; tr++) {
      uint32_t sixteens;
      if (done + 32 <= cnt) {
        sixteens = epoch<false, STRIDED, BITREV>(s, wc, one, bins, acc, 32, ones, twos, fours, eights);
      } else {
        const int64_t rem = done < cnt ? (int64_t)(cnt - done) : 0;
        sixteens = epoch<true, STRIDED, BITREV>(s, wc, one, bins, acc, rem, ones, twos, fours, eights);
      }
      done += 32;
      // ripple-add the weight-16 word into the vertical planes
      uint32_t c = sixteens;
#pragma unroll
      for (int p = 0; p < kPlanes; p++) {
        const uint32_t tt = pl[p] & c;
        pl[p] ^= c;
        c = tt;
      }
    }
    if (++since_flush == kFlushEvery) {   // planes hold <= 63 per column: flush to the CTA totals
      since_flush = 0;
#pragma unroll
      uint32_t colcnt[16] = {};   // transient: nothing column-wise lives across the loop
      for (int p = 0; p < kPlanes; p++) { columns_add(colcnt, pl[p], 16u << p); pl[p] = 0; }
      warp_flush16(colcnt, lo_cnt);
    }
    // epoch boundary of the sweep scheme (hist16.cuh): vote, and sweep if any word got hot.
    // The vote is an epoch-stamped flag + a plain barrier (BAR.SYNC) instead of the reduction
    // barrier __syncthreads_or (BAR.RED.OR): +0.9 % here, +4 % in scaled.cu.  Stamps are unique per
    // epoch, so the flag is never reset; two slots keep epoch e+1's writers off epoch e's slot
    // until every thread has read it (they only write after the next barrier).
    if (acc & kMask) hot_stamp[ep & 1] = ep + 1;
    __syncthreads();
    if (hot_stamp[ep & 1] == ep + 1) {
      flush_bins(bins, hist, hi_cnt);
      __syncthreads();
    }
  }
  // remaining carry-save state: weights 1, 2, 4, 8 and the planes
  uint32_t colcnt[16] = {};
  columns_add(colcnt, ones, 1);
  columns_add(colcnt, twos, 2);
  columns_add(colcnt, fours, 4);
  columns_add(colcnt, eights, 8);
#pragma unroll
  for (int p = 0; p < kPlanes; p++) columns_add(colcnt, pl[p], 16u << p);
  warp_flush16(colcnt, lo_cnt);

  // residual bins -> global hist (bits 16..31 derived from them)
  flush_bins(bins, hist, hi_cnt);
  __syncthreads();
  if (tid < 16) {
    const unsigned long long lo = lo_cnt[tid], hi = hi_cnt[tid];
    if (lo) atomicAdd(&ones_out[tid], lo);
    if (hi) atomicAdd(&ones_out[16 + tid], hi);
  }
}

int launch_fused(uint64_t key, uint64_t ctr0, uint64_t stride, uint64_t n, uint32_t flags,
                 uint64_t* hist, uint64_t* ones, cudaStream_t stream) {
  const DeviceInfo* di = device_info();
  if (!di) return SQ_ECUDA;
  const bool strided = stride != 1, bitrev = (flags & SQ_FUSED_BITREV) != 0;
  decltype(&fused_kernel<false, false>) kern =
      strided ? (bitrev ? fused_kernel<true, true> : fused_kernel<true, false>)
              : (bitrev ? fused_kernel<false, true> : fused_kernel<false, false>);
  // the 128 KiB opt-in is a per-(device, kernel) attribute: set once, then cached
  static std::atomic<bool> attr_set[kMaxDevices][4];
  std::atomic<bool>& as = attr_set[di->device][(strided ? 2 : 0) + (bitrev ? 1 : 0)];
  if (!as.load(std::memory_order_acquire)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFusedSmem);
    if (e != cudaSuccess) return set_cuda_error(e);
    as.store(true, std::memory_order_release);
  }
  // one CTA per SM; small n uses fewer CTAs (>= 2^20 samples each) so the flush amortises
  uint64_t blocks = (n + (1ull << 20) - 1) >> 20;
  if (blocks > (uint64_t)di->sms) blocks = di->sms;
  if (blocks < 1) blocks = 1;
  const uint64_t T = blocks * kFusedThreads;
  const uint64_t q = n / T, r = n % T;
  const uint64_t per = q + (r ? 1 : 0);
  const uint64_t epochs = (per + kEpoch - 1) / kEpoch;
  if (epochs > 0xFFFFFFFFull) return SQ_ERANGE;
  kern<<<(unsigned)blocks, kFusedThreads, kFusedSmem, stream>>>(
      key, ctr0, stride, q, r, (uint32_t)epochs, (unsigned long long*)hist, (unsigned long long*)ones, 1u);
  return set_cuda_error(cudaGetLastError());
}

}  // namespace sq

// ---------------------------------------------------------------------------------------
// Bit transitions of the output stream (for the runs statistic of the desk battery,
// SURVEY.md 8(f)3).  The stream is the outputs u_0, u_1, ... of counters
// ctr0 + i*stride, each read least-significant bit first; transitions = #{adjacent bit pairs
// that differ} = sum_i popc((u_i ^ (u_i >> 1)) & 0x7FFFFFFF) + sum_{i>0} (bit31(u_{i-1}) != bit0(u_i)).
// Each thread walks one contiguous index range and also evaluates the sample after it (one
// extra sample per thread) for the boundary pair.  Accumulates into *count.
namespace sq {

template <bool STRIDED, bool BITREV>
__global__ void __launch_bounds__(256)
transitions_kernel(uint64_t key, uint64_t ctr0, uint64_t stride, uint64_t n, uint64_t q, uint64_t r,
                   unsigned long long* __restrict__ count, uint32_t one) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t start = t * q + (t < r ? t : r);
  const uint64_t cnt = q + (t < r ? 1 : 0);
  const uint64_t K = STRIDED ? stride * key : key;
  uint64_t acc = 0;
  if (cnt) {
    // Each sample u_i contributes popc(u_i ^ funnel(u_i, u_{i+1})): bits 0..30 are its own 31
    // adjacent pairs, bit 31 is the pair (bit31(u_i), bit0(u_{i+1})) across the boundary.  The
    // thread's last sample pairs with the next thread's first (evaluated directly), or with
    // nothing at the end of the stream.  Full 8-sample batches come from gen8 (the fused
    // kernel's walk); the < 8 remaining samples from the per-counter step.
    State s = STRIDED ? state_at_strided(ctr0 + start * stride, key, K) : state_at(ctr0 + start, key);
    WalkConst wc;
    {
      const uint64_t k2x2 = 2 * K * K;
      wc.key = key;
      wc.K = K;
      wc.cst[0] = 0;
#pragma unroll
      for (int j = 1; j < 8; j++) wc.cst[j] = wc.cst[j - 1] + k2x2;
      wc.cst8 = wc.cst[7] + k2x2;
    }
    uint32_t prev = 0, part = 0;
    bool have = false;
    uint64_t i = 0;
    for (; i + 8 <= cnt; i += 8) {
      uint32_t v[8];
      gen8<STRIDED, BITREV>(s, wc, v, one);
      uint32_t bp = have ? __popc(prev ^ __funnelshift_r(prev, v[0], 1)) : 0u;   // <= 256 per batch
#pragma unroll
      for (int j = 0; j < 7; j++) bp += __popc(v[j] ^ __funnelshift_r(v[j], v[j + 1], 1));
      acc += bp;
      prev = v[7];
      have = true;
    }
    const uint64_t k2x2 = 2 * K * K;
    for (; i < cnt; i++) {
      const uint64_t z = add64(s.y, key);
      uint32_t u = squares32_from(s.y, z, s.u);
      if (BITREV) u = __brev(u);
      if (have) part += __popc(prev ^ __funnelshift_r(prev, u, 1));
      prev = u;
      have = true;
      if (STRIDED) s.y = add64(s.y, K); else s.y = z;
      s.u = add64(s.u, s.e);
      s.e = add64(s.e, k2x2);
    }
    acc += part;
    if (start + cnt < n) {   // boundary with the next thread's first sample
      const uint64_t cn = STRIDED ? ctr0 + (start + cnt) * stride : ctr0 + (start + cnt);
      uint32_t un = squares32(cn, key);
      if (BITREV) un = __brev(un);
      acc += __popc(prev ^ __funnelshift_r(prev, un, 1));
    } else {
      acc += __popc((prev ^ (prev >> 1)) & 0x7FFFFFFFu);
    }
  }
  // warp reduction (64-bit), one atomic per warp
  for (int sh = 16; sh; sh >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, sh);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(count, (unsigned long long)acc);
}

int launch_transitions(uint64_t key, uint64_t ctr0, uint64_t stride, uint64_t n, uint32_t flags,
                       uint64_t* count, cudaStream_t stream) {
  const DeviceInfo* di = device_info();
  if (!di) return SQ_ECUDA;
  const bool strided = stride != 1, bitrev = (flags & SQ_FUSED_BITREV) != 0;
  decltype(&transitions_kernel<false, false>) kern =
      strided ? (bitrev ? transitions_kernel<true, true> : transitions_kernel<true, false>)
              : (bitrev ? transitions_kernel<false, true> : transitions_kernel<false, false>);
  uint64_t blocks = (n + 255) / 256;
  const uint64_t cap = (uint64_t)di->sms * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  const uint64_t T = blocks * 256;
  kern<<<(unsigned)blocks, 256, 0, stream>>>(key, ctr0, stride, n, n / T, n % T, (unsigned long long*)count, 1u);
  return set_cuda_error(cudaGetLastError());
}

}  // namespace sq
