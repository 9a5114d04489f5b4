// fused.cu -- sq_fused_stats: generate squares32 and reduce without storing
// (BASELINE.json config 5; the GPU analogue of PAPER.md P:45's "basic uniformity test").
//
//   hist[b] += #{i : u_i >> 16 == b},  ones[j] += #{i : bit j of u_i},  u_i = squares32(ctr0+i, key)
//
// Design:
//  * One CTA of 1024 threads per SM (persistent), each thread owning one contiguous counter
//    range, walked with the multiply-free Weyl/finite-difference step (include/squares_dev.cuh).
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
#include "../../include/squares_dev.cuh"
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
// u(c+j+1) = u(c+j) + e(c) + j*2k^2 (include/squares_dev.cuh), e advances once per group.
// STRIDED: counters advance by `stride` (y by K, z = y + key separately); BITREV: each
// output is bit-reversed before it is counted ("bits-reversed tests").
#ifndef SQ_FUSED_PIPE
#define SQ_FUSED_PIPE 1
#endif
// Cross-term form per round (squares_dev.cuh cross_add): rounds 2 and 3 as form 6 (the
// product xl*xh first, off the chain through the IMAD.WIDE, then doubled and added), round 4 as
// form 3 (funnel-shift doubling on the ALU).  Measured on B200 (round 2, c5 at 2^34,
// warp-specialised kernel): 6/6/3 1117.6 Gsamples/s; 6/6/1 1112.7; 6/0/3 1097.6;
// 6/6/6 1092; 0/6/3 1090; 0/0/3 1084.6; 0/3/0 1083.9; 6/6/0 1077.5; 3/0/0 1077.2; 3/6/3 1057;
// 0/0/0 1055.5; the lock-step kernel with 6/6/3: 1057.8.
//   with the carry-chain addend of form 8 added in rounds 2-3 (14/14/3): 1148.9 vs 1145.9, and
//   one SASS instruction per sample fewer (the VIADD copies disappear) -- adopted.
#ifndef SQ_FUSED_MIX2
#define SQ_FUSED_MIX2 14
#define SQ_FUSED_MIX3 14
#define SQ_FUSED_MIX4 3
#endif
template <bool STRIDED, bool BITREV>
__device__ __forceinline__ void gen8(State& s, const WalkConst& wc, uint32_t (&v)[8], uint32_t one) {
  uint64_t y = s.y, u = s.u;
#pragma unroll
  for (int j = 0; j < 8; j++) {
    const uint64_t z = add64(y, wc.key);
    const uint32_t o = squares32_mix<SQ_FUSED_MIX2, SQ_FUSED_MIX3, SQ_FUSED_MIX4>(y, z, u, one);
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
__device__ __noinline__ void flush_bins(uint32_t* bins, unsigned long long* hist, unsigned long long* hi_cnt,
                                       uint32_t tid, uint32_t nthr) {
  uint32_t colcnt[16];
#pragma unroll
  for (int j = 0; j < 16; j++) colcnt[j] = 0;
  for (uint32_t w = tid; w < 32768; w += nthr) {
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
  // per thread <= 128 words (nthr >= 256) x 0x1FFFE per flush: no 32-bit overflow before warp_flush16
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
      uint32_t colcnt[16] = {};   // transient: nothing column-wise lives across the loop
#pragma unroll
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
      flush_bins(bins, hist, hi_cnt, tid, kFusedThreads);
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
  flush_bins(bins, hist, hi_cnt, tid, kFusedThreads);
  __syncthreads();
  if (tid < 16) {
    const unsigned long long lo = lo_cnt[tid], hi = hi_cnt[tid];
    if (lo) atomicAdd(&ones_out[tid], lo);
    if (hi) atomicAdd(&ones_out[16 + tid], hi);
  }
}


// ---------------------------------------------------------------------------------------
// Warp-specialised variant (round 2, the default c5 kernel).  The CTA's 32
// warps split into kWsGen = 24 generator warps and kWsRed = 8 reducer warps (the highest warp
// ids: the SMSP arbiter favours them, and they sit on every sub-partition).  A generator warp
// walks its lanes' counter ranges exactly like the kernel above (gen8), counts bits 0..15
// with the same carry-save tree, and hands each 32-sample tree (4 batches, 4 KiB per warp) to
// its reducer through a shared-memory ring of kWsDepth slots guarded by mbarriers (full: 32
// producer arrivals, empty: 32 consumer arrivals).  A reducer warp serves kWsGen / kWsRed
// generator warps round-robin and owns the histogram updates (ATOMS + sweep vote).  The sweep scheme's epoch barrier (hist16.cuh) is a named
// barrier among the reducers only, so the generators never stop at a barrier and the
// FMA-heavy generation and the ALU/LSU-heavy reduction run side by side on every SMSP
// instead of in lock-step phases.
// 1: warp-specialised kernel (default, measured faster); 0: the lock-step kernel above.
#ifndef SQ_FUSED_IMPL
#define SQ_FUSED_IMPL 1
#endif
#ifndef SQ_WS_GEN
#define SQ_WS_GEN 24
#endif
#ifndef SQ_WS_RED_FIRST
#define SQ_WS_RED_FIRST 0
#endif
#ifndef SQ_WS_MAXNREG
#define SQ_WS_MAXNREG 0     // e.g. 72 for the generators (then SQ_WS_REDNREG = 40 for the reducers)
#endif
#ifndef SQ_WS_REDNREG
#define SQ_WS_REDNREG 40
#endif
#ifndef SQ_WS_DEPTH
#define SQ_WS_DEPTH 1
#endif
#ifndef SQ_WS_EPOCH_STEPS
#define SQ_WS_EPOCH_STEPS 2
#endif
#ifndef SQ_WS_RED
#define SQ_WS_RED (32 - SQ_WS_GEN)
#endif
constexpr int kWsGen = SQ_WS_GEN;                       // generator warps
constexpr int kWsRed = SQ_WS_RED;                       // reducer warps
constexpr int kWsThreads = 32 * (kWsGen + kWsRed);
static_assert(kWsThreads <= 1024, "one CTA of at most 32 warps");
constexpr int kWsPer = kWsGen / kWsRed;                 // generator warps per reducer warp
constexpr int kWsDepth = SQ_WS_DEPTH;                   // ring slots per generator warp
constexpr int kWsEpochSteps = SQ_WS_EPOCH_STEPS;        // reducer steps (kWsPer slots each) per epoch
// SQ_WS_TREES carry-save trees per generator iteration, folded by more levels into one word
// (one plane ripple per 32*SQ_WS_TREES samples instead of per 32): 1 tree 1115, 2 trees 1135,
// 4 trees 1145 (adopted), 8 trees 1150 Gsamples/s with twice the code.
#ifndef SQ_WS_TREE2
#define SQ_WS_TREE2 1
#endif
#ifndef SQ_WS_TREES
#define SQ_WS_TREES 4
#endif
static_assert(SQ_WS_TREES == 2 || SQ_WS_TREES == 4 || SQ_WS_TREES == 8, "2, 4 or 8 trees per generator iteration");
#ifndef SQ_WS_SLOT_BATCHES
#define SQ_WS_SLOT_BATCHES 4
#endif
constexpr int kWsSB = SQ_WS_SLOT_BATCHES;               // batches (8 samples per lane) per ring slot
constexpr int kWsSlotWords = 256 * kWsSB;
static_assert(kWsSB == 1 || kWsSB == 2 || kWsSB == 4, "a slot holds 1, 2 or 4 batches (divides a 4-batch tree)");
constexpr uint32_t kWsEpochIncs = (uint32_t)kWsRed * 32 * kWsPer * 8 * kWsSB * kWsEpochSteps;
constexpr uint32_t kWsT = sweep_threshold(kWsEpochIncs);
constexpr uint32_t kWsMask = sweep_mask(kWsT);
static_assert(kWsGen % kWsRed == 0, "each reducer serves a whole number of generator warps");
static_assert(kWsT >= 0x100 && kWsT + kWsEpochIncs <= 0xFFFFu, "epoch bound of the sweep scheme (reducers)");
constexpr size_t kWsRingBytes = (size_t)kWsGen * kWsDepth * kWsSlotWords * 4;
constexpr size_t kWsBarOff = 32768 * 4 + kWsRingBytes;
// SQ_DEBUG_RING builds (tests only: SQ_LIB=<debug build>) tag every ring slot with its sequence
// number and trap on any out-of-order hand-off -- a protocol check in lieu of compute-sanitizer's
// racecheck, which is closed on this pool.  SQ_DEBUG_RING_BREAK (negative control)
// drops one of the generators' waits on the empty barrier, which the check must catch.
#ifdef SQ_DEBUG_RING
constexpr size_t kWsTagBytes = (size_t)kWsGen * kWsDepth * 4;
#define SQ_RING_TAG_ARG , volatile uint32_t* tag_g
#define SQ_RING_TAG_PASS(x) , (x)
#else
constexpr size_t kWsTagBytes = 0;
#define SQ_RING_TAG_ARG
#define SQ_RING_TAG_PASS(x)
#endif
constexpr size_t kWsSmem = kWsBarOff + (size_t)kWsGen * kWsDepth * 2 * 8 + 16 * 8 + 16 * 8 + 2 * 4 + kWsTagBytes;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
// Ring wait (both sides): one try_wait per pass (measured faster than a try_wait/branch spin
// loop: 1081 vs 1072 Gsamples/s); SQ_WS_SLEEP_NS > 0 adds a nanosleep back-off between polls
// (measured no better).
#ifndef SQ_WS_SLEEP_NS
#define SQ_WS_SLEEP_NS 0
#endif
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(smem_u32(b)), "r"(parity) : "memory");
  while (!ok) {
    if (SQ_WS_SLEEP_NS) __nanosleep(SQ_WS_SLEEP_NS);
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(smem_u32(b)), "r"(parity) : "memory");
  }
}
// Generator: one 32-sample Harley-Seal tree = 4 batches = 4 / kWsSB ring slots; each batch is
// stored as soon as it is generated.  MASKED: samples past this lane's count are zeroed for
// the bit counting (the reducer masks them in the histogram).  Slot layout: 2 kWsSB rows of 32
// lanes x uint4 (row = batch half), so every STS.128 / LDS.128 covers 512 contiguous bytes.
template <bool MASKED, bool STRIDED, bool BITREV>
__device__ __forceinline__ uint32_t ws_gen_tree(State& s, const WalkConst& wc, uint32_t one, uint32_t* ring_g,
                                                uint64_t* full_g, uint64_t* empty_g, uint32_t b0, int64_t rem,
                                                uint32_t lane, uint32_t& ones, uint32_t& twos, uint32_t& fours,
                                                uint32_t& eights SQ_RING_TAG_ARG) {
  uint32_t eightsAB[2], foursAB[2];
#pragma unroll
  for (int k = 0; k < 4; k++) {
    uint32_t v[8];
    gen8<STRIDED, BITREV>(s, wc, v, one);
    const uint32_t b = b0 + k, sl = b / kWsSB, sub = b % kWsSB, slot = sl % kWsDepth, round = sl / kWsDepth;
#ifndef SQ_DEBUG_RING_BREAK
    if (sub == 0 && round) mbar_wait_sleep(&empty_g[slot], (round - 1) & 1);
#else
    // negative control: skip the wait of round 1 only (the barrier phases stay consistent, so
    // nothing can hang; slot 0 may be rewritten while its reducer still reads round 0)
    if (sub == 0 && round > 1) mbar_wait_sleep(&empty_g[slot], (round - 1) & 1);
#endif
#ifdef SQ_DEBUG_RING
    if (sub == 0) {   // slot being rewritten: invalidate its tag first
      __syncwarp();
      if (lane == 0) tag_g[slot] = 0;
      __syncwarp();
    }
#endif
    uint4* dst = (uint4*)(ring_g + slot * kWsSlotWords) + sub * 64;
    dst[lane] = make_uint4(v[0], v[1], v[2], v[3]);
    dst[32 + lane] = make_uint4(v[4], v[5], v[6], v[7]);
#ifdef SQ_DEBUG_RING
    if (sub == kWsSB - 1) {
      __syncwarp();
      if (lane == 0) tag_g[slot] = sl + 1;
      __syncwarp();
    }
#endif
    if (sub == kWsSB - 1) mbar_arrive(&full_g[slot]);
    uint32_t w[4], twosA, twosB;
#pragma unroll
    for (int i = 0; i < 4; i++) {
      uint32_t a = v[2 * i], c = v[2 * i + 1];
      if (MASKED) {
        if (!(rem - 8 * k > 2 * i)) a = 0;
        if (!(rem - 8 * k > 2 * i + 1)) c = 0;
      }
      w[i] = __byte_perm(a, c, 0x5410);
    }
    const int blk = k >> 1, h = k & 1;
    csa(twosA, ones, ones, w[0], w[1]);
    csa(twosB, ones, ones, w[2], w[3]);
    csa(foursAB[h], twos, twos, twosA, twosB);
    if (h) csa(eightsAB[blk], fours, fours, foursAB[0], foursAB[1]);
  }
  uint32_t sixteens;
  csa(sixteens, eights, eights, eightsAB[0], eightsAB[1]);
  return sixteens;
}

// Histogram update for the reducers: the increment (v & 0x10000) | one as ONE LOP3 (`one` = 1
// in a register ptxas cannot see through; with two immediates it takes two).
__device__ __forceinline__ uint32_t ws_hist_add(uint32_t* bins, uint32_t v, uint32_t one, bool valid = true) {
  uint32_t inc;
  asm("lop3.b32 %0, %1, 0x10000, %2, 0xEA;" : "=r"(inc) : "r"(v), "r"(one));   // (a & b) | c
  if (!valid) inc = 0;
  return atomicAdd(&bins[v >> 17], inc);
}

// Reducer: one slot (kWsSB batches = 8 kWsSB samples per lane) of a generator warp.
template <bool MASKED>
__device__ __forceinline__ void ws_consume(const uint32_t* ring_g, uint64_t* full_g, uint64_t* empty_g, uint32_t sl,
                                           uint32_t lane, uint32_t* bins, uint32_t& acc, int64_t valid,
                                           uint32_t one SQ_RING_TAG_ARG) {
  const uint32_t slot = sl % kWsDepth, round = sl / kWsDepth;
  mbar_wait_sleep(&full_g[slot], round & 1);
#ifdef SQ_DEBUG_RING
  if (tag_g[slot] != sl + 1) __trap();   // handed over before it was written
#endif
  const uint4* src = (const uint4*)(ring_g + slot * kWsSlotWords);
  uint32_t v[8 * kWsSB];
#pragma unroll
  for (int r = 0; r < 2 * kWsSB; r++) {
    const uint4 p = src[32 * r + lane];
    v[4 * r] = p.x; v[4 * r + 1] = p.y; v[4 * r + 2] = p.z; v[4 * r + 3] = p.w;
  }
#ifdef SQ_DEBUG_RING
  __syncwarp();
  if (tag_g[slot] != sl + 1) __trap();   // overwritten while being read
#endif
  mbar_arrive(&empty_g[slot]);
#pragma unroll
  for (int i = 0; i < 8 * kWsSB; i += 2) {
    if (MASKED)
      acc |= ws_hist_add(bins, v[i], one, valid > i) | ws_hist_add(bins, v[i + 1], one, valid > i + 1);
    else
      acc |= ws_hist_add(bins, v[i], one) | ws_hist_add(bins, v[i + 1], one);
  }
}

// nb: batches per generator lane (a multiple of 4, the same for every lane of the grid);
// nfull: batches in which every lane of the grid has 8 valid samples.
template <bool STRIDED, bool BITREV>
__global__ void __launch_bounds__(kWsThreads, 1)
fused_ws_kernel(uint64_t key, uint64_t ctr0, uint64_t stride, uint64_t q, uint64_t r, uint32_t nb, uint32_t nfull,
                unsigned long long* __restrict__ hist, unsigned long long* __restrict__ ones_out, uint32_t one) {
  extern __shared__ __align__(16) uint32_t smem[];
  uint32_t* bins = smem;
  uint32_t* ring = smem + 32768;
  uint64_t* full = (uint64_t*)((char*)smem + kWsBarOff);
  uint64_t* empty = full + kWsGen * kWsDepth;
  unsigned long long* lo_cnt = (unsigned long long*)(empty + kWsGen * kWsDepth);
  unsigned long long* hi_cnt = lo_cnt + 16;
  volatile uint32_t* hot_stamp = (volatile uint32_t*)(hi_cnt + 16);
#ifdef SQ_DEBUG_RING
  volatile uint32_t* tags = (volatile uint32_t*)(hot_stamp + 2);
  for (uint32_t i = threadIdx.x; i < kWsGen * kWsDepth; i += blockDim.x) tags[i] = 0;
#endif
  const uint32_t tid = threadIdx.x, lane = tid & 31;
  // broadcast from lane 0 so that ptxas treats the role branch as warp-uniform (it then keeps
  // the walk constants in uniform registers inside it)
  const uint32_t warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  for (uint32_t i = tid; i < 32768; i += kWsThreads) bins[i] = 0;
  if (tid < 16) { lo_cnt[tid] = 0; hi_cnt[tid] = 0; }
  if (tid < 2) hot_stamp[tid] = 0;
  if (tid < kWsGen * kWsDepth) { mbar_init(&full[tid], 32); mbar_init(&empty[tid], 32); }
  // per-key walk constants, computed in convergent code from kernel parameters (uniform
  // registers; inside the role branch ptxas rematerialises them with IMAD.WIDE)
  const uint64_t K = STRIDED ? stride * key : key;
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
  __syncthreads();

  // role: generator warps gw = 0..kWsGen-1, reducer warps rw = 0..kWsRed-1.  SQ_WS_RED_FIRST
  // puts the reducers on the LOWEST warp ids (the SMSP arbiter favours high ids)
#if SQ_WS_RED_FIRST
  const bool is_gen = warp >= kWsRed;
  const uint32_t gw = warp - kWsRed, rw_ = warp;
#else
  const bool is_gen = warp < kWsGen;
  const uint32_t gw = warp, rw_ = warp - kWsGen;
#endif
  if (is_gen) {
    // ------------------------------------------------------------------ generator warp
#if SQ_WS_MAXNREG
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(SQ_WS_MAXNREG));
#endif
    const uint64_t t = (uint64_t)blockIdx.x * (kWsGen * 32) + gw * 32 + lane;
    const uint64_t start = t * q + (t < r ? t : r);
    const uint64_t cnt = q + (t < r ? 1 : 0);
    State st = STRIDED ? state_at_strided(ctr0 + start * stride, key, K) : state_at(ctr0 + start, key);
    uint32_t* ring_g = ring + gw * kWsDepth * kWsSlotWords;
    uint64_t* full_g = full + gw * kWsDepth;
    uint64_t* empty_g = empty + gw * kWsDepth;
    uint32_t ones = 0, twos = 0, fours = 0, eights = 0;
    uint32_t pl[kPlanes];
#pragma unroll
    for (int p = 0; p < kPlanes; p++) pl[p] = 0;
    int since_flush = 0;
#if SQ_WS_TREE2
    // SQ_WS_TREES (2 or 4) 32-sample trees per iteration, their weight-16 words folded by more
    // carry-save levels into one weight-16*SQ_WS_TREES word: one ripple into the count planes
    // per 32*SQ_WS_TREES samples instead of per 32
    constexpr int kTr = SQ_WS_TREES;
    constexpr uint32_t kW = 16u * kTr;   // weight of the rippled word
    uint32_t sx = 0, sx2 = 0, sx3 = 0;   // weight-16, -32 and -64 carry-save states
    for (uint32_t b = 0; b < nb; b += 4 * kTr) {
      uint32_t s16[kTr];
#pragma unroll
      for (int h = 0; h < kTr; h++) {
        const uint32_t bb = b + 4 * h;
        if (bb + 4 <= nfull) {
          s16[h] = ws_gen_tree<false, STRIDED, BITREV>(st, wc, one, ring_g, full_g, empty_g, bb, 32, lane, ones,
                                                       twos, fours, eights SQ_RING_TAG_PASS(tags + gw * kWsDepth));
        } else {
          const int64_t rem = 8 * (uint64_t)bb < cnt ? (int64_t)(cnt - 8 * (uint64_t)bb) : 0;
          s16[h] = ws_gen_tree<true, STRIDED, BITREV>(st, wc, one, ring_g, full_g, empty_g, bb, rem, lane, ones,
                                                      twos, fours, eights SQ_RING_TAG_PASS(tags + gw * kWsDepth));
        }
      }
      // carry-save levels: weight 16 -> 32 (state sx) -> 64 (sx2) -> 128 (sx3)
      uint32_t c;
      if (kTr == 2) {
        csa(c, sx, sx, s16[0], s16[1]);
      } else if (kTr == 4) {
        uint32_t c32a, c32b;
        csa(c32a, sx, sx, s16[0], s16[1]);
        csa(c32b, sx, sx, s16[2 % kTr], s16[3 % kTr]);
        csa(c, sx2, sx2, c32a, c32b);
      } else {
        uint32_t c32[4], c64[2];
#pragma unroll
        for (int i = 0; i < 4; i++) csa(c32[i], sx, sx, s16[(2 * i) % kTr], s16[(2 * i + 1) % kTr]);
        csa(c64[0], sx2, sx2, c32[0], c32[1]);
        csa(c64[1], sx2, sx2, c32[2], c32[3]);
        csa(c, sx3, sx3, c64[0], c64[1]);
      }
#pragma unroll
      for (int p = 0; p < kPlanes; p++) {
        const uint32_t tt = pl[p] & c;
        pl[p] ^= c;
        c = tt;
      }
      if (++since_flush == 63) {   // planes hold <= 63 per column
        since_flush = 0;
        uint32_t colcnt[16] = {};
#pragma unroll
        for (int p = 0; p < kPlanes; p++) { columns_add(colcnt, pl[p], kW << p); pl[p] = 0; }
        warp_flush16(colcnt, lo_cnt);
      }
    }
    uint32_t colcnt[16] = {};
    columns_add(colcnt, sx, 16);
    columns_add(colcnt, sx2, 32);
    columns_add(colcnt, sx3, 64);
#pragma unroll
    for (int p = 0; p < kPlanes; p++) { columns_add(colcnt, pl[p], kW << p); pl[p] = 0; }
#else
    for (uint32_t b = 0; b < nb; b += 4) {
      uint32_t sixteens;
      if (b + 4 <= nfull) {
        sixteens = ws_gen_tree<false, STRIDED, BITREV>(st, wc, one, ring_g, full_g, empty_g, b, 32, lane, ones, twos,
                                                       fours, eights SQ_RING_TAG_PASS(tags + gw * kWsDepth));
      } else {
        const int64_t rem = 8 * (uint64_t)b < cnt ? (int64_t)(cnt - 8 * (uint64_t)b) : 0;
        sixteens = ws_gen_tree<true, STRIDED, BITREV>(st, wc, one, ring_g, full_g, empty_g, b, rem, lane, ones, twos,
                                                      fours, eights SQ_RING_TAG_PASS(tags + gw * kWsDepth));
      }
      uint32_t c = sixteens;
#pragma unroll
      for (int p = 0; p < kPlanes; p++) {
        const uint32_t tt = pl[p] & c;
        pl[p] ^= c;
        c = tt;
      }
      if (++since_flush == 63) {   // planes hold <= 63 per column
        since_flush = 0;
        uint32_t colcnt[16] = {};
#pragma unroll
        for (int p = 0; p < kPlanes; p++) { columns_add(colcnt, pl[p], 16u << p); pl[p] = 0; }
        warp_flush16(colcnt, lo_cnt);
      }
    }
    uint32_t colcnt[16] = {};
#pragma unroll
    for (int p = 0; p < kPlanes; p++) columns_add(colcnt, pl[p], 16u << p);
#endif
    columns_add(colcnt, ones, 1);
    columns_add(colcnt, twos, 2);
    columns_add(colcnt, fours, 4);
    columns_add(colcnt, eights, 8);
    warp_flush16(colcnt, lo_cnt);
  } else {
    // ------------------------------------------------------------------ reducer warp
#if SQ_WS_MAXNREG
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(SQ_WS_REDNREG));
#endif
    const uint32_t rw = rw_, rtid = rw_ * 32 + lane;
    int64_t cnt_g[kWsPer];
#pragma unroll
    for (int j = 0; j < kWsPer; j++) {
      const uint64_t t = (uint64_t)blockIdx.x * (kWsGen * 32) + (rw * kWsPer + j) * 32 + lane;
      cnt_g[j] = (int64_t)(q + (t < r ? 1 : 0));
    }
    // slots: nb / kWsSB per generator warp; slot sl holds batches kWsSB*sl .. kWsSB*sl + kWsSB-1
    const uint32_t ns = nb / kWsSB, nsfull = nfull / kWsSB;
    uint32_t ep = 0;
    for (uint32_t sl = 0; sl < ns; ep++) {
      uint32_t acc = 0;
      const uint32_t se = (sl + kWsEpochSteps < ns) ? sl + kWsEpochSteps : ns;
      for (; sl < se; sl++) {
        if (sl < nsfull) {
#pragma unroll
          for (int j = 0; j < kWsPer; j++) {
            const uint32_t g = rw * kWsPer + j;
            ws_consume<false>(ring + g * kWsDepth * kWsSlotWords, full + g * kWsDepth, empty + g * kWsDepth, sl, lane,
                              bins, acc, 8 * kWsSB, one SQ_RING_TAG_PASS(tags + g * kWsDepth));
          }
        } else {
#pragma unroll
          for (int j = 0; j < kWsPer; j++) {
            const uint32_t g = rw * kWsPer + j;
            ws_consume<true>(ring + g * kWsDepth * kWsSlotWords, full + g * kWsDepth, empty + g * kWsDepth, sl, lane,
                             bins, acc, cnt_g[j] - 8 * kWsSB * (int64_t)sl, one SQ_RING_TAG_PASS(tags + g * kWsDepth));
          }
        }
      }
      // epoch boundary among the reducers (named barrier 1): vote, sweep if any word got hot
      if (acc & kWsMask) hot_stamp[ep & 1] = ep + 1;
      asm volatile("bar.sync 1, %0;" ::"n"(kWsRed * 32) : "memory");
      if (hot_stamp[ep & 1] == ep + 1) {
        flush_bins(bins, hist, hi_cnt, rtid, kWsRed * 32);
        asm volatile("bar.sync 1, %0;" ::"n"(kWsRed * 32) : "memory");
      }
    }
    flush_bins(bins, hist, hi_cnt, rtid, kWsRed * 32);
  }
  __syncthreads();
  if (tid < 16) {
    const unsigned long long lo = lo_cnt[tid], hi = hi_cnt[tid];
    if (lo) atomicAdd(&ones_out[tid], lo);
    if (hi) atomicAdd(&ones_out[16 + tid], hi);
  }
}

static int launch_fused_ws(uint64_t key, uint64_t ctr0, uint64_t stride, uint64_t n, uint32_t flags,
                           uint64_t* hist, uint64_t* ones, cudaStream_t stream, const DeviceInfo* di) {
  const bool strided = stride != 1, bitrev = (flags & SQ_FUSED_BITREV) != 0;
  decltype(&fused_ws_kernel<false, false>) kern =
      strided ? (bitrev ? fused_ws_kernel<true, true> : fused_ws_kernel<true, false>)
              : (bitrev ? fused_ws_kernel<false, true> : fused_ws_kernel<false, false>);
  static std::atomic<bool> attr_set[kMaxDevices][4];
  std::atomic<bool>& as = attr_set[di->device][(strided ? 2 : 0) + (bitrev ? 1 : 0)];
  if (!as.load(std::memory_order_acquire)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kWsSmem);
    if (e != cudaSuccess) return set_cuda_error(e);
    as.store(true, std::memory_order_release);
  }
  uint64_t blocks = (n + (1ull << 20) - 1) >> 20;
  if (blocks > (uint64_t)di->sms) blocks = di->sms;
  if (blocks < 1) blocks = 1;
  const uint64_t T = blocks * (kWsGen * 32);
  const uint64_t q = n / T, r = n % T;
  const uint64_t per = q + (r ? 1 : 0);
  // batches per lane, whole 4-batch trees (pairs of trees with SQ_WS_TREE2)
  const uint64_t nb = SQ_WS_TREE2 ? ((per + 32 * SQ_WS_TREES - 1) / (32 * SQ_WS_TREES)) * 4 * SQ_WS_TREES
                                   : ((per + 31) / 32) * 4;
  if (nb > 0xFFFFFFF0ull) return SQ_ERANGE;
  const uint64_t nfull = q / 8;
  kern<<<(unsigned)blocks, kWsThreads, kWsSmem, stream>>>(key, ctr0, stride, q, r, (uint32_t)nb,
                                                          (uint32_t)(nfull < nb ? nfull : nb),
                                                          (unsigned long long*)hist, (unsigned long long*)ones, 1u);
  return set_cuda_error(cudaGetLastError());
}

static int launch_fused_one(uint64_t key, uint64_t ctr0, uint64_t stride, uint64_t n, uint32_t flags,
                            uint64_t* hist, uint64_t* ones, cudaStream_t stream, const DeviceInfo* di) {
#if SQ_FUSED_IMPL == 1
  return launch_fused_ws(key, ctr0, stride, n, flags, hist, ones, stream, di);
#else
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
#endif
}

// Any n < 2^64: launches of at most 2^48 samples (the per-launch batch counters are 32-bit),
// accumulating into the same counts; counters continue mod 2^64 across the pieces.
int launch_fused(uint64_t key, uint64_t ctr0, uint64_t stride, uint64_t n, uint32_t flags,
                 uint64_t* hist, uint64_t* ones, cudaStream_t stream) {
  const DeviceInfo* di = device_info();
  if (!di) return SQ_ECUDA;
  constexpr uint64_t kPiece = 1ull << 48;
  while (n) {
    const uint64_t m = n < kPiece ? n : kPiece;
    const int rc = launch_fused_one(key, ctr0, stride, m, flags, hist, ones, stream, di);
    if (rc != SQ_OK) return rc;
    ctr0 += m * stride;
    n -= m;
  }
  return SQ_OK;
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
