// hist16.cuh -- a 65536-bin (or smaller) exact histogram in 128 KiB of shared memory:
// 16-bit counters packed two per 32-bit word, exact by a guard-bit + epoch scheme.
//
// Contract with the caller (fused.cu, scaled.cu): a CTA barrier separates epochs, and at most
// 0x8000 increments reach any bin per epoch.  Invariant: every half <= 0x7FFF at an epoch
// start, so during the epoch a half stays <= 0xFFFF (it never carries into its neighbour).
// The single thread whose ATOMS.ADD returns a half of 0x7FFF (the increment that makes it
// 0x8000) subtracts 0x8000 from that half and adds 0x8000 to the global bin before the next
// barrier, which restores the invariant.  A half has at most one pending crossing (a second
// one needs the half to fall below 0x8000 first, which only the owner's subtraction does),
// so every count is exact: final bin = 0x8000 * (fix-ups) + residual half.
#pragma once
#include <stdint.h>

namespace sq {

// Fix-up of one crossing of bin b (inc = 1 for the low half, 0x10000 for the high half).
// BITS: also count the fix-up per set bit of b (fused statistics derive ones[16..31] from the
// histogram and need each fix-up's weight per bin bit).
template <bool BITS>
__device__ __forceinline__ void guard_fixup(uint32_t* bins, uint32_t b, uint32_t inc,
                                            unsigned long long* hist, uint32_t* fix) {
  atomicSub(&bins[b >> 1], inc << 15);                 // half -= 0x8000
  atomicAdd(&hist[b], 0x8000ull);
  if (BITS) {
#pragma unroll 1
    for (int j = 0; j < 16; j++)
      if ((b >> j) & 1u) atomicAdd(&fix[j], 1u);
  }
}

// Count bin (v >> 16) of a 32-bit value v (bin index b < 65536; low half = even bins).  A lane
// with valid == false adds 0 (so callers need not diverge around masked samples).
template <bool BITS>
__device__ __forceinline__ void hist_add(uint32_t* bins, uint32_t v, unsigned long long* hist, uint32_t* fix,
                                         bool valid = true) {
  const uint32_t b = v >> 16;
  uint32_t inc = (v & 0x10000u) ? 0x10000u : 1u;
  if (!valid) inc = 0;
  const uint32_t old = atomicAdd(&bins[b >> 1], inc);
  if (((old + inc) ^ old) & 0x80008000u) guard_fixup<BITS>(bins, b, inc, hist, fix);
}

}  // namespace sq

namespace sq {

// ---------------------------------------------------------------------------------------
// Sweep scheme (fused statistics): 16-bit bins packed two per word, exact by a THRESHOLD
// invariant instead of a per-sample fix-up, so the hot loop never branches on an ATOMS result.
//
// Packing: word w (bins 2w and 2w+1) holds A = count(bin 2w) + count(bin 2w+1) in its low half
// and B = count(bin 2w+1) in its high half, so one increment is inc = 1 + (v & 0x10000) -- a
// predicate + SEL, or a single LOP3 `(v & 0x10000) | 1` -- and bin 2w = A - B, bin 2w+1 = B at
// flush time.
//
// Contract: a CTA barrier separates epochs and at most 0x8000 increments reach any word per
// epoch.  Invariant I: A <= T = 0x4000 in every word at an epoch start (B <= A).
// Each thread ORs the OLD word returned by each of its ATOMS into `acc`; at the epoch barrier
// the CTA votes (__syncthreads_or) on (acc & 0xC000C000) -- "some A (or B) was seen at >= 0x4000
// before an increment".  No vote => every increment found A < 0x4000, so every A ends the epoch
// <= 0x4000 and I holds.  A vote => the CTA sweeps all bins to the global histogram (every
// word -> 0), so I holds again.  Overflow: A starts <= 0x4000 and gains <= 0x8000 within an
// epoch, so it stays <= 0xC000 < 0x10000 and never carries into B.  With near-uniform bins a
// sweep happens about once per 2^29 samples per CTA.
// (General form: with at most I increments per epoch, T = the largest power of two with
// T + I <= 0xFFFF and the vote mask = the bits >= T of both halves.  I = 0x8000 gives the
// T = 0x4000, mask 0xC000C000 above.)
__host__ __device__ constexpr uint32_t sweep_threshold(uint32_t incs, uint32_t t = 0x8000) {
  return (t + incs <= 0xFFFFu || t <= 1) ? t : sweep_threshold(incs, t >> 1);
}
__host__ __device__ constexpr uint32_t sweep_mask(uint32_t t) {
  return ((0x10000u - t) & 0xFFFFu) * 0x10001u;
}
static_assert(sweep_threshold(0x8000) == 0x4000 && sweep_mask(0x4000) == 0xC000C000u, "sweep constants");

// Bin (v >> 16) += 1 (or += 0 for a masked lane); returns the old word for the vote.  The
// increment is a predicate test + SEL; the single-LOP3 form `(v & 0x10000) | one` (one = 1 in
// a register) is one instruction shorter but made ptxas cluster the ATOMS at the end of each
// epoch block: 955 vs 1032 Gsamples/s on B200 (SQ_INC_LOP3).
__device__ __forceinline__ uint32_t hist_add_sweep(uint32_t* bins, uint32_t v, uint32_t one, bool valid = true) {
#ifndef SQ_INC_LOP3
  uint32_t inc = (v & 0x10000u) ? 0x10001u : 1u;
#else
  uint32_t inc = (v & 0x10000u) | one;
#endif
  if (!valid) inc = 0;
  return atomicAdd(&bins[v >> 17], inc);
}

// Counts of bins 2w and 2w+1 from a swept word.
__device__ __forceinline__ void sweep_word_counts(uint32_t word, uint32_t& even, uint32_t& odd) {
  odd = word >> 16;
  even = (word & 0xFFFFu) - odd;
}

}  // namespace sq
