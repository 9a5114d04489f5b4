// hist16.cuh -- a 65536-bin (or smaller) exact histogram in 128 KiB of shared memory: 16-bit
// counters packed two per 32-bit word, exact by the sweep scheme below (fused.cu, scaled.cu).
// (Round 1's first design fixed every 0x7FFF -> 0x8000 crossing in place, one compare-and-branch
// on each ATOMS result; the sweep scheme removed that branch from the hot loop: +16 % on c5.)
#pragma once
#include <stdint.h>

namespace sq {

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
// the CTA votes on (acc & 0xC000C000) (an epoch-stamped shared flag + a plain barrier, see
// fused.cu) -- "some A (or B) was seen at >= 0x4000
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
