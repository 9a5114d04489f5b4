// keygen.cpp -- host-side key utility of libsquares.so: sq_validate_key and sq_keygen.
//
// PAPER.md P:37 (section 3): "The keys are chosen so the the upper 8 digits are different and
// also that the lower 8 digits are different ... The digits are also chosen randomly", "an
// irregular bit pattern with roughly half ones and half zeros"; "about 2 billion keys".
// The paper's utility is unpublished (P:37 footnote); this file implements the builder's
// documented mapping, which the test oracle re-implements
// independently (oracle/oracle.c) from the same description.
#include <stdint.h>

#include <array>
#include <new>
#include <unordered_set>

#include "../../include/squares.h"

namespace {

// SplitMix64 output finalizer (published constants 0xbf58476d1ce4e5b9, 0x94d049bb133111eb).
inline uint64_t finalize64(uint64_t v) {
  v ^= v >> 30;
  v *= 0xbf58476d1ce4e5b9ULL;
  v ^= v >> 27;
  v *= 0x94d049bb133111ebULL;
  return v ^ (v >> 31);
}

// Digit-draw stream of one (seed, index, attempt) triple.
class DrawStream {
 public:
  DrawStream(uint64_t seed, uint64_t index, uint64_t attempt) {
    uint64_t h = finalize64(seed ^ 0x53515541524553ULL);       // ASCII "SQUARES"
    h = finalize64(h + (index + 1) * 0x9E3779B97F4A7C15ULL);
    base_ = finalize64(h + (attempt + 1) * 0xD1B54A32D192ED03ULL);
  }
  // uniform integer in [0, bound): high 64 bits of r * bound
  uint32_t below(uint32_t bound) {
    const uint64_t r = finalize64(base_ + (++draw_) * 0x8CB92BA72F3D8DD7ULL);
    return (uint32_t)(((unsigned __int128)r * bound) >> 64);
  }

 private:
  uint64_t base_;
  uint64_t draw_ = 0;
};

uint64_t make_candidate(uint64_t seed, uint64_t index, uint64_t attempt) {
  DrawStream ds(seed, index, attempt);
  std::array<int, 16> d{};
  // upper half d15..d8: partial Fisher-Yates over {1..15}; position i of the shuffle -> d[15-i]
  std::array<int, 15> pool{};
  for (int i = 0; i < 15; i++) pool[i] = i + 1;
  for (int i = 0; i < 8; i++) {
    const int pick = i + (int)ds.below(15 - i);
    std::swap(pool[i], pool[pick]);
    d[15 - i] = pool[i];
  }
  // lower half: d0 odd, then d1..d7 by partial Fisher-Yates over the other 14 nonzero digits
  d[0] = 1 + 2 * (int)ds.below(8);
  std::array<int, 14> rest{};
  int nrest = 0;
  for (int v = 1; v <= 15; v++)
    if (v != d[0]) rest[nrest++] = v;
  for (int i = 0; i < 7; i++) {
    const int pick = i + (int)ds.below(14 - i);
    std::swap(rest[i], rest[pick]);
    d[1 + i] = rest[i];
  }
  uint64_t key = 0;
  for (int i = 15; i >= 0; i--) key = (key << 4) | (uint64_t)d[i];
  return key;
}

}  // namespace

extern "C" {

uint32_t sq_validate_key(uint64_t key) {
  uint32_t bad = 0;
  unsigned seen_hi = 0, seen_lo = 0;
  for (int i = 0; i < 16; i++) {
    const unsigned dig = (unsigned)((key >> (4 * i)) & 0xF);
    if (dig == 0) bad |= SQ_KEY_ZERO_DIGIT;
    unsigned& seen = (i < 8) ? seen_lo : seen_hi;
    if (seen & (1u << dig)) bad |= (i < 8) ? SQ_KEY_LOWER_REPEAT : SQ_KEY_UPPER_REPEAT;
    seen |= 1u << dig;
  }
  if ((key & 1) == 0) bad |= SQ_KEY_EVEN;
  const int pc = __builtin_popcountll(key);
  if (pc < 28 || pc > 36) bad |= SQ_KEY_POPCOUNT;
  return bad;
}

int sq_keygen(uint64_t seed, uint64_t count, uint64_t* keys_host) {
  if (count > (1ULL << 31)) return SQ_ERANGE;
  if (count == 0) return SQ_OK;
  if (!keys_host) return SQ_EINVAL;
  try {
    std::unordered_set<uint64_t> taken;
    taken.reserve((size_t)count);
    for (uint64_t j = 0; j < count; j++) {
      for (uint64_t attempt = 0;; attempt++) {
        const uint64_t key = make_candidate(seed, j, attempt);
        if (sq_validate_key(key) != 0) continue;
        if (!taken.insert(key).second) continue;   // distinct within the call
        keys_host[j] = key;
        break;
      }
    }
  } catch (const std::bad_alloc&) {
    return SQ_ENOMEM;
  }
  return SQ_OK;
}

}  // extern "C"
