/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for the Squares RNG hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2004_06278_b200/) never includes, links or calls anything in oracle/, and this
 * file includes nothing from the product (no shared headers, tables or helpers).
 *
 * Paper: B. Widynski, "Squares: A Fast Counter-Based RNG", arXiv 2004.06278.
 * Citations: P:n = /root/reference/PAPER.md line n (copied out of the repo at build time
 * is NOT required: the paper text is quoted below where it matters).  S:n = SPEC.md line n.
 *
 * Every function below is the paper's definition written out in its order and notation:
 * no strength reduction (ctr*key is recomputed per counter), no blocking, no fusion.
 * Arithmetic is uint64_t, i.e. mod 2^64, exactly as the C listings.
 *
 * Pins (tests/test_oracle_pins.py, -m "not gpu"):
 *   squares32 / squares64 : hand-evaluated values (tests/golden/hand_values.txt), the
 *       key = 2^32 closed form (c <= 1289), hi32(squares64) == squares32, key = 0 -> 0,
 *       cross-check against two independent multiplications (16-bit limbs, __int128).
 *   fill_* / f32          : per-element definition; f32 exact examples (0, 2^-24, 0.5, 1-2^-24).
 *   fused_stats           : key = 0 closed form, sum(hist) = n, ones[16+j] from hist,
 *       additivity over shards, equality with fill_u32 + numpy.bincount.
 *   scaled analogue       : hand-derived W = 8 and W = 16 values (tests/golden/scaled_values.txt);
 *       W = 64 equals squares32; key 0 -> constant 0; chi^2 p-value numerics against
 *       scipy.special.gammaincc.
 *   xorfold_u32           : n = 1 hand value, key 0 -> 0, the same fold of fill_u32 in numpy.
 *   partition             : SPEC examples, disjointness and coverage.
 *   validate_key          : SPEC examples and the rules of P:37.
 *   keygen                : rules, determinism, prefix stability, distinctness.
 *       "parity unpinned" for the *sequence*: the paper's key utility is unpublished
 *       (P:37 footnote), so the sequence is pinned only by the builder's documented
 *       mapping, re-implemented here independently.
 */
#include <stdint.h>
#include <stddef.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

/* ------------------------------------------------------------------------------------ */
/* The round primitive and the two generators, verbatim from the listings.               */
/* ------------------------------------------------------------------------------------ */

/* P:24 "x = (x>>32) | (x<<32)"; "a rotation (circular shift) by 32 bits is performed". */
uint64_t oracle_rot_half(uint64_t x) { return (x >> 32) | (x << 32); }

/* P:24-26 one round: x = x*x + w; x = (x>>32) | (x<<32). */
uint64_t oracle_round(uint64_t x, uint64_t w) {
  x = x * x + w;
  return (x >> 32) | (x << 32);
}

/* P:21-28, squares32 (section 2 listing), transcribed line by line. */
uint32_t oracle_squares32(uint64_t ctr, uint64_t key) {
  uint64_t x, y, z;
  y = x = ctr * key; z = y + key;
  x = x*x + y; x = (x>>32) | (x<<32);        /* round 1 */
  x = x*x + z; x = (x>>32) | (x<<32);        /* round 2 */
  x = x*x + y; x = (x>>32) | (x<<32);        /* round 3 */
  return (uint32_t)((x*x + z) >> 32);        /* round 4 */
}

/* P:56-64, squares64 (section 5 listing), transcribed line by line. */
uint64_t oracle_squares64(uint64_t ctr, uint64_t key) {
  uint64_t t, x, y, z;
  y = x = ctr * key; z = y + key;
  x = x*x + y; x = (x>>32) | (x<<32);        /* round 1 */
  x = x*x + z; x = (x>>32) | (x<<32);        /* round 2 */
  x = x*x + y; x = (x>>32) | (x<<32);        /* round 3 */
  t = x = x*x + z; x = (x>>32) | (x<<32);    /* round 4 */
  return t ^ ((x*x + y) >> 32);              /* round 5 */
}

/* ------------------------------------------------------------------------------------ */
/* Cross-check transcriptions: the same listings with the 64x64->64        */
/* product computed two other ways.  Used only by tests to pin the two above.            */
/* ------------------------------------------------------------------------------------ */

/* Generic schoolbook product mod 2^64 from four 16-bit limbs per operand.  Deliberately a
 * different decomposition from anything a GPU kernel would use (32-bit halves). */
static uint64_t mul64_limb16(uint64_t a, uint64_t b) {
  uint64_t al[4], bl[4], acc[8];
  int i, j;
  for (i = 0; i < 4; i++) { al[i] = (a >> (16 * i)) & 0xFFFFu; bl[i] = (b >> (16 * i)) & 0xFFFFu; }
  for (i = 0; i < 8; i++) acc[i] = 0;
  for (i = 0; i < 4; i++)
    for (j = 0; j < 4; j++)
      if (i + j < 4) acc[i + j] += al[i] * bl[j];   /* each product < 2^32; sums < 2^35 */
  /* propagate carries through 16-bit columns, keep the low four columns */
  uint64_t r = 0, carry = 0;
  for (i = 0; i < 4; i++) {
    uint64_t col = acc[i] + carry;
    r |= (col & 0xFFFFu) << (16 * i);
    carry = col >> 16;
  }
  return r;
}

static uint64_t mul64_i128(uint64_t a, uint64_t b) {
  unsigned __int128 p = (unsigned __int128)a * (unsigned __int128)b;
  return (uint64_t)p;   /* low 64 bits */
}

#define SQ_CROSS(NAME, MUL)                                                              \
  uint32_t oracle_squares32_##NAME(uint64_t ctr, uint64_t key) {                          \
    uint64_t x, y, z;                                                                     \
    y = x = MUL(ctr, key); z = y + key;                                                   \
    x = MUL(x, x) + y; x = (x >> 32) | (x << 32);                                         \
    x = MUL(x, x) + z; x = (x >> 32) | (x << 32);                                         \
    x = MUL(x, x) + y; x = (x >> 32) | (x << 32);                                         \
    return (uint32_t)((MUL(x, x) + z) >> 32);                                             \
  }                                                                                       \
  uint64_t oracle_squares64_##NAME(uint64_t ctr, uint64_t key) {                          \
    uint64_t t, x, y, z;                                                                  \
    y = x = MUL(ctr, key); z = y + key;                                                   \
    x = MUL(x, x) + y; x = (x >> 32) | (x << 32);                                         \
    x = MUL(x, x) + z; x = (x >> 32) | (x << 32);                                         \
    x = MUL(x, x) + y; x = (x >> 32) | (x << 32);                                         \
    t = x = MUL(x, x) + z; x = (x >> 32) | (x << 32);                                     \
    return t ^ ((MUL(x, x) + y) >> 32);                                                   \
  }
SQ_CROSS(limb, mul64_limb16)
SQ_CROSS(i128, mul64_i128)

/* Batch versions of the scalar functions over explicit (ctr[i], key[i]) pairs (fuzzing). */
void oracle_squares32_pairs(const uint64_t* ctr, const uint64_t* key, uint64_t n, uint32_t* out) {
  for (uint64_t i = 0; i < n; i++) out[i] = oracle_squares32(ctr[i], key[i]);
}
void oracle_squares64_pairs(const uint64_t* ctr, const uint64_t* key, uint64_t n, uint64_t* out) {
  for (uint64_t i = 0; i < n; i++) out[i] = oracle_squares64(ctr[i], key[i]);
}
void oracle_squares32_pairs_limb(const uint64_t* ctr, const uint64_t* key, uint64_t n, uint32_t* out) {
  for (uint64_t i = 0; i < n; i++) out[i] = oracle_squares32_limb(ctr[i], key[i]);
}
void oracle_squares64_pairs_limb(const uint64_t* ctr, const uint64_t* key, uint64_t n, uint64_t* out) {
  for (uint64_t i = 0; i < n; i++) out[i] = oracle_squares64_limb(ctr[i], key[i]);
}
void oracle_squares32_pairs_i128(const uint64_t* ctr, const uint64_t* key, uint64_t n, uint32_t* out) {
  for (uint64_t i = 0; i < n; i++) out[i] = oracle_squares32_i128(ctr[i], key[i]);
}
void oracle_squares64_pairs_i128(const uint64_t* ctr, const uint64_t* key, uint64_t n, uint64_t* out) {
  for (uint64_t i = 0; i < n; i++) out[i] = oracle_squares64_i128(ctr[i], key[i]);
}

/* ------------------------------------------------------------------------------------ */
/* Fills (BASELINE.json configs 1-4; "n sequential draws equal the batch").          */
/* out[k*ld + i] = G(ctr0 + i mod 2^64, keys[k]); ctr*key recomputed for every counter.   */
/* ------------------------------------------------------------------------------------ */

void oracle_fill_u32(const uint64_t* keys, uint64_t nkeys, uint64_t ctr0, uint64_t n,
                     uint32_t* out, uint64_t ld) {
  for (uint64_t k = 0; k < nkeys; k++)
    for (uint64_t i = 0; i < n; i++)
      out[k * ld + i] = oracle_squares32(ctr0 + i, keys[k]);
}

void oracle_fill_u64(const uint64_t* keys, uint64_t nkeys, uint64_t ctr0, uint64_t n,
                     uint64_t* out, uint64_t ld) {
  for (uint64_t k = 0; k < nkeys; k++)
    for (uint64_t i = 0; i < n; i++)
      out[k * ld + i] = oracle_squares64(ctr0 + i, keys[k]);
}

/* BASELINE.json config 4: "float32 uniform in [0,1) taken from the top 24 bits of squares32".
 * (float)(u >> 8) is exact (< 2^24) and the power-of-two scale 2^-24 is exact. */
float oracle_f32_from_u32(uint32_t u) { return (float)(u >> 8) * 0x1p-24f; }

void oracle_fill_f32(const uint64_t* keys, uint64_t nkeys, uint64_t ctr0, uint64_t n,
                     float* out, uint64_t ld) {
  for (uint64_t k = 0; k < nkeys; k++)
    for (uint64_t i = 0; i < n; i++)
      out[k * ld + i] = oracle_f32_from_u32(oracle_squares32(ctr0 + i, keys[k]));
}

/* BASELINE.json config 5 (the GPU analogue of P:45's "basic uniformity test"):
 * hist[b] += #{i : squares32(ctr0+i, key) >> 16 == b}, ones[j] += #{i : bit j of u_i set},
 * j = 0 the least significant bit.  Accumulates into the caller's arrays.  Every bit is
 * counted directly (bits 16..31 are NOT derived from hist here). */
void oracle_fused_stats(uint64_t key, uint64_t ctr0, uint64_t n, uint64_t* hist, uint64_t* ones) {
  for (uint64_t i = 0; i < n; i++) {
    uint32_t u = oracle_squares32(ctr0 + i, key);
    hist[u >> 16] += 1;
    for (int j = 0; j < 32; j++) ones[j] += (u >> j) & 1u;
  }
}

/* ------------------------------------------------------------------------------------ */
/* squares64-derived floats ("53-bit precision floating point" and "splits the 64 bits */
/* into two 32-bit halves"; formulas S:260 and S:269).                                      */
/* ------------------------------------------------------------------------------------ */

/* (v >> 11) * 2^-53: exact (a 53-bit integer times a power of two). */
double oracle_f64_from_u64(uint64_t v) { return (double)(v >> 11) * 0x1p-53; }

void oracle_fill_f64(const uint64_t* keys, uint64_t nkeys, uint64_t ctr0, uint64_t n,
                     double* out, uint64_t ld) {
  for (uint64_t k = 0; k < nkeys; k++)
    for (uint64_t i = 0; i < n; i++)
      out[k * ld + i] = oracle_f64_from_u64(oracle_squares64(ctr0 + i, keys[k]));
}

/* Two floats per squares64 output, low half first; ld counts float PAIRS. */
void oracle_fill_f32x2(const uint64_t* keys, uint64_t nkeys, uint64_t ctr0, uint64_t n,
                       float* out, uint64_t ld) {
  for (uint64_t k = 0; k < nkeys; k++)
    for (uint64_t i = 0; i < n; i++) {
      uint64_t v = oracle_squares64(ctr0 + i, keys[k]);
      out[2 * (k * ld + i)] = oracle_f32_from_u32((uint32_t)v);
      out[2 * (k * ld + i) + 1] = oracle_f32_from_u32((uint32_t)(v >> 32));
    }
}

/* One output of kind 0..4 (u32, u64, f32, f64, f32x2) for counter c, as 8 raw bytes
 * (4-byte kinds in the low word). */
static uint64_t oracle_one(int kind, uint64_t c, uint64_t key) {
  union { float f; uint32_t u; } a, b;
  union { double d; uint64_t u; } dd;
  switch (kind) {
    case 0: return oracle_squares32(c, key);
    case 1: return oracle_squares64(c, key);
    case 2: a.f = oracle_f32_from_u32(oracle_squares32(c, key)); return a.u;
    case 3: dd.d = oracle_f64_from_u64(oracle_squares64(c, key)); return dd.u;
    default: {
      uint64_t v = oracle_squares64(c, key);
      a.f = oracle_f32_from_u32((uint32_t)v);
      b.f = oracle_f32_from_u32((uint32_t)(v >> 32));
      return ((uint64_t)b.u << 32) | a.u;
    }
  }
}

/* Strided counters ("counter tests with increments other than one"):
 * element i of row k uses counter ctr0 + i*stride mod 2^64.  out is raw bytes of the kind's
 * element size (4 for u32/f32, 8 otherwise); ld in elements. */
void oracle_fill_strided(int kind, const uint64_t* keys, uint64_t nkeys, uint64_t ctr0, uint64_t stride,
                         uint64_t n, void* out, uint64_t ld) {
  for (uint64_t k = 0; k < nkeys; k++)
    for (uint64_t i = 0; i < n; i++) {
      uint64_t v = oracle_one(kind, ctr0 + i * stride, keys[k]);
      if (kind == 0 || kind == 2) ((uint32_t*)out)[k * ld + i] = (uint32_t)v;
      else ((uint64_t*)out)[k * ld + i] = v;
    }
}

/* Key-counter mode ("the counter was fixed and only the key changed"). */
void oracle_fill_keyctr(int kind, const uint64_t* keys, uint64_t nkeys, uint64_t ctr, void* out) {
  for (uint64_t j = 0; j < nkeys; j++) {
    uint64_t v = oracle_one(kind, ctr, keys[j]);
    if (kind == 0 || kind == 2) ((uint32_t*)out)[j] = (uint32_t)v;
    else ((uint64_t*)out)[j] = v;
  }
}

/* Bit reversal of a 32-bit word ("bits-reversed tests"), bit by bit. */
uint32_t oracle_bitrev32(uint32_t u) {
  uint32_t r = 0;
  for (int j = 0; j < 32; j++) r |= ((u >> j) & 1u) << (31 - j);
  return r;
}

/* Fused statistics over strided counters, optionally of the bit-reversed outputs. */
void oracle_fused_stats_ex(uint64_t key, uint64_t ctr0, uint64_t stride, uint64_t n, int bitrev,
                           uint64_t* hist, uint64_t* ones) {
  for (uint64_t i = 0; i < n; i++) {
    uint32_t u = oracle_squares32(ctr0 + i * stride, key);
    if (bitrev) u = oracle_bitrev32(u);
    hist[u >> 16] += 1;
    for (int j = 0; j < 32; j++) ones[j] += (u >> j) & 1u;
  }
}

/* XOR-fold of a u32 fill with no output buffer: the CPU-baseline timing kernel
 * ("dead-code-elimination guard").  Same per-counter definition as oracle_fill_u32. */
uint64_t oracle_xorfold_u32(uint64_t key, uint64_t ctr0, uint64_t n) {
  uint64_t acc = 0;
  for (uint64_t i = 0; i < n; i++) acc ^= (uint64_t)oracle_squares32(ctr0 + i, key) << (i & 31);
  return acc;
}

/* ------------------------------------------------------------------------------------ */
/* Weyl equivalence: "(w += s) is equivalent to w = i * s mod 2^64".               */
/* ------------------------------------------------------------------------------------ */
int oracle_weyl_check(uint64_t s, uint64_t n) {
  uint64_t w = 0;
  for (uint64_t i = 0; i < n; i++) {
    if (w != i * s) return 0;
    w += s;
  }
  return 1;
}

/* ------------------------------------------------------------------------------------ */
/* Key rules and the documented key-utility mapping.                  */
/* ------------------------------------------------------------------------------------ */

/* Rule bits (same meanings as documented in DESIGN.md; values are the interface). */
#define ORACLE_KEY_UPPER_REPEAT 1u   /* "the upper 8 digits are different" violated */
#define ORACLE_KEY_LOWER_REPEAT 2u   /* "the lower 8 digits are different" violated */
#define ORACLE_KEY_ZERO_DIGIT   4u   /* a zero hex digit (S:136-137 design decision) */
#define ORACLE_KEY_EVEN         8u   /* d0 even */
#define ORACLE_KEY_POPCOUNT    16u   /* popcount outside [28,36]: "roughly half ones" */

static int hexdigit(uint64_t key, int i) { return (int)((key >> (4 * i)) & 0xF); }

uint32_t oracle_validate_key(uint64_t key) {
  uint32_t v = 0;
  int i, j, pc = 0;
  for (i = 8; i < 16; i++)
    for (j = i + 1; j < 16; j++)
      if (hexdigit(key, i) == hexdigit(key, j)) v |= ORACLE_KEY_UPPER_REPEAT;
  for (i = 0; i < 8; i++)
    for (j = i + 1; j < 8; j++)
      if (hexdigit(key, i) == hexdigit(key, j)) v |= ORACLE_KEY_LOWER_REPEAT;
  for (i = 0; i < 16; i++)
    if (hexdigit(key, i) == 0) v |= ORACLE_KEY_ZERO_DIGIT;
  if ((hexdigit(key, 0) & 1) == 0) v |= ORACLE_KEY_EVEN;
  for (i = 0; i < 64; i++) pc += (int)((key >> i) & 1);
  if (pc < 28 || pc > 36) v |= ORACLE_KEY_POPCOUNT;
  return v;
}

/* SplitMix64 output finalizer, written from its published description
 * (z ^= z>>30; z *= 0xbf58476d1ce4e5b9; z ^= z>>27; z *= 0x94d049bb133111eb; z ^= z>>31). */
static uint64_t oracle_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* Draw number d of attempt a for key index j under seed s. */
static uint64_t oracle_key_draw(uint64_t seed, uint64_t j, uint64_t a, uint64_t d) {
  uint64_t h = oracle_mix64(seed ^ 0x53515541524553ULL);          /* "SQUARES" */
  h = oracle_mix64(h + (j + 1) * 0x9E3779B97F4A7C15ULL);
  h = oracle_mix64(h + (a + 1) * 0xD1B54A32D192ED03ULL);
  return oracle_mix64(h + (d + 1) * 0x8CB92BA72F3D8DD7ULL);
}

/* Uniform integer in [0, m): floor(r * m / 2^64) (multiply-high; bias < m / 2^64). */
static uint64_t oracle_below(uint64_t r, uint64_t m) {
  return (uint64_t)(((unsigned __int128)r * m) >> 64);
}

/* One candidate key for (seed, j, attempt): digits chosen as DESIGN.md describes. */
uint64_t oracle_key_candidate(uint64_t seed, uint64_t j, uint64_t a) {
  int pool[15], i, n, d = 0;
  int digit[16];
  /* upper half: 8 distinct digits from 1..15 by partial Fisher-Yates; d15 first */
  for (i = 0; i < 15; i++) pool[i] = i + 1;
  for (i = 0; i < 8; i++) {
    int pick = i + (int)oracle_below(oracle_key_draw(seed, j, a, (uint64_t)d++), (uint64_t)(15 - i));
    int t = pool[i]; pool[i] = pool[pick]; pool[pick] = t;
    digit[15 - i] = pool[i];
  }
  /* lower half: d0 from the odd digits {1,3,...,15}; d1..d7 from the other 14 nonzero digits */
  digit[0] = 2 * (int)oracle_below(oracle_key_draw(seed, j, a, (uint64_t)d++), 8) + 1;
  n = 0;
  for (i = 1; i <= 15; i++) if (i != digit[0]) pool[n++] = i;   /* ascending, 14 entries */
  for (i = 0; i < 7; i++) {
    int pick = i + (int)oracle_below(oracle_key_draw(seed, j, a, (uint64_t)d++), (uint64_t)(14 - i));
    int t = pool[i]; pool[i] = pool[pick]; pool[pick] = t;
    digit[1 + i] = pool[i];
  }
  uint64_t key = 0;
  for (i = 0; i < 16; i++) key |= (uint64_t)digit[i] << (4 * i);
  return key;
}

/* keys[j] = the first candidate (attempt 0, 1, ...) that passes oracle_validate_key and
 * differs from keys[0..j-1].  Returns 0 on success, 2 (range) if count > 2^31, 1 if out is
 * NULL with count > 0, 4 on allocation failure.  Duplicate test by a plain linear-probing set. */
int oracle_keygen(uint64_t seed, uint64_t count, uint64_t* out) {
  if (count > (1ULL << 31)) return 2;
  if (count == 0) return 0;
  if (!out) return 1;
  uint64_t cap = 16;
  while (cap < 2 * count) cap <<= 1;
  uint64_t* set = (uint64_t*)calloc(cap, sizeof(uint64_t));   /* 0 = empty (keys are nonzero) */
  if (!set) return 4;
  for (uint64_t j = 0; j < count; j++) {
    for (uint64_t a = 0;; a++) {
      uint64_t key = oracle_key_candidate(seed, j, a);
      if (oracle_validate_key(key) != 0) continue;
      uint64_t h = oracle_mix64(key) & (cap - 1);
      int dup = 0;
      while (set[h] != 0) {
        if (set[h] == key) { dup = 1; break; }
        h = (h + 1) & (cap - 1);
      }
      if (dup) continue;
      set[h] = key;
      out[j] = key;
      break;
    }
  }
  free(set);
  return 0;
}

/* ------------------------------------------------------------------------------------ */
/* Reduced-width analogue: 64 -> W and 32 -> W/2 everywhere.         */
/* ------------------------------------------------------------------------------------ */
uint64_t oracle_squares32_scaled(uint64_t ctr, uint64_t key, int W) {
  uint64_t M = (W == 64) ? ~0ULL : ((1ULL << W) - 1);
  int h = W / 2;
  uint64_t x, y, z;
  ctr &= M; key &= M;
  y = x = (ctr * key) & M; z = (y + key) & M;
  x = (x*x + y) & M; x = ((x >> h) | (x << h)) & M;        /* round 1 */
  x = (x*x + z) & M; x = ((x >> h) | (x << h)) & M;        /* round 2 */
  x = (x*x + y) & M; x = ((x >> h) | (x << h)) & M;        /* round 3 */
  return ((x*x + z) & M) >> h;                              /* round 4 */
}

/* Regularized upper incomplete gamma Q(a, x) (series for x < a+1, continued
 * fraction otherwise).  Textbook forms (Abramowitz & Stegun 6.5.29 series; Legendre
 * continued fraction 6.5.31 evaluated by the modified Lentz method). */
double oracle_gammaq(double a, double x) {
  if (x <= 0.0) return 1.0;
  double lg = lgamma(a);
  if (x < a + 1.0) {
    double ap = a, sum = 1.0 / a, del = sum;
    for (int n = 1; n < 100000; n++) {
      ap += 1.0; del *= x / ap; sum += del;
      if (fabs(del) < fabs(sum) * 1e-16) break;
    }
    double P = sum * exp(-x + a * log(x) - lg);
    return 1.0 - P;
  } else {
    const double tiny = 1e-300;
    double b = x + 1.0 - a, c = 1.0 / tiny, d = 1.0 / b, h = d;
    for (int i = 1; i < 100000; i++) {
      double an = -i * (i - a);
      b += 2.0;
      d = an * d + b; if (fabs(d) < tiny) d = tiny;
      c = b + an / c; if (fabs(c) < tiny) c = tiny;
      d = 1.0 / d;
      double del = d * c;
      h *= del;
      if (fabs(del - 1.0) < 1e-16) break;
    }
    return exp(-x + a * log(x) - lg) * h;
  }
}

/* Histogram of squares32_scaled over the counters [c0, c0 + n) (a piece of the exhaustive
 * enumeration; pieces add up).  hist has 2^(W/2) entries. */
void oracle_scaled_hist_range(uint64_t key, int W, uint64_t c0, uint64_t n, uint64_t* hist) {
  for (uint64_t c = c0; c < c0 + n; c++) hist[oracle_squares32_scaled(c, key, W)]++;
}

/* Exhaustive enumeration of all 2^W counters (W even, 8 <= W <= 24), histogram of the
 * 2^(W/2) outputs, chi-square against uniform; p = Q(df/2, chi2/2).  Returns 0 or 1 (bad W). */
int oracle_scaled_uniformity(uint64_t key, int W, double* chi2_out, double* p_out) {
  if (W < 8 || W > 24 || (W & 1)) return 1;
  uint64_t nb = 1ULL << (W / 2), nc = 1ULL << W;
  uint64_t* h = (uint64_t*)calloc(nb, sizeof(uint64_t));
  if (!h) return 1;
  for (uint64_t c = 0; c < nc; c++) h[oracle_squares32_scaled(c, key, W)]++;
  double e = (double)nc / (double)nb, chi2 = 0.0;
  for (uint64_t b = 0; b < nb; b++) { double d = (double)h[b] - e; chi2 += d * d / e; }
  free(h);
  *chi2_out = chi2;
  *p_out = oracle_gammaq((double)(nb - 1) / 2.0, chi2 / 2.0);
  return 0;
}

/* ------------------------------------------------------------------------------------ */
/* Partition ("If the 2^64 is divided equally among all the cores"):      */
/* start = idx * floor(N / P); the last part absorbs the remainder.  N up to 2^64 is      */
/* passed as (n_hi, n_lo).  Returns 0, or 1 on P == 0 / idx >= P.                        */
/* ------------------------------------------------------------------------------------ */
int oracle_partition(uint64_t n_hi, uint64_t n_lo, uint64_t parts, uint64_t idx,
                     uint64_t* start_hi, uint64_t* start_lo, uint64_t* len_hi, uint64_t* len_lo) {
  if (parts == 0 || idx >= parts) return 1;
  unsigned __int128 N = ((unsigned __int128)n_hi << 64) | n_lo;
  unsigned __int128 q = N / parts;
  unsigned __int128 s = q * idx;
  unsigned __int128 len = (idx == parts - 1) ? (N - s) : q;
  *start_hi = (uint64_t)(s >> 64); *start_lo = (uint64_t)s;
  *len_hi = (uint64_t)(len >> 64); *len_lo = (uint64_t)len;
  return 0;
}
