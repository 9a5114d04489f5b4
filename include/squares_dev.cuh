// squares_dev.cuh -- header-only DEVICE API of the Squares counter-based RNG (B. Widynski,
// arXiv 2004.06278) for sm_100a, and the arithmetic core of libsquares.so's kernels.
//
// Use inside your own kernels ("This generator would be used in a similar way as Philox",
// PAPER.md P:33):
//     #include "squares_dev.cuh"
//     uint32_t r = sq::squares32(ctr, key);
//     uint64_t s = sq::squares64(ctr, key);
//     sq::Stream st(ctr0, key);                       // consecutive counters, Weyl-stepped
//     float f = st.next_f32();  uint32_t u = st.next_u32();  st.skip(1 << 20);
//
// The listings square a 64-bit x mod 2^64, add y = ctr*key or z = y + key, and rotate by 32.
// This header evaluates the same map with 32-bit integer-multiply instructions, in a different
// ORDER of operations (never a different result):
//
//  * x*x mod 2^64 with x = xh*2^32 + xl is xl*xl + (2*xl*xh mod 2^32)*2^32.  One round
//    x <- rot32(x*x + w) is therefore
//        {lo, hi} = xl*xl + w            (IMAD.WIDE.U32 with the 64-bit addend folded in)
//        hi      += xl * (2*xh)          (IMAD)
//        (xh, xl) = (lo, hi)             (the rotation is a register rename, 0 instructions)
//  * Round 1's input is y itself ("y = x = ctr * key"), so round 1's sum is
//        u(c) = y^2 + y,  y = c*key  --  a quadratic polynomial in the counter c.
//    Along consecutive counters it is stepped exactly by finite differences (all mod 2^64):
//        y(c+1) = y(c) + key                       (the Weyl step)
//        u(c+1) = u(c) + e(c),   e(c) = 2*key*y(c) + key^2 + key
//        e(c+1) = e(c) + 2*key^2
//    so round 1 costs 64-bit adds and no multiply.  z(c) = y(c) + key = y(c+1).
//  * A jump of J counters (J a power of two) is also multiply-free:
//        y += J*key;  u += J*e + J(J-1)*key^2;  e += J*2*key^2,   J*e = e << log2(J).
//
// Per squares32 sample: rounds 2-4 = 2 IMAD.WIDE.U32 + 1 IMAD.HI.U32 + 3 IMAD (9 FMA-heavy
// pipe slots: IMAD 64 lanes/clk/SM, WIDE/HI 2 slots each -- 24-27 lanes/clk/SM measured in
// dependent loops on B200) plus 3 doublings and the two 64-bit walk adds.  squares64 adds
// round 4's full sum and round 5.  A Stream draw runs at ~1.33 Tsamples/s per B200 when the
// value is consumed in registers (tools/bench_next.py).
#pragma once
#include <stdint.h>

namespace sq {

// NOTE: written as plain C on purpose.  ptxas (CUDA 12.9, sm_100a) folds the 64-bit addend of
// `(uint64_t)a * b + c` into one IMAD.WIDE.U32 (or IMAD.HI.U32 when only the high word is
// used), but splits an inline-PTX `mad.wide.u32` into IMAD.WIDE + IADD3 + IADD3.X/IMAD.X,
// which costs two extra ops per round (checked with tools/sass_mix.py).
__device__ __forceinline__ uint64_t mad_wide(uint32_t a, uint32_t b, uint64_t c) {
  return (uint64_t)a * b + c;
}

__device__ __forceinline__ uint32_t mad_lo(uint32_t a, uint32_t b, uint32_t c) { return a * b + c; }

__device__ __forceinline__ uint32_t lo32(uint64_t v) { return (uint32_t)v; }
__device__ __forceinline__ uint32_t hi32(uint64_t v) { return (uint32_t)(v >> 32); }

// 64-bit add through inline PTX: opaque to NVVM's induction-variable analysis, which would
// otherwise rewrite the stepped sequences into closed forms (u_j = u_0 + j*e_0 + ...) that
// cost extra IMADs on the FMA-heavy pipe -- the pipe that bounds this kernel.
__device__ __forceinline__ uint64_t add64(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.u64 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// a + b + c mod 2^64 (one IADD3 with two carry-outs + one IADD3.X).
__device__ __forceinline__ uint64_t add64_3(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("add.u64 %0, %1, %2;\n\tadd.u64 %0, %0, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

// hi + lo32(2 * xl * xh): the cross term of a square.  `one` is the value 1 held in a register
// the compiler cannot see through (a kernel argument); FORM selects the instruction shape:
//   0  IMAD(xl, xh << 1, hi)                 -- the shortest form; ptxas may place the doubling
//                                               on the IMAD pipe
//   1  IMAD(xl, xh << one, hi)               -- the doubling is a variable shift: ALU only
//   2  hi + ((xl * xh) << one)               -- IMAD without addend runs beside the round's
//                                               IMAD.WIDE; only an IADD3 follows the WIDE on the
//                                               dependency chain (shorter latency per round)
//   3  IMAD(xl, SHF(RZ:xh, 1), hi)           -- the doubling as a funnel shift with an immediate
//                                               amount: ALU pipe, one register read
//   6  hi + ((xl * xh) << 1)                 -- product first, doubling and add after it (LEA)
//   +8 (round_rot only) the square's 64-bit addend added through an explicit carry chain (see
//      round_rot): removes the VIADD copy ptxas otherwise puts after every IMAD.WIDE.U32
// Measured on B200, per round 2 / 3 / 4: 11 / 11 / 3 for the library's 32-bit
// fills, 14 / 14 / 3 for the fused statistics walk, 14 / 14 / 6 for Stream::next_u32; form 0
// is the default of squares32_from / squares64_from.
#ifndef SQ_ROUND_FORM
#define SQ_ROUND_FORM 0
#endif
template <int FORM = SQ_ROUND_FORM>
__device__ __forceinline__ uint32_t cross_add(uint32_t xl, uint32_t xh, uint32_t hi, uint32_t one) {
  if (FORM == 0) return mad_lo(xl, xh << 1, hi);
  if (FORM == 6) {
    // hi + ((xl * xh) << 1): the product without the doubling (IMAD with no addend, off the
    // chain through the IMAD.WIDE), then shift-and-add; ptxas emits LEA / IMAD-by-2 forms here
    uint32_t p, r;
    asm("mul.lo.u32 %0, %1, %2;" : "=r"(p) : "r"(xl), "r"(xh));
    asm("shl.b32 %0, %1, 1;\n\tadd.u32 %0, %0, %2;" : "=r"(r) : "r"(p), "r"(hi));
    return r;
  }
  uint32_t d;
  if (FORM == 3) {
    asm("shf.l.clamp.b32 %0, 0, %1, 1;" : "=r"(d) : "r"(xh));
    return mad_lo(xl, d, hi);
  }
  if (FORM == 1) {
    asm("shl.b32 %0, %1, %2;" : "=r"(d) : "r"(xh), "r"(one));
    return mad_lo(xl, d, hi);
  }
  uint32_t c;
  asm("mul.lo.u32 %0, %1, %2;" : "=r"(c) : "r"(xl), "r"(xh));
  asm("shl.b32 %0, %1, %2;" : "=r"(d) : "r"(c), "r"(one));
  asm("add.u32 %0, %1, %2;" : "=r"(c) : "r"(hi), "r"(d));
  return c;
}

// x <- rot32(x*x + w), x held as (xh, xl).  P:24-26.
template <int FORM = SQ_ROUND_FORM>
__device__ __forceinline__ void round_rot(uint32_t& xh, uint32_t& xl, uint64_t w, uint32_t one = 1) {
  if (FORM & 8) {
    // +8: the 64-bit sum xl*xl + w written as a 32-bit product pair and an explicit add.cc /
    // addc carry chain (PTX), the cross term then in form FORM & 7.  ptxas still emits ONE
    // IMAD.WIDE.U32 with the addend folded in, but no longer inserts the VIADD copy of its high
    // register before the cross-term instruction (measured: u32 fill 15.25 -> 14.06 SASS
    // instructions per sample, c2 +5 %, c4 +6 %).
    uint32_t plo, phi, tlo, thi;
    asm("mul.lo.u32 %0, %2, %2;\n\tmul.hi.u32 %1, %2, %2;" : "=r"(plo), "=r"(phi) : "r"(xl));
    asm("add.cc.u32 %0, %2, %4;\n\taddc.u32 %1, %3, %5;"
        : "=r"(tlo), "=r"(thi) : "r"(plo), "r"(phi), "r"(lo32(w)), "r"(hi32(w)));
    const uint32_t hi = cross_add<(FORM & 7)>(xl, xh, thi, one);
    xh = tlo;
    xl = hi;
    return;
  }
  uint64_t t = mad_wide(xl, xl, w);
  uint32_t hi = cross_add<FORM>(xl, xh, hi32(t), one);
  xh = lo32(t);
  xl = hi;
}

// High 32 bits of x*x + w (the final extraction of P:27 and P:63).
template <int FORM = SQ_ROUND_FORM>
__device__ __forceinline__ uint32_t round_hi(uint32_t xh, uint32_t xl, uint64_t w, uint32_t one = 1) {
  uint64_t t = mad_wide(xl, xl, w);   // IMAD.HI: its result needs no copy, so the +8 bit is moot
  return cross_add<(FORM & 7)>(xl, xh, hi32(t), one);
}

// squares32 given y = ctr*key, z = y + key and u = y*y + y (round 1's sum).  P:21-28.
template <int FORM = SQ_ROUND_FORM>
__device__ __forceinline__ uint32_t squares32_from(uint64_t y, uint64_t z, uint64_t u, uint32_t one = 1) {
  uint32_t xh = lo32(u), xl = hi32(u);  // round 1: rot32(u)
  round_rot<FORM>(xh, xl, z, one);      // round 2
  round_rot<FORM>(xh, xl, y, one);      // round 3
  return round_hi<FORM>(xh, xl, z, one);  // round 4
}

// squares32 with a cross-term form per round (F2, F3, F4 for rounds 2, 3, 4): lets a kernel
// balance the doublings between the ALU and FMA pipes.  Same result as squares32_from.
template <int F2, int F3, int F4>
__device__ __forceinline__ uint32_t squares32_mix(uint64_t y, uint64_t z, uint64_t u, uint32_t one = 1) {
  uint32_t xh = lo32(u), xl = hi32(u);
  round_rot<F2>(xh, xl, z, one);
  round_rot<F3>(xh, xl, y, one);
  return round_hi<F4>(xh, xl, z, one);
}

// squares64 given y, z, u as above.  P:56-64: t = x*x + z (round 4, kept before rotating),
// result t ^ ((rot32(t)^2 + y) >> 32); only t's low half changes.
template <int FORM = SQ_ROUND_FORM>
__device__ __forceinline__ uint64_t squares64_from(uint64_t y, uint64_t z, uint64_t u, uint32_t one = 1) {
  uint32_t xh = lo32(u), xl = hi32(u);
  round_rot<FORM>(xh, xl, z, one);      // round 2
  round_rot<FORM>(xh, xl, y, one);      // round 3
  // round 4 (full 64-bit sum): round_rot without the rotation -- after it (xh, xl) holds
  // (lo, hi) of t, i.e. rot32(t), which is exactly round 5's input
  round_rot<FORM>(xh, xl, z, one);
  const uint32_t tl = xh, th = xl;
  const uint32_t r5 = round_hi<FORM>(tl, th, y, one);  // round 5 on rot32(t) = (tl, th)
  return ((uint64_t)th << 32) | (uint64_t)(tl ^ r5);
}

// Finite-difference state at counter c for key k (see header comment).
struct State {
  uint64_t y;  // c*k
  uint64_t u;  // y*y + y
  uint64_t e;  // u(c+1) - u(c) = 2*k*y + k*k + k
};

__device__ __forceinline__ State state_at(uint64_t c, uint64_t k) {
  State s;
  s.y = c * k;
  s.u = s.y * s.y + s.y;
  s.e = 2 * k * s.y + k * k + k;
  return s;
}

// Strided walk (counter c, c + stride, c + 2*stride, ...): y steps by K = stride*k, so
// u(i+1) - u(i) = 2*K*y(i) + K^2 + K and the second difference is 2*K^2.  (z = y + k still
// uses the key itself.)
__device__ __forceinline__ State state_at_strided(uint64_t c, uint64_t k, uint64_t K) {
  State s;
  s.y = c * k;
  s.u = s.y * s.y + s.y;
  s.e = 2 * K * s.y + K * K + K;
  return s;
}

// One counter forward.  k2x2 = 2*k*k.
__device__ __forceinline__ void step(State& s, uint64_t k, uint64_t k2x2) {
  s.y = add64(s.y, k);
  s.u = add64(s.u, s.e);
  s.e = add64(s.e, k2x2);
}

// Jump by J = 2^LOGJ counters.  jk = J*k, cj = J*(J-1)*k*k, dj = J*2*k*k (all mod 2^64).
template <int LOGJ>
__device__ __forceinline__ void jump(State& s, uint64_t jk, uint64_t cj, uint64_t dj) {
  s.u = add64_3(s.u, s.e << LOGJ, cj);
  s.y = add64(s.y, jk);
  s.e = add64(s.e, dj);
}

// (u >> 8) * 2^-24: top 24 bits of u as a float in [0, 1).  Exact (BASELINE.json config 4).
__device__ __forceinline__ float u32_to_unit_f32(uint32_t u) {
  return __uint2float_rn(u >> 8) * 0x1p-24f;
}

// (v >> 11) * 2^-53: top 53 bits of a squares64 output as a double in [0, 1).  Exact.
__device__ __forceinline__ double u64_to_unit_f64(uint64_t v) {
  return __ull2double_rn(v >> 11) * 0x1p-53;
}

// ---------------------------------------------------------------------------------------
// Direct evaluation of one (ctr, key) pair (no walk): y = ctr*key (a full 64x64 product) and
// round 1 as a square; then the same rounds.  P:21-28 / P:56-64.
__device__ __forceinline__ uint32_t squares32(uint64_t ctr, uint64_t key) {
  const uint64_t y = ctr * key;
  return squares32_from(y, y + key, y * y + y);
}

__device__ __forceinline__ uint64_t squares64(uint64_t ctr, uint64_t key) {
  const uint64_t y = ctr * key;
  return squares64_from(y, y + key, y * y + y);
}

// Cross-term forms per round of Stream::next_u32 (rounds 2, 3, 4): the carry-chain addend with
// the product-first cross term in rounds 2-3 (14 = 8 + 6), form 6 in round 4.  Measured on
// B200 (XOR-folded draws, 303104 threads x 4096): 14/14/6 1327 Gsamples/s, 14/14/2 1326,
// 0/0/0 1256, 14/14/0 1253, 11/11/3 1240, 14/14/3 1234.
#ifndef SQ_STREAM_MIX2
#define SQ_STREAM_MIX2 14
#define SQ_STREAM_MIX3 14
#define SQ_STREAM_MIX4 6
#endif
// A per-thread stream over consecutive counters ctr, ctr+1, ... of one key (the batch of
// n sequential draws equal the batch evaluation).  Each draw costs the round
// multiplies only; the counter walk is the Weyl/finite-difference step.  Counters wrap mod
// 2^64.  skip(n) is O(1) (a fresh state at the new counter).
class Stream {
 public:
  __device__ __forceinline__ Stream(uint64_t ctr, uint64_t key) : ctr_(ctr), key_(key), k2x2_(2 * key * key) {
    s_ = state_at(ctr, key);
  }
  __device__ __forceinline__ uint32_t next_u32() {
    const uint64_t z = add64(s_.y, key_);
    const uint32_t o = squares32_mix<SQ_STREAM_MIX2, SQ_STREAM_MIX3, SQ_STREAM_MIX4>(s_.y, z, s_.u);
    advance();
    return o;
  }
  __device__ __forceinline__ uint64_t next_u64() {
    const uint64_t z = add64(s_.y, key_);
    const uint64_t o = squares64_from(s_.y, z, s_.u);
    advance();
    return o;
  }
  __device__ __forceinline__ float next_f32() { return u32_to_unit_f32(next_u32()); }
  __device__ __forceinline__ double next_f64() { return u64_to_unit_f64(next_u64()); }
  __device__ __forceinline__ void skip(uint64_t n) {
    ctr_ += n;
    s_ = state_at(ctr_, key_);
  }
  __device__ __forceinline__ uint64_t counter() const { return ctr_; }

 private:
  __device__ __forceinline__ void advance() {
    step(s_, key_, k2x2_);
    ctr_ += 1;
  }
  State s_;
  uint64_t ctr_, key_, k2x2_;
};

}  // namespace sq

