/*
 * squares.h -- C ABI of libsquares.so, the B200 (sm_100a) bulk evaluator of the Squares
 * counter-based RNG (B. Widynski, arXiv 2004.06278).
 *
 * Citations: P:n = PAPER.md line n (the paper text), S:n = SPEC.md line n.
 *
 *   squares32(ctr, key)  P:21-28 (section 2 listing): y = x = ctr*key; z = y + key;
 *                        rounds x = rot32(x*x + w) with w = y, z, y; return (x*x + z) >> 32.
 *   squares64(ctr, key)  P:56-64 (section 5 listing): rounds 1-3 as above,
 *                        t = x = x*x + z; x = rot32(x); return t ^ ((x*x + y) >> 32).
 *   All arithmetic is mod 2^64 ("uint64_t"); rot32 swaps the 32-bit halves.
 *
 * Conventions for every entry point below:
 *   - Device pointers are CUDA device (or managed) memory of the CURRENT device; host pointers
 *     are ordinary host memory.  The caller owns every buffer; the library allocates nothing
 *     that outlives a call.
 *   - GPU entry points are asynchronous on `stream` (a cudaStream_t; NULL = legacy default
 *     stream).  They only enqueue work: they never synchronize, never change the current
 *     device, and return as soon as the launch is queued.  Asynchronous device faults surface
 *     at the caller's next synchronization.
 *   - All functions are reentrant and may be called concurrently on any number of streams.
 *   - Counters wrap mod 2^64: element i of a fill uses counter ctr0 + i mod 2^64.
 *   - Keys are NOT validated on the GPU paths: the generators are total over (ctr, key).
 *     Validation belongs to sq_validate_key / sq_keygen.
 *   - Return value: SQ_OK, or an error code (nothing is launched when an error is returned).
 */
#ifndef SQUARES_H_
#define SQUARES_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Opaque stream handle, ABI-compatible with cudaStream_t / CUstream. */
typedef struct CUstream_st* sq_stream_t;

/* Status codes. */
#define SQ_OK 0      /* success (also returned, with no launch, when there is nothing to do) */
#define SQ_EINVAL 1  /* bad argument: NULL pointer with work to do, ld < n with nkeys > 1,
                        misaligned output, size overflow */
#define SQ_ERANGE 2  /* argument out of the supported range (e.g. keygen count > 2^31) */
#define SQ_ECUDA 3   /* a CUDA call failed (launch/config error, no device); see sq_last_cuda_error */
#define SQ_ENOMEM 4  /* host allocation failed */

/* Human-readable name of a status code (static string, never NULL). */
const char* sq_strerror(int code);

/* cudaError_t value of the most recent SQ_ECUDA returned on the calling thread (0 if none). */
int sq_last_cuda_error(void);

/* Library ABI version (major*10000 + minor*100 + patch). */
int sq_version(void);

/* ----------------------------------------------------------------------------------------
 * Key utility -- the "different digits" rules of P:37 (section 3):
 *   "The keys are chosen so the the upper 8 digits are different and also that the lower 8
 *    digits are different", "The digits are also chosen randomly", "an irregular bit pattern
 *    with roughly half ones and half zeros".
 * Builder's readings: every hex digit nonzero, the
 * least significant digit odd, and popcount in [28, 36] ("roughly half ones").
 * -------------------------------------------------------------------------------------- */

/* Rule bits returned by sq_validate_key (0 = valid key). */
#define SQ_KEY_UPPER_REPEAT 1u /* two of the upper 8 hex digits are equal */
#define SQ_KEY_LOWER_REPEAT 2u /* two of the lower 8 hex digits are equal */
#define SQ_KEY_ZERO_DIGIT 4u   /* some hex digit is 0 */
#define SQ_KEY_EVEN 8u         /* least significant digit is even */
#define SQ_KEY_POPCOUNT 16u    /* popcount outside [28, 36] ("roughly half ones") */

/* Host only.  Bitmask of the rules above that `key` violates; 0 iff `key` is valid. */
uint32_t sq_validate_key(uint64_t key);

/* Host only.  keys_host[j], j < count, = the j-th key of stream `seed` under the documented
 * deterministic mapping: candidates are drawn digit by digit
 * from a SplitMix64-finalizer hash of (seed, j, attempt, draw); the first candidate that passes
 * sq_validate_key and differs from keys_host[0..j-1] is kept.  Properties: deterministic,
 * prefix-stable (the first k keys do not depend on count), pairwise distinct, all valid.
 * Not sequence-compatible with the paper's unpublished utility (P:37 footnote).
 * Errors: SQ_ERANGE if count > 2^31 ("about 2 billion keys"); SQ_EINVAL if
 * keys_host is NULL with count > 0; SQ_ENOMEM if the O(count) duplicate set cannot be
 * allocated.  count == 0 is SQ_OK. */
int sq_keygen(uint64_t seed, uint64_t count, uint64_t* keys_host);

/* ----------------------------------------------------------------------------------------
 * Bulk fills (BASELINE.json configs 1-4).  Row-major [key][ctr] layout:
 *   out[k*ld + i] = G(ctr0 + i mod 2^64, keys[k])   for k < nkeys, i < n;
 * elements i in [n, ld) of each row are left untouched.
 *   keys_dev  device, nkeys uint64 keys (read only), 8-byte aligned
 *   nkeys     number of rows
 *   ctr0      first counter of every row
 *   n         counters per row
 *   out_dev   device output, must be aligned to its element size; rows of `ld` elements
 *   ld        leading dimension in ELEMENTS (ld >= n required when nkeys > 1; ignored when
 *             nkeys == 1)
 * Returns SQ_OK without launching when n == 0 or nkeys == 0.
 * Errors: SQ_EINVAL on NULL pointers with work to do, ld < n with nkeys > 1, a misaligned
 * out_dev or keys_dev, or nkeys*ld*elem overflowing size_t; SQ_ECUDA if the launch fails.
 * -------------------------------------------------------------------------------------- */

/* G = squares32, uint32 output. */
int sq_fill_u32(const uint64_t* keys_dev, uint64_t nkeys, uint64_t ctr0, uint64_t n,
                uint32_t* out_dev, uint64_t ld, sq_stream_t stream);

/* G = squares64, uint64 output (little-endian words). */
int sq_fill_u64(const uint64_t* keys_dev, uint64_t nkeys, uint64_t ctr0, uint64_t n,
                uint64_t* out_dev, uint64_t ld, sq_stream_t stream);

/* G = (float)(squares32 >> 8) * 2^-24: the top 24 bits of squares32 as a float32 in
 * [0, 1 - 2^-24] (BASELINE.json config 4).  Exact: no rounding occurs. */
int sq_fill_f32(const uint64_t* keys_dev, uint64_t nkeys, uint64_t ctr0, uint64_t n,
                float* out_dev, uint64_t ld, sq_stream_t stream);

/* Single-key fills with the key passed BY VALUE (same map, one row, ld = n).  The key travels
 * in the launch parameters, so the kernel holds it and every per-key constant of the counter
 * walk in uniform registers.  Same errors as above (no keys pointer to check). */
int sq_fill_u32_k(uint64_t key, uint64_t ctr0, uint64_t n, uint32_t* out_dev, sq_stream_t stream);
int sq_fill_u64_k(uint64_t key, uint64_t ctr0, uint64_t n, uint64_t* out_dev, sq_stream_t stream);
int sq_fill_f32_k(uint64_t key, uint64_t ctr0, uint64_t n, float* out_dev, sq_stream_t stream);

/* ----------------------------------------------------------------------------------------
 * Output kinds and the generic fill (squares64-derived floats, strided
 * counters).  Kinds:
 *   SQ_KIND_U32    squares32, uint32                                  4 bytes
 *   SQ_KIND_U64    squares64, uint64                                  8 bytes
 *   SQ_KIND_F32    (float)(squares32 >> 8) * 2^-24 in [0,1)  (BASELINE.json config 4)   4 bytes
 *   SQ_KIND_F64    (double)(squares64 >> 11) * 2^-53 in [0,1) ("53-bit precision floating
 *                  point"; formula S:260), exact                          8 bytes
 *   SQ_KIND_F32X2  squares64 split into two 32-bit halves, each (h >> 8) * 2^-24, LOW half
 *                  first ("splits the 64 bits into two 32-bit halves"; order S:269).
 *                  One element = a pair of floats (8 bytes): n counters give 2n floats and
 *                  `ld` counts pairs.
 * All conversions are exact (no rounding): the integer fits the float's significand and the
 * scale is a power of two.
 * -------------------------------------------------------------------------------------- */
#define SQ_KIND_U32 0
#define SQ_KIND_U64 1
#define SQ_KIND_F32 2
#define SQ_KIND_F64 3
#define SQ_KIND_F32X2 4

int sq_fill_f64(const uint64_t* keys_dev, uint64_t nkeys, uint64_t ctr0, uint64_t n,
                double* out_dev, uint64_t ld, sq_stream_t stream);
int sq_fill_f32x2(const uint64_t* keys_dev, uint64_t nkeys, uint64_t ctr0, uint64_t n,
                  float* out_dev, uint64_t ld, sq_stream_t stream);
int sq_fill_f64_k(uint64_t key, uint64_t ctr0, uint64_t n, double* out_dev, sq_stream_t stream);
int sq_fill_f32x2_k(uint64_t key, uint64_t ctr0, uint64_t n, float* out_dev, sq_stream_t stream);

/* Generic fill: out[k*ld + i] = G_kind(ctr0 + i*stride mod 2^64, key_k) where key_k =
 * keys_dev[k] (k < nkeys), or, when keys_dev is NULL, the single key `key_imm` (nkeys must
 * be 1).  stride = 1 is the consecutive walk of the fills above; stride > 1 evaluates "counter
 * tests with increments other than one".  stride = 0 is rejected (SQ_EINVAL:
 * use sq_fill_keyctr for a fixed counter).  Other errors as for sq_fill_u32. */
int sq_fill_ex(int kind, const uint64_t* keys_dev, uint64_t nkeys, uint64_t key_imm, uint64_t ctr0,
               uint64_t stride, uint64_t n, void* out_dev, uint64_t ld, sq_stream_t stream);

/* Key-counter mode ("the counter was fixed and only the key changed"):
 * out[j] = G_kind(ctr, keys_dev[j]) for j < nkeys, densely packed (element size of `kind`).
 * nkeys == 0 is SQ_OK without a launch; NULL pointers or a misaligned out_dev: SQ_EINVAL. */
int sq_fill_keyctr(int kind, const uint64_t* keys_dev, uint64_t nkeys, uint64_t ctr, void* out_dev,
                   sq_stream_t stream);

/* CUDA graphs: every device entry point only enqueues work on `stream` (no synchronisation, no
 * allocation, no host callback), so calls can be captured into a CUDA graph and replayed
 * (tests/test_gpu_graph.py); per-(device, kernel) attributes are set on the first call, so make
 * one eager call before capturing.  In the launch-bound small-n regime a replayed fill of 2^20
 * samples costs ~2.6 us vs ~7 us issued eagerly from Python (tools/small_n.py). */

/* ----------------------------------------------------------------------------------------
 * Fused generate-and-reduce (BASELINE.json config 5; the GPU analogue of P:45's "basic
 * uniformity test").  With u_i = squares32(ctr0 + i mod 2^64, key), i < n, ACCUMULATES
 *   hist_dev[b] += #{i : u_i >> 16 == b}            b < 65536
 *   ones_dev[j] += #{i : (u_i >> j) & 1 == 1}        j < 32, j = 0 the least significant bit
 * into caller-initialised device arrays (uint64).  No sample is stored.  Accumulation makes
 * chunked and sharded runs compose by addition.  hist_dev and ones_dev must be 8-byte aligned.
 * Any n < 2^64 (runs above 2^48 samples are split into several launches internally).
 * Returns SQ_OK without launching when n == 0.  Errors: SQ_EINVAL (NULL / misaligned),
 * SQ_ECUDA (launch failure).
 * -------------------------------------------------------------------------------------- */
int sq_fused_stats(uint64_t key, uint64_t ctr0, uint64_t n, uint64_t* hist_dev,
                   uint64_t* ones_dev, sq_stream_t stream);

/* Fused statistics over the strided counters ctr0 + i*stride (i < n; stride >= 1) with an
 * optional output transform: flags & SQ_FUSED_BITREV counts bitrev32(u_i) instead of u_i
 * ("bits-reversed tests"), i.e. hist over the reversed low 16 bits.
 * stride = 0 or unknown flag bits: SQ_EINVAL. */
#define SQ_FUSED_BITREV 1u
int sq_fused_stats_ex(uint64_t key, uint64_t ctr0, uint64_t stride, uint64_t n, uint32_t flags,
                      uint64_t* hist_dev, uint64_t* ones_dev, sq_stream_t stream);

/* Bit transitions of the output stream, for the runs statistic of the desk battery:
 * with u_i = squares32(ctr0 + i*stride, key) (bit-reversed if flags & SQ_FUSED_BITREV) read
 * least-significant bit first, ACCUMULATES into *count_dev (uint64, 8-byte aligned)
 *   sum_i popc((u_i ^ (u_i >> 1)) & 0x7FFFFFFF) + sum_{0<i<n} [bit31(u_{i-1}) != bit0(u_i)],
 * i.e. (number of runs) - 1 of the 32n-bit stream.  Errors as for sq_fused_stats_ex. */
int sq_transitions(uint64_t key, uint64_t ctr0, uint64_t stride, uint64_t n, uint32_t flags,
                   uint64_t* count_dev, sq_stream_t stream);

/* Exhaustive reduced-width uniformity (the desk-scale stand-in for
 * footnote 1 of P:17, "The probability of any given output is 1/2^32").  For each key k < nkeys
 * (taken mod 2^W) and EVERY counter c in [0, 2^W), evaluates the W-bit analogue of squares32
 * (64 -> W and 32 -> W/2 in every square, add, rotation and the final shift) and ACCUMULATES
 *   hist_dev[k * 2^(W/2) + v] += #{c : squares32_scaled(c, key_k, W) == v}
 * into caller-zeroed uint64 device memory (nkeys * 2^(W/2) entries).  W even in [8, 32], else
 * SQ_EINVAL; nkeys <= 65535 per call (else SQ_ERANGE). */
int sq_scaled_hist(int W, const uint64_t* keys_dev, uint64_t nkeys, uint64_t* hist_dev, sq_stream_t stream);

/* ----------------------------------------------------------------------------------------
 * Host-buffer fill (the end-to-end path): the same map as sq_fill_u32 / sq_fill_u64 /
 * sq_fill_f32 for ONE key, written to HOST memory.  The library generates chunks of
 * `chunk_elems` elements into the caller's device scratch (two ping-pong halves of
 * scratch_bytes) and copies each chunk to out_host with cudaMemcpyAsync on `stream`,
 * overlapping generation of chunk c+1 with the copy of chunk c via `copy_stream`.  The call is
 * SYNCHRONOUS: it returns after out_host holds all n elements.  out_host should be pinned
 * (cudaHostAlloc / cudaHostRegister) for full PCIe bandwidth.
 *   kind        SQ_KIND_* (0 = u32, 1 = u64, 2 = f32, 3 = f64, 4 = f32x2)
 *   key         the key (host value)
 *   scratch_dev device scratch, aligned to the element size; the library starts its two
 *               halves at the first 32-byte boundary inside it, so it needs >= 2 * 32 bytes
 *               plus that offset (256-byte aligned recommended)
 * Errors: SQ_EINVAL (bad kind, NULL pointers with n > 0, scratch misaligned to the element
 * size or too small), SQ_ECUDA.
 * -------------------------------------------------------------------------------------- */
int sq_fill_host(int kind, uint64_t key, uint64_t ctr0, uint64_t n, void* out_host,
                 void* scratch_dev, size_t scratch_bytes, sq_stream_t stream,
                 sq_stream_t copy_stream);

#ifdef __cplusplus
}
#endif

#endif /* SQUARES_H_ */
