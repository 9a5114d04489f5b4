// M1 microbenchmarks: pipe rates that set the roofline
// denominators for the squares kernels on B200 (sm_100a).
//
//   IMAD / IMAD.WIDE.U32 / IMAD.HI.U32 / IADD3 / LOP3 / I2F lane-ops per clock per SM,
//   the squaring-round instruction mix, ATOMS.ADD on a 128 KiB shared table
//   (random and conflict-free addresses), and write-only HBM bandwidth
//   (cudaMemsetAsync, STG.128, STG.256, with and without the .cs hint).
//
// Standalone executable; prints one JSON object on stdout.  Not part of the product path.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o tools/microbench tools/microbench.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <algorithm>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

enum Op { OP_IMAD, OP_WIDE, OP_HI, OP_IADD, OP_LOP3, OP_I2F, OP_ROUND, OP_SHL, OP_WIDEF, OP_HI64, OP_IADD64 };

template <int OP>
__global__ void k_pipe(uint32_t* out, int iters, unsigned long long* cyc) {
  uint32_t a[8];
  uint64_t w[8];
  uint32_t m = 0x9E3779B9u ^ threadIdx.x, c = 12345u + blockIdx.x;
#pragma unroll
  for (int j = 0; j < 8; j++) { a[j] = threadIdx.x * 7 + j; w[j] = ((uint64_t)a[j] << 32) | (a[j] * 3u); }
  float f[8];
#pragma unroll
  for (int j = 0; j < 8; j++) f[j] = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 8; j++) {
      // every chain depends on a neighbouring chain so ptxas cannot fold or hoist it
      const int j1 = (j + 1) & 7, j2 = (j + 2) & 7;
      if (OP == OP_IMAD) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[j]) : "r"(m), "r"(a[j1]));
      if (OP == OP_WIDE) {
        uint32_t lo = (uint32_t)w[j], hi = (uint32_t)(w[j] >> 32);
        asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(w[j]) : "r"(lo), "r"(hi ^ (uint32_t)w[j1]));
      }
      if (OP == OP_WIDEF) {  // folded 64-bit addend (plain C so ptxas emits IMAD.WIDE.U32 d, a, b, c64)
        w[j] = (uint64_t)(uint32_t)w[j] * (uint32_t)(w[j1] >> 32) + w[j2];
      }
      if (OP == OP_HI64) {   // high word of a*b + c64: IMAD.HI.U32 with a 64-bit addend
        a[j] = (uint32_t)(((uint64_t)a[j] * a[j1] + w[j]) >> 32);
      }
      if (OP == OP_IADD64) { // 64-bit add chain (IADD3 + IADD3.X or IMAD.X)
        w[j] = w[j] + w[j1];
      }
      if (OP == OP_HI)   asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(a[j]) : "r"(m), "r"(a[j1]));
      if (OP == OP_IADD) asm volatile("add.u32 %0, %0, %1;" : "+r"(a[j]) : "r"(a[j1]));
      if (OP == OP_LOP3) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[j]) : "r"(a[j1]), "r"(a[j2]));
      if (OP == OP_SHL)  asm volatile("shf.l.wrap.b32 %0, %0, %1, %2;" : "+r"(a[j]) : "r"(a[j1]), "r"(a[j2]));
      if (OP == OP_I2F) {
        float t;
        asm volatile("cvt.rn.f32.u32 %0, %1;" : "=f"(t) : "r"(a[j]));
        f[j] += t;  // FADD on the FMA pipe; compare with the I2F-only rate
        a[j] ^= m;
      }
      if (OP == OP_ROUND) {
        // one squaring round: {lo,hi} = xl*xl + w (IMAD.WIDE), hi += xl*(2xh) (IMAD), swap
        uint32_t xl = (uint32_t)(w[j] >> 32), xh = (uint32_t)w[j];
        uint64_t t;
        asm volatile("mad.wide.u32 %0, %1, %1, %2;" : "=l"(t) : "r"(xl), "l"(w[(j + 1) & 7]));
        uint32_t lo = (uint32_t)t, hi = (uint32_t)(t >> 32);
        asm volatile("mad.lo.u32 %0, %1, %2, %0;" : "+r"(hi) : "r"(xl), "r"(xh << 1));
        w[j] = ((uint64_t)lo << 32) | hi;
      }
    }
  }
  long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int j = 0; j < 8; j++) s += a[j] + (uint32_t)w[j] + (uint32_t)(w[j] >> 32) + __float_as_uint(f[j]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = (unsigned long long)(t1 - t0);
}

// ATOMS on a 32768-word (128 KiB) shared table.  MODE 0: random address, return value used.
// MODE 1: random address, no return (red).  MODE 2: conflict-free (lane-strided), return used.
template <int MODE>
__global__ void k_atoms(uint32_t* out, int iters, unsigned long long* cyc) {
  extern __shared__ uint32_t tab[];
  for (int i = threadIdx.x; i < 32768; i += blockDim.x) tab[i] = 0;
  __syncthreads();
  uint32_t st = 0x12345u * (threadIdx.x + 1) + blockIdx.x * 977u, acc = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 4; j++) {
      st = st * 1664525u + 1013904223u;
      uint32_t addr = (MODE == 2) ? (((st >> 20) & ~31u) | (threadIdx.x & 31)) & 32767u : (st >> 17);
      if (MODE == 1) {
        asm volatile("red.shared.add.u32 [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(&tab[addr])), "r"(1u) : "memory");
      } else {
        uint32_t old;
        asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"((uint32_t)__cvta_generic_to_shared(&tab[addr])), "r"(1u) : "memory");
        acc += old;
      }
    }
  }
  long long t1 = clock64();
  __syncthreads();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc + tab[threadIdx.x];
  if (threadIdx.x == 0) cyc[blockIdx.x] = (unsigned long long)(t1 - t0);
}

template <int VEC, bool CS>
__global__ void k_write(uint32_t* out, size_t nwords) {
  size_t nvec = nwords / VEC;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  uint32_t v = threadIdx.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < nvec; i += stride) {
    uint32_t* p = out + i * VEC;
    uint32_t a = v + (uint32_t)i;
    if (VEC == 4) {
      if (CS) asm volatile("st.global.cs.v4.b32 [%0], {%1,%2,%3,%4};" :: "l"(p), "r"(a), "r"(a+1), "r"(a+2), "r"(a+3) : "memory");
      else    asm volatile("st.global.v4.b32 [%0], {%1,%2,%3,%4};" :: "l"(p), "r"(a), "r"(a+1), "r"(a+2), "r"(a+3) : "memory");
    } else {
      if (CS) asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" :: "l"(p), "r"(a), "r"(a+1), "r"(a+2), "r"(a+3), "r"(a+4), "r"(a+5), "r"(a+6), "r"(a+7) : "memory");
      else    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" :: "l"(p), "r"(a), "r"(a+1), "r"(a+2), "r"(a+3), "r"(a+4), "r"(a+5), "r"(a+6), "r"(a+7) : "memory");
    }
  }
}


// Each warp owns one contiguous range of 32*VEC-word chunks (the fill kernels' decomposition).
template <int VEC>
__global__ void k_write_warpseg(uint32_t* out, size_t nwords) {
  size_t chunks = nwords / (32 * VEC);
  size_t nw = (size_t)gridDim.x * (blockDim.x / 32);
  size_t w = (size_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  size_t c0 = w * chunks / nw, c1 = (w + 1) * chunks / nw;
  uint32_t lane = threadIdx.x & 31, a = lane;
  for (size_t c = c0; c < c1; c++) {
    uint32_t* p = out + (c * 32 + lane) * VEC;
    a += 3;
    if (VEC == 4) asm volatile("st.global.v4.b32 [%0], {%1,%2,%3,%4};" :: "l"(p), "r"(a), "r"(a+1), "r"(a+2), "r"(a+3) : "memory");
    else asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" :: "l"(p), "r"(a), "r"(a+1), "r"(a+2), "r"(a+3), "r"(a+4), "r"(a+5), "r"(a+6), "r"(a+7) : "memory");
  }
}

// TMA bulk store (cp.async.bulk.global.shared::cta): each CTA streams one smem tile
// over its contiguous range; one thread issues, up to all groups in flight.
template <int TILE>
__global__ void k_write_bulk(uint32_t* out, size_t nwords) {
  __shared__ __align__(128) uint32_t tile[TILE / 4];
  for (int i = threadIdx.x; i < TILE / 4; i += blockDim.x) tile[i] = i * 2654435761u;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  size_t tiles = nwords * 4 / TILE;
  size_t t0 = (size_t)blockIdx.x * tiles / gridDim.x, t1 = (size_t)(blockIdx.x + 1) * tiles / gridDim.x;
  if (threadIdx.x == 0) {
    uint32_t s = (uint32_t)__cvta_generic_to_shared(tile);
    for (size_t t = t0; t < t1; t++) {
      char* g = (char*)out + t * TILE;
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" :: "l"(g), "r"(s), "r"(TILE) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 8;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

// Data-dependence probe: MODE 0 constant 0, MODE 1 constant pattern, MODE 2 hashed (random-looking),
// MODE 3 hashed + L2 evict_first policy, MODE 4 hashed + .L1::no_allocate.
template <int MODE>
__global__ void k_write_data(uint32_t* out, size_t nwords) {
  size_t chunks = nwords / (32 * 8);
  size_t nw = (size_t)gridDim.x * (blockDim.x / 32);
  size_t w = (size_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  size_t c0 = w * chunks / nw, c1 = (w + 1) * chunks / nw;
  uint32_t lane = threadIdx.x & 31;
  uint64_t pol = 0;
  if (MODE == 3) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  for (size_t c = c0; c < c1; c++) {
    uint32_t* p = out + (c * 32 + lane) * 8;
    uint32_t v[8];
#pragma unroll
    for (int j = 0; j < 8; j++) {
      uint32_t h = (uint32_t)(c * 256 + lane * 8 + j) * 0x9E3779B1u;
      h ^= h >> 15; h *= 0x85EBCA77u; h ^= h >> 13;
      v[j] = MODE == 0 ? 0u : MODE == 1 ? 0x01010101u : h;
    }
    if (MODE == 3)
      asm volatile("st.global.L2::cache_hint.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8}, %9;" :: "l"(p), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "l"(pol) : "memory");
    else if (MODE == 4)
      asm volatile("st.global.L1::no_allocate.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" :: "l"(p), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]) : "memory");
    else
      asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" :: "l"(p), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]) : "memory");
  }
}

static int g_sms = 0;

template <typename K>
static double run_pipe(K kern, const char* name, int lane_ops_per_iter_per_thread, int threads, int blocks_per_sm,
                       int iters, size_t smem, double* clk_ghz_out, bool first) {
  int blocks = g_sms * blocks_per_sm;
  uint32_t* out; unsigned long long* cyc;
  CK(cudaMalloc(&out, (size_t)blocks * threads * 4));
  CK(cudaMalloc(&cyc, blocks * 8));
  if (smem) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<<<blocks, threads, smem>>>(out, iters, cyc);  // warm
  CK(cudaDeviceSynchronize());
  double best = 0, clk = 0;
  for (int rep = 0; rep < 3; rep++) {
    cudaEventRecord(e0);
    kern<<<blocks, threads, smem>>>(out, iters, cyc);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    std::vector<unsigned long long> h(blocks);
    CK(cudaMemcpy(h.data(), cyc, blocks * 8, cudaMemcpyDeviceToHost));
    double mean = 0; unsigned long long mx = 0;
    for (auto v : h) { mean += v; mx = std::max(mx, v); }
    mean /= blocks;
    double total = (double)blocks * threads * iters * lane_ops_per_iter_per_thread;
    double per_sm_clk = total / g_sms / (double)mx;
    double c = (double)mx / (ms * 1e6);  // GHz, slowest block cycles / wall
    if (per_sm_clk > best) { best = per_sm_clk; clk = c; }
  }
  printf("%s  \"%s\": {\"lane_ops_per_clk_per_sm\": %.2f, \"clk_ghz_est\": %.3f, \"blocks_per_sm\": %d, \"threads\": %d}\n",
         first ? "" : ",", name, best, clk, blocks_per_sm, threads);
  if (clk_ghz_out) *clk_ghz_out = clk;
  cudaFree(out); cudaFree(cyc);
  return best;
}

template <typename K>
static void run_write(K kern, const char* name, uint32_t* buf, size_t nwords, int vec, int threads = 256, int bps = 0) {
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, 0));
  if (bps > 0) occ = std::min(occ, bps);
  int blocks = g_sms * occ;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<<<blocks, threads>>>(buf, nwords);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int rep = 0; rep < 10; rep++) {
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(buf, nwords);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    best = std::min(best, ms);
  }
  printf(",  \"%s\": {\"GBps\": %.1f, \"ms\": %.4f, \"bytes\": %zu, \"vec\": %d}\n", name, nwords * 4.0 / (best * 1e6), best, nwords * 4, vec);
}

int main(int argc, char** argv) {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  g_sms = p.multiProcessorCount;
  int optin = 0; cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
  printf("{\"device\": \"%s\", \"sms\": %d, \"smem_optin\": %d, \"cc\": \"%d.%d\"\n", p.name, g_sms, optin, p.major, p.minor);
  const int it = 4096;
  if (argc > 1) {  // "writes": only the write-path probes (for ncu)
    size_t bytes = (size_t)1 << 30;
    uint32_t* buf; CK(cudaMalloc(&buf, bytes));
    for (int r = 0; r < 2; r++) CK(cudaMemsetAsync(buf, r + 1, bytes));
    run_write(k_write_data<2>, "data.hash", buf, bytes / 4, 8);
    run_write(k_write_bulk<16384>, "bulk16K.x4", buf, bytes / 4, 0, 32, 4);
    CK(cudaDeviceSynchronize());
    printf("}\n");
    return 0;
  }
  run_pipe(k_pipe<OP_IMAD>, "IMAD", 8, 256, 8, it, 0, nullptr, false);
  run_pipe(k_pipe<OP_WIDE>, "IMAD.WIDE.U32", 8, 256, 8, it, 0, nullptr, false);
  run_pipe(k_pipe<OP_HI>, "IMAD.HI.U32", 8, 256, 8, it, 0, nullptr, false);
  run_pipe(k_pipe<OP_WIDEF>, "IMAD.WIDE.U32.folded64", 8, 256, 8, it, 0, nullptr, false);
  run_pipe(k_pipe<OP_HI64>, "IMAD.HI.U32.addend64", 8, 256, 8, it, 0, nullptr, false);
  run_pipe(k_pipe<OP_IADD64>, "IADD64", 8, 256, 8, it, 0, nullptr, false);
  run_pipe(k_pipe<OP_IADD>, "IADD", 8, 256, 8, it, 0, nullptr, false);
  run_pipe(k_pipe<OP_LOP3>, "LOP3", 8, 256, 8, it, 0, nullptr, false);
  run_pipe(k_pipe<OP_SHL>, "SHL", 8, 256, 8, it, 0, nullptr, false);
  run_pipe(k_pipe<OP_I2F>, "I2F.U32(+FADD)", 8, 256, 8, it, 0, nullptr, false);
  run_pipe(k_pipe<OP_ROUND>, "ROUND(WIDE+IMAD+SHL)", 8, 256, 8, it, 0, nullptr, false);
  run_pipe(k_atoms<0>, "ATOMS.random.ret", 4, 1024, 1, 1024, 32768 * 4, nullptr, false);
  run_pipe(k_atoms<1>, "ATOMS.random.noret", 4, 1024, 1, 1024, 32768 * 4, nullptr, false);
  run_pipe(k_atoms<2>, "ATOMS.conflictfree.ret", 4, 1024, 1, 1024, 32768 * 4, nullptr, false);
  run_pipe(k_atoms<0>, "ATOMS.random.ret.512t", 4, 512, 1, 1024, 32768 * 4, nullptr, false);

  size_t bytes = (size_t)4 << 30;
  uint32_t* buf; CK(cudaMalloc(&buf, bytes));
  {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    CK(cudaMemsetAsync(buf, 0, bytes));
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int rep = 0; rep < 10; rep++) {
      cudaEventRecord(e0); cudaMemsetAsync(buf, rep, bytes); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1); best = std::min(best, ms);
    }
    printf(",  \"memset\": {\"GBps\": %.1f, \"ms\": %.4f, \"bytes\": %zu}\n", bytes / (best * 1e6), best, bytes);
  }
  run_write(k_write<4, false>, "STG.128", buf, bytes / 4, 4);
  run_write(k_write<4, true>, "STG.128.cs", buf, bytes / 4, 4);
  run_write(k_write<8, false>, "STG.256", buf, bytes / 4, 8);
  run_write(k_write<8, true>, "STG.256.cs", buf, bytes / 4, 8);
  run_write(k_write_warpseg<4>, "warpseg.STG.128", buf, bytes / 4, 4);
  run_write(k_write_warpseg<8>, "warpseg.STG.256", buf, bytes / 4, 8);
  run_write(k_write_warpseg<8>, "warpseg.STG.256.occ4", buf, bytes / 4, 8, 256, 4);
  run_write(k_write_warpseg<8>, "warpseg.STG.256.occ2", buf, bytes / 4, 8, 256, 2);
  run_write(k_write_data<0>, "data.zero", buf, bytes / 4, 8);
  run_write(k_write_data<1>, "data.const", buf, bytes / 4, 8);
  run_write(k_write_data<2>, "data.hash", buf, bytes / 4, 8);
  run_write(k_write_data<3>, "data.hash.evict_first", buf, bytes / 4, 8);
  run_write(k_write_data<4>, "data.hash.L1noalloc", buf, bytes / 4, 8);
  run_write(k_write_bulk<16384>, "bulk16K.x4", buf, bytes / 4, 0, 32, 4);
  run_write(k_write_bulk<16384>, "bulk16K.x8", buf, bytes / 4, 0, 32, 8);
  run_write(k_write_bulk<32768>, "bulk32K.x4", buf, bytes / 4, 0, 32, 4);
  run_write(k_write_bulk<8192>, "bulk8K.x8", buf, bytes / 4, 0, 32, 8);
  printf("}\n");
  cudaFree(buf);
  return 0;
}
