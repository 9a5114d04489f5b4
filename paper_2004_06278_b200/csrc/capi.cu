// capi.cu -- the extern "C" entry points of libsquares.so declared in include/squares.h:
// argument validation, error codes, device-property cache, and the host-buffer fill.
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>

#include "sq_internal.h"

namespace sq {

static thread_local int g_last_cuda_error = 0;

int set_cuda_error(cudaError_t e) {
  if (e == cudaSuccess) return SQ_OK;
  g_last_cuda_error = (int)e;
  return SQ_ECUDA;
}

static std::mutex g_dev_mu;
static DeviceInfo g_dev[kMaxDevices];
static bool g_dev_ok[kMaxDevices];

const DeviceInfo* device_info() {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) { set_cuda_error(e); return nullptr; }
  if (dev < 0 || dev >= kMaxDevices) { set_cuda_error(cudaErrorInvalidDevice); return nullptr; }
  std::lock_guard<std::mutex> lk(g_dev_mu);
  if (!g_dev_ok[dev]) {
    DeviceInfo d;
    d.device = dev;
    e = cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&d.smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (e != cudaSuccess) { set_cuda_error(e); return nullptr; }
    g_dev[dev] = d;
    g_dev_ok[dev] = true;
  }
  return &g_dev[dev];
}

// nkeys * ld * es must fit size_t and the address range of `out`.
static bool size_ok(uint64_t nkeys, uint64_t ld, uint64_t es) {
  if (ld == 0) return true;
  const unsigned __int128 bytes = (unsigned __int128)nkeys * ld * es;
  return bytes <= (unsigned __int128)SIZE_MAX;
}

static bool kind_ok(int kind) { return kind >= KIND_U32 && kind <= KIND_F32X2; }

// keys_dev == nullptr: single row with key key_imm (nkeys must be 1).
static int fill_any(int kind, const uint64_t* keys_dev, uint64_t nkeys, uint64_t key_imm, uint64_t ctr0,
                    uint64_t stride, uint64_t n, void* out_dev, uint64_t ld, cudaStream_t stream) {
  if (!kind_ok(kind) || stride == 0) return SQ_EINVAL;
  const uint64_t es = kind_elem_bytes(kind);
  if (n == 0 || nkeys == 0) return SQ_OK;
  if (!out_dev) return SQ_EINVAL;
  if (!keys_dev && nkeys != 1) return SQ_EINVAL;
  if (((uintptr_t)out_dev % es) != 0) return SQ_EINVAL;
  if (((uintptr_t)keys_dev & 7) != 0) return SQ_EINVAL;   // the kernels __ldg 8-byte keys
  if (nkeys == 1) ld = n;
  if (ld < n) return SQ_EINVAL;
  if (!size_ok(nkeys, ld, es)) return SQ_EINVAL;
  FillArgs a{};
  a.keys = keys_dev;
  a.key_imm = key_imm;
  a.ctr0 = ctr0;
  a.stride = stride;
  a.one = 1;
  a.n = n;
  a.out = (char*)out_dev;
  a.ld_bytes = ld * es;
  return launch_fill_kind(kind, a, nkeys, n, stream);
}

static int fill_entry(int kind, const uint64_t* keys_dev, uint64_t nkeys, uint64_t ctr0, uint64_t n,
                      void* out_dev, uint64_t ld, cudaStream_t stream) {
  if (n != 0 && nkeys != 0 && !keys_dev) return SQ_EINVAL;
  return fill_any(kind, keys_dev, nkeys, 0, ctr0, 1, n, out_dev, ld, stream);
}

}  // namespace sq

using namespace sq;

extern "C" {

const char* sq_strerror(int code) {
  switch (code) {
    case SQ_OK: return "SQ_OK: success";
    case SQ_EINVAL: return "SQ_EINVAL: invalid argument";
    case SQ_ERANGE: return "SQ_ERANGE: argument out of range";
    case SQ_ECUDA: return "SQ_ECUDA: CUDA error";
    case SQ_ENOMEM: return "SQ_ENOMEM: out of host memory";
    default: return "unknown squares status code";
  }
}

int sq_last_cuda_error(void) { return g_last_cuda_error; }

int sq_version(void) { return 200; }

int sq_fill_u32(const uint64_t* keys_dev, uint64_t nkeys, uint64_t ctr0, uint64_t n, uint32_t* out_dev,
                uint64_t ld, sq_stream_t stream) {
  return fill_entry(KIND_U32, keys_dev, nkeys, ctr0, n, out_dev, ld, (cudaStream_t)stream);
}

int sq_fill_u64(const uint64_t* keys_dev, uint64_t nkeys, uint64_t ctr0, uint64_t n, uint64_t* out_dev,
                uint64_t ld, sq_stream_t stream) {
  return fill_entry(KIND_U64, keys_dev, nkeys, ctr0, n, out_dev, ld, (cudaStream_t)stream);
}

int sq_fill_f32(const uint64_t* keys_dev, uint64_t nkeys, uint64_t ctr0, uint64_t n, float* out_dev,
                uint64_t ld, sq_stream_t stream) {
  return fill_entry(KIND_F32, keys_dev, nkeys, ctr0, n, out_dev, ld, (cudaStream_t)stream);
}

static int fill_key_entry(int kind, uint64_t key, uint64_t ctr0, uint64_t n, void* out_dev, cudaStream_t stream) {
  return fill_any(kind, nullptr, 1, key, ctr0, 1, n, out_dev, n, stream);
}

int sq_fill_u32_k(uint64_t key, uint64_t ctr0, uint64_t n, uint32_t* out_dev, sq_stream_t stream) {
  return fill_key_entry(KIND_U32, key, ctr0, n, out_dev, (cudaStream_t)stream);
}

int sq_fill_u64_k(uint64_t key, uint64_t ctr0, uint64_t n, uint64_t* out_dev, sq_stream_t stream) {
  return fill_key_entry(KIND_U64, key, ctr0, n, out_dev, (cudaStream_t)stream);
}

int sq_fill_f32_k(uint64_t key, uint64_t ctr0, uint64_t n, float* out_dev, sq_stream_t stream) {
  return fill_key_entry(KIND_F32, key, ctr0, n, out_dev, (cudaStream_t)stream);
}

int sq_fill_f64(const uint64_t* keys_dev, uint64_t nkeys, uint64_t ctr0, uint64_t n, double* out_dev,
                uint64_t ld, sq_stream_t stream) {
  return fill_entry(KIND_F64, keys_dev, nkeys, ctr0, n, out_dev, ld, (cudaStream_t)stream);
}

int sq_fill_f32x2(const uint64_t* keys_dev, uint64_t nkeys, uint64_t ctr0, uint64_t n, float* out_dev,
                  uint64_t ld, sq_stream_t stream) {
  return fill_entry(KIND_F32X2, keys_dev, nkeys, ctr0, n, out_dev, ld, (cudaStream_t)stream);
}

int sq_fill_f64_k(uint64_t key, uint64_t ctr0, uint64_t n, double* out_dev, sq_stream_t stream) {
  return fill_key_entry(KIND_F64, key, ctr0, n, out_dev, (cudaStream_t)stream);
}

int sq_fill_f32x2_k(uint64_t key, uint64_t ctr0, uint64_t n, float* out_dev, sq_stream_t stream) {
  return fill_key_entry(KIND_F32X2, key, ctr0, n, out_dev, (cudaStream_t)stream);
}

int sq_fill_ex(int kind, const uint64_t* keys_dev, uint64_t nkeys, uint64_t key_imm, uint64_t ctr0,
               uint64_t stride, uint64_t n, void* out_dev, uint64_t ld, sq_stream_t stream) {
  return fill_any(kind, keys_dev, nkeys, key_imm, ctr0, stride, n, out_dev, ld, (cudaStream_t)stream);
}

int sq_fill_keyctr(int kind, const uint64_t* keys_dev, uint64_t nkeys, uint64_t ctr, void* out_dev,
                   sq_stream_t stream) {
  if (!kind_ok(kind)) return SQ_EINVAL;
  if (nkeys == 0) return SQ_OK;
  if (!keys_dev || !out_dev) return SQ_EINVAL;
  if (((uintptr_t)out_dev % kind_elem_bytes(kind)) != 0 || ((uintptr_t)keys_dev & 7)) return SQ_EINVAL;
  if (!size_ok(1, nkeys, 8)) return SQ_EINVAL;
  return launch_keyctr(kind, keys_dev, nkeys, ctr, out_dev, (cudaStream_t)stream);
}

int sq_fused_stats_ex(uint64_t key, uint64_t ctr0, uint64_t stride, uint64_t n, uint32_t flags,
                      uint64_t* hist_dev, uint64_t* ones_dev, sq_stream_t stream) {
  if (stride == 0 || (flags & ~SQ_FUSED_BITREV)) return SQ_EINVAL;
  if (n == 0) return SQ_OK;
  if (!hist_dev || !ones_dev) return SQ_EINVAL;
  if (((uintptr_t)hist_dev & 7) || ((uintptr_t)ones_dev & 7)) return SQ_EINVAL;
  return launch_fused(key, ctr0, stride, n, flags, hist_dev, ones_dev, (cudaStream_t)stream);
}

int sq_transitions(uint64_t key, uint64_t ctr0, uint64_t stride, uint64_t n, uint32_t flags,
                   uint64_t* count_dev, sq_stream_t stream) {
  if (stride == 0 || (flags & ~SQ_FUSED_BITREV)) return SQ_EINVAL;
  if (n == 0) return SQ_OK;
  if (!count_dev || ((uintptr_t)count_dev & 7)) return SQ_EINVAL;
  return launch_transitions(key, ctr0, stride, n, flags, count_dev, (cudaStream_t)stream);
}

int sq_scaled_hist(int W, const uint64_t* keys_dev, uint64_t nkeys, uint64_t* hist_dev, sq_stream_t stream) {
  if (W < 8 || W > 32 || (W & 1)) return SQ_EINVAL;
  if (nkeys == 0) return SQ_OK;
  if (!keys_dev || !hist_dev || ((uintptr_t)hist_dev & 7) || ((uintptr_t)keys_dev & 7)) return SQ_EINVAL;
  if (nkeys > 65535) return SQ_ERANGE;
  return launch_scaled_hist(W, keys_dev, nkeys, hist_dev, (cudaStream_t)stream);
}

int sq_fused_stats(uint64_t key, uint64_t ctr0, uint64_t n, uint64_t* hist_dev, uint64_t* ones_dev,
                   sq_stream_t stream) {
  return sq_fused_stats_ex(key, ctr0, 1, n, 0, hist_dev, ones_dev, stream);
}

int sq_fill_host(int kind, uint64_t key, uint64_t ctr0, uint64_t n, void* out_host, void* scratch_dev,
                 size_t scratch_bytes, sq_stream_t stream, sq_stream_t copy_stream) {
  if (!kind_ok(kind)) return SQ_EINVAL;
  if (n == 0) return SQ_OK;
  if (!out_host || !scratch_dev) return SQ_EINVAL;
  const uint64_t es = kind_elem_bytes(kind);
  // the fill kernel corrects misalignment only in whole elements: an unaligned scratch
  // pointer would make its 256-bit stores fault (a sticky context error), so reject it
  if (((uintptr_t)scratch_dev % es) != 0) return SQ_EINVAL;
  // two ping-pong halves, each a multiple of 32 bytes, the first starting 32-byte aligned
  const uint64_t pad = (32 - ((uintptr_t)scratch_dev & 31)) & 31;
  if (scratch_bytes < pad) return SQ_EINVAL;
  scratch_dev = (char*)scratch_dev + pad;
  scratch_bytes -= pad;
  const uint64_t half = (scratch_bytes / 2) & ~(uint64_t)31;
  const uint64_t chunk = half / es;
  if (chunk == 0) return SQ_EINVAL;
  cudaStream_t gs = (cudaStream_t)stream, cs = (cudaStream_t)copy_stream;
  if (cs == gs) cs = nullptr;
  cudaEvent_t gen_done[2] = {nullptr, nullptr}, copy_done[2] = {nullptr, nullptr};
  auto destroy_events = [&]() {
    for (int i = 0; i < 2; i++) {
      if (gen_done[i]) cudaEventDestroy(gen_done[i]);
      if (copy_done[i]) cudaEventDestroy(copy_done[i]);
    }
  };
  for (int b = 0; b < 2; b++) {
    cudaError_t e = cudaEventCreateWithFlags(&gen_done[b], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&copy_done[b], cudaEventDisableTiming);
    if (e != cudaSuccess) {
      destroy_events();
      return set_cuda_error(e);
    }
  }
  int rc = SQ_OK;
  uint64_t done = 0;
  int b = 0;
  bool used[2] = {false, false};
  while (done < n && rc == SQ_OK) {
    const uint64_t m = (n - done < chunk) ? (n - done) : chunk;
    char* buf = (char*)scratch_dev + b * half;
    cudaError_t e = cudaSuccess;
    if (used[b]) e = cudaStreamWaitEvent(gs, copy_done[b], 0);   // buffer free again
    if (e != cudaSuccess) { rc = set_cuda_error(e); break; }
    FillArgs a{};
    a.keys = nullptr;
    a.key_imm = key;
    a.ctr0 = ctr0 + done;
    a.stride = 1;
    a.one = 1;
    a.n = m;
    a.out = buf;
    a.ld_bytes = m * es;
    rc = launch_fill_kind(kind, a, 1, m, gs);
    if (rc != SQ_OK) break;
    cudaStream_t copier = cs ? cs : gs;
    e = cudaEventRecord(gen_done[b], gs);
    if (e == cudaSuccess && cs) e = cudaStreamWaitEvent(cs, gen_done[b], 0);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync((char*)out_host + done * es, buf, m * es, cudaMemcpyDeviceToHost, copier);
    if (e == cudaSuccess) e = cudaEventRecord(copy_done[b], copier);
    if (e != cudaSuccess) { rc = set_cuda_error(e); break; }
    used[b] = true;
    done += m;
    b ^= 1;
  }
  cudaError_t e1 = cudaStreamSynchronize(gs);
  cudaError_t e2 = cs ? cudaStreamSynchronize(cs) : cudaSuccess;
  destroy_events();
  if (rc != SQ_OK) return rc;
  if (e1 != cudaSuccess) return set_cuda_error(e1);
  return set_cuda_error(e2);
}

}  // extern "C"
