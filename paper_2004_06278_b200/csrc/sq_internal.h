// sq_internal.h -- shared declarations of libsquares.so (not part of the public ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/squares.h"

namespace sq {

// Output kinds (the numeric values are the C ABI's SQ_KIND_* constants).
enum Kind { KIND_U32 = 0, KIND_U64 = 1, KIND_F32 = 2, KIND_F64 = 3, KIND_F32X2 = 4 };

__host__ __device__ constexpr int kind_elem_bytes(int kind) { return (kind == KIND_U32 || kind == KIND_F32) ? 4 : 8; }

#ifndef SQ_FILL_THREADS
#define SQ_FILL_THREADS 256
#endif
// Minimum resident CTAs per SM for the fill kernels (caps registers: 3 -> <= 85, 2 -> <= 128).
// Measured on B200 (tools/variant_bench.py): 3 for key-by-value, 2 for device keys.
#ifndef SQ_FILL_MINBLOCKS
#define SQ_FILL_MINBLOCKS 2
#endif
#ifndef SQ_FILL_MINBLOCKS_IMM
#define SQ_FILL_MINBLOCKS_IMM 3
#endif
constexpr int kFillThreads = SQ_FILL_THREADS;
constexpr int kFillMinBlocks = SQ_FILL_MINBLOCKS;         // device-keys kernels
constexpr int kFillMinBlocksImm = SQ_FILL_MINBLOCKS_IMM;  // key-by-value kernels
#ifndef SQ_FUSED_THREADS
#define SQ_FUSED_THREADS 1024
#endif
constexpr int kFusedThreads = SQ_FUSED_THREADS;   // 1024 (epochs of 32 samples) or 512 (64)

struct FillArgs {
  const uint64_t* keys;     // device keys, or nullptr to use key_imm (single row)
  uint64_t key_imm;
  uint64_t ctr0;
  uint64_t stride;          // counter increment between consecutive outputs (1 = consecutive)
  uint64_t n;
  char* out;                // row 0 base
  uint64_t ld_bytes;        // row pitch in bytes
  uint64_t chunks_per_row;  // set by the launcher
  uint64_t chunks_q, chunks_r;  // balanced split of all chunks over the grid's warps
  uint32_t one;             // always 1: the opaque shift amount of squares_dev.cuh cross_add
};

constexpr int kMaxDevices = 64;   // per-device caches (device_info, occupancy, attributes)

struct DeviceInfo {
  int device;
  int sms;
  int smem_optin;
};

// Cached per-device properties of the current device (nullptr + error recorded on failure).
const DeviceInfo* device_info();

// Record a CUDA error for sq_last_cuda_error(); returns SQ_OK for cudaSuccess else SQ_ECUDA.
int set_cuda_error(cudaError_t e);

int launch_fill_kind(int kind, const FillArgs& a, uint64_t nkeys, uint64_t n, cudaStream_t stream);

int launch_fused(uint64_t key, uint64_t ctr0, uint64_t stride, uint64_t n, uint32_t flags,
                 uint64_t* hist, uint64_t* ones, cudaStream_t stream);

int launch_transitions(uint64_t key, uint64_t ctr0, uint64_t stride, uint64_t n, uint32_t flags,
                       uint64_t* count, cudaStream_t stream);

int launch_scaled_hist(int W, const uint64_t* keys, uint64_t nkeys, uint64_t* hist, cudaStream_t stream);

int launch_keyctr(int kind, const uint64_t* keys, uint64_t nkeys, uint64_t ctr, void* out,
                  cudaStream_t stream);

}  // namespace sq
