// Shared helpers for the TokenFlow B200 library (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdio.h>

#include <string>
#include <vector>

#include "../../include/tokenflow_b200.h"

namespace tf {

// ------------------------------------------------------------ error state
void set_error(const char* fmt, ...);

#define TF_CHECK_ARG(cond, ...)          \
  do {                                   \
    if (!(cond)) {                       \
      ::tf::set_error(__VA_ARGS__);      \
      return TF_EINVAL;                  \
    }                                    \
  } while (0)

#define TF_CUDA(expr)                                                                          \
  do {                                                                                         \
    cudaError_t _e = (expr);                                                                   \
    if (_e != cudaSuccess) {                                                                   \
      ::tf::set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e), __FILE__, __LINE__); \
      return TF_EIO;                                                                           \
    }                                                                                          \
  } while (0)

// every kernel launch of the library passes here: counted for tf_launch_count()
void count_launch();

#define TF_LAUNCH_CHECK()                                                                       \
  do {                                                                                          \
    ::tf::count_launch();                                                                       \
    cudaError_t _e = cudaGetLastError();                                                        \
    if (_e != cudaSuccess) {                                                                    \
      ::tf::set_error("kernel launch failed: %s (%s:%d)", cudaGetErrorString(_e), __FILE__, __LINE__); \
      return TF_EIO;                                                                            \
    }                                                                                           \
  } while (0)

// --------------------------------------------------------------- pool
struct Pool {
  uint16_t* gpu;        // device pointer, bf16 bits
  uint16_t* host;       // host pointer (pinned)
  uint16_t* host_dev;   // device-visible alias of host (UVA / mapped)
  int32_t n_blocks, n_host_blocks;
  int32_t n_layers, block_tokens, kv_heads, head_dim;
  int64_t block_elems;  // elements per block (all layers)
  int64_t tile_elems;   // block_tokens * head_dim (one (block,layer,kv,head) tile)
  std::vector<int32_t> free_gpu, free_host;  // LIFO stacks (back = next)
  std::vector<uint8_t> used_gpu, used_host;  // per-block allocation state (double-free check)
  alignas(64) unsigned char tmap[128];       // CUtensorMap of the HBM pool (v5 attention), built lazily
  bool tmap_ok = false;
  // copy-engine swaps: one auxiliary stream per direction (0 = d2h, 1 = h2d)
  // so consecutive runs of a chunk alternate between two copy queues and the
  // per-copy setup of one overlaps the transfer of the other; created lazily
  cudaStream_t aux[2] = {nullptr, nullptr};
  cudaEvent_t fork_ev[2] = {nullptr, nullptr}, join_ev[2] = {nullptr, nullptr};
  ~Pool() {
    for (int i = 0; i < 2; ++i) {
      if (aux[i]) cudaStreamDestroy(aux[i]);
      if (fork_ev[i]) cudaEventDestroy(fork_ev[i]);
      if (join_ev[i]) cudaEventDestroy(join_ev[i]);
    }
  }

  // element offset of (block, layer, kv, head, slot, dim=0)
  __host__ __device__ int64_t off(int64_t b, int l, int kv, int h, int s) const {
    return b * block_elems + ((((int64_t)l * 2 + kv) * kv_heads + h) * block_tokens + s) * head_dim;
  }
};

Pool* get_pool(int64_t handle);

// Plain-old-data view passed to kernels.
struct PoolView {
  uint16_t* gpu;
  uint16_t* host;
  int64_t block_elems;
  int32_t n_layers, block_tokens, kv_heads, head_dim;
  __host__ __device__ int64_t off(int64_t b, int l, int kv, int h, int s) const {
    return b * block_elems + ((((int64_t)l * 2 + kv) * kv_heads + h) * block_tokens + s) * head_dim;
  }
};

inline PoolView view_of(const Pool& p) {
  PoolView v;
  v.gpu = p.gpu;
  v.host = p.host_dev;
  v.block_elems = p.block_elems;
  v.n_layers = p.n_layers;
  v.block_tokens = p.block_tokens;
  v.kv_heads = p.kv_heads;
  v.head_dim = p.head_dim;
  return v;
}

// ------------------------------------------------- synthetic KV contents
// Must match oracle/dataplane.py kv_bits bit for bit.
__host__ __device__ __forceinline__ uint32_t fmix32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x85EBCA6Bu;
  x ^= x >> 13;
  x *= 0xC2B2AE35u;
  x ^= x >> 16;
  return x;
}

__host__ __device__ __forceinline__ uint16_t kv_bits(uint32_t rid, uint32_t pos, uint32_t layer, uint32_t kv,
                                                     uint32_t head, uint32_t dim, uint32_t seed) {
  uint32_t x = rid * 0x9E3779B1u + pos * 0x85EBCA77u + layer * 0xC2B2AE3Du + kv * 0x27D4EB2Fu +
               head * 0x165667B1u + dim * 0x61C88647u + seed * 0x2545F491u;
  x = fmix32(x);
  return (uint16_t)((x & 0x807Fu) | 0x3F00u);
}

}  // namespace tf
