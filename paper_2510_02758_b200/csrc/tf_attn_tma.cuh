// v5 paged decode attention (tf_attn_tma.cu): TMA tensor loads + stream-K warps.
#pragma once
#include "tf_common.cuh"

namespace tf {

constexpr int kAttn5MaxB = 1024;  // requests per launch (prefix sums in shared memory)
constexpr int kAttn5MinPer = 4;   // minimum blocks per warp (bounds the partials per segment)

struct Attn5Args {
  const uint16_t* pool;  // HBM pool base (L2 prefetch addresses)
  const uint16_t* q;
  const int32_t* table;
  const int32_t* rows;
  const int32_t* ctx;
  uint16_t* out;
  float* ws_acc;      // [B*kv][kmax][G][D] partial accumulators
  float* ws_ml;       // [B*kv][kmax][G][2] partial (max, sum)
  int32_t* counters;  // [B*kv] self-resetting merge counters
  unsigned long long* ticket;  // dispatch-order CTA ticket (monotonic; grid size is fixed per process)
  int* diag;                   // expired-wait diagnostics (workspace bytes [8, 64))
  int32_t stride, n_layers, kv_heads, layer, hq, B, kmax, min_per;
  float scale_log2;
  int32_t mutate;     // test-only fault injection (TF_ATTN_MUTATE), 0 in production
};

bool attn5_supported(const Pool* p, int G, int B);
int64_t attn5_workspace(const Pool* p, int B, int max_ctx, int G);
int attn5_launch(Pool* p, Attn5Args a, int G, int max_ctx, void* workspace, int64_t workspace_bytes, int sms,
                 cudaStream_t st);

}  // namespace tf
