// KV append into the paged pool (decode growth / prefill) and synthetic KV.
//
// Reference: a decode iteration adds one KV token per member
// (tokensim/engine.py:510-540), a prefill prompt_len+1 (:484-508); in the
// reference these are counter increments, here they write real bytes.
#include <algorithm>

#include "tf_common.cuh"

namespace tf {

// One warp per (token, kv, head) row of head_dim elements.
__global__ void append_kernel(PoolView pv, const int32_t* __restrict__ table, int32_t stride,
                              const int32_t* __restrict__ rows, const int32_t* __restrict__ pos, int32_t n,
                              int32_t layer, const uint16_t* __restrict__ k, const uint16_t* __restrict__ v,
                              int64_t kv_stride) {
  const int warps = blockDim.x / 32;
  const int64_t wid = (int64_t)blockIdx.x * warps + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  const int64_t total = (int64_t)n * 2 * pv.kv_heads;
  if (wid >= total) return;
  const int tok = (int)(wid / (2 * pv.kv_heads));
  const int kv = (int)((wid / pv.kv_heads) & 1);
  const int h = (int)(wid % pv.kv_heads);
  const int p = pos[tok];
  const int blk = table[(int64_t)rows[tok] * stride + p / pv.block_tokens];
  const uint16_t* src = (kv ? v : k) + (int64_t)tok * kv_stride + (int64_t)h * pv.head_dim;
  uint16_t* dst = pv.gpu + pv.off(blk, layer, kv, h, p % pv.block_tokens);
  for (int d = lane * 8; d < pv.head_dim; d += 32 * 8)
    *reinterpret_cast<uint4*>(dst + d) = *reinterpret_cast<const uint4*>(src + d);
}

// Fused decode epilogue of the QKV projection: rotary embedding of q and k
// (interleaved pairs, angle = pos * inv_freq[i]) + append of k, v into the
// paged pool + q written contiguously for the attention kernel (+ the
// contiguous k / v copy a prefill's attention reads, + the host-store slot
// when write-through is fused).  One CTA per token: the token's sin / cos
// table (head_dim / 2 angles) is computed ONCE into shared memory and shared
// by all its rotated heads (q and k), its pool / host block is looked up
// once, and every head moves as 16-byte vectors (the earlier one-warp-per-
// (token, head) version recomputed sincosf per head and moved 4-byte words).
// The arithmetic per element is unchanged (bit-identical output).
constexpr int kRopeThreads = 256;
constexpr int kRopeMaxPairs = 128;  // head_dim <= 256

__global__ void __launch_bounds__(kRopeThreads) rope_append_kernel(
    PoolView pv, const int32_t* __restrict__ table, int32_t stride, const int32_t* __restrict__ rows,
    const int32_t* __restrict__ pos, int32_t n, int32_t layer, const uint16_t* __restrict__ qkv, int32_t hq,
    const float* __restrict__ inv_freq, uint16_t* __restrict__ q_out, uint16_t* __restrict__ kv_out,
    const int32_t* __restrict__ host_table) {
  __shared__ float sn_sh[kRopeMaxPairs], cs_sh[kRopeMaxPairs];
  const int tok = blockIdx.x;
  const int D = pv.head_dim, hkv = pv.kv_heads;
  const int heads = hq + 2 * hkv;
  const int p = __ldg(pos + tok);
  const int row = __ldg(rows + tok);
  const int lb = p / pv.block_tokens, slot = p % pv.block_tokens;
  for (int i = threadIdx.x; i < D / 2; i += blockDim.x) {
    float sn, cs;
    sincosf((float)p * __ldg(inv_freq + i), &sn, &cs);
    sn_sh[i] = sn;
    cs_sh[i] = cs;
  }
  const int blk = __ldg(table + (int64_t)row * stride + lb);
  const int hb = host_table ? __ldg(host_table + (int64_t)row * stride + lb) : -1;
  __syncthreads();
  const int vph = D / 8;  // 16-byte vectors per head
  const uint4* src = reinterpret_cast<const uint4*>(qkv + (int64_t)tok * heads * D);
  for (int v = threadIdx.x; v < heads * vph; v += blockDim.x) {
    const int h = v / vph, d = (v - h * vph) * 8;
    uint4 w = __ldg(src + v);
    const bool is_q = h < hq;
    const int kv = is_q ? 0 : (h - hq) / hkv, kvh = is_q ? 0 : (h - hq) % hkv;
    if (is_q || kv == 0) {
      uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int i = d / 2 + k;
        const float x1 = __uint_as_float(ws[k] << 16), x2 = __uint_as_float(ws[k] & 0xFFFF0000u);
        const float sn = sn_sh[i], cs = cs_sh[i];
        const uint32_t o1 = __bfloat16_as_ushort(__float2bfloat16_rn(x1 * cs - x2 * sn));
        const uint32_t o2 = __bfloat16_as_ushort(__float2bfloat16_rn(x1 * sn + x2 * cs));
        ws[k] = o1 | (o2 << 16);
      }
      w = make_uint4(ws[0], ws[1], ws[2], ws[3]);
    }
    if (is_q) {
      *reinterpret_cast<uint4*>(q_out + ((int64_t)tok * hq + h) * D + d) = w;
      continue;
    }
    *reinterpret_cast<uint4*>(pv.gpu + pv.off(blk, layer, kv, kvh, slot) + d) = w;
    if (kv_out) *reinterpret_cast<uint4*>(kv_out + (((int64_t)kv * n + tok) * hkv + kvh) * D + d) = w;
    // fused write-through: the same slot of the request's host block, written
    // straight over PCIe into the mapped pinned store (posted writes)
    if (hb >= 0) *reinterpret_cast<uint4*>(pv.host + pv.off(hb, layer, kv, kvh, slot) + d) = w;
  }
}

constexpr int kMaxSpans = 1536;
struct SpanArgs {
  int32_t n;
  uint32_t seed;
  int32_t stride;
  int32_t row[kMaxSpans], rid[kMaxSpans], lo[kMaxSpans], hi[kMaxSpans];
};

// blockIdx.y = span, elements of the span strided over blockIdx.x / threads.
__global__ void fill_synth_kernel(PoolView pv, const int32_t* __restrict__ table, const __grid_constant__ SpanArgs a) {
  const int s = blockIdx.y;
  const int npos = a.hi[s] - a.lo[s];
  const int64_t per_pos = (int64_t)pv.n_layers * 2 * pv.kv_heads * pv.head_dim;
  const int64_t total = per_pos * npos;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    int d = (int)(e % pv.head_dim);
    int64_t r = e / pv.head_dim;
    int h = (int)(r % pv.kv_heads);
    r /= pv.kv_heads;
    int kv = (int)(r & 1);
    r >>= 1;
    int l = (int)(r % pv.n_layers);
    int p = a.lo[s] + (int)(r / pv.n_layers);
    int blk = table[(int64_t)a.row[s] * a.stride + p / pv.block_tokens];
    pv.gpu[pv.off(blk, l, kv, h, p % pv.block_tokens) + d] =
        kv_bits((uint32_t)a.rid[s], (uint32_t)p, (uint32_t)l, (uint32_t)kv, (uint32_t)h, (uint32_t)d, a.seed);
  }
}

__global__ void q_synth_kernel(uint16_t* q, const int32_t* __restrict__ rids, const int32_t* __restrict__ pos, int B,
                               int layer, int hq, int hd, uint32_t seed) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t total = (int64_t)B * hq * hd;
  if (e >= total) return;
  int d = (int)(e % hd);
  int h = (int)((e / hd) % hq);
  int b = (int)(e / ((int64_t)hd * hq));
  // q_bits(rid, pos, layer, qhead, dim) = kv_bits(rid + 0x5000, pos, layer, 2, qhead, dim)
  q[e] = kv_bits((uint32_t)rids[b] + 0x5000u, (uint32_t)pos[b], (uint32_t)layer, 2u, (uint32_t)h, (uint32_t)d, seed);
}

// Zero-copy small transfer (step inputs / sampled ids): one CTA moves the
// bytes through the SMs over mapped pinned memory, so a decode step never
// queues behind bulk KV copies on the copy engines.
__global__ void copy_small_kernel(unsigned char* __restrict__ dst, const unsigned char* __restrict__ src,
                                  int64_t bytes) {
  const bool vec = ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0;
  const int64_t nv = vec ? bytes / 16 : 0;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = tid; i < nv; i += nt) reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
  for (int64_t i = nv * 16 + tid; i < bytes; i += nt) dst[i] = src[i];
}

}  // namespace tf

using namespace tf;

extern "C" {

int tf_copy_small(void* dst, const void* src, int64_t bytes, void* stream) {
  TF_CHECK_ARG(bytes >= 0 && bytes <= (64 << 20), "tf_copy_small: bytes %lld out of range", (long long)bytes);
  if (bytes == 0) return TF_OK;
  TF_CHECK_ARG(dst && src, "tf_copy_small: NULL pointer");
  // one CTA for step-sized copies; up to 32 for prefill inputs (PCIe latency-bound)
  const int grid = (int)std::min<int64_t>(32, std::max<int64_t>(1, bytes / (16 << 10)));
  copy_small_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>((unsigned char*)dst, (const unsigned char*)src, bytes);
  TF_LAUNCH_CHECK();
  return TF_OK;
}

int tf_kv_append(int64_t pool, const int32_t* dev_table, int32_t row_stride, const int32_t* dev_rows,
                 const int32_t* dev_pos, int32_t n, int32_t layer, const void* k, const void* v, int64_t kv_row_stride,
                 void* stream) {
  Pool* p = get_pool(pool);
  TF_CHECK_ARG(p, "tf_kv_append: unknown pool");
  TF_CHECK_ARG(layer >= 0 && layer < p->n_layers, "tf_kv_append: bad layer %d", layer);
  TF_CHECK_ARG(n >= 0, "tf_kv_append: n < 0");
  if (n == 0) return TF_OK;
  TF_CHECK_ARG(dev_table && dev_rows && dev_pos && k && v, "tf_kv_append: NULL pointer");
  TF_CHECK_ARG(kv_row_stride % 8 == 0, "tf_kv_append: row stride must keep 16-byte alignment");
  int64_t warps = (int64_t)n * 2 * p->kv_heads;
  int threads = 256;
  int64_t blocks = (warps * 32 + threads - 1) / threads;
  append_kernel<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(
      view_of(*p), dev_table, row_stride, dev_rows, dev_pos, n, layer, (const uint16_t*)k, (const uint16_t*)v,
      kv_row_stride);
  TF_LAUNCH_CHECK();
  return TF_OK;
}

int tf_rope_kv_append(int64_t pool, const int32_t* dev_table, int32_t row_stride, const int32_t* dev_rows,
                      const int32_t* dev_pos, int32_t n, int32_t layer, const void* qkv, int32_t n_q_heads,
                      const float* inv_freq, void* q_out, void* kv_out, void* stream) {
  Pool* p = get_pool(pool);
  TF_CHECK_ARG(p, "tf_rope_kv_append: unknown pool");
  TF_CHECK_ARG(layer >= 0 && layer < p->n_layers, "tf_rope_kv_append: bad layer %d", layer);
  TF_CHECK_ARG(n >= 0, "tf_rope_kv_append: n < 0");
  if (n == 0) return TF_OK;
  TF_CHECK_ARG(dev_table && dev_rows && dev_pos && qkv && inv_freq && q_out, "tf_rope_kv_append: NULL pointer");
  TF_CHECK_ARG(p->head_dim % 8 == 0 && p->head_dim / 2 <= kRopeMaxPairs, "tf_rope_kv_append: head_dim %d",
               p->head_dim);
  rope_append_kernel<<<(unsigned)n, kRopeThreads, 0, (cudaStream_t)stream>>>(
      view_of(*p), dev_table, row_stride, dev_rows, dev_pos, n, layer, (const uint16_t*)qkv, n_q_heads, inv_freq,
      (uint16_t*)q_out, (uint16_t*)kv_out, nullptr);
  TF_LAUNCH_CHECK();
  return TF_OK;
}

int tf_rope_kv_append_wt(int64_t pool, const int32_t* dev_table, const int32_t* dev_host_table, int32_t row_stride,
                         const int32_t* dev_rows, const int32_t* dev_pos, int32_t n, int32_t layer, const void* qkv,
                         int32_t n_q_heads, const float* inv_freq, void* q_out, void* kv_out, void* stream) {
  Pool* p = get_pool(pool);
  TF_CHECK_ARG(p, "tf_rope_kv_append_wt: unknown pool");
  TF_CHECK_ARG(p->host_dev, "tf_rope_kv_append_wt: pool has no host tier");
  TF_CHECK_ARG(layer >= 0 && layer < p->n_layers, "tf_rope_kv_append_wt: bad layer %d", layer);
  TF_CHECK_ARG(n >= 0, "tf_rope_kv_append_wt: n < 0");
  if (n == 0) return TF_OK;
  TF_CHECK_ARG(dev_table && dev_host_table && dev_rows && dev_pos && qkv && inv_freq && q_out,
               "tf_rope_kv_append_wt: NULL pointer");
  TF_CHECK_ARG(p->head_dim % 8 == 0 && p->head_dim / 2 <= kRopeMaxPairs, "tf_rope_kv_append_wt: head_dim %d",
               p->head_dim);
  rope_append_kernel<<<(unsigned)n, kRopeThreads, 0, (cudaStream_t)stream>>>(
      view_of(*p), dev_table, row_stride, dev_rows, dev_pos, n, layer, (const uint16_t*)qkv, n_q_heads, inv_freq,
      (uint16_t*)q_out, (uint16_t*)kv_out, dev_host_table);
  TF_LAUNCH_CHECK();
  return TF_OK;
}

int tf_kv_fill_synthetic(int64_t pool, const int32_t* dev_table, int32_t row_stride, const tf_span* spans,
                         int32_t n_spans, uint32_t seed, void* stream) {
  Pool* p = get_pool(pool);
  TF_CHECK_ARG(p, "tf_kv_fill_synthetic: unknown pool");
  TF_CHECK_ARG(n_spans >= 0 && (n_spans == 0 || (spans && dev_table)), "tf_kv_fill_synthetic: bad args");
  for (int32_t base = 0; base < n_spans; base += kMaxSpans) {
    SpanArgs a;
    a.n = std::min<int32_t>(kMaxSpans, n_spans - base);
    a.seed = seed;
    a.stride = row_stride;
    int64_t max_e = 0;
    int m = 0;
    for (int i = 0; i < a.n; ++i) {
      const tf_span& s = spans[base + i];
      TF_CHECK_ARG(s.pos_begin >= 0 && s.pos_end >= s.pos_begin, "tf_kv_fill_synthetic: bad span");
      if (s.pos_end == s.pos_begin) continue;
      a.row[m] = s.row;
      a.rid[m] = s.rid;
      a.lo[m] = s.pos_begin;
      a.hi[m] = s.pos_end;
      max_e = std::max<int64_t>(max_e, (int64_t)(s.pos_end - s.pos_begin) * p->n_layers * 2 * p->kv_heads * p->head_dim);
      ++m;
    }
    a.n = m;
    if (m == 0) continue;
    unsigned gx = (unsigned)std::min<int64_t>(256, (max_e + 255) / 256);
    fill_synth_kernel<<<dim3(gx, m), 256, 0, (cudaStream_t)stream>>>(view_of(*p), dev_table, a);
    TF_LAUNCH_CHECK();
  }
  return TF_OK;
}

int tf_q_fill_synthetic(void* q, const int32_t* dev_rids, const int32_t* dev_pos, int32_t B, int32_t layer,
                        int32_t n_q_heads, int32_t head_dim, uint32_t seed, void* stream) {
  TF_CHECK_ARG(q && dev_rids && dev_pos && B >= 0, "tf_q_fill_synthetic: bad args");
  int64_t total = (int64_t)B * n_q_heads * head_dim;
  if (total == 0) return TF_OK;
  q_synth_kernel<<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      (uint16_t*)q, dev_rids, dev_pos, B, layer, n_q_heads, head_dim, seed);
  TF_LAUNCH_CHECK();
  return TF_OK;
}

}  // extern "C"
