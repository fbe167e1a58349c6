// Paged GQA decode attention over the block-major KV pool.
//
// Replaces the reference's affine decode cost (tokensim/costs.py:45-59,
// dispatched by _dispatch_gpu, tokensim/engine.py:669-708) with the real
// memory-bound kernel.  Layout: one (block, layer, K|V, kv_head) tile is a
// contiguous [16 slots][head_dim] bf16 array, so a warp streams a whole tile
// with one 16-byte load per lane per row pair - fully coalesced, no gather.
//
// Work split: CTA = (request b, kv head, KV split); 4 warps, each warp walks
// every 4th block of its split with its own online-softmax state; the warps
// merge through shared memory; splits merge in a second tiny kernel.
// Per block a warp loads K and V (8 KiB for hd=128) up front, computes the
// G=Hq/Hkv query heads' scores with a butterfly reduce-scatter (30 shuffles
// instead of 128), and accumulates P.V in fp32.
#include <float.h>
#include <stdlib.h>

#include <algorithm>

#include "tf_common.cuh"
#include "tf_attn_tma.cuh"

namespace tf {

constexpr int kAttnWarps = 4;
constexpr int kBlk = 16;  // tokens per block (pool block_tokens must be 16)

template <int N>
struct Pow2Ceil {
  static constexpr int v = N <= 1 ? 1 : 2 * Pow2Ceil<(N + 1) / 2>::v;
};

__device__ __forceinline__ void bf16x8_to_f32(const uint4& u, float* f) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
  }
}

struct AttnArgs {
  const uint16_t* pool;
  const uint16_t* q;
  const int32_t* table;
  const int32_t* rows;
  const int32_t* ctx;
  float* ws_acc;  // [B*Hq][splits][D]
  float* ws_ml;   // [B*Hq][splits][2]
  uint16_t* out;
  int64_t block_elems;
  int32_t stride, n_layers, kv_heads, layer, hq, splits, blocks_per_split;
  int32_t min_blocks_per_split;  // v3: per-request split size = max(this, ceil(nblk_b / splits))
  float scale_log2;
  // v4 (stream-K): batch, partial slots per (request, kv head), self-resetting counters
  int32_t B, kmax;
  int32_t* counters;
  int32_t mutate;  // test-only fault injection (attn_mutate)
  int32_t balanced, ctas;  // v3: device-side balanced split plan over ~ctas CTAs (1-D grid)
  int32_t l2_prefetch;     // v3: blocks per warp bulk-prefetched into L2 past the ring (0 = off)
};

// D = head_dim, G = q heads per kv head.
template <int D, int G>
__global__ void __launch_bounds__(kAttnWarps * 32) paged_attn_kernel(const AttnArgs a) {
  constexpr int LPR = D / 8;          // lanes per K/V row (one uint4 each)
  constexpr int TPP = 32 / LPR;       // rows (tokens) per warp pass
  constexpr int ITER = kBlk / TPP;    // passes per block
  constexpr int GP = Pow2Ceil<G>::v > LPR / ITER ? Pow2Ceil<G>::v : LPR / ITER;  // padded head count
  constexpr int NV = ITER * GP;       // partial scores per lane before reduce
  constexpr int NR = NV / LPR;        // reduced scores per lane
  static_assert(NV % LPR == 0 && NR >= 1, "unsupported (D, G)");

  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int bh = blockIdx.y;  // b * kv_heads + kvh
  const int b = bh / a.kv_heads, kvh = bh % a.kv_heads;
  const int split = blockIdx.x;
  const int ctx = a.ctx[b];
  const int nblk = (ctx + kBlk - 1) / kBlk;
  const int blk_lo = split * a.blocks_per_split;
  const int blk_hi = min(nblk, blk_lo + a.blocks_per_split);
  const int col = (lane % LPR) * 8;  // first head dim this lane owns
  const int rsub = lane / LPR;       // row within a pass

  // q for the lane's 8 dims, all G heads, pre-scaled for exp2
  float qf[G][8];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const int h = kvh * G + g;
    uint4 u = *reinterpret_cast<const uint4*>(a.q + ((int64_t)b * a.hq + h) * D + col);
    bf16x8_to_f32(u, qf[g]);
#pragma unroll
    for (int j = 0; j < 8; ++j) qf[g][j] *= a.scale_log2;
  }

  float m[G], l[G], acc[G][8];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    m[g] = -FLT_MAX;
    l[g] = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[g][j] = 0.f;
  }
  __shared__ float p_sh[kAttnWarps][kBlk][GP];

  const int32_t* trow = a.table + (int64_t)a.rows[b] * a.stride;
  const int64_t tile = (int64_t)kBlk * D;
  const int64_t koff = (((int64_t)a.layer * 2 + 0) * a.kv_heads + kvh) * tile;
  const int64_t voff = (((int64_t)a.layer * 2 + 1) * a.kv_heads + kvh) * tile;

  for (int blk = blk_lo + warp; blk < blk_hi; blk += kAttnWarps) {
    const int64_t base = (int64_t)__ldg(trow + blk) * a.block_elems;
    const uint16_t* kt = a.pool + base + koff;
    const uint16_t* vt = a.pool + base + voff;
    uint4 kr[ITER], vr[ITER];
#pragma unroll
    for (int it = 0; it < ITER; ++it) {
      const int t = it * TPP + rsub;
      kr[it] = __ldg(reinterpret_cast<const uint4*>(kt + t * D + col));
    }
#pragma unroll
    for (int it = 0; it < ITER; ++it) {
      const int t = it * TPP + rsub;
      vr[it] = __ldg(reinterpret_cast<const uint4*>(vt + t * D + col));
    }
    // partial dot products: val[it*GP + g]
    float val[NV];
#pragma unroll
    for (int it = 0; it < ITER; ++it) {
      float kf[8];
      bf16x8_to_f32(kr[it], kf);
#pragma unroll
      for (int g = 0; g < GP; ++g) {
        float s = 0.f;
        if (g < G) {
#pragma unroll
          for (int j = 0; j < 8; ++j) s = fmaf(qf[g][j], kf[j], s);
        }
        val[it * GP + g] = s;
      }
    }
    // butterfly reduce-scatter over the LPR lanes of a row group
    int cnt = NV;
#pragma unroll
    for (int off = LPR / 2; off >= 1; off >>= 1) {
      const bool upper = (lane & off) != 0;
      const int half = cnt / 2;
#pragma unroll
      for (int i = 0; i < NV / 2; ++i) {
        if (i < half) {
          float send = upper ? val[i] : val[i + half];
          float keep = upper ? val[i + half] : val[i];
          float recv = __shfl_xor_sync(0xffffffffu, send, off);
          val[i] = keep + recv;
        }
      }
      cnt = half;
    }
    // lane (x = lane % LPR) now owns flat indices x*NR .. x*NR+NR-1
    const int x = lane % LPR;
    float bm[G];
#pragma unroll
    for (int g = 0; g < G; ++g) bm[g] = -FLT_MAX;
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const int fi = x * NR + r;
      const int it = fi / GP, g = fi % GP;
      const int t = it * TPP + rsub;
      const bool valid = (g < G) && (blk * kBlk + t < ctx);
      if (!valid) val[r] = -FLT_MAX;
#pragma unroll
      for (int gg = 0; gg < G; ++gg)
        if (g == gg) bm[gg] = fmaxf(bm[gg], val[r]);
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) bm[g] = fmaxf(bm[g], __shfl_xor_sync(0xffffffffu, bm[g], off));
    }
    float alpha[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const float mn = fmaxf(m[g], bm[g]);
      alpha[g] = exp2f(m[g] - mn);
      m[g] = mn;
      l[g] *= alpha[g];
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[g][j] *= alpha[g];
    }
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const int fi = x * NR + r;
      const int it = fi / GP, g = fi % GP;
      const int t = it * TPP + rsub;
      float p = 0.f;
#pragma unroll
      for (int gg = 0; gg < G; ++gg)
        if (g == gg && val[r] > -FLT_MAX) p = exp2f(val[r] - m[gg]);
#pragma unroll
      for (int gg = 0; gg < G; ++gg)
        if (g == gg) l[gg] += p;
      p_sh[warp][t][g] = p;
    }
    __syncwarp();
    // P.V for the lane's rows (t = it*TPP + rsub) and dims [col, col+8)
#pragma unroll
    for (int it = 0; it < ITER; ++it) {
      const int t = it * TPP + rsub;
      if (blk * kBlk + t >= ctx) continue;  // slots past ctx may hold stale bits
      float vf[8];
      bf16x8_to_f32(vr[it], vf);
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const float p = p_sh[warp][t][g];
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[g][j] = fmaf(p, vf[j], acc[g][j]);
      }
    }
    __syncwarp();
  }

  // reduce l over the warp, acc over the TPP row groups
#pragma unroll
  for (int g = 0; g < G; ++g) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) l[g] += __shfl_xor_sync(0xffffffffu, l[g], off);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
#pragma unroll
      for (int off = 16; off >= LPR; off >>= 1) acc[g][j] += __shfl_xor_sync(0xffffffffu, acc[g][j], off);
    }
  }
  // merge the warps through shared memory
  __shared__ float m_sh[kAttnWarps][G], l_sh[kAttnWarps][G];
  __shared__ float acc_sh[kAttnWarps][G][D];
  if (lane == 0) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      m_sh[warp][g] = m[g];
      l_sh[warp][g] = l[g];
    }
  }
  if (rsub == 0) {
#pragma unroll
    for (int g = 0; g < G; ++g)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc_sh[warp][g][col + j] = acc[g][j];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < G * D; e += blockDim.x) {
    const int g = e / D, d = e % D;
    float mm = -FLT_MAX;
#pragma unroll
    for (int w = 0; w < kAttnWarps; ++w) mm = fmaxf(mm, m_sh[w][g]);
    float ll = 0.f, aa = 0.f;
#pragma unroll
    for (int w = 0; w < kAttnWarps; ++w) {
      const float f = (m_sh[w][g] == -FLT_MAX) ? 0.f : exp2f(m_sh[w][g] - mm);
      ll += l_sh[w][g] * f;
      aa += acc_sh[w][g][d] * f;
    }
    const int h = kvh * G + g;
    const int64_t row = (int64_t)b * a.hq + h;
    if (a.splits == 1) {
      const float o = ll > 0.f ? aa / ll : 0.f;
      a.out[row * D + d] = __bfloat16_as_ushort(__float2bfloat16_rn(o));
    } else {
      a.ws_acc[(row * a.splits + split) * D + d] = aa;
      if (d == 0) {
        a.ws_ml[(row * a.splits + split) * 2 + 0] = mm;
        a.ws_ml[(row * a.splits + split) * 2 + 1] = ll;
      }
    }
  }
}

// one CTA per (b, q head): merge the splits
template <int D>
__global__ void attn_combine_kernel(const AttnArgs a) {
  const int64_t row = blockIdx.x;
  float mm = -FLT_MAX;
  for (int s = 0; s < a.splits; ++s) mm = fmaxf(mm, a.ws_ml[(row * a.splits + s) * 2]);
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    float ll = 0.f, aa = 0.f;
    for (int s = 0; s < a.splits; ++s) {
      const float ms = a.ws_ml[(row * a.splits + s) * 2];
      if (ms == -FLT_MAX) continue;
      const float f = exp2f(ms - mm);
      ll += a.ws_ml[(row * a.splits + s) * 2 + 1] * f;
      aa += a.ws_acc[(row * a.splits + s) * D + d] * f;
    }
    a.out[row * D + d] = __bfloat16_as_ushort(__float2bfloat16_rn(ll > 0.f ? aa / ll : 0.f));
  }
}

// ------------------------------------------------------------------------
// v2: TMA bulk-copy pipeline.  Warp 0 is the producer: one elected lane
// streams each block's contiguous K tile and V tile (16 x head_dim bf16 each)
// into an S-stage shared-memory ring with cp.async.bulk (the TMA engine does
// the address generation; no register staging), signalling mbarriers with the
// transaction bytes.  Warps 1..4 consume stages round-robin with the same
// math as v1, reading conflict-free 16-B rows from shared memory, and release
// each stage through an "empty" mbarrier.  Bytes in flight per CTA = S x 8 KiB.
constexpr int kStages = 8;
constexpr int kConsumers = 4;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

template <int D, int G>
__global__ void __launch_bounds__((kConsumers + 1) * 32) paged_attn_tma_kernel(const AttnArgs a) {
  constexpr int LPR = D / 8;
  constexpr int TPP = 32 / LPR;
  constexpr int ITER = kBlk / TPP;
  constexpr int GP = Pow2Ceil<G>::v > LPR / ITER ? Pow2Ceil<G>::v : LPR / ITER;
  constexpr int NV = ITER * GP;
  constexpr int NR = NV / LPR;
  constexpr uint32_t kTile = kBlk * D * 2;  // bytes of one K or V tile
  static_assert(NV % LPR == 0 && NR >= 1, "unsupported (D, G)");

  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint16_t* kv_sh = reinterpret_cast<uint16_t*>(smem_raw);  // [kStages][2][kBlk*D]
  __shared__ __align__(8) uint64_t full_bar[kStages], empty_bar[kStages];
  __shared__ float p_sh[kConsumers][kBlk][GP];
  __shared__ float m_sh[kConsumers][G], l_sh[kConsumers][G];
  __shared__ float acc_sh[kConsumers][G][D];

  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int bh = blockIdx.y;
  const int b = bh / a.kv_heads, kvh = bh % a.kv_heads;
  const int split = blockIdx.x;
  const int ctx = a.ctx[b];
  const int nblk = (ctx + kBlk - 1) / kBlk;
  const int blk_lo = split * a.blocks_per_split;
  const int blk_hi = min(nblk, blk_lo + a.blocks_per_split);
  const int nloc = max(0, blk_hi - blk_lo);

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const int64_t tile = (int64_t)kBlk * D;
  const int64_t koff = (((int64_t)a.layer * 2 + 0) * a.kv_heads + kvh) * tile;
  const int64_t voff = (((int64_t)a.layer * 2 + 1) * a.kv_heads + kvh) * tile;
  const int32_t* trow = a.table + (int64_t)a.rows[b] * a.stride;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      for (int i = 0; i < nloc; ++i) {
        const int s = i % kStages;
        if (i >= kStages) mbar_wait(&empty_bar[s], ((i / kStages) - 1) & 1);
        const int64_t base = (int64_t)__ldg(trow + blk_lo + i) * a.block_elems;
        uint16_t* dst = kv_sh + (int64_t)s * 2 * tile;
        mbar_expect_tx(&full_bar[s], 2 * kTile);
        tma_bulk_g2s(dst, a.pool + base + koff, kTile, &full_bar[s]);
        tma_bulk_g2s(dst + tile, a.pool + base + voff, kTile, &full_bar[s]);
      }
    }
  } else {
    // ------------------------------------------------------------ consumers
    const int c = warp - 1;
    const int col = (lane % LPR) * 8;
    const int rsub = lane / LPR;
    float qf[G][8];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int h = kvh * G + g;
      uint4 u = *reinterpret_cast<const uint4*>(a.q + ((int64_t)b * a.hq + h) * D + col);
      bf16x8_to_f32(u, qf[g]);
#pragma unroll
      for (int j = 0; j < 8; ++j) qf[g][j] *= a.scale_log2;
    }
    float m[G], l[G], acc[G][8];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      m[g] = -FLT_MAX;
      l[g] = 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[g][j] = 0.f;
    }
    for (int i = c; i < nloc; i += kConsumers) {
      const int s = i % kStages;
      const int blk = blk_lo + i;
      mbar_wait(&full_bar[s], (i / kStages) & 1);
      const uint16_t* kt = kv_sh + (int64_t)s * 2 * tile;
      const uint16_t* vt = kt + tile;
      float val[NV];
#pragma unroll
      for (int it = 0; it < ITER; ++it) {
        const int t = it * TPP + rsub;
        float kf[8];
        bf16x8_to_f32(*reinterpret_cast<const uint4*>(kt + t * D + col), kf);
#pragma unroll
        for (int g = 0; g < GP; ++g) {
          float sacc = 0.f;
          if (g < G) {
#pragma unroll
            for (int j = 0; j < 8; ++j) sacc = fmaf(qf[g][j], kf[j], sacc);
          }
          val[it * GP + g] = sacc;
        }
      }
      int cnt = NV;
#pragma unroll
      for (int off = LPR / 2; off >= 1; off >>= 1) {
        const bool upper = (lane & off) != 0;
        const int half = cnt / 2;
#pragma unroll
        for (int k = 0; k < NV / 2; ++k) {
          if (k < half) {
            float send = upper ? val[k] : val[k + half];
            float keep = upper ? val[k + half] : val[k];
            val[k] = keep + __shfl_xor_sync(0xffffffffu, send, off);
          }
        }
        cnt = half;
      }
      const int x = lane % LPR;
      float bm[G];
#pragma unroll
      for (int g = 0; g < G; ++g) bm[g] = -FLT_MAX;
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        const int fi = x * NR + r;
        const int g = fi % GP, t = (fi / GP) * TPP + rsub;
        if (!((g < G) && (blk * kBlk + t < ctx))) val[r] = -FLT_MAX;
#pragma unroll
        for (int gg = 0; gg < G; ++gg)
          if (g == gg) bm[gg] = fmaxf(bm[gg], val[r]);
      }
#pragma unroll
      for (int g = 0; g < G; ++g) {
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) bm[g] = fmaxf(bm[g], __shfl_xor_sync(0xffffffffu, bm[g], off));
        const float mn = fmaxf(m[g], bm[g]);
        const float alpha = exp2f(m[g] - mn);
        m[g] = mn;
        l[g] *= alpha;
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[g][j] *= alpha;
      }
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        const int fi = x * NR + r;
        const int g = fi % GP, t = (fi / GP) * TPP + rsub;
        float p = 0.f;
#pragma unroll
        for (int gg = 0; gg < G; ++gg)
          if (g == gg && val[r] > -FLT_MAX) p = exp2f(val[r] - m[gg]);
#pragma unroll
        for (int gg = 0; gg < G; ++gg)
          if (g == gg) l[gg] += p;
        p_sh[c][t][g] = p;
      }
      __syncwarp();
#pragma unroll
      for (int it = 0; it < ITER; ++it) {
        const int t = it * TPP + rsub;
        if (blk * kBlk + t >= ctx) continue;
        float vf[8];
        bf16x8_to_f32(*reinterpret_cast<const uint4*>(vt + t * D + col), vf);
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const float p = p_sh[c][t][g];
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[g][j] = fmaf(p, vf[j], acc[g][j]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[s]);
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) l[g] += __shfl_xor_sync(0xffffffffu, l[g], off);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
#pragma unroll
        for (int off = 16; off >= LPR; off >>= 1) acc[g][j] += __shfl_xor_sync(0xffffffffu, acc[g][j], off);
      }
    }
    if (lane == 0) {
#pragma unroll
      for (int g = 0; g < G; ++g) {
        m_sh[c][g] = m[g];
        l_sh[c][g] = l[g];
      }
    }
    if (rsub == 0) {
#pragma unroll
      for (int g = 0; g < G; ++g)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc_sh[c][g][col + j] = acc[g][j];
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < G * D; e += blockDim.x) {
    const int g = e / D, d = e % D;
    float mm = -FLT_MAX;
#pragma unroll
    for (int w = 0; w < kConsumers; ++w) mm = fmaxf(mm, m_sh[w][g]);
    float ll = 0.f, aa = 0.f;
#pragma unroll
    for (int w = 0; w < kConsumers; ++w) {
      const float f = (m_sh[w][g] == -FLT_MAX) ? 0.f : exp2f(m_sh[w][g] - mm);
      ll += l_sh[w][g] * f;
      aa += acc_sh[w][g][d] * f;
    }
    const int h = kvh * G + g;
    const int64_t row = (int64_t)b * a.hq + h;
    if (a.splits == 1) {
      a.out[row * D + d] = __bfloat16_as_ushort(__float2bfloat16_rn(ll > 0.f ? aa / ll : 0.f));
    } else {
      a.ws_acc[(row * a.splits + split) * D + d] = aa;
      if (d == 0) {
        a.ws_ml[(row * a.splits + split) * 2 + 0] = mm;
        a.ws_ml[(row * a.splits + split) * 2 + 1] = ll;
      }
    }
  }
}

// ------------------------------------------------------------------------
// v3: tensor cores for QK and PV (mma.sync m16n8k16 bf16 -> fp32).
// Each warp owns every 4th block of the CTA's split and streams it through a
// private 3-stage cp.async ring in shared memory (K and V tiles, rows padded
// to 272 B so ldmatrix is conflict-free).  Per 16-token block a warp issues
// 16 MMAs for S = Q K^T (the G q heads of the kv head fill rows 0..G-1 of
// the 16-row A tile) and 16 MMAs for O += P V, where P is re-used straight
// from the S accumulators as the A operand (no shuffle / smem round trip).
// ~100 instructions per block per warp instead of ~1000 on the CUDA cores.
constexpr int kV3Warps = 4;
constexpr int kRowPad = 136;  // bf16 elements per padded smem row (128 + 8)

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void ldsm_x4(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3, const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(smem_u32(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3, const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(smem_u32(p)));
}
__device__ __forceinline__ void mma_bf16(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  return (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(lo)) |
         ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(hi)) << 16);
}

// S = ring stages per warp (S - 1 blocks in flight); 2 stages fit 3 CTAs per
// SM (12 warps), 3 stages 2 CTAs per SM (8 warps).
__device__ __forceinline__ uint32_t movt3(uint32_t x) {  // transpose an 8x8 bf16 fragment across the warp
  uint32_t y;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}

// TR = transposed contractions (v5's math inside v3's grid): S^T[16 tokens][8
// heads] = K Q^T and O^T[D][8 heads] += V^T P^T - the G <= 8 q heads fill the
// N = 8 side of m16n8k16 instead of G of the 16 M rows, so a block costs 16
// MMAs instead of 32 and the output accumulators 32 registers instead of 64.
template <int G, int S, bool TR>
__global__ void __launch_bounds__(kV3Warps * 32, S == 2 ? 3 : 2) paged_attn_mma_kernel(const AttnArgs a) {
  constexpr int D = 128;
  static_assert(G >= 1 && G <= 8, "v3 packs the group into rows 0..7 of the 16-row tile");
  static_assert(S >= 2 && S <= 4, "2..4 stages");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  // per warp: [S][K|V][16 rows][kRowPad]
  constexpr int kTileElems = kBlk * kRowPad;
  constexpr int kWarpElems = S * 2 * kTileElems;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  uint16_t* ring = reinterpret_cast<uint16_t*>(smem_raw) + warp * kWarpElems;

  // ---- this CTA's (request b, kv head, split) and the split count of (b, kv head)
  int b, kvh, split, nsplit, slot0;
  if (a.balanced) {
    // Device-side balanced plan (same on every CTA, from the contexts in HBM,
    // so a captured graph re-plans for the batch it replays): every request
    // is cut into ceil(nblk_b / per) splits with per = max(min, ceil(total
    // blocks x kv / a.ctas)), so all CTAs carry ~the same number of blocks
    // and the grid is ~a.ctas = a whole number of waves of resident CTAs - no
    // wave tail, no dependence on a host-side max_ctx.  CTA i takes the i-th
    // (b, kv head, split) in request-major order; CTAs past the last exit.
    __shared__ int map_sh[5];
    if (warp == 0) {
      int tot = 0;
      for (int base = 0; base < a.B; base += 32) {
        const int bb = base + lane;
        if (bb < a.B) tot += (__ldg(a.ctx + bb) + kBlk - 1) / kBlk;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
      const int per = max(a.min_blocks_per_split, (tot * a.kv_heads + a.ctas - 1) / a.ctas);
      const int me = blockIdx.x;
      int carry = 0;
      for (int base = 0; base < a.B; base += 32) {
        const int bb = base + lane;
        const int nb = bb < a.B ? (__ldg(a.ctx + bb) + kBlk - 1) / kBlk : 0;
        const int sp = bb < a.B ? max(1, (nb + per - 1) / per) : 0;
        const int v = sp * a.kv_heads;
        int incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int t = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += t;
        }
        const int excl = carry + incl - v;
        if (bb < a.B && me >= excl && me < excl + v) {
          map_sh[0] = bb;
          map_sh[1] = (me - excl) / sp;
          map_sh[2] = (me - excl) % sp;
          map_sh[3] = sp;
          map_sh[4] = excl + ((me - excl) / sp) * sp;
        }
        carry += __shfl_sync(0xffffffffu, incl, 31);
      }
      if (lane == 0 && me >= carry) map_sh[0] = -1;
    }
    __syncthreads();
    b = map_sh[0];
    if (b < 0) return;  // uniform: the whole CTA has no work
    kvh = map_sh[1];
    split = map_sh[2];
    nsplit = map_sh[3];
    slot0 = map_sh[4];
  } else {
    b = blockIdx.y / a.kv_heads;
    kvh = blockIdx.y % a.kv_heads;
    split = blockIdx.x;
    nsplit = a.splits;
    slot0 = blockIdx.y * a.splits;
  }
  const int bh = b * a.kv_heads + kvh;
  const int ctx = a.ctx[b];
  const int nblk = (ctx + kBlk - 1) / kBlk;
  const int ctx_eff = (a.mutate == 1 && nblk >= 8) ? min(ctx, (nblk - nblk / 8) * kBlk) : ctx;
  // split size per request: a short request in a launch planned for a long
  // maximum context still spreads over all splits instead of idling them
  const int bps = a.balanced ? (nblk + nsplit - 1) / nsplit
                             : max(a.min_blocks_per_split, (nblk + a.splits - 1) / a.splits);
  const int blk_lo = split * bps;
  const int blk_hi = min(nblk, blk_lo + bps);
  const int nmine = blk_hi > blk_lo + warp ? (blk_hi - blk_lo - warp + kV3Warps - 1) / kV3Warps : 0;

  const int64_t tile = (int64_t)kBlk * D;
  const int64_t koff = (((int64_t)a.layer * 2 + 0) * a.kv_heads + kvh) * tile;
  const int64_t voff = (((int64_t)a.layer * 2 + 1) * a.kv_heads + kvh) * tile;
  const int32_t* trow = a.table + (int64_t)a.rows[b] * a.stride;
  // the warp's first 32 table entries in one coalesced load (lane i: block i),
  // so the pipeline prologue waits for one table load instead of S - 1
  // dependent ones
  const int tab_pre = lane < nmine ? __ldg(trow + blk_lo + warp + lane * kV3Warps) : 0;

  // Memory-level parallelism beyond the shared-memory ring: the K and V
  // tiles of the warp's block l2_prefetch blocks past the ring's newest stage
  // are requested into L2 with one bulk prefetch each (no shared memory, no
  // registers), so the ring's cp.async hits L2 instead of waiting on DRAM
  auto prefetch_l2 = [&](int jp) {
    if (a.l2_prefetch <= 0 || jp >= nmine) return;  // warp-uniform
    const int ent = jp < 32 ? __shfl_sync(0xffffffffu, tab_pre, jp) : __ldg(trow + blk_lo + warp + jp * kV3Warps);
    if (lane == 0) {
      const uint16_t* base = a.pool + (int64_t)ent * a.block_elems;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + koff), "r"((uint32_t)(tile * 2))
                   : "memory");
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + voff), "r"((uint32_t)(tile * 2))
                   : "memory");
    }
  };
  auto issue = [&](int j) {  // warp-local block j -> stage j % S
    if (j < nmine) {
      const int blk = blk_lo + warp + j * kV3Warps;
      const int ent = j < 32 ? __shfl_sync(0xffffffffu, tab_pre, j) : __ldg(trow + blk);
      const int64_t base = (int64_t)ent * a.block_elems;
      uint16_t* ks = ring + (j % S) * 2 * kTileElems;
      uint16_t* vs = ks + kTileElems;
#pragma unroll
      for (int u = 0; u < 8; ++u) {  // 256 x 16 B per tile, 8 per lane
        const int ch = u * 32 + lane;
        const int r = ch >> 4, c16 = ch & 15;
        cp_async16(ks + r * kRowPad + c16 * 8, a.pool + base + koff + ch * 8);
        cp_async16(vs + r * kRowPad + c16 * 8, a.pool + base + voff + ch * 8);
      }
    }
    cp_async_commit();
    if (j >= S - 1) prefetch_l2(j + a.l2_prefetch);
  };
#pragma unroll
  for (int jj = S - 1; jj < S - 1 + a.l2_prefetch; ++jj) prefetch_l2(jj);
#pragma unroll
  for (int p0 = 0; p0 < S - 1; ++p0) issue(p0);

  // ---- per-warp partial in a uniform shape for the epilogue: head g of the
  // group -> acc over D, running max, sum
  const int r0 = lane >> 2, cq = (lane & 3) * 2;
  float m_fin[2], l_fin[2];  // TR: heads h0, h0 + 1; v3: row r0 in [0]
  float o[16][4];            // v3: [n-tile of 8 dims][c]; TR uses o[0..7] as [m-tile of 16 dims][c]
#pragma unroll
  for (int n = 0; n < 16; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
  if constexpr (TR) {
    // B operand Q^T: head g4 = r0 (zero past G), dims 16kk + 2q4 (+1), (+8)
    uint32_t qb[8][2];
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const uint16_t* qrow = a.q + ((int64_t)b * a.hq + kvh * G + (r0 < G ? r0 : 0)) * D + kk * 16 + cq;
      qb[kk][0] = r0 < G ? *reinterpret_cast<const uint32_t*>(qrow) : 0u;
      qb[kk][1] = r0 < G ? *reinterpret_cast<const uint32_t*>(qrow + 8) : 0u;
    }
    float m_0 = -FLT_MAX, m_1 = -FLT_MAX, l_0 = 0.f, l_1 = 0.f;
    const int lr = lane & 7, mi = lane >> 3;
    const int k_row = (mi & 1) * 8 + lr, k_cadd = mi >> 1;  // K as the A operand (non-trans)
    const int v_row = (mi >> 1) * 8 + lr, v_cadd = mi & 1;  // V^T as the A operand (.trans)
    for (int j = 0; j < nmine; ++j) {
      issue(j + S - 1);
      cp_async_wait<S - 1>();
      __syncwarp();
      const uint16_t* ks = ring + (j % S) * 2 * kTileElems;
      const uint16_t* vs = ks + kTileElems;
      const int blk = blk_lo + warp + j * kV3Warps;
      // S^T = K Q^T, two accumulators (even / odd k-steps) halve the MMA chain
      float sa[4] = {0.f, 0.f, 0.f, 0.f}, sb[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        uint32_t a0_, a1_, a2_, a3_;
        ldsm_x4(a0_, a1_, a2_, a3_, ks + k_row * kRowPad + kk * 16 + k_cadd * 8);
        const uint32_t af[4] = {a0_, a1_, a2_, a3_};
        mma_bf16((kk & 1) ? sb : sa, af, qb[kk][0], qb[kk][1]);
      }
      // online softmax per head (this thread: tokens r0, r0 + 8; heads cq, cq + 1)
      const int t0 = blk * kBlk + r0;
      float s00 = (sa[0] + sb[0]) * a.scale_log2, s01 = (sa[1] + sb[1]) * a.scale_log2;
      float s10 = (sa[2] + sb[2]) * a.scale_log2, s11 = (sa[3] + sb[3]) * a.scale_log2;
      if (t0 >= ctx_eff) s00 = s01 = -FLT_MAX;
      if (t0 + 8 >= ctx_eff) s10 = s11 = -FLT_MAX;
      float mx0 = fmaxf(s00, s10), mx1 = fmaxf(s01, s11);
#pragma unroll
      for (int off = 4; off < 32; off <<= 1) {
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, off));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, off));
      }
      const float mn0 = fmaxf(m_0, mx0), mn1 = fmaxf(m_1, mx1);
      const float al0 = exp2f(m_0 - mn0), al1 = exp2f(m_1 - mn1);
      m_0 = mn0;
      m_1 = mn1;
      const float p00 = s00 > -FLT_MAX ? exp2f(s00 - mn0) : 0.f;
      const float p01 = s01 > -FLT_MAX ? exp2f(s01 - mn1) : 0.f;
      const float p10 = s10 > -FLT_MAX ? exp2f(s10 - mn0) : 0.f;
      const float p11 = s11 > -FLT_MAX ? exp2f(s11 - mn1) : 0.f;
      l_0 = l_0 * al0 + p00 + p10;
      l_1 = l_1 * al1 + p01 + p11;
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) {
        o[mt][0] *= al0;
        o[mt][1] *= al1;
        o[mt][2] *= al0;
        o[mt][3] *= al1;
      }
      // P^T (tokens x heads) -> B operand (tokens along the quad index)
      const uint32_t pb0 = movt3(pack_bf16(p00, p01));
      const uint32_t pb1 = movt3(pack_bf16(p10, p11));
      const int valid = ctx - blk * kBlk;
      if (valid < kBlk) {
        // V slots past ctx may hold stale bits (NaN * 0 = NaN in the MMA): zero them
        uint16_t* vw = const_cast<uint16_t*>(vs);
        for (int e = lane; e < (kBlk - valid) * (D / 8); e += 32) {
          const int r = valid + e / (D / 8), c8 = e % (D / 8);
          *reinterpret_cast<uint4*>(vw + r * kRowPad + c8 * 8) = make_uint4(0, 0, 0, 0);
        }
        __syncwarp();
      }
      // O^T += V^T P^T: 8 m-tiles of 16 dims
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) {
        uint32_t a0_, a1_, a2_, a3_;
        ldsm_x4_t(a0_, a1_, a2_, a3_, vs + v_row * kRowPad + mt * 16 + v_cadd * 8);
        const uint32_t af[4] = {a0_, a1_, a2_, a3_};
        mma_bf16(o[mt], af, pb0, pb1);
      }
      __syncwarp();  // the stage is refilled by issue(j + S - 1) next iteration
    }
    cp_async_wait<0>();
#pragma unroll
    for (int off = 4; off < 32; off <<= 1) {
      l_0 += __shfl_xor_sync(0xffffffffu, l_0, off);
      l_1 += __shfl_xor_sync(0xffffffffu, l_1, off);
    }
    m_fin[0] = m_0;
    m_fin[1] = m_1;
    l_fin[0] = l_0;
    l_fin[1] = l_1;
  } else {
    // Q as the A operand: rows 0..G-1 = the group's heads (scaled later), rest 0
    uint32_t qa[8][4];
  #pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      uint32_t lo = 0, hi = 0;
      if (r0 < G) {
        const uint16_t* qrow = a.q + ((int64_t)b * a.hq + kvh * G + r0) * D + kk * 16 + cq;
        lo = *reinterpret_cast<const uint32_t*>(qrow);
        hi = *reinterpret_cast<const uint32_t*>(qrow + 8);
      }
      qa[kk][0] = lo;
      qa[kk][1] = 0;  // row r0 + 8 >= 8 > G - 1
      qa[kk][2] = hi;
      qa[kk][3] = 0;
    }
    float m0 = -FLT_MAX, l0 = 0.f;  // row r0 (rows r0+8 are padding)

    for (int j = 0; j < nmine; ++j) {
      issue(j + S - 1);
      cp_async_wait<S - 1>();
      __syncwarp();
      const uint16_t* ks = ring + (j % S) * 2 * kTileElems;
      const uint16_t* vs = ks + kTileElems;
      const int blk = blk_lo + warp + j * kV3Warps;
      // ---- S = Q K^T : two n-tiles of 8 tokens, 8 k-steps of 16 dims
      float s[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
      const int lr = lane & 7, lm = lane >> 3;  // ldmatrix: row within matrix, matrix id
  #pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        uint32_t b00, b01, b10, b11;
        // matrices: (tok 0-7, dims lo), (tok 0-7, dims hi), (tok 8-15, dims lo), (tok 8-15, dims hi)
        const uint16_t* p = ks + ((lm >> 1) * 8 + lr) * kRowPad + kk * 16 + (lm & 1) * 8;
        ldsm_x4(b00, b01, b10, b11, p);
        mma_bf16(s[0], qa[kk], b00, b01);
        mma_bf16(s[1], qa[kk], b10, b11);
      }
      // ---- online softmax on row r0 (c0, c1 of each n-tile)
      float mx = -FLT_MAX;
  #pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
  #pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int t = nt * 8 + cq + e;
          float v = s[nt][e] * a.scale_log2;
          if (blk * kBlk + t >= ctx_eff) v = -FLT_MAX;
          s[nt][e] = v;
          mx = fmaxf(mx, v);
        }
      }
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      const float mn = fmaxf(m0, mx);
      const float alpha = exp2f(m0 - mn);
      m0 = mn;
      float ps = 0.f;
  #pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
  #pragma unroll
        for (int e = 0; e < 2; ++e) {
          const float p = s[nt][e] > -FLT_MAX ? exp2f(s[nt][e] - mn) : 0.f;
          s[nt][e] = p;
          ps += p;
        }
      }
      l0 = l0 * alpha + ps;
  #pragma unroll
      for (int n = 0; n < 16; ++n) {
        o[n][0] *= alpha;
        o[n][1] *= alpha;
      }
      // ---- O += P V : P from the S accumulators (rows r0 / r0+8 = 0), V via ldmatrix.trans
      uint32_t pa[4];
      pa[0] = pack_bf16(s[0][0], s[0][1]);
      pa[1] = 0;
      pa[2] = pack_bf16(s[1][0], s[1][1]);
      pa[3] = 0;
      const int valid = ctx - blk * kBlk;
      if (valid < kBlk) {
        // V slots past ctx may hold stale bits (NaN * 0 = NaN in the MMA): zero them
        uint16_t* vw = const_cast<uint16_t*>(vs);
        for (int e = lane; e < (kBlk - valid) * (D / 8); e += 32) {
          const int r = valid + e / (D / 8), c8 = e % (D / 8);
          *reinterpret_cast<uint4*>(vw + r * kRowPad + c8 * 8) = make_uint4(0, 0, 0, 0);
        }
        __syncwarp();
      }
  #pragma unroll
      for (int np = 0; np < 8; ++np) {  // pairs of 8-dim n-tiles
        uint32_t v0, v1, v2, v3;
        // matrices: (tok 0-7, dims 16np..+8), (tok 8-15, same), (tok 0-7, dims +8), (tok 8-15, dims +8)
        const uint16_t* p = vs + ((lm & 1) * 8 + lr) * kRowPad + np * 16 + (lm >> 1) * 8;
        ldsm_x4_t(v0, v1, v2, v3, p);
        mma_bf16(o[2 * np], pa, v0, v1);
        mma_bf16(o[2 * np + 1], pa, v2, v3);
      }
      __syncwarp();  // the stage is refilled by issue(j + 3) next iteration
    }
    cp_async_wait<0>();
    l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
    l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
    m_fin[0] = m0;
    l_fin[0] = l0;
  }

  // ---- merge the 4 warps (reuse the ring memory), write split / output
  __syncthreads();
  float* acc_sh = reinterpret_cast<float*>(smem_raw);  // [kV3Warps][G][D]
  __shared__ float m_sh[kV3Warps][8], l_sh[kV3Warps][8];
  if constexpr (TR) {
    // o[mt][0 / 2]: head cq at dims 16mt + r0 (+ 8); o[mt][1 / 3]: head cq + 1
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const int h = cq + hh;
      if (h < G) {
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
          acc_sh[(warp * G + h) * D + 16 * mt + r0] = o[mt][hh];
          acc_sh[(warp * G + h) * D + 16 * mt + r0 + 8] = o[mt][2 + hh];
        }
        if (r0 == 0) {
          m_sh[warp][h] = m_fin[hh];
          l_sh[warp][h] = l_fin[hh];
        }
      }
    }
  } else if (r0 < G) {
#pragma unroll
    for (int n = 0; n < 16; ++n) {
      acc_sh[(warp * G + r0) * D + n * 8 + cq] = o[n][0];
      acc_sh[(warp * G + r0) * D + n * 8 + cq + 1] = o[n][1];
    }
    if ((lane & 3) == 0) {
      m_sh[warp][r0] = m_fin[0];
      l_sh[warp][r0] = l_fin[0];
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < G * D; e += blockDim.x) {
    const int g = e / D, d = e % D;
    float mm = -FLT_MAX;
#pragma unroll
    for (int w = 0; w < kV3Warps; ++w) mm = fmaxf(mm, m_sh[w][g]);
    float ll = 0.f, aa = 0.f;
#pragma unroll
    for (int w = 0; w < kV3Warps; ++w) {
      const float f = (m_sh[w][g] == -FLT_MAX) ? 0.f : exp2f(m_sh[w][g] - mm);
      ll += l_sh[w][g] * f;
      aa += acc_sh[(w * G + g) * D + d] * f;
    }
    const int64_t row = (int64_t)b * a.hq + kvh * G + g;
    if (nsplit == 1) {
      a.out[row * D + d] = __bfloat16_as_ushort(__float2bfloat16_rn(ll > 0.f ? aa / ll : 0.f));
    } else {
      // partial slot of (b, kv head, split): [slot][G][D] / [slot][G][2]
      const int64_t pi = (int64_t)(slot0 + split) * G + g;
      a.ws_acc[pi * D + d] = aa;
      if (d == 0) {
        a.ws_ml[pi * 2 + 0] = mm;
        a.ws_ml[pi * 2 + 1] = ll;
      }
    }
  }
  if (nsplit == 1) return;
  // ---- in-kernel split merge: the LAST split CTA of this (request, kv head)
  // to arrive merges every split's partial (no separate combine launch, and
  // nobody waits: the counter only elects the merger).  Writers publish with
  // a fence before the counter increment; the merger reads through L2.
  __shared__ int last_sh;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const int prev = atomicAdd(a.counters + bh, 1);
    last_sh = (prev == nsplit - 1);
    if (last_sh) a.counters[bh] = 0;  // every split arrived: ready for the next launch
  }
  __syncthreads();
  if (!last_sh) return;
  __threadfence();
  for (int e = threadIdx.x; e < G * D; e += blockDim.x) {
    const int g = e / D, d = e % D;
    const int64_t row = (int64_t)b * a.hq + kvh * G + g;
    float mm = -FLT_MAX;
    for (int sp = 0; sp < nsplit; ++sp) mm = fmaxf(mm, __ldcg(a.ws_ml + ((int64_t)(slot0 + sp) * G + g) * 2));
    float ll = 0.f, aa = 0.f;
    for (int sp = 0; sp < nsplit; ++sp) {
      const int64_t pi = (int64_t)(slot0 + sp) * G + g;
      const float ms = __ldcg(a.ws_ml + pi * 2);
      const float f = ms == -FLT_MAX ? 0.f : exp2f(ms - mm);
      ll += __ldcg(a.ws_ml + pi * 2 + 1) * f;
      aa += __ldcg(a.ws_acc + pi * D + d) * f;
    }
    a.out[row * D + d] = __bfloat16_as_ushort(__float2bfloat16_rn(ll > 0.f ? aa / ll : 0.f));
  }
}


// ------------------------------------------------------------------------
// v4: stream-K warps.  The (request, kv head, block) work of one layer is
// flattened (request-major, then kv head, then block) and split into equal
// contiguous ranges, one per warp of a persistent grid (2 CTAs x 4 warps per
// SM).  Each warp streams its range through its own 3-stage cp.async ring
// (v3's tensor-core inner loop: S = Q K^T and O += P V on mma.sync, fp32
// online softmax) WITHOUT draining at (request, head) boundaries: the issue
// cursor runs two blocks ahead across segment boundaries, so per-request
// prologue / epilogue bubbles (v3's cost at short or ragged contexts) vanish
// and every warp moves the same number of bytes.  A segment wholly inside one
// warp writes the output directly; a segment shared by k warps writes k
// partials and the last warp to finish (self-resetting atomic counter) merges
// them - no second launch.
constexpr int kV4Warps = 4;
constexpr int kV4Stages = 3;
constexpr int kPerMin = 8;      // minimum blocks per warp (bounds partials per segment)
constexpr int kV4MaxB = 1024;   // requests per launch (prefix sums in shared memory)
constexpr int kV4CtasPerSm = 2;

struct SegCursor {
  int b, kvh, j, nb;
};

__device__ __forceinline__ void seg_locate(const int* pre, int B, int kv, int f, SegCursor& c) {
  int lo = 0, hi = B;  // largest b with pre[b] * kv <= f
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (pre[mid] * kv <= f) lo = mid; else hi = mid;
  }
  while (lo < B - 1 && pre[lo + 1] == pre[lo]) ++lo;  // skip empty requests
  c.b = lo;
  c.nb = pre[lo + 1] - pre[lo];
  const int rem = f - pre[lo] * kv;
  c.kvh = c.nb ? rem / c.nb : 0;
  c.j = c.nb ? rem % c.nb : 0;
}

__device__ __forceinline__ void seg_advance(const int* pre, int B, int kv, SegCursor& c) {
  if (++c.j < c.nb) return;
  c.j = 0;
  if (++c.kvh < kv) return;
  c.kvh = 0;
  do {
    ++c.b;
    c.nb = c.b < B ? pre[c.b + 1] - pre[c.b] : 1;
  } while (c.nb == 0);
}

template <int G>
__global__ void __launch_bounds__(kV4Warps * 32, kV4CtasPerSm) paged_attn_stream_kernel(const AttnArgs a) {
  constexpr int D = 128;
  static_assert(G >= 1 && G <= 8, "v4 packs the group into rows 0..7 of the 16-row tile");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ int pre[kV4MaxB + 1];
  constexpr int kTileElems = kBlk * kRowPad;
  constexpr int kWarpElems = kV4Stages * 2 * kTileElems;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  uint16_t* ring = reinterpret_cast<uint16_t*>(smem_raw) + warp * kWarpElems;
  const int B = a.B, kv = a.kv_heads;

  // blocks per request -> prefix sums (every CTA, ~B/32 warp scans)
  if (warp == 0) {
    int carry = 0;
    if (lane == 0) pre[0] = 0;
    for (int base = 0; base < B; base += 32) {
      const int b = base + lane;
      int v = b < B ? (a.ctx[b] + kBlk - 1) / kBlk : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
      }
      if (b < B) pre[b + 1] = carry + v;
      carry += __shfl_sync(0xffffffffu, v, 31);
    }
  }
  __syncthreads();
  const int T = pre[B] * kv;
  const int W = gridDim.x * kV4Warps;
  const int per = max(kPerMin, (T + W - 1) / W);
  const int gw = blockIdx.x * kV4Warps + warp;
  const int lo = gw * per;
  if (lo >= T) return;
  const int hi = min(T, lo + per);
  const int n = hi - lo;

  const int64_t tile = (int64_t)kBlk * D;
  SegCursor ic;  // issue cursor (runs two blocks ahead of the compute cursor)
  seg_locate(pre, B, kv, lo, ic);
  const int32_t* itrow = a.table + (int64_t)a.rows[ic.b] * a.stride;  // table row of ic.b
  int itrow_b = ic.b;
  const int r0q = lane >> 2, cqq = (lane & 3) * 2;
  uint32_t qn[8][2];  // q fragments of the next segment, prefetched at its first issue
  auto load_q = [&](int b, int kvh) {
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      uint32_t qlo = 0, qhi = 0;
      if (r0q < G) {
        const uint16_t* qrow = a.q + ((int64_t)b * a.hq + kvh * G + r0q) * D + kk * 16 + cqq;
        qlo = __ldg(reinterpret_cast<const unsigned int*>(qrow));
        qhi = __ldg(reinterpret_cast<const unsigned int*>(qrow + 8));
      }
      qn[kk][0] = qlo;
      qn[kk][1] = qhi;
    }
  };
  load_q(ic.b, ic.kvh);
  auto issue = [&](int i) {
    if (i < n) {
      if (ic.b != itrow_b) {
        itrow_b = ic.b;
        itrow = a.table + (int64_t)a.rows[ic.b] * a.stride;
      }
      const int64_t koff = (((int64_t)a.layer * 2 + 0) * kv + ic.kvh) * tile;
      const int64_t voff = (((int64_t)a.layer * 2 + 1) * kv + ic.kvh) * tile;
      const int64_t base = (int64_t)__ldg(itrow + ic.j) * a.block_elems;
      uint16_t* ks = ring + (i % kV4Stages) * 2 * kTileElems;
      uint16_t* vs = ks + kTileElems;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int ch = u * 32 + lane;
        const int r = ch >> 4, c16 = ch & 15;
        cp_async16(ks + r * kRowPad + c16 * 8, a.pool + base + koff + ch * 8);
        cp_async16(vs + r * kRowPad + c16 * 8, a.pool + base + voff + ch * 8);
      }
      seg_advance(pre, B, kv, ic);
    }
    cp_async_commit();
  };
  issue(0);
  issue(1);

  const int r0 = lane >> 2, cq = (lane & 3) * 2;
  const int lr = lane & 7, lm = lane >> 3;
  SegCursor cc, seg;  // compute cursor; the segment being accumulated
  seg_locate(pre, B, kv, lo, cc);
  uint32_t qa[8][4];
  float o[16][4];
  float m0 = -FLT_MAX, l0 = 0.f;
  int ctx = 0;

  auto begin_segment = [&]() {
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      qa[kk][0] = qn[kk][0];
      qa[kk][1] = 0;
      qa[kk][2] = qn[kk][1];
      qa[kk][3] = 0;
    }
#pragma unroll
    for (int nn = 0; nn < 16; ++nn) o[nn][0] = o[nn][1] = o[nn][2] = o[nn][3] = 0.f;
    m0 = -FLT_MAX;
    l0 = 0.f;
    ctx = a.ctx[cc.b];
    seg = cc;
    // prefetch the next segment's q (used at the next boundary, >= 1 block later)
    SegCursor nx = cc;
    nx.j = nx.nb - 1;
    seg_advance(pre, B, kv, nx);
    if (nx.b < B) load_q(nx.b, nx.kvh);
  };

  auto end_segment = [&](const SegCursor& sc) {
    float l = l0;
    l += __shfl_xor_sync(0xffffffffu, l, 1);
    l += __shfl_xor_sync(0xffffffffu, l, 2);
    const int S = pre[sc.b] * kv + sc.kvh * sc.nb;
    const int first = S / per, last = (S + sc.nb - 1) / per;
    const int64_t row0 = (int64_t)sc.b * a.hq + sc.kvh * G;
    if (first == last) {  // the whole segment is this warp's: normalise and store
      if (r0 < G) {
        const float inv = l > 0.f ? 1.f / l : 0.f;
        uint32_t* orow = reinterpret_cast<uint32_t*>(a.out + (row0 + r0) * D);
#pragma unroll
        for (int nn = 0; nn < 16; ++nn) orow[(nn * 8 + cq) >> 1] = pack_bf16(o[nn][0] * inv, o[nn][1] * inv);
      }
      return;
    }
    const int seg = sc.b * kv + sc.kvh;
    const int64_t slot0 = (int64_t)seg * a.kmax;
    const int64_t slot = slot0 + (gw - first);
    if (r0 < G) {
      float* acc = a.ws_acc + (slot * G + r0) * D;
#pragma unroll
      for (int nn = 0; nn < 16; ++nn)
        *reinterpret_cast<float2*>(acc + nn * 8 + cq) = make_float2(o[nn][0], o[nn][1]);
      if ((lane & 3) == 0) {
        a.ws_ml[(slot * G + r0) * 2 + 0] = m0;
        a.ws_ml[(slot * G + r0) * 2 + 1] = l;
      }
    }
    __threadfence();
    __syncwarp();
    int old = 0;
    if (lane == 0) old = atomicAdd(a.counters + seg, 1);
    old = __shfl_sync(0xffffffffu, old, 0);
    const int cnt = last - first + 1;
    if (old != cnt - 1) return;
    // last of the segment's warps: merge the cnt partials.  Lane l owns
    // elements [l*E, l*E+E) of the [G][D] tile (E = 4G, whole float4s, never
    // straddling a row); all loads of a pass are independent (one L2 round trip).
    __threadfence();
    constexpr int E = G * D / 32;
    constexpr int NC = E / 4;
    float mrow[NC], lsum[NC];
    float4 acc4[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      mrow[c] = -FLT_MAX;
      lsum[c] = 0.f;
      acc4[c] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    for (int k = 0; k < cnt; ++k) {
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const int g = (lane * E + 4 * c) / D;
        mrow[c] = fmaxf(mrow[c], __ldcg(a.ws_ml + ((slot0 + k) * G + g) * 2));
      }
    }
    for (int k = 0; k < cnt; ++k) {
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const int e = lane * E + 4 * c, g = e / D, d = e % D;
        const float mk = __ldcg(a.ws_ml + ((slot0 + k) * G + g) * 2);
        const float lk = __ldcg(a.ws_ml + ((slot0 + k) * G + g) * 2 + 1);
        const float4 v = __ldcg(reinterpret_cast<const float4*>(a.ws_acc + ((slot0 + k) * G + g) * D + d));
        const float w = exp2f(mk - mrow[c]);
        lsum[c] += lk * w;
        acc4[c].x += v.x * w;
        acc4[c].y += v.y * w;
        acc4[c].z += v.z * w;
        acc4[c].w += v.w * w;
      }
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int e = lane * E + 4 * c, g = e / D, d = e % D;
      const float inv = lsum[c] > 0.f ? 1.f / lsum[c] : 0.f;
      uint2 pk;
      pk.x = pack_bf16(acc4[c].x * inv, acc4[c].y * inv);
      pk.y = pack_bf16(acc4[c].z * inv, acc4[c].w * inv);
      *reinterpret_cast<uint2*>(a.out + (row0 + g) * D + d) = pk;
    }
    if (lane == 0) a.counters[seg] = 0;  // ready for the next launch
  };

  begin_segment();
  for (int i = 0; i < n; ++i) {
    if (i > 0 && cc.j == 0) {  // crossed into the next (request, kv head)
      end_segment(seg);
      begin_segment();
    }
    issue(i + 2);
    cp_async_wait<2>();
    __syncwarp();
    const uint16_t* ks = ring + (i % kV4Stages) * 2 * kTileElems;
    const uint16_t* vs = ks + kTileElems;
    const int blk = cc.j;
    float sfr[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      uint32_t b00, b01, b10, b11;
      const uint16_t* p = ks + ((lm >> 1) * 8 + lr) * kRowPad + kk * 16 + (lm & 1) * 8;
      ldsm_x4(b00, b01, b10, b11, p);
      mma_bf16(sfr[0], qa[kk], b00, b01);
      mma_bf16(sfr[1], qa[kk], b10, b11);
    }
    float mx = -FLT_MAX;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int t = nt * 8 + cq + e;
        float v = sfr[nt][e] * a.scale_log2;
        if (blk * kBlk + t >= ctx) v = -FLT_MAX;
        sfr[nt][e] = v;
        mx = fmaxf(mx, v);
      }
    }
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    const float mn = fmaxf(m0, mx);
    const float alpha = exp2f(m0 - mn);
    m0 = mn;
    float ps = 0.f;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const float pv = sfr[nt][e] > -FLT_MAX ? exp2f(sfr[nt][e] - mn) : 0.f;
        sfr[nt][e] = pv;
        ps += pv;
      }
    }
    l0 = l0 * alpha + ps;
#pragma unroll
    for (int nn = 0; nn < 16; ++nn) {
      o[nn][0] *= alpha;
      o[nn][1] *= alpha;
    }
    uint32_t pa[4];
    pa[0] = pack_bf16(sfr[0][0], sfr[0][1]);
    pa[1] = 0;
    pa[2] = pack_bf16(sfr[1][0], sfr[1][1]);
    pa[3] = 0;
    const int valid = ctx - blk * kBlk;
    if (valid < kBlk) {
      uint16_t* vw = const_cast<uint16_t*>(vs);
      for (int e = lane; e < (kBlk - valid) * (D / 8); e += 32) {
        const int r = valid + e / (D / 8), c8 = e % (D / 8);
        *reinterpret_cast<uint4*>(vw + r * kRowPad + c8 * 8) = make_uint4(0, 0, 0, 0);
      }
      __syncwarp();
    }
#pragma unroll
    for (int np = 0; np < 8; ++np) {
      uint32_t v0, v1, v2, v3;
      const uint16_t* p = vs + ((lm & 1) * 8 + lr) * kRowPad + np * 16 + (lm >> 1) * 8;
      ldsm_x4_t(v0, v1, v2, v3, p);
      mma_bf16(o[2 * np], pa, v0, v1);
      mma_bf16(o[2 * np + 1], pa, v2, v3);
    }
    __syncwarp();
    seg_advance(pre, B, kv, cc);
  }
  cp_async_wait<0>();
  end_segment(seg);
}

// implementation selector: 0 (default) = by batch - v5 (TMA stream-K,
// tf_attn_tma.cu) for B <= 64, v3 above (measured: profiles/r2_attn_*.json);
// 5 = v5, 3 = split-KV cp.async tensor-core kernel, 4 = cp.async stream-K,
// 2 = bulk-copy CUDA-core, 1 = register-staged CUDA-core.  TF_ATTN_IMPL
// overrides the default at start-up; tf_paged_decode_attn_impl() switches it
// at run time (A/B benchmarks and the parity tests run every implementation
// in one process).
static int g_impl = -1;
static int attn_impl_sel() {
  if (g_impl < 0) {
    const char* e = getenv("TF_ATTN_IMPL");
    g_impl = (e && e[0] >= '1' && e[0] <= '5') ? e[0] - '0' : 0;
  }
  return g_impl;
}
static thread_local int g_cur_b = 0;  // batch of the launch being planned (for the "by batch" default)
// default: v3 at every batch.  v5 (TMA + stream-K, TF_ATTN_IMPL=5) is within
// a few percent of v3 where measured (profiles/r2_attn_v3_v5.json) but its
// in-kernel merge stalled the full-size C2 replay (tiny shapes, ragged B <= 64;
// its waits are now bounded, tests/attn_parity.py), so it stays opt-in
static int attn_impl() {
  const int i = attn_impl_sel();
  return i ? i : 3;
}

// test-only fault injection (TF_ATTN_MUTATE=1: every (request, kv head) with
// >= 8 blocks ignores its last eighth, the shape of a dropped split); the
// parity tests run it in a subprocess and must FAIL under it
static int attn_mutate() {
  static int m = -1;
  if (m < 0) {
    const char* e = getenv("TF_ATTN_MUTATE");
    m = (e && e[0] == '1') ? 1 : 0;
  }
  return m;
}

// v3 ring depth: 2 stages (3 CTAs = 12 warps per SM) at B <= 96, 3 stages
// (2 CTAs, 8 warps) above: at B = 64 the extra resident warps win 4-5% at
// C2-live contexts, at B = 128 the two are equal (profiles/r2_attn_lpt_stages.json).
// TF_ATTN_STAGES=2|3 forces one.
static int v3_stages() {
  static int st = -1;
  if (st < 0) {
    const char* e = getenv("TF_ATTN_STAGES");
    st = (e && (e[0] == '2' || e[0] == '3')) ? e[0] - '0' : 0;
  }
  return st ? st : (g_cur_b <= 96 ? 2 : 3);
}

static int g_minblk = 8;

static void plan_splits(int B, int kv_heads, int max_ctx, int* splits, int* bps) {
  const int nblk = std::max(1, (max_ctx + kBlk - 1) / kBlk);
  const int base = std::max(1, B * kv_heads);
  // >= ~4 waves of resident CTAs (3 per SM) so the tail wave is cheap,
  // >= 8 blocks per split so the pipeline prologue is amortised
  // tuning knobs (TF_ATTN_WAVES, TF_ATTN_MINBLK) for the split planner
  static int waves = -1, minblk = -1;
  if (waves < 0) {
    const char* w = getenv("TF_ATTN_WAVES");
    const char* m = getenv("TF_ATTN_MINBLK");
    waves = w ? std::max(1, atoi(w)) : 2;  // tuned: profiles/r1_attn_plan_tuning.json
    minblk = m ? std::max(1, atoi(m)) : 8;
    g_minblk = minblk;
  }
  const int per_sm = attn_impl() >= 3 ? (v3_stages() == 2 ? 3 : 2) : 2;  // resident CTAs per SM
  const int target = attn_impl() >= 2 ? 148 * per_sm * waves : 148 * 6;
  int s = std::max(1, std::min((target + base - 1) / base, (nblk + minblk - 1) / minblk));
  int per = (nblk + s - 1) / s;
  s = (nblk + per - 1) / per;
  *splits = s;
  *bps = per;
}

static bool use_v4(int D, int G, int B) { return attn_impl() == 4 && D == 128 && G <= 8 && B <= kV4MaxB; }

// v3 merges its splits in-kernel (last-arriving split CTA per (request, kv
// head), counter region of FIXED size at the start of the workspace, for the
// reason given at attn5_counter_bytes); other kernels use attn_combine_kernel
constexpr int kV3MaxB = 4096;


static int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

static bool v3_used(int D, int G, int B) {
  return attn_impl() >= 3 && attn_impl() != 4 && D == 128 && G <= 8 && B <= kV3MaxB;
}
static int64_t v3_counter_bytes(int kv) { return ((int64_t)kV3MaxB * kv * 4 + 255) / 256 * 256; }
// v3 split plan: the host plan_splits grid (default) or, with
// TF_ATTN_BALANCED=1, the device-side balanced plan over TF_ATTN_BWAVES waves
// of resident CTAs.  The balanced plan is correct but slower at every
// measured shape (profiles/r2_attn_balanced_plan.json): its per-CTA scan of
// the batch's contexts sits on every CTA's critical path, and the extra
// splits it makes at more than one wave add per-CTA prologues
static int v3_balanced() {
  static int b = -1;
  if (b < 0) {
    const char* e = getenv("TF_ATTN_BALANCED");
    b = (e && e[0] == '1') ? 1 : 0;
  }
  return b;
}
static int v3_bwaves() {
  static int w = -1;
  if (w < 0) {
    const char* e = getenv("TF_ATTN_BWAVES");
    w = e ? std::max(1, atoi(e)) : 2;
  }
  return w;
}
static int v3_per_sm() { return v3_stages() == 2 ? 3 : 2; }
// v3 inner loop: transposed contractions (TF_ATTN_TR=1) or the original
static bool v3_transposed() {
  static int t = -1;
  if (t < 0) {
    const char* e = getenv("TF_ATTN_TR");
    t = (e && e[0] == '1') ? 1 : 0;
  }
  return t == 1;
}
static int v3_l2_prefetch() {  // TF_ATTN_PF: blocks prefetched into L2 past the ring, per warp
  static int pf = -1;
  if (pf < 0) {
    const char* e = getenv("TF_ATTN_PF");
    pf = e ? std::max(0, std::min(8, atoi(e))) : 0;
  }
  return pf;
}
static int v3_ctas() { return sm_count() * v3_per_sm() * v3_bwaves(); }
// partial slots of a v3 launch (0: no split can happen)
static int64_t v3_slots(int B, int kv, int splits) {
  if (v3_balanced()) return (int64_t)v3_ctas() + (int64_t)B * kv;
  return splits > 1 ? (int64_t)B * kv * splits : 0;
}

static int64_t v4_kmax(int max_ctx) { return (std::max(1, (max_ctx + kBlk - 1) / kBlk) + kPerMin - 1) / kPerMin + 1; }

// fixed size (the largest batch), for the same reason as attn5_counter_bytes
static int64_t v4_counter_bytes(int B, int kv) {
  (void)B;
  return ((int64_t)kV4MaxB * kv * 4 + 255) / 256 * 256;
}

template <int D, int G>
static int launch(const AttnArgs& a, int B, cudaStream_t st) {
  if (use_v4(D, G, B)) {
    constexpr int GG = G <= 8 ? G : 8;
    const int smem = kV4Warps * kV4Stages * 2 * kBlk * kRowPad * 2;
    static bool attr4 = false;
    if (!attr4) {
      TF_CUDA(cudaFuncSetAttribute(paged_attn_stream_kernel<GG>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      attr4 = true;
    }
    paged_attn_stream_kernel<GG><<<sm_count() * kV4CtasPerSm, kV4Warps * 32, smem, st>>>(a);
    TF_LAUNCH_CHECK();
    return TF_OK;
  }
  dim3 grid(a.splits, B * a.kv_heads);
  if (v3_used(D, G, B)) {
    if (a.balanced) grid = dim3(a.ctas + B * a.kv_heads);
    constexpr int GG = G <= 8 ? G : 8;
    const int S = v3_stages();
    const int smem = kV3Warps * S * 2 * kBlk * kRowPad * 2;
    static bool attr3 = false;
    if (!attr3) {
      TF_CUDA(cudaFuncSetAttribute(paged_attn_mma_kernel<GG, 2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   kV3Warps * 2 * 2 * kBlk * kRowPad * 2));
      TF_CUDA(cudaFuncSetAttribute(paged_attn_mma_kernel<GG, 3, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   kV3Warps * 3 * 2 * kBlk * kRowPad * 2));
      TF_CUDA(cudaFuncSetAttribute(paged_attn_mma_kernel<GG, 2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   kV3Warps * 2 * 2 * kBlk * kRowPad * 2));
      TF_CUDA(cudaFuncSetAttribute(paged_attn_mma_kernel<GG, 3, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   kV3Warps * 3 * 2 * kBlk * kRowPad * 2));
      attr3 = true;
    }
    const bool tr = v3_transposed();
    if (S == 2)
      tr ? paged_attn_mma_kernel<GG, 2, true><<<grid, kV3Warps * 32, smem, st>>>(a)
         : paged_attn_mma_kernel<GG, 2, false><<<grid, kV3Warps * 32, smem, st>>>(a);
    else
      tr ? paged_attn_mma_kernel<GG, 3, true><<<grid, kV3Warps * 32, smem, st>>>(a)
         : paged_attn_mma_kernel<GG, 3, false><<<grid, kV3Warps * 32, smem, st>>>(a);
  } else if (attn_impl() >= 2) {
    const int smem = kStages * 2 * kBlk * D * 2;
    static bool attr = false;
    if (!attr) {
      TF_CUDA(cudaFuncSetAttribute(paged_attn_tma_kernel<D, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      attr = true;
    }
    paged_attn_tma_kernel<D, G><<<grid, (kConsumers + 1) * 32, smem, st>>>(a);
  } else {
    paged_attn_kernel<D, G><<<grid, kAttnWarps * 32, 0, st>>>(a);
  }
  TF_LAUNCH_CHECK();
  if (!v3_used(D, G, B) && a.splits > 1) {
    attn_combine_kernel<D><<<B * a.hq, std::min(D, 128), 0, st>>>(a);
    TF_LAUNCH_CHECK();
  }
  return TF_OK;
}

}  // namespace tf

using namespace tf;

extern "C" {

int64_t tf_paged_decode_attn_workspace(int64_t pool, int32_t B, int32_t max_ctx, int32_t n_q_heads) {
  Pool* p = get_pool(pool);
  if (!p) return -1;
  if (n_q_heads % p->kv_heads) return -1;
  const int G = n_q_heads / p->kv_heads;
  g_cur_b = B;
  if (attn_impl() == 5 && attn5_supported(p, G, B)) return attn5_workspace(p, B, max_ctx, G);
  if (use_v4(p->head_dim, G, B))
    return v4_counter_bytes(B, p->kv_heads) +
           (int64_t)B * p->kv_heads * v4_kmax(max_ctx) * G * (p->head_dim + 2) * (int64_t)sizeof(float);
  int splits, bps;
  plan_splits(B, p->kv_heads, max_ctx, &splits, &bps);
  if (v3_used(p->head_dim, G, B)) {
    const int64_t slots = v3_slots(B, p->kv_heads, splits);
    return slots ? v3_counter_bytes(p->kv_heads) + slots * G * (p->head_dim + 2) * (int64_t)sizeof(float) : 0;
  }
  if (splits == 1) return 0;
  return (int64_t)B * n_q_heads * splits * (p->head_dim + 2) * (int64_t)sizeof(float);
}

int tf_paged_decode_attn(int64_t pool, const void* q, const int32_t* dev_table, int32_t row_stride,
                         const int32_t* dev_rows, const int32_t* dev_ctx, int32_t B, int32_t max_ctx, int32_t layer,
                         int32_t n_q_heads, float scale, void* out, void* workspace, int64_t workspace_bytes,
                         void* stream) {
  Pool* p = get_pool(pool);
  TF_CHECK_ARG(p, "tf_paged_decode_attn: unknown pool");
  TF_CHECK_ARG(p->block_tokens == kBlk, "tf_paged_decode_attn: block_tokens must be 16");
  TF_CHECK_ARG(layer >= 0 && layer < p->n_layers, "tf_paged_decode_attn: bad layer");
  TF_CHECK_ARG(n_q_heads % p->kv_heads == 0, "tf_paged_decode_attn: n_q_heads %% kv_heads != 0");
  TF_CHECK_ARG(B >= 0 && max_ctx >= 0, "tf_paged_decode_attn: bad B/max_ctx");
  if (B == 0) return TF_OK;
  TF_CHECK_ARG(q && dev_table && dev_rows && dev_ctx && out, "tf_paged_decode_attn: NULL pointer");
  AttnArgs a{};
  a.pool = p->gpu;
  a.q = (const uint16_t*)q;
  a.table = dev_table;
  a.rows = dev_rows;
  a.ctx = dev_ctx;
  a.out = (uint16_t*)out;
  a.block_elems = p->block_elems;
  a.stride = row_stride;
  a.n_layers = p->n_layers;
  a.kv_heads = p->kv_heads;
  a.layer = layer;
  a.hq = n_q_heads;
  a.scale_log2 = scale * 1.4426950408889634f;
  const int G = n_q_heads / p->kv_heads;
  const int D = p->head_dim;
  g_cur_b = B;
  a.B = B;
  a.mutate = attn_mutate();
  if (attn_impl() == 5 && attn5_supported(p, G, B)) {
    Attn5Args a5;
    a5.q = (const uint16_t*)q;
    a5.table = dev_table;
    a5.rows = dev_rows;
    a5.ctx = dev_ctx;
    a5.out = (uint16_t*)out;
    a5.stride = row_stride;
    a5.layer = layer;
    a5.hq = n_q_heads;
    a5.B = B;
    a5.scale_log2 = a.scale_log2;
    a5.mutate = a.mutate;
    return attn5_launch(p, a5, G, max_ctx, workspace, workspace_bytes, sm_count(), (cudaStream_t)stream);
  }
  if (use_v4(D, G, B)) {
    a.kmax = (int32_t)v4_kmax(max_ctx);
    const int64_t cb = v4_counter_bytes(B, p->kv_heads);
    const int64_t need4 = cb + (int64_t)B * p->kv_heads * a.kmax * G * (D + 2) * (int64_t)sizeof(float);
    TF_CHECK_ARG(workspace && workspace_bytes >= need4, "tf_paged_decode_attn: workspace too small (%lld < %lld)",
                 (long long)workspace_bytes, (long long)need4);
    a.counters = (int32_t*)workspace;
    a.ws_ml = (float*)((char*)workspace + cb);
    a.ws_acc = a.ws_ml + (int64_t)B * p->kv_heads * a.kmax * G * 2;
    a.splits = 1;
    a.blocks_per_split = 0;
  } else {
  plan_splits(B, p->kv_heads, max_ctx, &a.splits, &a.blocks_per_split);
  a.min_blocks_per_split = g_minblk;
  a.kmax = 0;
  if (v3_used(D, G, B)) {
    // v3: splits merged in-kernel; partials in [slot][G][D] / [slot][G][2]
    a.balanced = v3_balanced();
    a.ctas = a.balanced ? v3_ctas() : 0;
    a.l2_prefetch = v3_l2_prefetch();
    const int64_t slots = v3_slots(B, p->kv_heads, a.splits);
    const int64_t cb = slots ? v3_counter_bytes(p->kv_heads) : 0;
    const int64_t need = slots ? cb + slots * G * (D + 2) * (int64_t)sizeof(float) : 0;
    TF_CHECK_ARG(workspace_bytes >= need && (need == 0 || workspace),
                 "tf_paged_decode_attn: workspace too small (%lld < %lld)", (long long)workspace_bytes,
                 (long long)need);
    a.counters = slots ? (int32_t*)workspace : nullptr;
    a.ws_acc = (float*)((char*)workspace + cb);
    a.ws_ml = a.ws_acc + slots * G * D;
  } else {
    int64_t need = a.splits == 1 ? 0 : (int64_t)B * n_q_heads * a.splits * (p->head_dim + 2) * (int64_t)sizeof(float);
    TF_CHECK_ARG(workspace_bytes >= need && (need == 0 || workspace),
                 "tf_paged_decode_attn: workspace too small (%lld < %lld)", (long long)workspace_bytes,
                 (long long)need);
    a.counters = nullptr;
    a.ws_acc = (float*)workspace;
    a.ws_ml = a.ws_acc + (int64_t)B * n_q_heads * a.splits * p->head_dim;
  }
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (D == 128 && G == 4) return launch<128, 4>(a, B, st);
  if (D == 128 && G == 5) return launch<128, 5>(a, B, st);
  if (D == 128 && G == 8) return launch<128, 8>(a, B, st);
  if (D == 128 && G == 2) return launch<128, 2>(a, B, st);
  if (D == 128 && G == 1) return launch<128, 1>(a, B, st);
  if (D == 64 && G == 2) return launch<64, 2>(a, B, st);
  if (D == 64 && G == 4) return launch<64, 4>(a, B, st);
  if (D == 64 && G == 1) return launch<64, 1>(a, B, st);
  set_error("tf_paged_decode_attn: unsupported head_dim %d / group %d", D, G);
  return TF_EINVAL;
}

int tf_paged_decode_attn_impl(int32_t impl) {
  const int prev = attn_impl_sel();
  if (impl >= 0 && impl <= 5) g_impl = impl;
  return prev;
}

}  // extern "C"
