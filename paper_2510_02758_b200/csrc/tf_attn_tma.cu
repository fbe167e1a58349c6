// v5 paged decode attention: TMA tensor loads into swizzled shared memory,
// transposed tensor-core contractions, stream-K warps over the whole layer.
//
// Replaces the reference's affine decode cost (tokensim/costs.py:45-59, as
// dispatched by _dispatch_gpu, tokensim/engine.py:669-708).
//
// Data movement (Blackwell TMA).  The block-major pool (tf_common.cuh Pool)
// is described ONCE per pool by a rank-3 tensor map: dim0 = 64 bf16 of a
// head-dim half (128 B), dim1 = the halves of a row (stride 128 B), dim2 =
// every 16-slot row of every (block, layer, K|V, kv head) tile (stride
// head_dim*2 B).  One elected lane per warp issues, per 16-token block,
// 2*(head_dim/64) `cp.async.bulk.tensor` loads of a [16 rows][64] box with the
// 128-byte swizzle (16-B chunk c of row r lands at chunk c ^ (r & 7)), so the
// ldmatrix reads below are bank-conflict free without the 272-B row padding
// of v3, and completion is signalled through one mbarrier per ring stage
// (transaction bytes).  No LDGSTS, no per-lane address arithmetic.
//
// Math (mma.sync bf16 -> fp32; tensor cores only for the two contractions):
//   S^T[16 tokens][8 heads] = K[16][D] . Q^T[D][8]      8 MMAs (A = K tile via ldmatrix,
//                                                         B = the group's q rows, in registers)
//   P^T = exp2(S^T*scale - m) (fp32 online softmax per head; masked past ctx)
//   O^T[D][8 heads] += V^T[D][16] . P^T[16][8]          8 MMAs (A = V tile via ldmatrix.trans,
//                                                         B = P^T re-laid out by 2 movmatrix)
// i.e. 16 MMAs and 32 fp32 accumulators per thread per block instead of v3's
// 32 MMAs / 64 accumulators (the G <= 8 q heads of a kv head fill the N=8
// side of the tile instead of 4 of 16 M rows).
//
// Work split (stream-K, as v4): the layer's (request, kv head, block) work is
// flattened and cut into equal contiguous ranges, one per warp of a
// persistent grid; each warp's TMA cursor runs S-1 blocks ahead ACROSS
// (request, head) boundaries, so no warp drains its pipeline between
// segments.  A segment wholly inside one warp is normalised and stored
// directly; a segment shared by k warps leaves k fp32 partials and the last
// warp to finish (self-resetting counter) merges them in the same launch.
#include <cuda.h>
#include <float.h>
#include <stdlib.h>

#include <algorithm>
#include <mutex>

#include "tf_common.cuh"
#include "tf_attn_tma.cuh"

namespace tf {

namespace {

constexpr int kBlk5 = 16;

__device__ __forceinline__ uint32_t s_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init5(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx5(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ unsigned long long now5() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
constexpr unsigned long long kWait5Ns = 2000ull * 1000 * 1000;  // 2 s: a wait that long is a bug, not load

// Diagnostics of a bounded wait that expired (workspace bytes [8, 64), see
// attn5_counter_bytes): int32 [0] = number of expired waits, [2..9] = the
// first one's (kind 1 = TMA stage / 2 = merge counter, logical CTA, warp, B,
// segment, observed, expected, iteration).  The kernel then continues with
// whatever the buffer holds - wrong output instead of a hung GPU.
__device__ __forceinline__ void wait5_expired(int* diag, int kind, int lid, int warp, int B, int sid, int seen,
                                              int want, int it) {
  if (atomicAdd(diag, 1) == 0) {
    int* r = diag + 2;
    r[0] = kind; r[1] = lid; r[2] = warp; r[3] = B; r[4] = sid; r[5] = seen; r[6] = want; r[7] = it;
    __threadfence();
  }
}

__device__ __forceinline__ bool mbar_try5(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(s_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// true when the phase completed; false after kWait5Ns
__device__ __forceinline__ bool mbar_wait5(uint64_t* bar, uint32_t parity) {
  if (mbar_try5(bar, parity)) return true;
  const unsigned long long t0 = now5();
  while (!mbar_try5(bar, parity))
    if (now5() - t0 > kWait5Ns) return false;
  return true;
}
__device__ __forceinline__ void ldsm4(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3, uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm4t(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3, uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ uint32_t movt(uint32_t x) {
  uint32_t y;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ void mma16816(float* c, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pk_bf16(float lo, float hi) {
  return (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(lo)) |
         ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(hi)) << 16);
}

struct Cursor {
  int b, kvh, j, nb;
};

__device__ __forceinline__ void cur_locate(const int* pre, int B, int kv, int f, Cursor& c) {
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

__device__ __forceinline__ void cur_advance(const int* pre, int B, int kv, Cursor& c) {
  if (++c.j < c.nb) return;
  c.j = 0;
  if (++c.kvh < kv) return;
  c.kvh = 0;
  do {
    ++c.b;
    c.nb = c.b < B ? pre[c.b + 1] - pre[c.b] : 1;
  } while (c.nb == 0);
}

// blocks per request -> prefix sums in shared memory (B <= 1024).  Every
// thread of the CTA loads its share of the contexts first (ONE memory round
// trip, not B/32 dependent ones), then warp 0 scans them; ends with a CTA barrier.
template <int NT>
__device__ __forceinline__ void block_prefix(const int32_t* __restrict__ ctx, int B, int* pre) {
  for (int b = threadIdx.x; b < B; b += NT) pre[b + 1] = (__ldg(ctx + b) + kBlk5 - 1) / kBlk5;
  __syncthreads();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    int carry = 0;
    if (lane == 0) pre[0] = 0;
    for (int base = 0; base < B; base += 32) {
      const int b = base + lane;
      int v = b < B ? pre[b + 1] : 0;
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
}

// Programmatic dependent launch (PDL): the prologue of a launch overlaps the
// tail of the kernel before it on the stream; griddep_wait() blocks until
// that kernel has completed and its writes are visible.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// G = q heads per kv head (<= 8), NH = head_dim / 64, S = ring stages per
// warp, W = warps per CTA, CPS = CTAs per SM
template <int G, int NH, int S, int W, int CPS>
__global__ void __launch_bounds__(W * 32, CPS) paged_attn_tma5_kernel(const __grid_constant__ CUtensorMap map,
                                                                        const Attn5Args a) {
  constexpr int D = 64 * NH;
  constexpr uint32_t kHalf = kBlk5 * 64 * 2;          // one [16][64] bf16 box = 2 KiB
  constexpr uint32_t kStage = 2 * NH * kHalf;         // K and V of one block
  static_assert(G >= 1 && G <= 8, "the group fills the N=8 side of the tile");
  extern __shared__ __align__(1024) unsigned char smem5[];
  __shared__ int pre[kAttn5MaxB + 1];
  __shared__ int rows_sh[kAttn5MaxB];
  __shared__ __align__(8) uint64_t bars[W][S];

  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  // 1024-B aligned ring (the 128-B swizzle pattern repeats every 1024 B)
  const uint32_t ring_base = (s_u32(smem5) + 1023u) & ~1023u;
  const uint32_t ring = ring_base + (uint32_t)warp * S * kStage;
  const int B = a.B, kv = a.kv_heads;

  // ---- prologue: reads only what the kernels BEFORE the previous one wrote
  // (contexts, rows, block tables), so under PDL it overlaps that kernel
  __shared__ int lid_sh;
  if (threadIdx.x < W * S) mbar_init5(&bars[threadIdx.x / S][threadIdx.x % S], 1);
  if (threadIdx.x == 0) {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map)) : "memory");
    // logical CTA index in DISPATCH order (ticket): a warp only ever waits on
    // warps of lower logical index, which are resident or finished - no
    // deadlock even when other kernels share the SMs
    lid_sh = (int)(atomicAdd(a.ticket, 1ull) % gridDim.x);
  }
  for (int b = threadIdx.x; b < B; b += W * 32) rows_sh[b] = __ldg(a.rows + b);
  block_prefix<W * 32>(a.ctx, B, pre);
  const int T = pre[B] * kv;
  const int NWt = gridDim.x * W;
  const int per = max(a.min_per, (T + NWt - 1) / NWt);
  const int gw = lid_sh * W + warp;
  const int lo = gw * per;
  const int hi = min(T, lo + per);
  const int n = hi - lo;
  uint64_t* bar = bars[warp];

  // Processing order: the range is ROTATED to start at its tail piece (the
  // first part of a segment continued by higher warps) and wrap to `lo`, so
  // both split pieces of every warp are done first and their partials are
  // published long before anyone merges them.  rot = offset of that piece.
  int rot = 0;
  if (n > 0) {
    Cursor t;
    cur_locate(pre, B, kv, hi - 1, t);
    const int seg_lo = hi - 1 - t.j;  // first position of the last segment touched
    if (t.j != t.nb - 1 && seg_lo > lo) rot = seg_lo - lo;  // partial tail piece, not the whole range
  }
  auto pos_of = [&](int r) { return lo + (r + rot < n ? r + rot : r + rot - n); };

  // Block ids of this warp's range, 32 at a time: lane L of chunk c holds the
  // packed (block << 8 | kv head) of sequence index 32c + L.  Two chunks live
  // in registers; the next is loaded 32 issues before it is needed, so the
  // dependent table load is never on the critical path.
  auto load_chunk = [&](int c) -> int {
    const int r = 32 * c + lane;
    if (r >= n) return 0;
    Cursor t;
    cur_locate(pre, B, kv, pos_of(r), t);
    return (__ldg(a.table + (int64_t)rows_sh[t.b] * a.stride + t.j) << 8) | t.kvh;
  };
  int e_cur = 0, e_nxt = 0, cur_chunk = 0;
  if (n > 0) {
    e_cur = load_chunk(0);
    e_nxt = load_chunk(1);
  }
  // everything below reads q / the KV the previous kernel (rope + append) wrote
  griddep_wait();
  if (n <= 0) return;

  const int64_t tile_rows = (int64_t)kv * kBlk5;  // rows between K and V of one layer
  auto issue = [&](int i) {  // all lanes (uniform); lane 0 issues the TMA
    if (i >= n) return;
    if (i == 32 * (cur_chunk + 1)) {  // all of cur_chunk issued: rotate, fetch chunk + 2
      e_cur = e_nxt;
      ++cur_chunk;
      e_nxt = load_chunk(cur_chunk + 1);
    }
    const int e = __shfl_sync(0xffffffffu, e_cur, i & 31);
    if (lane == 0) {
      const int64_t krow = ((((int64_t)(e >> 8) * a.n_layers + a.layer) * 2) * kv + (e & 255)) * kBlk5;
      const int s = i % S;
      const uint32_t dst = ring + s * kStage;
      mbar_expect_tx5(&bar[s], kStage);
#pragma unroll
      for (int h = 0; h < NH; ++h) {
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
            "%4}], [%5];" ::"r"(dst + h * kHalf),
            "l"(reinterpret_cast<uint64_t>(&map)), "r"(0), "r"(h), "r"((int)krow), "r"(s_u32(&bar[s]))
            : "memory");
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
            "%4}], [%5];" ::"r"(dst + (NH + h) * kHalf),
            "l"(reinterpret_cast<uint64_t>(&map)), "r"(0), "r"(h), "r"((int)(krow + tile_rows)), "r"(s_u32(&bar[s]))
            : "memory");
      }
    }
  };
#pragma unroll
  for (int p0 = 0; p0 < S - 1; ++p0) issue(p0);

  // ---------------------------------------------------------------- math
  const int g4 = lane >> 2, q4 = lane & 3;  // fragment row group / quad index
  const int h0 = 2 * q4;                    // this thread's two heads: h0, h0 + 1
  Cursor cc, seg;
  cur_locate(pre, B, kv, pos_of(0), cc);
  uint32_t qb[4 * NH][2];  // B operand Q^T: head g4, dims 16kk + 2q4 (+1), (+8)
  float o[4 * NH][4];      // O^T accumulators: dims 16mt + g4 (+8), heads h0, h0+1
  float m_0 = -FLT_MAX, m_1 = -FLT_MAX, l_0 = 0.f, l_1 = 0.f;
  int ctx = 0, ctx_eff = 0;

  uint32_t qn[4 * NH][2];  // the NEXT segment's q fragments, loaded one segment ahead
  auto load_q = [&](int b, int kvh) {
    const uint16_t* qrow = a.q + ((int64_t)b * a.hq + kvh * G + (g4 < G ? g4 : 0)) * D + 2 * q4;
#pragma unroll
    for (int kk = 0; kk < 4 * NH; ++kk) {
      qn[kk][0] = g4 < G ? *reinterpret_cast<const unsigned int*>(qrow + kk * 16) : 0u;
      qn[kk][1] = g4 < G ? *reinterpret_cast<const unsigned int*>(qrow + kk * 16 + 8) : 0u;
    }
  };
  load_q(cc.b, cc.kvh);
  auto begin_segment = [&]() {
    seg = cc;
    ctx = __ldg(a.ctx + cc.b);
    ctx_eff = ctx;
    if (a.mutate == 1 && cc.nb >= 8) ctx_eff = min(ctx, (cc.nb - cc.nb / 8) * kBlk5);  // test-only: drop 1/8
#pragma unroll
    for (int kk = 0; kk < 4 * NH; ++kk) {
      qb[kk][0] = qn[kk][0];
      qb[kk][1] = qn[kk][1];
    }
    // prefetch the next segment's q (first used >= 1 block later)
    Cursor nx = cc;
    nx.j = nx.nb - 1;
    cur_advance(pre, B, kv, nx);
    if (nx.b < B) load_q(nx.b, nx.kvh);
#pragma unroll
    for (int mt = 0; mt < 4 * NH; ++mt) o[mt][0] = o[mt][1] = o[mt][2] = o[mt][3] = 0.f;
    m_0 = m_1 = -FLT_MAX;
    l_0 = l_1 = 0.f;
  };

  // A segment wholly inside this warp is normalised and stored.  A segment
  // split over warps first..last: every piece leaves its fp32 partial
  // (accumulator, max, sum) in slot gw - first; the pieces below `last`
  // publish theirs (fence + counter increment) two blocks LATER, when their
  // stores have completed (cheap fence, no stall on the stream); warp `last`
  // merges at its end, after waiting on the counter (only lower warps, see
  // the ticket).  With the rotated order every published piece is one of a
  // warp's first two, so the merger practically never waits.
  int pub_sid = -1, pub_at = 0;     // partial written, published at iteration pub_at
  int mrg_sid = -1, mrg_cnt = 0, mrg_b = 0, mrg_kvh = 0;  // segment this warp merges at its end
  auto publish = [&]() {
    if (pub_sid < 0) return;
    __syncwarp();
    if (lane == 0) {
      __threadfence();
      atomicAdd(a.counters + pub_sid, 1);
    }
    pub_sid = -1;
  };
  auto end_segment = [&](const Cursor& sc, int i_now) {
    publish();
    float l0 = l_0, l1 = l_1;
#pragma unroll
    for (int off = 4; off < 32; off <<= 1) {
      l0 += __shfl_xor_sync(0xffffffffu, l0, off);
      l1 += __shfl_xor_sync(0xffffffffu, l1, off);
    }
    const int Sg = pre[sc.b] * kv + sc.kvh * sc.nb;
    const int first = Sg / per, last = (Sg + sc.nb - 1) / per;
    const int64_t row0 = (int64_t)sc.b * a.hq + sc.kvh * G;
    if (first == last) {
      const float i0 = l0 > 0.f ? 1.f / l0 : 0.f, i1 = l1 > 0.f ? 1.f / l1 : 0.f;
#pragma unroll
      for (int mt = 0; mt < 4 * NH; ++mt) {
        const int d = 16 * mt + g4;
        if (h0 < G) {
          a.out[(row0 + h0) * D + d] = __bfloat16_as_ushort(__float2bfloat16_rn(o[mt][0] * i0));
          a.out[(row0 + h0) * D + d + 8] = __bfloat16_as_ushort(__float2bfloat16_rn(o[mt][2] * i0));
        }
        if (h0 + 1 < G) {
          a.out[(row0 + h0 + 1) * D + d] = __bfloat16_as_ushort(__float2bfloat16_rn(o[mt][1] * i1));
          a.out[(row0 + h0 + 1) * D + d + 8] = __bfloat16_as_ushort(__float2bfloat16_rn(o[mt][3] * i1));
        }
      }
      return;
    }
    const int sid = sc.b * kv + sc.kvh;
    const int64_t slot = (int64_t)sid * a.kmax + (gw - first);
#pragma unroll
    for (int mt = 0; mt < 4 * NH; ++mt) {
      const int d = 16 * mt + g4;
      if (h0 < G) {
        a.ws_acc[(slot * G + h0) * D + d] = o[mt][0];
        a.ws_acc[(slot * G + h0) * D + d + 8] = o[mt][2];
      }
      if (h0 + 1 < G) {
        a.ws_acc[(slot * G + h0 + 1) * D + d] = o[mt][1];
        a.ws_acc[(slot * G + h0 + 1) * D + d + 8] = o[mt][3];
      }
    }
    if (g4 == 0) {
      if (h0 < G) *reinterpret_cast<float2*>(a.ws_ml + (slot * G + h0) * 2) = make_float2(m_0, l0);
      if (h0 + 1 < G) *reinterpret_cast<float2*>(a.ws_ml + (slot * G + h0 + 1) * 2) = make_float2(m_1, l1);
    }
    if (gw == last) {
      mrg_sid = sid;
      mrg_cnt = last - first + 1;
      mrg_b = sc.b;
      mrg_kvh = sc.kvh;
    } else {
      pub_sid = sid;
      pub_at = i_now + 2;
    }
  };

  auto merge = [&]() {
    // wait until the cnt - 1 lower pieces are published (acquire), then merge
    if (lane == 0) {
      unsigned int v = 0;
      unsigned long long t0 = 0;
      for (;;) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.counters + mrg_sid) : "memory");
        if ((int)v == mrg_cnt - 1) break;
        if (!t0) {
          t0 = now5();
        } else if (now5() - t0 > kWait5Ns) {
          wait5_expired(a.diag, 2, lid_sh, warp, B, mrg_sid, (int)v, mrg_cnt - 1, n);
          break;
        }
      }
    }
    __syncwarp();
    const int64_t slot0 = (int64_t)mrg_sid * a.kmax;
    const int64_t row0 = (int64_t)mrg_b * a.hq + mrg_kvh * G;
    // lane owns G*D/32 consecutive elements of the [G][D] tile, in float4s
    constexpr int E = G * D / 32;
    constexpr int NC = (E + 3) / 4;
    float mrow[NC], lsum[NC];
    float4 acc4[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      mrow[c] = -FLT_MAX;
      lsum[c] = 0.f;
      acc4[c] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    for (int k = 0; k < mrg_cnt; ++k) {
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const int e = lane * E + 4 * c;
        if (4 * c < E) mrow[c] = fmaxf(mrow[c], __ldcg(a.ws_ml + ((slot0 + k) * G + e / D) * 2));
      }
    }
    for (int k = 0; k < mrg_cnt; ++k) {
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        if (4 * c >= E) continue;
        const int e = lane * E + 4 * c, g = e / D, d = e % D;
        const float2 ml = __ldcg(reinterpret_cast<const float2*>(a.ws_ml + ((slot0 + k) * G + g) * 2));
        const float4 v = __ldcg(reinterpret_cast<const float4*>(a.ws_acc + ((slot0 + k) * G + g) * D + d));
        const float w = ml.x == -FLT_MAX ? 0.f : exp2f(ml.x - mrow[c]);
        lsum[c] += ml.y * w;
        acc4[c].x += v.x * w;
        acc4[c].y += v.y * w;
        acc4[c].z += v.z * w;
        acc4[c].w += v.w * w;
      }
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      if (4 * c >= E) continue;
      const int e = lane * E + 4 * c, g = e / D, d = e % D;
      const float inv = lsum[c] > 0.f ? 1.f / lsum[c] : 0.f;
      uint2 pk;
      pk.x = pk_bf16(acc4[c].x * inv, acc4[c].y * inv);
      pk.y = pk_bf16(acc4[c].z * inv, acc4[c].w * inv);
      *reinterpret_cast<uint2*>(a.out + (row0 + g) * D + d) = pk;
    }
    if (lane == 0) a.counters[mrg_sid] = 0;  // every piece has arrived: ready for the next launch
  };

  // ldmatrix lane addressing inside a [16 rows][64] swizzled box
  const int lr = lane & 7, mi = lane >> 3;
  // K (A operand, non-trans): matrix mi -> rows (mi&1)*8.., chunk +(mi>>1)
  const int k_row = (mi & 1) * 8 + lr, k_cadd = mi >> 1;
  // V (A operand of V^T, .trans): matrix mi -> rows (mi>>1)*8.., chunk +(mi&1)
  const int v_row = (mi >> 1) * 8 + lr, v_cadd = mi & 1;

  begin_segment();
  for (int i = 0; i < n; ++i) {
    if (i > 0 && (cc.j == 0 || i == n - rot)) {  // next (request, kv head), or the wrap to `lo`
      end_segment(seg, i);
      if (i == n - rot) {  // wrap: the head piece at `lo` (its q was not the prefetched successor)
        cur_locate(pre, B, kv, lo, cc);
        load_q(cc.b, cc.kvh);
      }
      begin_segment();
    }
    if (i == pub_at) publish();
    issue(i + S - 1);
    const int s = i % S;
    if (!mbar_wait5(&bar[s], (uint32_t)((i / S) & 1)) && lane == 0)
      wait5_expired(a.diag, 1, lid_sh, warp, B, -1, i % S, (i / S) & 1, i);
    const uint32_t kst = ring + s * kStage;
    const uint32_t vst = kst + NH * kHalf;
    const int blk = cc.j;

    // ---- S^T = K Q^T: two accumulators (even / odd k-steps) halve the MMA chain
    float sa[4] = {0.f, 0.f, 0.f, 0.f}, sb[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int kk = 0; kk < 4 * NH; ++kk) {
      const int half = kk >> 2, c = ((kk & 3) << 1) + k_cadd;
      uint32_t a0, a1, a2, a3;
      ldsm4(a0, a1, a2, a3, kst + half * kHalf + k_row * 128 + ((c ^ (k_row & 7)) << 4));
      mma16816((kk & 1) ? sb : sa, a0, a1, a2, a3, qb[kk][0], qb[kk][1]);
    }
    // ---- online softmax per head (this thread: tokens g4, g4+8; heads h0, h0+1)
    const int t0 = blk * kBlk5 + g4;
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
    if (__any_sync(0xffffffffu, al0 != 1.f || al1 != 1.f)) {
#pragma unroll
      for (int mt = 0; mt < 4 * NH; ++mt) {
        o[mt][0] *= al0;
        o[mt][1] *= al1;
        o[mt][2] *= al0;
        o[mt][3] *= al1;
      }
    }
    // P^T (tokens x heads) -> B operand (tokens along the quad index): transpose
    // the two 8x8 bf16 fragments in registers
    const uint32_t pb0 = movt(pk_bf16(p00, p01));
    const uint32_t pb1 = movt(pk_bf16(p10, p11));
    // V slots past ctx may hold stale bits (NaN * 0 = NaN in the MMA): zero them
    const int valid = ctx - blk * kBlk5;
    if (valid < kBlk5) {
      for (int e = lane; e < (kBlk5 - valid) * 8 * NH; e += 32) {
        const int r = valid + e / (8 * NH), rest = e % (8 * NH);
        const uint32_t addr = vst + (rest >> 3) * kHalf + r * 128 + ((rest & 7) << 4);
        asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(addr), "r"(0u) : "memory");
      }
      __syncwarp();
    }
    // ---- O^T += V^T P^T
#pragma unroll
    for (int mt = 0; mt < 4 * NH; ++mt) {
      const int half = mt >> 2, c = ((mt & 3) << 1) + v_cadd;
      uint32_t a0, a1, a2, a3;
      ldsm4t(a0, a1, a2, a3, vst + half * kHalf + v_row * 128 + ((c ^ (v_row & 7)) << 4));
      mma16816(o[mt], a0, a1, a2, a3, pb0, pb1);
    }
    __syncwarp();  // every lane is done with stage s before lane 0 refills it
    if (valid < kBlk5 && lane == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    cur_advance(pre, B, kv, cc);
  }
  end_segment(seg, n);
  publish();
  if (mrg_sid >= 0) merge();
}

// launched with the PDL attribute: the prologue may run while the previous
// kernel on the stream drains (griddepcontrol.wait before touching its
// outputs); captured into CUDA graphs as a programmatic edge
template <typename K, typename... Args>
int launch_pdl(K kernel, dim3 grid, dim3 block, int smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  TF_CUDA(cudaLaunchKernelEx(&cfg, kernel, args...));
  TF_LAUNCH_CHECK();
  return TF_OK;
}

template <int G, int NH, int S, int W, int CPS>
int launch5(const CUtensorMap& map, const Attn5Args& a, int sms, cudaStream_t st) {
  constexpr int kStage = 2 * NH * kBlk5 * 64 * 2;
  const int smem = W * S * kStage + 1024;
  static bool attr = false;
  if (!attr) {
    TF_CUDA(cudaFuncSetAttribute(paged_attn_tma5_kernel<G, NH, S, W, CPS>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = true;
  }
  return launch_pdl(paged_attn_tma5_kernel<G, NH, S, W, CPS>, dim3(sms * CPS), dim3(W * 32), smem, st, map, a);
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
    else
      cudaGetLastError();
  });
  return fn;
}

}  // namespace

// The pool's tensor map (built once per pool, host-only: no GPU work, so it
// is safe during CUDA-graph capture).
static int pool_tmap(Pool* p, const CUtensorMap** out) {
  static_assert(sizeof(CUtensorMap) <= sizeof(p->tmap), "tmap storage");
  if (!p->tmap_ok) {
    EncodeTiledFn enc = encode_fn();
    TF_CHECK_ARG(enc, "tf_paged_decode_attn: cuTensorMapEncodeTiled unavailable in the driver");
    const cuuint64_t rows = (cuuint64_t)p->n_blocks * p->n_layers * 2 * p->kv_heads * p->block_tokens;
    cuuint64_t dims[3] = {64, (cuuint64_t)(p->head_dim / 64), rows};
    cuuint64_t strides[2] = {128, (cuuint64_t)p->head_dim * 2};
    cuuint32_t box[3] = {64, 1, (cuuint32_t)kBlk5};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(reinterpret_cast<CUtensorMap*>(p->tmap), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, p->gpu, dims,
                     strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      set_error("tf_paged_decode_attn: cuTensorMapEncodeTiled failed (%d)", (int)r);
      return TF_EIO;
    }
    p->tmap_ok = true;
  }
  *out = reinterpret_cast<const CUtensorMap*>(p->tmap);
  return TF_OK;
}

bool attn5_supported(const Pool* p, int G, int B) {
  const bool inst = p->head_dim == 128 ? (G == 1 || G == 2 || G == 4 || G == 5 || G == 8)
                                        : (p->head_dim == 64 && (G == 1 || G == 2 || G == 4));
  return inst && B <= kAttn5MaxB &&
         p->block_tokens == kBlk5 && p->n_blocks > 0 &&
         (int64_t)p->n_blocks * p->n_layers * 2 * p->kv_heads * p->block_tokens < (1LL << 31);
}

int64_t attn5_kmax(int max_ctx) {
  return (std::max(1, (max_ctx + kBlk5 - 1) / kBlk5) + kAttn5MinPer - 1) / kAttn5MinPer + 1;
}

// workspace: [ticket u64 | diagnostics int32[14] | pad to 256][merge counters kAttn5MaxB*kv int32, to 256]
//            [(max, sum) partials][acc partials]
// The counter region has a FIXED size (the largest batch), independent of this
// launch's B: the counters must read zero at every launch, and the mergers
// reset only the ones they used - if the region grew with B, a larger batch
// would find the previous launch's partials where its counters are and wait
// for a count that never comes.
int64_t attn5_counter_bytes(int B, int kv) {
  (void)B;
  return 256 + ((int64_t)kAttn5MaxB * kv * 4 + 255) / 256 * 256;
}

int64_t attn5_workspace(const Pool* p, int B, int max_ctx, int G) {
  return attn5_counter_bytes(B, p->kv_heads) +
         (int64_t)B * p->kv_heads * attn5_kmax(max_ctx) * G * (p->head_dim + 2) * (int64_t)sizeof(float);
}

int attn5_launch(Pool* p, Attn5Args a, int G, int max_ctx, void* workspace, int64_t workspace_bytes, int sms,
                 cudaStream_t st) {
  const CUtensorMap* map = nullptr;
  int rc = pool_tmap(p, &map);
  if (rc != TF_OK) return rc;
  a.kmax = (int32_t)attn5_kmax(max_ctx);
  a.min_per = kAttn5MinPer;
  const int64_t cb = attn5_counter_bytes(a.B, p->kv_heads);
  const int64_t need = attn5_workspace(p, a.B, max_ctx, G);
  TF_CHECK_ARG(workspace && workspace_bytes >= need, "tf_paged_decode_attn: workspace too small (%lld < %lld)",
               (long long)workspace_bytes, (long long)need);
  a.ticket = (unsigned long long*)workspace;
  a.diag = (int*)((char*)workspace + 8);
  a.counters = (int32_t*)((char*)workspace + 256);
  a.ws_ml = (float*)((char*)workspace + cb);
  a.ws_acc = a.ws_ml + (int64_t)a.B * p->kv_heads * a.kmax * G * 2;
  a.n_layers = p->n_layers;
  a.kv_heads = p->kv_heads;
  a.pool = p->gpu;
  // ring configuration (TF_ATTN5_CFG): 1 (default) = 2 stages per warp x 4
  // warps x 3 CTAs per SM (12 warps, 24 blocks = 192 KiB in flight per SM);
  // 0 = 3 stages x 4 warps x 2 CTAs (8 warps, 16 blocks in flight): cfg 1 is
  // 3-5% faster at B = 64-128 (profiles/r2_attn_cfg.json)
  static const int cfg = getenv("TF_ATTN5_CFG") ? atoi(getenv("TF_ATTN5_CFG")) : 1;
#define TF_A5(G_, NH_) \
  return cfg == 1 ? launch5<G_, NH_, 2, 4, 3>(*map, a, sms, st) : launch5<G_, NH_, 3, 4, 2>(*map, a, sms, st)
  if (p->head_dim == 128) {
    switch (G) {
      case 1: TF_A5(1, 2);
      case 2: TF_A5(2, 2);
      case 4: TF_A5(4, 2);
      case 5: TF_A5(5, 2);
      case 8: TF_A5(8, 2);
    }
  } else {
    switch (G) {
      case 1: TF_A5(1, 1);
      case 2: TF_A5(2, 1);
      case 4: TF_A5(4, 1);
    }
  }
#undef TF_A5
  set_error("tf_paged_decode_attn: v5 has no instance for head_dim %d / group %d", p->head_dim, G);
  return TF_EINVAL;
}

}  // namespace tf
