// Swap engine: token-granular paged KV movement between the HBM pool and the
// pinned host store.
//
// Replaces the reference's simulated PCIe channels (tokensim/engine.py:235-247,
// :736-779) and transfer_time (tokensim/costs.py:69-75): a write-through /
// evict chunk becomes one gather (HBM -> host), a load chunk one scatter
// (host -> HBM).  Two engines:
//   TF_ENGINE_SM  - SM-driven zero-copy kernel: 16-byte vectorised, fully
//                   coalesced reads of the block-major pool, posted writes
//                   straight into mapped pinned memory (d2h) or deep batches
//                   of outstanding sysmem loads (h2d).  Grid capped to a few
//                   dozen CTAs: PCIe, not the SMs, is the bound, and the
//                   decode step keeps the rest of the machine.
//   TF_ENGINE_CE / CE2D / AUTO - copy engines only: whole blocks (all
//                   layers) are coalesced into maximal contiguous runs (a
//                   whole block is a single 2 MiB run in this layout, LIFO-
//                   adjacent blocks merge into longer ones), one cudaMemcpyAsync
//                   per run; every partial block is ONE 2-D copy (its runs are
//                   equally spaced).  No SM is used.
#include <algorithm>

#include "tf_common.cuh"

namespace tf {

constexpr int kMaxSegs = 1536;
constexpr int kSwapThreads = 256;
constexpr int kUnroll = 8;

// Segment capacity is a template parameter so a small chunk (write-through
// tails: 1-3 segments) launches with a few hundred bytes of parameters
// instead of 18 KB.
template <int CAP>
struct SwapArgs {
  PoolView pv;
  int32_t layer_begin, layer_end, n_segs, to_host;
  int32_t gpu_block[CAP];
  int32_t host_block[CAP];
  int16_t slot_begin[CAP];
  int16_t n_slots[CAP];
};

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ uint4 ld_sysmem(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.cv.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

__device__ __forceinline__ void st_stream(uint4* p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// blockIdx.y = segment; the segment's vectors (16 B) are enumerated as
// run-major (layer, kv, head) x (slot, dim/8) and strided over blockIdx.x.
template <int CAP>
__global__ void __launch_bounds__(kSwapThreads) swap_kernel(const __grid_constant__ SwapArgs<CAP> a) {
  const int s = blockIdx.y;
  const PoolView& pv = a.pv;
  const int ns = a.n_slots[s];
  const int vpr = ns * pv.head_dim / 8;            // vectors per run
  const int runs = (a.layer_end - a.layer_begin) * 2 * pv.kv_heads;
  const int64_t total = (int64_t)runs * vpr;
  const int64_t gb = a.gpu_block[s], hb = a.host_block[s];
  const int sb = a.slot_begin[s];
  const int64_t stride = (int64_t)gridDim.x * kSwapThreads;
  for (int64_t v0 = (int64_t)blockIdx.x * kSwapThreads + threadIdx.x; v0 < total; v0 += stride * kUnroll) {
    uint4 buf[kUnroll];
    int64_t dst_off[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      int64_t v = v0 + (int64_t)u * stride;
      dst_off[u] = -1;
      if (v < total) {
        int rho = (int)(v / vpr), i = (int)(v - (int64_t)rho * vpr);
        int l = a.layer_begin + rho / (2 * pv.kv_heads);
        int kv = (rho / pv.kv_heads) & 1, h = rho % pv.kv_heads;
        int64_t g = pv.off(gb, l, kv, h, sb) + (int64_t)i * 8;
        int64_t c = pv.off(hb, l, kv, h, sb) + (int64_t)i * 8;
        if (a.to_host) {
          buf[u] = ld_stream(reinterpret_cast<const uint4*>(pv.gpu + g));
          dst_off[u] = c;
        } else {
          buf[u] = ld_sysmem(reinterpret_cast<const uint4*>(pv.host + c));
          dst_off[u] = g;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      if (dst_off[u] >= 0) {
        uint16_t* base = a.to_host ? pv.host : pv.gpu;
        st_stream(reinterpret_cast<uint4*>(base + dst_off[u]), buf[u]);
      }
    }
  }
}

template <int CAP>
static int swap_sm_launch(const Pool& p, const tf_seg* segs, int32_t n, int32_t l0, int32_t l1, int to_host,
                          cudaStream_t st) {
  SwapArgs<CAP> a;
  a.pv = view_of(p);
  a.layer_begin = l0;
  a.layer_end = l1;
  a.to_host = to_host;
  a.n_segs = n;
  int64_t max_vec = 0;
  for (int i = 0; i < n; ++i) {
    const tf_seg& s = segs[i];
    a.gpu_block[i] = s.gpu_block;
    a.host_block[i] = s.host_block;
    a.slot_begin[i] = (int16_t)s.slot_begin;
    a.n_slots[i] = (int16_t)s.n_slots;
    max_vec = std::max(max_vec, (int64_t)(l1 - l0) * 2 * p.kv_heads * s.n_slots * p.head_dim / 8);
  }
  // PCIe-bound: ~128 CTAs of 256 threads x 8 x 16 B keep > 4 MB in flight.
  int64_t want = (max_vec + (int64_t)kSwapThreads * kUnroll - 1) / ((int64_t)kSwapThreads * kUnroll);
  int64_t cap = std::max<int64_t>(1, 128 / std::max<int32_t>(1, n));
  dim3 grid((unsigned)std::max<int64_t>(1, std::min(want, cap)), (unsigned)n);
  swap_kernel<CAP><<<grid, kSwapThreads, 0, st>>>(a);
  TF_LAUNCH_CHECK();
  return TF_OK;
}

static int swap_sm(const Pool& p, const tf_seg* segs, int32_t n, int32_t l0, int32_t l1, int to_host,
                   cudaStream_t st) {
  for (int32_t base = 0; base < n; base += kMaxSegs) {
    const int32_t m = std::min<int32_t>(kMaxSegs, n - base);
    int rc = m <= 8 ? swap_sm_launch<8>(p, segs + base, m, l0, l1, to_host, st)
             : m <= 64 ? swap_sm_launch<64>(p, segs + base, m, l0, l1, to_host, st)
                       : swap_sm_launch<kMaxSegs>(p, segs + base, m, l0, l1, to_host, st);
    if (rc != TF_OK) return rc;
  }
  return TF_OK;
}

// Copy-engine path.  Whole blocks (all layers) become maximal contiguous 1-D
// runs (a block is one 2 MiB run; LIFO-adjacent blocks merge).  A PARTIAL
// block is ONE 2-D copy: the n slots of one (block, layer, K|V, head) tile sit
// at the same offset in every tile, and the tiles of a block are consecutive
// (block_tokens * head_dim elements apart), so a partial block over layers
// [l0, l1) is width n_slots * head_dim * 2 B x height (l1 - l0) * 2 * kv_heads
// rows at a pitch of one tile - instead of that many separate runs or an SM
// kernel.  No SM is used.
//
// Copies alternate between the caller's stream and the pool's auxiliary copy
// stream of this direction (fork / join through events, so the chunk still
// completes on the caller's stream): every copy carries a fixed setup cost
// (~4 us per 2 MiB block on one queue: 51 vs 57 GB/s) that the other queue's
// transfer then covers.
struct CopyOp {
  void* dst;
  const void* src;
  size_t width, height, pitch;  // height 1 = a 1-D run of `width` bytes
};

static int swap_ce(const Pool& p, const tf_seg* segs, int32_t n, int32_t l0, int32_t l1, int to_host,
                   cudaStream_t st) {
  std::vector<CopyOp> ops;
  const bool all_layers = (l0 == 0 && l1 == p.n_layers);
  auto push_run = [&](int64_t goff, int64_t hoff, int64_t elems) {
    uint16_t* g = p.gpu + goff;
    uint16_t* h = p.host + hoff;
    const size_t bytes = (size_t)elems * 2;
    void* d = to_host ? (void*)h : (void*)g;
    const void* sp = to_host ? (const void*)g : (const void*)h;
    // merge with the previous 1-D run when both sides continue contiguously
    if (!ops.empty() && ops.back().height == 1 && (char*)ops.back().dst + ops.back().width == (char*)d &&
        (const char*)ops.back().src + ops.back().width == (const char*)sp) {
      ops.back().width += bytes;
      return;
    }
    ops.push_back({d, sp, bytes, 1, bytes});
  };
  const size_t pitch = (size_t)p.tile_elems * 2;
  const size_t rows = (size_t)(l1 - l0) * 2 * p.kv_heads;
  for (int32_t i = 0; i < n; ++i) {
    const tf_seg& s = segs[i];
    if (all_layers && s.n_slots == p.block_tokens && s.slot_begin == 0) {
      push_run(p.off(s.gpu_block, 0, 0, 0, 0), p.off(s.host_block, 0, 0, 0, 0), p.block_elems);
    } else if (s.n_slots == p.block_tokens && s.slot_begin == 0) {
      // whole block over a layer range: its tiles for [l0, l1) are contiguous
      push_run(p.off(s.gpu_block, l0, 0, 0, 0), p.off(s.host_block, l0, 0, 0, 0), (int64_t)rows * p.tile_elems);
    } else {
      uint16_t* g = p.gpu + p.off(s.gpu_block, l0, 0, 0, s.slot_begin);
      uint16_t* h = p.host + p.off(s.host_block, l0, 0, 0, s.slot_begin);
      ops.push_back({to_host ? (void*)h : (void*)g, to_host ? (const void*)g : (const void*)h,
                     (size_t)s.n_slots * p.head_dim * 2, rows, pitch});
    }
  }
  if (ops.empty()) return TF_OK;
  const cudaMemcpyKind kind = to_host ? cudaMemcpyDeviceToHost : cudaMemcpyHostToDevice;
  Pool& pm = const_cast<Pool&>(p);
  const int dir = to_host ? 0 : 1;
  cudaStream_t st2 = nullptr;
  if (ops.size() >= 2) {
    if (!pm.aux[dir]) {
      int lo = 0, hi = 0;
      TF_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      TF_CUDA(cudaStreamCreateWithPriority(&pm.aux[dir], cudaStreamNonBlocking, hi));
      TF_CUDA(cudaEventCreateWithFlags(&pm.fork_ev[dir], cudaEventDisableTiming));
      TF_CUDA(cudaEventCreateWithFlags(&pm.join_ev[dir], cudaEventDisableTiming));
    }
    st2 = pm.aux[dir];
    TF_CUDA(cudaEventRecord(pm.fork_ev[dir], st));
    TF_CUDA(cudaStreamWaitEvent(st2, pm.fork_ev[dir], 0));
  }
  for (size_t i = 0; i < ops.size(); ++i) {
    const CopyOp& o = ops[i];
    cudaStream_t q = (st2 && (i & 1)) ? st2 : st;
    if (o.height == 1)
      TF_CUDA(cudaMemcpyAsync(o.dst, o.src, o.width, kind, q));
    else
      TF_CUDA(cudaMemcpy2DAsync(o.dst, o.pitch, o.src, o.pitch, o.width, o.height, kind, q));
  }
  if (st2) {
    TF_CUDA(cudaEventRecord(pm.join_ev[dir], st2));
    TF_CUDA(cudaStreamWaitEvent(st, pm.join_ev[dir], 0));
  }
  return TF_OK;
}

static int swap_entry(int64_t pool, const tf_seg* segs, int32_t n, int32_t l0, int32_t l1, int32_t engine,
                      int to_host, void* stream) {
  Pool* p = get_pool(pool);
  TF_CHECK_ARG(p, "swap: unknown pool");
  TF_CHECK_ARG(p->host && p->gpu, "swap: pool has no host tier");
  TF_CHECK_ARG(n >= 0 && (n == 0 || segs), "swap: bad segment list");
  TF_CHECK_ARG(0 <= l0 && l0 < l1 && l1 <= p->n_layers, "swap: bad layer range [%d,%d)", l0, l1);
  for (int32_t i = 0; i < n; ++i) {
    const tf_seg& s = segs[i];
    TF_CHECK_ARG(s.gpu_block >= 0 && s.gpu_block < p->n_blocks, "swap: gpu block %d out of range", s.gpu_block);
    TF_CHECK_ARG(s.host_block >= 0 && s.host_block < p->n_host_blocks, "swap: host block %d out of range",
                 s.host_block);
    TF_CHECK_ARG(s.slot_begin >= 0 && s.n_slots > 0 && s.slot_begin + s.n_slots <= p->block_tokens,
                 "swap: bad slot range [%d,+%d)", s.slot_begin, s.n_slots);
  }
  if (n == 0) return TF_OK;
  cudaStream_t st = (cudaStream_t)stream;
  // every copy-engine mode is the same path now (TF_ENGINE_CE used to move a
  // partial block as 2 x kv_heads x layers separate 1-D runs): the copy
  // engines beat the SM kernel at every chunk size
  // (profiles/r2_wt_chunks_ce2d.json) and leave the SMs to the decode step
  if (engine == TF_ENGINE_CE || engine == TF_ENGINE_CE2D || engine == TF_ENGINE_AUTO)
    return swap_ce(*p, segs, n, l0, l1, to_host, st);
  TF_CHECK_ARG(engine == TF_ENGINE_SM, "swap: unknown engine %d", engine);
  return swap_sm(*p, segs, n, l0, l1, to_host, st);
}

}  // namespace tf

extern "C" {

int tf_kv_gather_d2h(int64_t pool, const tf_seg* segs, int32_t n_segs, int32_t layer_begin, int32_t layer_end,
                     int32_t engine, void* stream) {
  return tf::swap_entry(pool, segs, n_segs, layer_begin, layer_end, engine, 1, stream);
}

int tf_kv_scatter_h2d(int64_t pool, const tf_seg* segs, int32_t n_segs, int32_t layer_begin, int32_t layer_end,
                      int32_t engine, void* stream) {
  return tf::swap_entry(pool, segs, n_segs, layer_begin, layer_end, engine, 0, stream);
}

}  // extern "C"
