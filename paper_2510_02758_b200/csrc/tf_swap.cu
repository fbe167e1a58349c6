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

// Copy-engine path: maximal contiguous runs, one submission per run.
static int swap_ce(const Pool& p, const tf_seg* segs, int32_t n, int32_t l0, int32_t l1, int to_host,
                   cudaStream_t st) {
  std::vector<void*> dst, src;
  std::vector<size_t> sz;
  const bool all_layers = (l0 == 0 && l1 == p.n_layers);
  auto push = [&](int64_t goff, int64_t hoff, int64_t elems) {
    uint16_t* g = p.gpu + goff;
    uint16_t* h = p.host + hoff;
    size_t bytes = (size_t)elems * 2;
    // merge with the previous run when both sides continue contiguously
    if (!sz.empty()) {
      char* pd = (char*)dst.back() + sz.back();
      char* ps = (char*)src.back() + sz.back();
      if (pd == (char*)(to_host ? (void*)h : (void*)g) && ps == (char*)(to_host ? (void*)g : (void*)h)) {
        sz.back() += bytes;
        return;
      }
    }
    dst.push_back(to_host ? (void*)h : (void*)g);
    src.push_back(to_host ? (void*)g : (void*)h);
    sz.push_back(bytes);
  };
  for (int32_t i = 0; i < n; ++i) {
    const tf_seg& s = segs[i];
    if (all_layers && s.n_slots == p.block_tokens && s.slot_begin == 0) {
      push(p.off(s.gpu_block, 0, 0, 0, 0), p.off(s.host_block, 0, 0, 0, 0), p.block_elems);
      continue;
    }
    for (int l = l0; l < l1; ++l)
      for (int kv = 0; kv < 2; ++kv)
        for (int h = 0; h < p.kv_heads; ++h)
          push(p.off(s.gpu_block, l, kv, h, s.slot_begin), p.off(s.host_block, l, kv, h, s.slot_begin),
               (int64_t)s.n_slots * p.head_dim);
  }
  // One plain async copy per maximal run: few, large submissions (a chunk of
  // whole blocks is typically a handful of multi-MiB runs).
  for (size_t i = 0; i < sz.size(); ++i)
    TF_CUDA(cudaMemcpyAsync(dst[i], src[i], sz[i], to_host ? cudaMemcpyDeviceToHost : cudaMemcpyHostToDevice, st));
  return TF_OK;
}

// Copy-engine path for PARTIAL blocks: the n slots of one (block, layer, K|V,
// head) run sit at the same offset in every run, and the runs of a block are
// consecutive tiles of block_tokens * head_dim elements - so a partial block
// over layers [l0, l1) is ONE 2-D copy (width n_slots * head_dim * 2 bytes,
// height (l1 - l0) * 2 * kv_heads rows, pitch one tile) for the DMA engine,
// instead of 2 * kv_heads * layers separate runs or an SM kernel.
static int swap_ce2d(const Pool& p, const tf_seg* segs, int32_t n, int32_t l0, int32_t l1, int to_host,
                     cudaStream_t st) {
  const size_t pitch = (size_t)p.tile_elems * 2;
  const size_t rows = (size_t)(l1 - l0) * 2 * p.kv_heads;
  for (int32_t i = 0; i < n; ++i) {
    const tf_seg& s = segs[i];
    uint16_t* g = p.gpu + p.off(s.gpu_block, l0, 0, 0, s.slot_begin);
    uint16_t* h = p.host + p.off(s.host_block, l0, 0, 0, s.slot_begin);
    const size_t width = (size_t)s.n_slots * p.head_dim * 2;
    if (to_host)
      TF_CUDA(cudaMemcpy2DAsync(h, pitch, g, pitch, width, rows, cudaMemcpyDeviceToHost, st));
    else
      TF_CUDA(cudaMemcpy2DAsync(g, pitch, h, pitch, width, rows, cudaMemcpyHostToDevice, st));
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
  if (engine == TF_ENGINE_CE || engine == TF_ENGINE_CE2D || engine == TF_ENGINE_AUTO) {
    // (TF_ENGINE_CE used to move a partial block as 2 x kv_heads x layers
    // separate 1-D runs; one submission each made it ~100x slower than this)
    // whole blocks (all layers): merged 1-D runs; every other
    // segment: one 2-D copy each.  No SM is used at all (the copy engines
    // beat the SM kernel at every chunk size, profiles/r2_wt_chunks_ce2d.json,
    // and leave the SMs to the decode step).
    std::vector<tf_seg> full, part;
    const bool all_layers = (l0 == 0 && l1 == p->n_layers);
    for (int32_t i = 0; i < n; ++i)
      (all_layers && segs[i].n_slots == p->block_tokens ? full : part).push_back(segs[i]);
    if (!full.empty()) {
      int rc = swap_ce(*p, full.data(), (int32_t)full.size(), l0, l1, to_host, st);
      if (rc != TF_OK) return rc;
    }
    return part.empty() ? TF_OK : swap_ce2d(*p, part.data(), (int32_t)part.size(), l0, l1, to_host, st);
  }
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
