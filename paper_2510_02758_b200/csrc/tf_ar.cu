// C4 tensor-parallel data path: one-shot all-reduce over peer memory, fused
// with the residual add and the RMSNorm that follow it in the decoder.
//
// the only real exchange step of the hot path is the sum of the
// TP ranks' partial projections after o_proj and after down_proj (each rank
// holds a row slice of wo / wd).  In the decoder the all-reduce is always
// followed by `x += sum` and `h = rmsnorm(x) * gamma` (the next sub-layer's
// input), so ONE kernel does all three:
//
//   x[r]  <- bf16( x[r] + sum_{p = 0..TP-1} part_p[r] )        (fp32, rank order)
//   h[r]  <- rmsnorm(x[r]) * gamma                              (tf_rmsnorm's arithmetic)
//
// where part_p is rank p's GEMM output, written by cuBLAS straight into p's
// registered buffer.  Every rank reads every peer's buffer through NVLink
// (P2P loads of IPC-mapped memory; on one device the "peers" are plain
// device pointers), sums in rank order - so all ranks hold bit-identical x -
// and writes only local memory.  No NCCL call, no staging copy, no separate
// residual / norm launches, and the kernel is graph-capturable (its barrier
// state is device-resident and advances by itself on every replay).
//
// Synchronisation: per CTA c, two flag barriers over the ranks.  Each rank
// keeps an epoch counter per CTA (device memory, local); a call increments
// it to e, stores e into every peer's sig[phase][my_rank][c] (release, system
// scope) and waits until its own sig[phase][p][c] reached e for every p
// (acquire).  Phase 0 (start): every rank's partial is complete.  Phase 1
// (end): every rank finished reading this CTA's rows of every buffer, so
// the next GEMM may overwrite them.  Waits are bounded (10 s of globaltimer):
// a missing peer sets the error flag (tf_ar_status) instead of hanging.
#include <stdint.h>

#include <cstring>
#include <memory>
#include <mutex>
#include <unordered_map>

#include "tf_common.cuh"

namespace tf {

constexpr int kArMaxRanks = 8;
constexpr int kArMaxCtas = 148;      // one per SM; grid = min(rows, this) - identical on every rank
constexpr int kArThreads = 256;
constexpr int kArMaxVec = 4;         // 16-B vectors per thread in registers: dim <= 256*4*8 = 8192
constexpr unsigned long long kArTimeoutNs = 10ull * 1000 * 1000 * 1000;

struct ArCtl {
  uint32_t sig[2][kArMaxRanks][kArMaxCtas];  // written by peers (and self)
  uint32_t epoch[kArMaxCtas];                // local per-CTA call counter
  int32_t err;                               // 1 = a barrier timed out
};

struct ArComm {
  int rank = 0, world = 1, device = 0;
  int max_ctas = kArMaxCtas;  // grid cap (identical on every rank)
  int64_t capacity = 0;  // bytes of the data buffer
  void* data = nullptr;  // this rank's registered buffer (cudaMalloc: IPC-exportable)
  ArCtl* ctl = nullptr;
  void* peer_data[kArMaxRanks] = {};
  ArCtl* peer_ctl[kArMaxRanks] = {};
  bool opened[kArMaxRanks] = {};  // peer mapping owned by us (cudaIpcOpenMemHandle)
};

struct ArArgs {
  const uint16_t* part[kArMaxRanks];
  ArCtl* ctl[kArMaxRanks];
  int32_t rank, world, rows, dim;
  uint16_t* x;            // residual in/out (may be NULL: h_out receives the plain sum)
  const uint16_t* gamma;  // NULL: no norm
  uint16_t* h_out;
  float eps;
};

static std::mutex g_ar_mu;
static std::unordered_map<int64_t, std::unique_ptr<ArComm>> g_ars;
static int64_t g_ar_next = 1;

static ArComm* get_ar(int64_t h) {
  std::lock_guard<std::mutex> lk(g_ar_mu);
  auto it = g_ars.find(h);
  return it == g_ars.end() ? nullptr : it->second.get();
}

__device__ __forceinline__ unsigned long long ar_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Flag barrier of CTA blockIdx.x over the ranks (threads 0..world-1 each
// handle one peer).  Returns after every rank reached the same phase of call e.
__device__ __forceinline__ void ar_barrier(const ArArgs& a, int phase, uint32_t e) {
  const int c = blockIdx.x;
  // every thread's earlier accesses (phase 1: its reads of the peers' buffers)
  // happen before the release below
  __syncthreads();
  if (threadIdx.x < (unsigned)a.world) {
    const int p = threadIdx.x;
    __threadfence_system();
    st_release_sys(&a.ctl[p]->sig[phase][a.rank][c], e);
    const uint32_t* mine = &a.ctl[a.rank]->sig[phase][p][c];
    const unsigned long long t0 = ar_now();
    while ((int32_t)(ld_acquire_sys(mine) - e) < 0) {
      if (ar_now() - t0 > kArTimeoutNs) {
        atomicExch(&a.ctl[a.rank]->err, 1);
        break;
      }
    }
  }
  __syncthreads();
}

__device__ __forceinline__ void unpack8f(const uint4& u, float* f) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
  }
}

__device__ __forceinline__ uint4 pack8f(const float* f) {
  uint32_t w[4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
    w[i] = (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(f[2 * i])) |
           ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(f[2 * i + 1])) << 16);
  return make_uint4(w[0], w[1], w[2], w[3]);
}

__global__ void __launch_bounds__(kArThreads) ar_residual_rmsnorm_kernel(const __grid_constant__ ArArgs a) {
  __shared__ uint32_t s_epoch;
  __shared__ float s_part[kArThreads / 32];
  if (threadIdx.x == 0) {
    uint32_t* ep = &a.ctl[a.rank]->epoch[blockIdx.x];
    s_epoch = *ep + 1;
    *ep = s_epoch;
  }
  __syncthreads();
  const uint32_t e = s_epoch;
  const int nv = a.dim / 8;
  // the norm weights (local, not written by peers): loaded once per CTA, while
  // the start barrier waits
  uint4 gw[kArMaxVec];
#pragma unroll
  for (int k = 0; k < kArMaxVec; ++k) {
    const int i = threadIdx.x + k * kArThreads;
    gw[k] = (a.gamma && i < nv) ? __ldg(reinterpret_cast<const uint4*>(a.gamma) + i) : make_uint4(0, 0, 0, 0);
  }
  ar_barrier(a, 0, e);

  for (int r = blockIdx.x; r < a.rows; r += gridDim.x) {
    const int64_t base = (int64_t)r * a.dim;
    float v[kArMaxVec][8];
    float ss = 0.f;
#pragma unroll
    for (int k = 0; k < kArMaxVec; ++k) {
      const int i = threadIdx.x + k * kArThreads;
      if (i < nv) {
#pragma unroll
        for (int j = 0; j < 8; ++j) v[k][j] = 0.f;
        // every rank sums the partials in the same (rank) order: identical x everywhere
        for (int p = 0; p < a.world; ++p) {
          float f[8];
          unpack8f(__ldcg(reinterpret_cast<const uint4*>(a.part[p] + base) + i), f);
#pragma unroll
          for (int j = 0; j < 8; ++j) v[k][j] += f[j];
        }
        if (a.x) {
          float f[8];
          unpack8f(reinterpret_cast<const uint4*>(a.x + base)[i], f);
#pragma unroll
          for (int j = 0; j < 8; ++j) v[k][j] += f[j];
        }
        // the new residual is a bf16 tensor: round once, normalise the rounded values
        const uint4 packed = pack8f(v[k]);
        unpack8f(packed, v[k]);
        if (a.x)
          reinterpret_cast<uint4*>(a.x + base)[i] = packed;
        else if (!a.gamma)
          reinterpret_cast<uint4*>(a.h_out + base)[i] = packed;
#pragma unroll
        for (int j = 0; j < 8; ++j) ss += v[k][j] * v[k][j];
      }
    }
    if (a.gamma) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = ss;
      __syncthreads();
      float tot = 0.f;
#pragma unroll
      for (int i = 0; i < kArThreads / 32; ++i) tot += s_part[i];
      const float rs = rsqrtf(tot / (float)a.dim + a.eps);
#pragma unroll
      for (int k = 0; k < kArMaxVec; ++k) {
        const int i = threadIdx.x + k * kArThreads;
        if (i < nv) {
          float g[8], o[8];
          unpack8f(gw[k], g);
#pragma unroll
          for (int j = 0; j < 8; ++j) o[j] = __bfloat162float(__float2bfloat16_rn(v[k][j] * rs)) * g[j];
          reinterpret_cast<uint4*>(a.h_out + base)[i] = pack8f(o);
        }
      }
      __syncthreads();  // s_part is reused by the next row
    }
  }
  ar_barrier(a, 1, e);
}

}  // namespace tf

using namespace tf;

extern "C" {

int tf_ar_create(int32_t rank, int32_t world, int64_t capacity_bytes, int32_t max_ctas, int64_t* out_handle) {
  TF_CHECK_ARG(out_handle, "tf_ar_create: out_handle is NULL");
  TF_CHECK_ARG(world >= 1 && world <= kArMaxRanks && rank >= 0 && rank < world, "tf_ar_create: rank %d of %d",
               rank, world);
  TF_CHECK_ARG(capacity_bytes > 0 && capacity_bytes % 16 == 0, "tf_ar_create: bad capacity %lld",
               (long long)capacity_bytes);
  TF_CHECK_ARG(max_ctas >= 0 && max_ctas <= kArMaxCtas, "tf_ar_create: max_ctas %d not in [0, %d]", max_ctas,
               kArMaxCtas);
  auto c = std::make_unique<ArComm>();
  c->max_ctas = max_ctas ? max_ctas : kArMaxCtas;
  c->rank = rank;
  c->world = world;
  c->capacity = capacity_bytes;
  TF_CUDA(cudaGetDevice(&c->device));
  TF_CUDA(cudaMalloc(&c->data, capacity_bytes));
  void* ctl = nullptr;
  cudaError_t e = cudaMalloc(&ctl, sizeof(ArCtl));
  if (e != cudaSuccess) {
    cudaFree(c->data);
    TF_CUDA(e);
  }
  c->ctl = (ArCtl*)ctl;
  TF_CUDA(cudaMemset(c->ctl, 0, sizeof(ArCtl)));
  TF_CUDA(cudaMemset(c->data, 0, capacity_bytes));
  TF_CUDA(cudaDeviceSynchronize());
  c->peer_data[rank] = c->data;
  c->peer_ctl[rank] = c->ctl;
  std::lock_guard<std::mutex> lk(g_ar_mu);
  *out_handle = g_ar_next++;
  g_ars[*out_handle] = std::move(c);
  return TF_OK;
}

void* tf_ar_buffer(int64_t h) {
  ArComm* c = get_ar(h);
  return c ? c->data : nullptr;
}

void* tf_ar_ctl(int64_t h) {
  ArComm* c = get_ar(h);
  return c ? (void*)c->ctl : nullptr;
}

int tf_ar_export(int64_t h, void* out128) {
  ArComm* c = get_ar(h);
  TF_CHECK_ARG(c && out128, "tf_ar_export: bad handle / NULL output");
  cudaIpcMemHandle_t a, b;
  TF_CUDA(cudaIpcGetMemHandle(&a, c->data));
  TF_CUDA(cudaIpcGetMemHandle(&b, c->ctl));
  memcpy(out128, &a, 64);
  memcpy((char*)out128 + 64, &b, 64);
  return TF_OK;
}

int tf_ar_open(int64_t h, const void* all) {
  ArComm* c = get_ar(h);
  TF_CHECK_ARG(c && all, "tf_ar_open: bad handle / NULL handles");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  for (int p = 0; p < c->world; ++p) {
    if (p == c->rank) continue;
    cudaIpcMemHandle_t a, b;
    memcpy(&a, (const char*)all + 128 * p, 64);
    memcpy(&b, (const char*)all + 128 * p + 64, 64);
    void *d = nullptr, *s = nullptr;
    TF_CUDA(cudaIpcOpenMemHandle(&d, a, cudaIpcMemLazyEnablePeerAccess));
    TF_CUDA(cudaIpcOpenMemHandle(&s, b, cudaIpcMemLazyEnablePeerAccess));
    c->peer_data[p] = d;
    c->peer_ctl[p] = (ArCtl*)s;
    c->opened[p] = true;
  }
  return TF_OK;
}

int tf_ar_set_peers(int64_t h, void* const* data, void* const* ctl) {
  ArComm* c = get_ar(h);
  TF_CHECK_ARG(c && data && ctl, "tf_ar_set_peers: bad handle / NULL arrays");
  for (int p = 0; p < c->world; ++p) {
    TF_CHECK_ARG(data[p] && ctl[p], "tf_ar_set_peers: NULL pointer of rank %d", p);
    c->peer_data[p] = data[p];
    c->peer_ctl[p] = (ArCtl*)ctl[p];
  }
  return TF_OK;
}

int tf_ar_residual_rmsnorm(int64_t h, void* x, const void* gamma, void* h_out, int32_t rows, int32_t dim, float eps,
                           void* stream) {
  ArComm* c = get_ar(h);
  TF_CHECK_ARG(c, "tf_ar_residual_rmsnorm: unknown communicator");
  TF_CHECK_ARG(rows >= 0 && dim > 0 && dim % 8 == 0 && dim <= kArThreads * kArMaxVec * 8,
               "tf_ar_residual_rmsnorm: bad shape %d x %d", rows, dim);
  TF_CHECK_ARG((int64_t)rows * dim * 2 <= c->capacity, "tf_ar_residual_rmsnorm: %d x %d exceeds the %lld-byte buffer",
               rows, dim, (long long)c->capacity);
  TF_CHECK_ARG(x || h_out, "tf_ar_residual_rmsnorm: no output");
  TF_CHECK_ARG(!gamma || h_out, "tf_ar_residual_rmsnorm: gamma without h_out");
  if (rows == 0) return TF_OK;
  ArArgs a;
  for (int p = 0; p < c->world; ++p) {
    TF_CHECK_ARG(c->peer_data[p] && c->peer_ctl[p], "tf_ar_residual_rmsnorm: rank %d not mapped", p);
    a.part[p] = (const uint16_t*)c->peer_data[p];
    a.ctl[p] = c->peer_ctl[p];
  }
  a.rank = c->rank;
  a.world = c->world;
  a.rows = rows;
  a.dim = dim;
  a.x = (uint16_t*)x;
  a.gamma = (const uint16_t*)gamma;
  a.h_out = (uint16_t*)h_out;
  a.eps = eps;
  const int grid = rows < c->max_ctas ? rows : c->max_ctas;
  ar_residual_rmsnorm_kernel<<<grid, kArThreads, 0, (cudaStream_t)stream>>>(a);
  TF_LAUNCH_CHECK();
  return TF_OK;
}

int tf_ar_status(int64_t h) {
  ArComm* c = get_ar(h);
  TF_CHECK_ARG(c, "tf_ar_status: unknown communicator");
  int32_t err = 0;
  TF_CUDA(cudaMemcpy(&err, &c->ctl->err, sizeof(err), cudaMemcpyDeviceToHost));
  return err;
}

int tf_ar_destroy(int64_t h) {
  std::unique_ptr<ArComm> c;
  {
    std::lock_guard<std::mutex> lk(g_ar_mu);
    auto it = g_ars.find(h);
    TF_CHECK_ARG(it != g_ars.end(), "tf_ar_destroy: unknown communicator");
    c = std::move(it->second);
    g_ars.erase(it);
  }
  for (int p = 0; p < c->world; ++p) {
    if (!c->opened[p]) continue;
    cudaIpcCloseMemHandle(c->peer_data[p]);
    cudaIpcCloseMemHandle(c->peer_ctl[p]);
  }
  cudaFree(c->data);
  cudaFree(c->ctl);
  return TF_OK;
}

}  // extern "C"
