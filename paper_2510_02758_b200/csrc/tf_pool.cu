// KV pool descriptor, deterministic block allocator and device block tables.
//
// Replaces the reference's token-denominated ledger (tokensim/engine.py:325-365)
// with real blocks: the ledger stays token-exact on the host (decisions
// depend on it) while this allocator hands out physical blocks in a fixed
// LIFO order so block tables are reproducible bit for bit (oracle/dataplane.py).
#include <stdarg.h>

#include <memory>
#include <mutex>
#include <unordered_map>

#include <atomic>

#include "tf_common.cuh"

namespace tf {

static thread_local char g_err[1024] = "";

static std::atomic<long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

static std::mutex g_mu;
static std::unordered_map<int64_t, std::unique_ptr<Pool>> g_pools;
static int64_t g_next = 1;

Pool* get_pool(int64_t handle) {
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_pools.find(handle);
  return it == g_pools.end() ? nullptr : it->second.get();
}

// (row, lb, block) triples applied by one thread each.
// Launch parameters sized to the delta: a typical decode step changes a few
// table entries, and a 24 KB parameter block would dominate the launch cost.
template <int CAP>
struct TableOps {
  int32_t n;
  int32_t v[3 * CAP];
};

template <int CAP>
__global__ void table_apply_kernel(int32_t* table, int32_t stride, const __grid_constant__ TableOps<CAP> ops) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < ops.n) {
    int32_t row = ops.v[3 * i], lb = ops.v[3 * i + 1], blk = ops.v[3 * i + 2];
    table[(int64_t)row * stride + lb] = blk;
  }
}

__global__ void noop_kernel() {}

}  // namespace tf

using namespace tf;

extern "C" {

const char* tf_last_error(void) { return g_err; }

int64_t tf_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }
int tf_abi_version(void) { return 1; }

double tf_host_glibc_exp(double x);

int tf_pool_init(void* gpu_pool, int32_t n_blocks, void* host_pool, int32_t n_host_blocks, int32_t n_layers,
                 int32_t block_tokens, int32_t kv_heads, int32_t head_dim, int32_t dtype, int64_t* out_handle) {
  TF_CHECK_ARG(out_handle != nullptr, "tf_pool_init: out_handle is NULL");
  TF_CHECK_ARG(dtype == TF_DTYPE_BF16, "tf_pool_init: only bf16 KV is supported (dtype=%d)", dtype);
  TF_CHECK_ARG(n_blocks >= 0 && n_host_blocks >= 0, "tf_pool_init: negative block count");
  TF_CHECK_ARG(n_layers > 0 && block_tokens > 0 && kv_heads > 0, "tf_pool_init: bad shape");
  TF_CHECK_ARG(head_dim % 8 == 0 && head_dim <= 256, "tf_pool_init: head_dim must be a multiple of 8, <= 256");
  TF_CHECK_ARG(n_blocks == 0 || gpu_pool != nullptr, "tf_pool_init: gpu_pool is NULL");
  TF_CHECK_ARG(n_host_blocks == 0 || host_pool != nullptr, "tf_pool_init: host_pool is NULL");
  auto p = std::make_unique<Pool>();
  p->gpu = (uint16_t*)gpu_pool;
  p->host = (uint16_t*)host_pool;
  p->host_dev = nullptr;
  if (host_pool) {
    void* dptr = nullptr;
    cudaError_t e = cudaHostGetDevicePointer(&dptr, host_pool, 0);
    if (e != cudaSuccess) {
      cudaGetLastError();
      set_error("tf_pool_init: host_pool is not pinned/mapped host memory (%s)", cudaGetErrorString(e));
      return TF_EINVAL;
    }
    p->host_dev = (uint16_t*)dptr;
  }
  p->n_blocks = n_blocks;
  p->n_host_blocks = n_host_blocks;
  p->n_layers = n_layers;
  p->block_tokens = block_tokens;
  p->kv_heads = kv_heads;
  p->head_dim = head_dim;
  p->tile_elems = (int64_t)block_tokens * head_dim;
  p->block_elems = (int64_t)n_layers * 2 * kv_heads * p->tile_elems;
  p->free_gpu.resize(n_blocks);
  for (int32_t i = 0; i < n_blocks; ++i) p->free_gpu[i] = n_blocks - 1 - i;
  p->free_host.resize(n_host_blocks);
  for (int32_t i = 0; i < n_host_blocks; ++i) p->free_host[i] = n_host_blocks - 1 - i;
  p->used_gpu.assign(n_blocks, 0);
  p->used_host.assign(n_host_blocks, 0);
  std::lock_guard<std::mutex> lk(g_mu);
  int64_t h = g_next++;
  g_pools[h] = std::move(p);
  *out_handle = h;
  return TF_OK;
}

int tf_pool_destroy(int64_t pool) {
  std::lock_guard<std::mutex> lk(g_mu);
  TF_CHECK_ARG(g_pools.erase(pool) == 1, "tf_pool_destroy: unknown pool %lld", (long long)pool);
  return TF_OK;
}

int64_t tf_pool_block_bytes(int64_t pool) {
  Pool* p = get_pool(pool);
  return p ? p->block_elems * 2 : -1;
}

int tf_blocks_alloc(int64_t pool, int32_t tier, int32_t n, int32_t* out_ids) {
  Pool* p = get_pool(pool);
  TF_CHECK_ARG(p, "tf_blocks_alloc: unknown pool");
  TF_CHECK_ARG(tier == TF_TIER_GPU || tier == TF_TIER_HOST, "tf_blocks_alloc: bad tier %d", tier);
  TF_CHECK_ARG(n >= 0 && (n == 0 || out_ids), "tf_blocks_alloc: bad n/out");
  auto& st = tier == TF_TIER_GPU ? p->free_gpu : p->free_host;
  auto& used = tier == TF_TIER_GPU ? p->used_gpu : p->used_host;
  if ((int64_t)st.size() < n) {
    set_error("tf_blocks_alloc: %s tier exhausted (%d requested, %zu free)", tier ? "host" : "gpu", n, st.size());
    return TF_ENOMEM;
  }
  for (int32_t i = 0; i < n; ++i) {
    out_ids[i] = st.back();
    used[st.back()] = 1;
    st.pop_back();
  }
  return TF_OK;
}

int tf_blocks_free(int64_t pool, int32_t tier, const int32_t* ids, int32_t n) {
  Pool* p = get_pool(pool);
  TF_CHECK_ARG(p, "tf_blocks_free: unknown pool");
  TF_CHECK_ARG(tier == TF_TIER_GPU || tier == TF_TIER_HOST, "tf_blocks_free: bad tier %d", tier);
  TF_CHECK_ARG(n >= 0 && (n == 0 || ids), "tf_blocks_free: bad n/ids");
  auto& st = tier == TF_TIER_GPU ? p->free_gpu : p->free_host;
  auto& used = tier == TF_TIER_GPU ? p->used_gpu : p->used_host;
  int32_t cap = tier == TF_TIER_GPU ? p->n_blocks : p->n_host_blocks;
  // validate the whole list before touching the stack: a rejected call leaves
  // the allocator unchanged (no partial push); state 2 marks "listed in this
  // call" so a duplicate id inside the list is caught as well
  for (int32_t i = 0; i < n; ++i) {
    const bool in_range = ids[i] >= 0 && ids[i] < cap;
    if (!in_range || used[ids[i]] != 1) {
      for (int32_t k = 0; k < i; ++k) used[ids[k]] = 1;
      if (!in_range)
        set_error("tf_blocks_free: block %d out of range", ids[i]);
      else
        set_error("tf_blocks_free: double free of block %d", ids[i]);
      return TF_EINVAL;
    }
    used[ids[i]] = 2;
  }
  for (int32_t i = 0; i < n; ++i) {
    used[ids[i]] = 0;
    st.push_back(ids[i]);
  }
  return TF_OK;
}

int tf_launch_floor(void* stream) {
  noop_kernel<<<1, 32, 0, (cudaStream_t)stream>>>();
  TF_LAUNCH_CHECK();
  return TF_OK;
}

int tf_blocks_free_count(int64_t pool, int32_t tier) {
  Pool* p = get_pool(pool);
  TF_CHECK_ARG(p, "tf_blocks_free_count: unknown pool");
  return (int)(tier == TF_TIER_GPU ? p->free_gpu.size() : p->free_host.size());
}

int tf_table_apply(int32_t* dev_table, int32_t row_stride, const int32_t* triples, int32_t n_triples, void* stream) {
  TF_CHECK_ARG(dev_table && row_stride > 0, "tf_table_apply: bad table");
  TF_CHECK_ARG(n_triples >= 0 && (n_triples == 0 || triples), "tf_table_apply: bad triples");
  for (int32_t base = 0; base < n_triples; base += 2048) {
    const int32_t n = n_triples - base < 2048 ? n_triples - base : 2048;
    if (n <= 64) {
      TableOps<64> ops;
      ops.n = n;
      memcpy(ops.v, triples + 3 * base, sizeof(int32_t) * 3 * n);
      table_apply_kernel<64><<<1, 128, 0, (cudaStream_t)stream>>>(dev_table, row_stride, ops);
    } else {
      TableOps<2048> ops;
      ops.n = n;
      memcpy(ops.v, triples + 3 * base, sizeof(int32_t) * 3 * n);
      table_apply_kernel<2048><<<(n + 127) / 128, 128, 0, (cudaStream_t)stream>>>(dev_table, row_stride, ops);
    }
    TF_LAUNCH_CHECK();
  }
  return TF_OK;
}

}  // extern "C"
