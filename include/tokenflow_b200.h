/*
 * tokenflow_b200.h - C ABI of the B200-native TokenFlow KV-movement hot path.
 *
 * One shared library (paper_2510_02758_b200/_tf_b200.so, sm_100a) exporting
 * plain-C entry points: raw pointers, sizes, cudaStream_t passed as void*.
 * No torch types cross this boundary; the Python host (ctypes) and any other
 * FFI bind it directly (INTEGRATION.md shows the bindings).
 *
 * Reference interfaces replaced (paths relative to /root/reference/pkg/src):
 *   tf_pool_* / tf_blocks_* / tf_table_apply
 *       token-denominated ledger + KvResidency      tokensim/engine.py:325-365,
 *                                                    tokensim/kvstore.py:35-59
 *   tf_kv_gather_d2h   writethrough + evict chunks  tokensim/engine.py:781-813, :843-848
 *                      transfer_time (d2h)          tokensim/costs.py:69-75
 *   tf_kv_scatter_h2d  load chunks                  tokensim/engine.py:880-888, :607-615
 *   tf_kv_append / tf_kv_fill_synthetic
 *                      KV growth of prefill/decode  tokensim/engine.py:484-540
 *   tf_paged_decode_attn
 *                      decode_iteration_time        tokensim/costs.py:45-59
 *                      (as dispatched by _dispatch_gpu, engine.py:669-708)
 *   tf_policy_tick     BufferAwarePolicy.on_tick    tokensim/scheduler.py:513-772
 *   tf_policy_fastpath BufferAwarePolicy.opportunistic  scheduler.py:774-809
 *   tf_iteration_batch BufferAwarePolicy.iteration_batch scheduler.py:811-823
 *   tf_select_batch    select_batch                 tokensim/scheduler.py:205-269
 *
 * Status codes: 0 ok, TF_EINVAL bad arguments, TF_ENOMEM no free block,
 * TF_EIO CUDA error.  tf_last_error() returns the text of the last failure
 * on the calling thread.  The Python shim maps them to the reference's
 * exceptions (ValueError, MemoryError, InvariantError).
 *
 * Threading: every launch is asynchronous on the given stream unless noted;
 * entry points are not re-entrant per pool handle.
 */
#ifndef TOKENFLOW_B200_H
#define TOKENFLOW_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TF_OK 0
#define TF_EINVAL (-22)
#define TF_ENOMEM (-12)
#define TF_EIO (-5)

#define TF_DTYPE_BF16 0
#define TF_TIER_GPU 0
#define TF_TIER_HOST 1
#define TF_ENGINE_SM 0 /* SM-driven zero-copy gather/scatter kernel */
#define TF_ENGINE_CE 1 /* copy engines (= TF_ENGINE_CE2D since ABI v1.1) */
#define TF_ENGINE_AUTO 2 /* = TF_ENGINE_CE2D (kept for callers of ABI v1) */
#define TF_ENGINE_CE2D 3 /* copy engines only: whole blocks as merged 1-D runs, each partial block one 2-D copy */

const char* tf_last_error(void);
int tf_abi_version(void);
/* Kernel launches issued through this library so far (captured launches
 * count once, at capture - a graph replay re-runs them without calling in). */
int64_t tf_launch_count(void);
/* Launch one empty kernel on the stream: the launch-latency floor that the
 * selector's per-tick latency is reported against. */
int tf_launch_floor(void* stream);

/* ------------------------------------------------------------------ pool --
 * Block-major KV layout shared by HBM pool and pinned host store:
 *   block[b] = [layer][kv(K=0,V=1)][kv_head][slot][head_dim]  (bf16)
 * so one block (all layers) is one contiguous run of
 *   n_layers*2*kv_heads*block_tokens*head_dim*2 bytes (2 MiB for Llama3-8B)
 * and one (block, layer, kv, head) tile is block_tokens*head_dim*2 bytes. */
int tf_pool_init(void* gpu_pool, int32_t n_blocks, void* host_pool, int32_t n_host_blocks,
                 int32_t n_layers, int32_t block_tokens, int32_t kv_heads, int32_t head_dim,
                 int32_t dtype, int64_t* out_handle);
int tf_pool_destroy(int64_t pool);
int64_t tf_pool_block_bytes(int64_t pool);

/* Deterministic LIFO block allocator per tier (initial stack [N-1..0]:
 * block 0 is handed out first).  Host-side bookkeeping, no launch. */
int tf_blocks_alloc(int64_t pool, int32_t tier, int32_t n, int32_t* out_ids);
int tf_blocks_free(int64_t pool, int32_t tier, const int32_t* ids, int32_t n);
int tf_blocks_free_count(int64_t pool, int32_t tier);

/* Device-resident block tables: table[row*row_stride + lb] = physical block.
 * Applies (row, lb, block|-1) triples (host array) in one launch per 2048. */
int tf_table_apply(int32_t* dev_table, int32_t row_stride, const int32_t* triples, int32_t n_triples,
                   void* stream);

/* ------------------------------------------------------------ swap engine --
 * One segment = n_slots consecutive token slots [slot_begin, slot_begin+n)
 * of one GPU block <-> the same slots of one host block, for layers
 * [layer_begin, layer_end).  Segments are passed by value in the launch
 * (no H2D staging); a whole step's chunks go in one call. */
typedef struct {
  int32_t gpu_block;
  int32_t host_block;
  int32_t slot_begin;
  int32_t n_slots;
} tf_seg;

int tf_kv_gather_d2h(int64_t pool, const tf_seg* segs, int32_t n_segs, int32_t layer_begin, int32_t layer_end,
                     int32_t engine, void* stream);
int tf_kv_scatter_h2d(int64_t pool, const tf_seg* segs, int32_t n_segs, int32_t layer_begin, int32_t layer_end,
                      int32_t engine, void* stream);

/* Zero-copy small copy through one CTA (either side may be pinned host memory,
 * which is device-addressable under UVA): the per-step token ids / positions
 * in and sampled ids out, so a decode step never waits behind bulk KV
 * transfers queued on the copy engines.  bytes <= 64 MiB. */
int tf_copy_small(void* dst, const void* src, int64_t bytes, void* stream);

/* Fused decode-forward ops between the library GEMMs (bf16 in / out, fp32
 * math): y = x * rsqrt(mean(x^2) + eps) * w per row (dim % 8 == 0, dim <=
 * 8192), and y = silu(gu[:, :ffn]) * gu[:, ffn:] for gu [rows][2*ffn]. */
int tf_rmsnorm(const void* x, const void* w, void* y, int32_t rows, int32_t dim, float eps, void* stream);
int tf_silu_mul(const void* gu, void* y, int32_t rows, int32_t ffn, void* stream);
/* x[r] = bf16(x[r] + y[r]) (in place), h[r] = rmsnorm(x[r]) * w; rows x dim bf16,
 * dim % 8 == 0, dim <= 8192.  The TP=1 decoder's residual + next-norm after
 * its output projections (plain GEMMs into y). */
int tf_residual_rmsnorm(void* x, const void* y, const void* w, void* h, int32_t rows, int32_t dim, float eps,
                        void* stream);

/* ---------------------------------------------------------------- KV append --
 * Model path: write K/V rows of n tokens for one layer, token i at
 * (table[rows[i]], pos[i]).  k/v: [n][kv_heads][head_dim] bf16 with a row
 * stride of kv_row_stride elements (so a fused QKV output can be passed). */
int tf_kv_append(int64_t pool, const int32_t* dev_table, int32_t row_stride, const int32_t* dev_rows,
                 const int32_t* dev_pos, int32_t n, int32_t layer, const void* k, const void* v,
                 int64_t kv_row_stride, void* stream);

/* Decode epilogue of the fused QKV projection: qkv [n][n_q_heads + 2*kv_heads]
 * [head_dim] bf16 -> rotary embedding (interleaved pairs, angle = pos *
 * inv_freq[i], inv_freq fp32 [head_dim/2] on device) of q and k; k and v
 * appended at (table[rows[i]], pos[i]) of `layer`; rotated q written to
 * q_out [n][n_q_heads][head_dim]; if kv_out is not NULL the rotated k and v
 * are also written contiguously to kv_out [2][n][kv_heads][head_dim] (the
 * prefill attention input).  One launch per layer. */
int tf_rope_kv_append(int64_t pool, const int32_t* dev_table, int32_t row_stride, const int32_t* dev_rows,
                      const int32_t* dev_pos, int32_t n, int32_t layer, const void* qkv, int32_t n_q_heads,
                      const float* inv_freq, void* q_out, void* kv_out, void* stream);

/* Same as tf_rope_kv_append for decode, with the write-through fused into
 * the epilogue (reference write-through: engine.py:781-813):
 * when dev_host_table[rows[i]][pos[i]/block] >= 0 the appended k/v are also
 * stored into that block of the pinned host store (same slot, same layout),
 * so a token's KV is mirrored to the host in the step that makes it
 * (prefill or decode).  kv_out as in tf_rope_kv_append (may be NULL). */
int tf_rope_kv_append_wt(int64_t pool, const int32_t* dev_table, const int32_t* dev_host_table, int32_t row_stride,
                         const int32_t* dev_rows, const int32_t* dev_pos, int32_t n, int32_t layer, const void* qkv,
                         int32_t n_q_heads, const float* inv_freq, void* q_out, void* kv_out, void* stream);

/* Synthetic KV (parity / swap benchmarks): positions [pos_begin,pos_end) of
 * request rid, all layers, value = tf_kv_bits(seed, rid, pos, layer, kv,
 * head, dim) (identical to oracle/dataplane.py kv_bits). */
typedef struct {
  int32_t row;
  int32_t rid;
  int32_t pos_begin;
  int32_t pos_end;
} tf_span;

int tf_kv_fill_synthetic(int64_t pool, const int32_t* dev_table, int32_t row_stride, const tf_span* spans,
                         int32_t n_spans, uint32_t seed, void* stream);
int tf_q_fill_synthetic(void* q, const int32_t* dev_rids, const int32_t* dev_pos, int32_t B, int32_t layer,
                        int32_t n_q_heads, int32_t head_dim, uint32_t seed, void* stream);

/* ------------------------------------------------------- decode attention --
 * out[b][h] = softmax(q[b][h] . K[0:ctx[b]]^T * scale) V[0:ctx[b]] over the
 * paged KV of layer `layer` of request row rows[b]; GQA head h reads kv head
 * h / (n_q_heads/kv_heads).  q/out: [B][n_q_heads][head_dim] bf16, fp32
 * accumulation on tensor cores (mma.sync bf16 for the QK^T / PV contractions).
 * Implementations (tf_paged_decode_attn_impl): v5 (tf_attn_tma.cu; head_dim
 * 128 with group 1/2/4/5/8 or head_dim 64 with group 1/2/4, B <= 1024) is a
 * persistent grid of stream-K warps - the layer's (request, kv head, block)
 * work is split evenly over the warps; each warp's elected lane streams its
 * 16-token K/V tiles with TMA tensor loads (128-B swizzle) into a per-warp
 * mbarrier ring, running ahead across (request, head) boundaries; a (request,
 * head) shared by several warps is merged in-kernel.  v3 (head_dim 128) is a
 * split-KV grid of (request, kv head, split) CTAs with cp.async rings and is
 * the default at every batch (2-stage rings at B <= 96, 3 above); v5 is
 * opt-in (impl 5): its waits are bounded (2 s; an expired wait is counted in
 * workspace bytes [8, 64) instead of hanging the GPU).  Other shapes use the
 * CUDA-core / bulk-copy kernels.
 * max_ctx must bound every ctx[b].  The workspace (size from
 * tf_paged_decode_attn_workspace for the same B / max_ctx / n_q_heads, under
 * the same implementation) must be ZERO-filled before its first use; every
 * launch leaves its counters zero, so it can be reused (and captured in CUDA
 * graphs) without re-zeroing.
 * Replaces the affine decode cost of tokensim/costs.py:45-59. */
int tf_paged_decode_attn(int64_t pool, const void* q, const int32_t* dev_table, int32_t row_stride,
                         const int32_t* dev_rows, const int32_t* dev_ctx, int32_t B, int32_t max_ctx,
                         int32_t layer, int32_t n_q_heads, float scale, void* out, void* workspace,
                         int64_t workspace_bytes, void* stream);
int64_t tf_paged_decode_attn_workspace(int64_t pool, int32_t B, int32_t max_ctx, int32_t n_q_heads);
/* Select the implementation for subsequent launches (0 = the default by
 * batch, 1..5 = that version; any other value only queries).  Returns the
 * previous selection.  For A/B benchmarks and for tests that check every
 * implementation in one process. */
int tf_paged_decode_attn_impl(int32_t impl);

/* ----------------------------------------------------------------- selector --
 * Bit-exact GPU restatement of the buffer-aware policy's decisions (IEEE
 * float64 in the reference's operation order, CPython 3.12 sum() semantics,
 * glibc exp).  Synchronous: copies in, one single-CTA launch, copies out. */
typedef struct {
  int32_t request_id;
  int32_t prompt_len;
  int32_t output_len;
  int32_t running;
  int32_t pinned;
  int32_t has_tprime;
  int64_t generated;
  int64_t consumed;
  int64_t ctx_tokens;
  int64_t gpu_resident;
  double arrival_time;
  double rate;
  double busy_since_tick;
  double t_io;
  double t_recompute;
  double last_iter_time; /* 0.0 encodes None (same truthiness) */
  double t_prime;        /* policy EMA state (in), ignored unless has_tprime */
} tf_member;

typedef struct {
  int32_t request_id;
  int32_t prompt_len;
  double waited_s;
} tf_waiter;

typedef struct {
  int32_t n_members;
  int32_t n_waiting;
  int32_t free_slots;
  int32_t max_batch;
  int32_t offload_enabled;
  int32_t mode; /* in: current policy mode (0 buffer_aware, 1 fcfs_fallback) */
  int64_t h2d_blocked_tokens;
  double now;
  double gpu_mem_free;
  double gpu_mem_total;
  double cpu_mem_total;
  double gamma;
  /* SchedulerConfig */
  double schedule_interval;
  double per_request_mem_estimate;
  double workingset_adjust_rate;
  double buffer_safety_factor;
  double penalty_weight;
  double tau_schedule;
  double critical_buffer_seconds;
  double value_threshold_frac;
  double value_decay_alpha;
  double pacing_buffer_seconds;
  double ema_factor;
} tf_tick_params;

/* On-device snapshot builder input: the engine's raw
 * per-request counters in request-id order (the engine packs only requests
 * in service and not generation-complete; rows of other requests are
 * accepted and skipped; n_rows <= the selector's max_members <= 1024, the
 * concurrent-member capacity of the single-CTA kernels); the device derives
 * the MemberView rows of tokensim/engine.py:993-1061 (membership = in service
 * and not generation-complete; t_io = io_overhead_estimate, kvstore.py:173-193;
 * t_recompute = prefill_s_per_token * total_kv) in the reference's operation
 * order, compacts them and hands them to the tick kernel without a host
 * round trip. */
enum { TF_ST_PENDING = 0, TF_ST_WAITING = 1, TF_ST_PREFILL_WAIT = 2, TF_ST_PREFILLING = 3, TF_ST_RUNNING = 4,
       TF_ST_PREEMPTED = 5, TF_ST_LOADING = 6, TF_ST_RECOMPUTING = 7, TF_ST_GEN_DONE = 8, TF_ST_DONE = 9 };

typedef struct {
  int32_t request_id;
  int32_t status; /* TF_ST_* */
  int32_t prompt_len;
  int32_t output_len;
  int32_t has_tprime;
  int32_t pad_;
  int64_t generated;
  int64_t consumed;
  int64_t total_kv;
  int64_t gpu_resident;
  int64_t cpu_synced;
  int64_t inflight_d2h;
  double arrival_time;
  double rate;
  double busy_since_tick;
  double last_iter_time; /* 0.0 encodes None */
  double t_prime;
} tf_req_row;

typedef struct {
  int64_t q_d2h_tokens; /* tokens queued or in service per channel */
  int64_t q_h2d_tokens;
  double d2h_rate;      /* measured EMA, or the configured bandwidth before the first sample */
  double h2d_rate;
  double prefill_s_per_token;
} tf_snap_globals;

/* Result arrays (caller-owned host memory, capacity n_members / n_waiting):
 * counts[0]=mode, [1]=n_preempt, [2]=n_resume, [3]=n_admitted,
 * [4]=n_recomputed, [5]=n_batches.  resume_how: 0 load, 1 recompute.
 * batch_sizes[n_batches] partitions batch_ids (prefill sub-batches).
 * t_prime_out[i] / t_prime_set[i]: EMA state after the tick per member. */
typedef struct {
  int32_t* counts;
  int32_t* preempt;
  int32_t* resume_ids;
  int32_t* resume_how;
  int32_t* admitted;
  int32_t* recomputed;
  int32_t* batch_sizes;
  int32_t* batch_ids;
  double* t_prime_out;
  int32_t* t_prime_set;
} tf_tick_result;

int64_t tf_selector_workspace_bytes(int32_t max_members, int32_t max_waiting);
int tf_selector_init(void* dev_ws, int64_t dev_bytes, void* host_pinned_ws, int64_t host_bytes, int32_t max_members,
                     int32_t max_waiting, int64_t* out_handle);
int tf_selector_destroy(int64_t sel);
int tf_policy_tick(int64_t sel, const tf_tick_params* p, const tf_member* members, const tf_waiter* waiting,
                   tf_tick_result* out, void* stream);
/* on_tick from raw request rows: builds the member view on the device
 * (p->n_members is ignored and set by the builder); member_ids (capacity
 * n_rows) receives the request id of every member, in member order. */
int tf_policy_tick_rows(int64_t sel, const tf_tick_params* p, const tf_req_row* rows, int32_t n_rows,
                        const tf_snap_globals* g, const tf_waiter* waiting, tf_tick_result* out, int32_t* member_ids,
                        int32_t* n_members, void* stream);
int tf_policy_fastpath(int64_t sel, const tf_tick_params* p, const tf_member* members, const tf_waiter* waiting,
                       tf_tick_result* out, void* stream);

/* Pacing filter over (id, b_rem, rate) triples -> kept ids (in input order).
 * Returns the number kept via *n_out. */
int tf_iteration_batch(int64_t sel, const int32_t* ids, const int64_t* b_rem, const double* rates, int32_t n,
                       int32_t contention, int32_t mode, double pacing_buffer_seconds, int32_t* out_ids,
                       int32_t* n_out, void* stream);

/* select_batch on priority views (phi, value, t_prime, rate, utility, length
 * per candidate) -> chosen flags. */
typedef struct {
  int32_t request_id;
  int32_t pad;
  int64_t length;
  double phi;
  double value;
  double t_prime;
  double rate;
  double utility;
} tf_prio;

int tf_select_batch(int64_t sel, const tf_prio* views, int32_t n, double gpu_mem, int32_t max_batch,
                    uint8_t* out_chosen, void* stream);

/* glibc-exact exp, exported for the oracle checks */
double tf_host_glibc_exp(double x);


/* ---- C4 tensor-parallel data path: peer-memory all-reduce
 * fused with the residual add and the next RMSNorm.  Replaces the NCCL
 * all-reduce after o_proj / down_proj of the TP decoder (the reference has
 * no TP: tokensim/engine.py:1089-1091 runs one replica per GPU; C4 is the
 * north-star configuration built on top of it).
 *
 * tf_ar_create   this rank's communicator on the current device: a cudaMalloc'ed
 *                data buffer of capacity_bytes (the rank's GEMM partial goes
 *                there: tf_ar_buffer) + a zeroed control block (barrier flags).
 *                max_ctas caps the grid (0 = one CTA per SM, 148); every rank
 *                must pass the same value.  A small cap keeps the spinning
 *                CTAs from starving the other ranks' kernels when several
 *                ranks share ONE device (tests).
 * tf_ar_export   128 bytes: IPC handles of the data buffer and control block.
 * tf_ar_open     all_handles = world x 128 bytes in rank order: maps every
 *                peer's buffer and control block (cudaIpcOpenMemHandle; P2P
 *                over NVLink between GPUs, plain aliases on one device).
 * tf_ar_set_peers  same-process ranks (tests): peers' device pointers directly.
 * tf_ar_residual_rmsnorm
 *                x[r] = bf16(x[r] + sum_p part_p[r]) (fp32, rank order: bit-identical
 *                on every rank); h_out[r] = rmsnorm(x[r]) * gamma.  x NULL: the
 *                plain sum (to h_out when gamma is NULL).  rows x dim bf16,
 *                dim % 8 == 0, dim <= 8192.  Every rank must issue the same
 *                sequence of calls with the same rows; graph-capturable.
 * tf_ar_status   1 if a barrier wait timed out (10 s) since creation, else 0 (syncs).
 */
int tf_ar_create(int32_t rank, int32_t world, int64_t capacity_bytes, int32_t max_ctas, int64_t* out_handle);
void* tf_ar_buffer(int64_t ar);
void* tf_ar_ctl(int64_t ar);
int tf_ar_export(int64_t ar, void* out128);
int tf_ar_open(int64_t ar, const void* all_handles);
int tf_ar_set_peers(int64_t ar, void* const* data, void* const* ctl);
int tf_ar_residual_rmsnorm(int64_t ar, void* x, const void* gamma, void* h_out, int32_t rows, int32_t dim, float eps,
                           void* stream);
int tf_ar_status(int64_t ar);
int tf_ar_destroy(int64_t ar);

#ifdef __cplusplus
}
#endif
#endif /* TOKENFLOW_B200_H */
