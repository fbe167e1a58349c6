// Batch-priority selector: the buffer-aware policy's decisions on the GPU.
//
// Restates BufferAwarePolicy.on_tick / opportunistic / iteration_batch and
// select_batch (tokensim/scheduler.py:205-269, :513-823) as ONE single-CTA
// launch per call.  Every request is scored in parallel (phi, token value,
// utility, buffer-coverage safety), orderings are computed by parallel rank
// sorts over (key..., id) tuples, and select_batch's adjacent-swap local
// search evaluates all swap trials of a pass in parallel (one thread per
// trial, resuming from the shared prefix state) and accepts the first
// strict improvement - the same trajectory as the sequential search.
//
// Bit-exactness rules (compiled with -fmad=false):
//  * float64 everywhere, operations in the reference's order;
//  * Python max/min argument semantics (max(a,b) = b if b > a else a);
//  * CPython 3.12 sum() (Neumaier) for the float sums (utilities, rates);
//  * CPython float floor division for working_set_size;
//  * glibc's exp (tf_glibc_exp.h) for phi.
#include <algorithm>
#include <cstring>

#include "tf_common.cuh"
#include "tf_glibc_exp.h"

namespace tf {

constexpr int kSelThreads = 512;
constexpr int kMaxN = 1024;  // members (and select candidates)
constexpr int kMaxW = 2048;  // waiting requests

__device__ __forceinline__ double pmax(double a, double b) { return b > a ? b : a; }
__device__ __forceinline__ double pmin(double a, double b) { return b < a ? b : a; }

// CPython float floor division (Objects/floatobject.c float_divmod).
__device__ double py_floordiv(double vx, double wx) {
  double mod = fmod(vx, wx);
  double div = __ddiv_rn(__dsub_rn(vx, mod), wx);
  if (mod != 0.0) {
    if ((wx < 0) != (mod < 0)) div = __dsub_rn(div, 1.0);
  }
  double fl;
  if (div != 0.0) {
    fl = floor(div);
    if (__dsub_rn(div, fl) > 0.5) fl = __dadd_rn(fl, 1.0);
  } else {
    fl = copysign(0.0, __ddiv_rn(vx, wx));
  }
  return fl;
}

// CPython 3.12 sum(): int start 0, then Neumaier compensation.
struct PySum {
  int n;
  double f, c;
  __device__ void init() { n = 0; f = 0.0; c = 0.0; }
  __device__ void add(double x) {
    if (n == 0) {
      f = __dadd_rn(0.0, x);
      c = 0.0;
    } else {
      double t = __dadd_rn(f, x);
      if (fabs(f) >= fabs(x))
        c = __dadd_rn(c, __dadd_rn(__dsub_rn(f, t), x));
      else
        c = __dadd_rn(c, __dadd_rn(__dsub_rn(x, t), f));
      f = t;
    }
    ++n;
  }
  __device__ double result() const {
    if (n == 0) return 0.0;
    double r = f;
    if (c != 0.0 && isfinite(c)) r = __dadd_rn(r, c);
    return r;
  }
};

struct SelWork {
  tf_tick_params p;
  int32_t n, w;
};

// Per-member derived values (shared memory).
struct Smem {
  double drain[kMaxN];
  double phi[kMaxN];
  double vt[kMaxN];      // value * t_prime (priority key)
  double util[kMaxN];
  double tprime[kMaxN];
  long long brem[kMaxN];
  int8_t safe[kMaxN];
  int8_t flag[kMaxN];    // bit0 preempted-now, bit1 resumed-now, bit2 in proposal, bit3 filter
  int16_t ord[kMaxN];    // sort output
  int16_t ord2[kMaxN];
  // select_batch scratch
  int16_t cand[kMaxN];
  int16_t sorder[kMaxN];
  double pre_used[kMaxN + 1];
  double pre_f[kMaxN + 1];
  double pre_c[kMaxN + 1];
  int16_t pre_cnt[kMaxN + 1];
  double trial_u[kMaxN];
  int best_i;
  // scalar control state
  int slots;
  double mem;
  int n_pre, n_res, n_adm, n_rc, n_bat;
  int stop;
};

// Results live in global memory, laid out by the host wrapper.
struct SelOut {
  int32_t* counts;
  int32_t* preempt;
  int32_t* resume_ids;
  int32_t* resume_how;
  int32_t* admitted;
  int32_t* recomputed;
  int32_t* batch_sizes;
  int32_t* batch_ids;
  double* tprime_out;
  int32_t* tprime_set;
};

// rank sort of the members whose flag bit3 is set, by comparator less(i, j)
template <typename Less>
__device__ int rank_sort(Smem& s, int n, int16_t* out, Less less) {
  __shared__ int cnt;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    if (!(s.flag[i] & 8)) continue;
    int r = 0;
    for (int j = 0; j < n; ++j)
      if ((s.flag[j] & 8) && j != i && less(j, i)) ++r;
    out[r] = (int16_t)i;
    atomicAdd(&cnt, 1);
  }
  __syncthreads();
  int c = cnt;
  __syncthreads();
  return c;
}

// --------------------------------------------------------- select_batch
// Candidates s.cand[0..nc) (member indices or view indices), keys in s.phi /
// s.vt / rates / ids, utilities in s.util, lengths via len[].  Output: flag
// bit2 set on chosen candidates.
__device__ void select_batch_dev(Smem& s, int nc, const double* rate, const int32_t* ids, const long long* len,
                                 double gpu_mem, int max_batch) {
  // 1. greedy order: (-phi, -(value*t'), -rate, id)
  for (int a = threadIdx.x; a < nc; a += blockDim.x) {
    const int i = s.cand[a];
    int r = 0;
    for (int b = 0; b < nc; ++b) {
      const int j = s.cand[b];
      if (j == i) continue;
      double ki = -s.phi[i], kj = -s.phi[j];
      bool lt;
      if (kj != ki) lt = kj < ki;
      else if (-s.vt[j] != -s.vt[i]) lt = -s.vt[j] < -s.vt[i];
      else if (-rate[j] != -rate[i]) lt = -rate[j] < -rate[i];
      else lt = ids[j] < ids[i];
      if (lt) ++r;
    }
    s.sorder[r] = (int16_t)i;
  }
  __syncthreads();
  const int max_passes = nc > 1 ? nc : 1;
  int passes = 0, start = 0;
  bool moved = false;
  double best_u = 0.0;
  while (true) {
    // prefix states of the current order (thread 0, O(n))
    if (threadIdx.x == 0) {
      double used = 0.0;
      int cnt = 0;
      PySum ps;
      ps.init();
      for (int k = 0; k < nc; ++k) {
        s.pre_used[k] = used;
        s.pre_cnt[k] = (int16_t)cnt;
        s.pre_f[k] = ps.n ? ps.f : 0.0;
        s.pre_c[k] = ps.c;
        if (cnt < max_batch) {
          const int i = s.sorder[k];
          const double need = (double)len[i];
          if (__dadd_rn(used, need) <= gpu_mem) {
            ps.add(s.util[i]);
            used = __dadd_rn(used, need);
            ++cnt;
          }
        }
      }
      s.pre_used[nc] = used;
      s.pre_cnt[nc] = (int16_t)cnt;
      s.pre_f[nc] = ps.n ? ps.f : 0.0;
      s.pre_c[nc] = ps.c;
      s.trial_u[0] = ps.result();  // base utility scratch
      s.best_i = nc;
    }
    __syncthreads();
    if (passes == 0 && start == 0 && !moved) best_u = s.trial_u[0];
    __syncthreads();
    // evaluate trials i in [start, nc-2] against the current order
    for (int i = start + threadIdx.x; i <= nc - 2; i += blockDim.x) {
      double used = s.pre_used[i];
      int cnt = s.pre_cnt[i];
      PySum ps;
      ps.n = cnt;
      ps.f = s.pre_f[i];
      ps.c = s.pre_c[i];
      for (int k = i; k < nc; ++k) {
        if (cnt >= max_batch) break;
        const int e = (k == i) ? s.sorder[i + 1] : (k == i + 1 ? s.sorder[i] : s.sorder[k]);
        const double need = (double)len[e];
        if (__dadd_rn(used, need) <= gpu_mem) {
          ps.add(s.util[e]);
          used = __dadd_rn(used, need);
          ++cnt;
        }
      }
      const double u = ps.result();
      if (u > best_u) atomicMin(&s.best_i, i);
    }
    __syncthreads();
    const int bi = s.best_i;
    __syncthreads();
    if (bi < nc) {
      // accept the first improving swap; recompute its utility exactly
      if (threadIdx.x == 0) {
        int16_t t = s.sorder[bi];
        s.sorder[bi] = s.sorder[bi + 1];
        s.sorder[bi + 1] = t;
      }
      __syncthreads();
      moved = true;
      start = bi + 1;
      // best_u := utility of the new order's selection (identical to the trial's)
      if (threadIdx.x == 0) {
        double used = 0.0;
        int cnt = 0;
        PySum ps;
        ps.init();
        for (int k = 0; k < nc && cnt < max_batch; ++k) {
          const int e = s.sorder[k];
          const double need = (double)len[e];
          if (__dadd_rn(used, need) <= gpu_mem) {
            ps.add(s.util[e]);
            used = __dadd_rn(used, need);
            ++cnt;
          }
        }
        s.trial_u[0] = ps.result();
      }
      __syncthreads();
      best_u = s.trial_u[0];
      __syncthreads();
      if (start <= nc - 2) continue;
    }
    // the pass is over
    ++passes;
    if (!moved || passes >= max_passes) break;
    moved = false;
    start = 0;
  }
  // mark the selection of the final order
  if (threadIdx.x == 0) {
    double used = 0.0;
    int cnt = 0;
    for (int k = 0; k < nc && cnt < max_batch; ++k) {
      const int e = s.sorder[k];
      const double need = (double)len[e];
      if (__dadd_rn(used, need) <= gpu_mem) {
        s.flag[e] |= 4;
        used = __dadd_rn(used, need);
        ++cnt;
      }
    }
  }
  __syncthreads();
}

// ------------------------------------------------------------ policy views
__device__ double token_value(long long b, int out_len, double frac, double alpha) {
  const double thr = __dmul_rn(frac, (double)out_len);
  if ((double)b <= thr) return 1.0;
  return pmax(__dsub_rn(1.0, __dmul_rn(alpha, __dsub_rn((double)b, thr))), 0.0);
}

__device__ double overhead_of(const tf_member& m, int offload) {
  return offload ? pmin(m.t_io, m.t_recompute) : m.t_recompute;
}

__device__ int restore_how(const tf_member& m, int offload) {  // 0 load, 1 recompute
  if (!offload) return 1;
  return m.t_io > m.t_recompute ? 1 : 0;
}

__device__ int ws_size(const tf_tick_params& p, int n_running) {
  const double total = __dadd_rn(p.gpu_mem_total, p.cpu_mem_total);
  const long long cap = (long long)py_floordiv(total, p.per_request_mem_estimate);
  if (n_running >= cap) return (int)(cap > 1 ? cap : 1);
  const double adj = __dsub_rn((double)cap, __dmul_rn(p.workingset_adjust_rate, (double)(cap - n_running)));
  long long w = (long long)floor(__dadd_rn(adj, 0.5));
  if (w > cap) w = cap;
  return (int)(w > 1 ? w : 1);
}

// Scores every member: EMA of t', drain, phi, value*t', utility, safety.
__device__ void score_members(Smem& s, const tf_member* mem, int n, const tf_tick_params& p, bool ema) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const tf_member& m = mem[i];
    double tp = m.has_tprime ? m.t_prime : p.schedule_interval;
    if (ema && m.running && !m.pinned) tp = __dadd_rn(tp, __dmul_rn(p.ema_factor, __dsub_rn(m.busy_since_tick, tp)));
    s.tprime[i] = tp;
    const long long b = m.generated - m.consumed;
    s.brem[i] = b;
    s.drain[i] = __ddiv_rn((double)b, m.rate);
    const double ov = overhead_of(m, p.offload_enabled);
    const double v = token_value(b, m.output_len, p.value_threshold_frac, p.value_decay_alpha);
    const double sc = pmax(__dmul_rn(m.rate, p.schedule_interval), 1e-9);
    const double phi = tf_glibc_exp(__ddiv_rn(-pmax((double)b, 0.0), sc));
    s.phi[i] = phi;
    s.vt[i] = __dmul_rn(v, tp);
    const double teff = pmax(__dsub_rn(tp, ov), 0.0);
    s.util[i] = __dsub_rn(__dmul_rn(v, teff), __dmul_rn(p.penalty_weight, phi));
    const double need = __dmul_rn(__dmul_rn(p.buffer_safety_factor, m.rate), __dadd_rn(__dadd_rn(ov, 0.0), p.tau_schedule));
    s.safe[i] = (double)b >= need ? 1 : 0;
    s.flag[i] = 0;
  }
  __syncthreads();
}

// argmax over members with flag bit3 by (b_rem, -id): largest b_rem, ties -> smaller id
__device__ int argmax_brem(Smem& s, const tf_member* mem, int n) {
  __shared__ unsigned long long best;
  if (threadIdx.x == 0) best = ~0ull;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    if (!(s.flag[i] & 8)) continue;
    // encode: larger b_rem first, then smaller id -> minimise (MAXB - b, id)
    unsigned long long key = ((unsigned long long)(0x7FFFFFFFll - s.brem[i]) << 32) | (unsigned)mem[i].request_id;
    atomicMin(&best, key);
  }
  __syncthreads();
  int res = -1;
  if (best != ~0ull) {
    unsigned id = (unsigned)(best & 0xFFFFFFFFu);
    for (int i = 0; i < n; ++i)
      if ((unsigned)mem[i].request_id == id) { res = i; break; }
  }
  __syncthreads();
  return res;
}

__device__ void emit_preempt(Smem& s, SelOut& o, const tf_member* mem, int v) {
  if (threadIdx.x == 0) {
    o.preempt[s.n_pre++] = mem[v].request_id;
    s.flag[v] |= 1;
    s.slots += 1;
    s.mem = __dadd_rn(s.mem, (double)mem[v].gpu_resident);
  }
  __syncthreads();
}

__device__ void emit_resume(Smem& s, SelOut& o, const tf_member* mem, int i, int offload) {
  if (threadIdx.x == 0) {
    const int how = restore_how(mem[i], offload);
    o.resume_ids[s.n_res] = mem[i].request_id;
    o.resume_how[s.n_res] = how;
    s.n_res++;
    if (how == 1) o.recomputed[s.n_rc++] = mem[i].request_id;
    s.flag[i] |= 2;
    s.slots -= 1;
    s.mem = __dsub_rn(s.mem, (double)mem[i].ctx_tokens);
  }
  __syncthreads();
}

// ------------------------------------------------------------------ kernels
struct TickArgs {
  const tf_tick_params* p;
  const tf_member* mem;
  const tf_waiter* wait;
  SelOut o;
  int fastpath;
};

__global__ void __launch_bounds__(kSelThreads) tick_kernel(TickArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>(smem_raw);
  const tf_tick_params p = *a.p;
  const tf_member* mem = a.mem;
  const tf_waiter* wait = a.wait;
  SelOut o = a.o;
  const int n = p.n_members, nw = p.n_waiting;
  if (threadIdx.x == 0) {
    s.slots = p.free_slots;
    s.mem = p.gpu_mem_free;
    s.n_pre = s.n_res = s.n_adm = s.n_rc = s.n_bat = 0;
  }
  // ------------------------------------------------ fast path (opportunistic)
  if (a.fastpath) {
    score_members(s, mem, n, p, false);
    if (p.mode == 1) {
      if (threadIdx.x == 0) for (int k = 0; k < 6; ++k) o.counts[k] = 0;
      if (threadIdx.x == 0) o.counts[0] = 1;
      return;
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) s.flag[i] = (!mem[i].running && !mem[i].pinned) ? 8 : 0;
    __syncthreads();
    const int np = rank_sort(s, n, s.ord, [&](int j, int i) {
      return s.drain[j] != s.drain[i] ? s.drain[j] < s.drain[i] : mem[j].request_id < mem[i].request_id;
    });
    if (threadIdx.x == 0) {
      for (int k = 0; k < np; ++k) {
        const int i = s.ord[k];
        if (s.slots <= 0 || (double)mem[i].ctx_tokens > s.mem) break;
        const int how = restore_how(mem[i], p.offload_enabled);
        o.resume_ids[s.n_res] = mem[i].request_id;
        o.resume_how[s.n_res] = how;
        s.n_res++;
        if (how == 1) o.recomputed[s.n_rc++] = mem[i].request_id;
        s.slots -= 1;
        s.mem = __dsub_rn(s.mem, (double)mem[i].ctx_tokens);
      }
      int n_run = 0;
      for (int i = 0; i < n; ++i) n_run += mem[i].running ? 1 : 0;
      s.stop = n_run;
    }
    __syncthreads();
    const int room = ws_size(p, s.stop);
    if (threadIdx.x == 0) {
      int in_service = n + s.n_res;
      int nb = 0;
      for (int k = 0; k < nw; ++k) {
        const double need = (double)wait[k].prompt_len + 1.0;
        if (s.slots <= 0 || need > s.mem || in_service >= room) break;
        o.batch_ids[nb++] = wait[k].request_id;
        s.slots -= 1;
        s.mem = __dsub_rn(s.mem, need);
        in_service += 1;
      }
      if (nb) {
        o.batch_sizes[0] = nb;
        s.n_bat = 1;
      }
      o.counts[0] = 0;
      o.counts[1] = 0;
      o.counts[2] = s.n_res;
      o.counts[3] = 0;
      o.counts[4] = s.n_rc;
      o.counts[5] = s.n_bat;
    }
    return;
  }

  // ------------------------------------------------------------ on_tick
  score_members(s, mem, n, p, true);
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    o.tprime_out[i] = s.tprime[i];
    o.tprime_set[i] = (mem[i].has_tprime || (mem[i].running && !mem[i].pinned)) ? 1 : 0;
  }
  // mode: sum(rates of running members) <= gamma (CPython sum)
  if (threadIdx.x == 0) {
    PySum ps;
    ps.init();
    int any = 0;
    for (int i = 0; i < n; ++i)
      if (mem[i].running) {
        ps.add(mem[i].rate);
        any = 1;
      }
    const double tot = any ? ps.result() : 0.0;
    s.stop = tot <= p.gamma ? 0 : 1;
  }
  __syncthreads();
  const int mode = s.stop;
  if (mode == 1) {
    // _fallback_tick: arrival order within device memory (scheduler.py:738-772)
    for (int i = threadIdx.x; i < n; i += blockDim.x) s.flag[i] = mem[i].pinned ? 0 : 8;
    __syncthreads();
    const int np = rank_sort(s, n, s.ord, [&](int j, int i) {
      return mem[j].arrival_time != mem[i].arrival_time ? mem[j].arrival_time < mem[i].arrival_time
                                                        : mem[j].request_id < mem[i].request_id;
    });
    if (threadIdx.x == 0) {
      int pinned = 0;
      for (int i = 0; i < n; ++i) pinned += mem[i].pinned ? 1 : 0;
      const int budget = p.max_batch - pinned;
      double used = 0.0;
      int nt = 0;
      for (int k = 0; k < np; ++k) {
        if (nt >= budget) break;
        const int i = s.ord[k];
        if (__dadd_rn(used, (double)mem[i].ctx_tokens) <= p.gpu_mem_total) {
          s.flag[i] |= 4;
          s.ord2[nt++] = (int16_t)i;
          used = __dadd_rn(used, (double)mem[i].ctx_tokens);
        }
      }
      for (int i = 0; i < n; ++i)
        if (!mem[i].pinned && mem[i].running && !(s.flag[i] & 4)) o.preempt[s.n_pre++] = mem[i].request_id;
      for (int k = 0; k < nt; ++k) {
        const int i = s.ord2[k];
        if (!mem[i].running) {
          const int how = restore_how(mem[i], p.offload_enabled);
          o.resume_ids[s.n_res] = mem[i].request_id;
          o.resume_how[s.n_res] = how;
          s.n_res++;
          if (how == 1) o.recomputed[s.n_rc++] = mem[i].request_id;
        }
      }
      o.counts[0] = 1;
      o.counts[1] = s.n_pre;
      o.counts[2] = s.n_res;
      o.counts[3] = 0;
      o.counts[4] = s.n_rc;
      o.counts[5] = 0;
    }
    return;
  }

  const double crit = p.critical_buffer_seconds;
  // ---- step 1: critical rescue (scheduler.py:549-572)
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    s.flag[i] = (!mem[i].pinned && !mem[i].running && s.drain[i] < crit) ? 8 : 0;
  __syncthreads();
  const int ncrit = rank_sort(s, n, s.ord2, [&](int j, int i) {
    return s.drain[j] != s.drain[i] ? s.drain[j] < s.drain[i] : mem[j].request_id < mem[i].request_id;
  });
  for (int i = threadIdx.x; i < n; i += blockDim.x) s.flag[i] &= ~8;
  __syncthreads();
  for (int k = 0; k < ncrit; ++k) {
    const int m = s.ord2[k];
    if (s.slots <= 0) {
      // candidates: running, not preempted now, strictly fatter drain
      __shared__ int n_cand, n_safe;
      if (threadIdx.x == 0) n_cand = n_safe = 0;
      __syncthreads();
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        s.flag[i] &= ~8;
        if (!mem[i].pinned && mem[i].running && !(s.flag[i] & 1) && s.drain[i] > s.drain[m]) {
          atomicAdd(&n_cand, 1);
          if (s.safe[i]) atomicAdd(&n_safe, 1);
        }
      }
      __syncthreads();
      if (n_cand == 0) continue;
      const bool use_safe = n_safe > 0;
      for (int i = threadIdx.x; i < n; i += blockDim.x)
        if (!mem[i].pinned && mem[i].running && !(s.flag[i] & 1) && s.drain[i] > s.drain[m] &&
            (!use_safe || s.safe[i]))
          s.flag[i] |= 8;
      __syncthreads();
      const int v = argmax_brem(s, mem, n);
      for (int i = threadIdx.x; i < n; i += blockDim.x) s.flag[i] &= ~8;
      __syncthreads();
      emit_preempt(s, o, mem, v);
    }
    emit_resume(s, o, mem, m, p.offload_enabled);
  }

  // ---- step 2: working-set admission (scheduler.py:574-607)
  __shared__ int n_running_all;
  if (threadIdx.x == 0) {
    int c = 0;
    for (int i = 0; i < n; ++i) c += mem[i].running ? 1 : 0;
    n_running_all = c;
  }
  __syncthreads();
  const int room = ws_size(p, n_running_all);
  for (int k = 0; k < nw; ++k) {
    if (n + s.n_adm >= room) break;
    const double need = (double)wait[k].prompt_len + 1.0;
    if (!(s.slots > 0 && need <= s.mem)) {
      __shared__ int n_v;
      if (threadIdx.x == 0) n_v = 0;
      __syncthreads();
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        s.flag[i] &= ~8;
        if (!mem[i].pinned && mem[i].running && !(s.flag[i] & 3) && s.safe[i]) {
          s.flag[i] |= 8;
          atomicAdd(&n_v, 1);
        }
      }
      __syncthreads();
      if (n_v == 0) break;
      const int v = argmax_brem(s, mem, n);
      for (int i = threadIdx.x; i < n; i += blockDim.x) s.flag[i] &= ~8;
      __syncthreads();
      emit_preempt(s, o, mem, v);
    }
    if (threadIdx.x == 0) {
      s.slots -= 1;
      s.mem = __dsub_rn(s.mem, need);
      o.admitted[s.n_adm++] = k;  // waiting index for now; mapped to ids below
    }
    __syncthreads();
  }

  // ---- step 3: memory headroom (scheduler.py:609-652)
  if (threadIdx.x == 0) {
    bool contention = nw > 0;
    for (int i = 0; i < n && !contention; ++i)
      if (!mem[i].pinned && !mem[i].running) contention = true;
    double growth = 0.0;
    int n_active = 0;
    for (int i = 0; i < n; ++i) {
      const tf_member& m = mem[i];
      if (m.pinned || !m.running || (s.flag[i] & 3)) continue;
      ++n_active;
      if (m.last_iter_time == 0.0) continue;
      double sl = __ddiv_rn(p.schedule_interval, m.last_iter_time);
      if (contention) {
        const double ceil_ = __dmul_rn(m.rate, __dadd_rn(p.pacing_buffer_seconds, p.schedule_interval));
        sl = pmin(sl, pmax(0.0, __dsub_rn(ceil_, (double)s.brem[i])));
      }
      growth = __dadd_rn(growth, pmin(sl, (double)(m.output_len - m.generated)));
    }
    s.pre_used[0] = growth;
    s.pre_used[1] = __dadd_rn(growth, (double)p.h2d_blocked_tokens);
    s.stop = n_active;
  }
  __syncthreads();
  {
    const double growth = s.pre_used[0];
    const double target = s.pre_used[1];
    const int n_active = s.stop;
    __syncthreads();
    if (target > s.mem) {
      for (int i = threadIdx.x; i < n; i += blockDim.x)
        s.flag[i] = (s.flag[i] & ~8) |
                    ((!mem[i].pinned && mem[i].running && !(s.flag[i] & 3) && s.safe[i]) ? 8 : 0);
      __syncthreads();
      const int nv = rank_sort(s, n, s.ord, [&](int j, int i) {
        return s.brem[j] != s.brem[i] ? s.brem[j] > s.brem[i] : mem[j].request_id < mem[i].request_id;
      });
      for (int k = 0; k < nv; ++k) {
        if (s.mem >= target) break;
        emit_preempt(s, o, mem, s.ord[k]);
      }
      if (s.mem <= 0.0 && (p.h2d_blocked_tokens > 0 || growth > 0.0)) {
        // active = running, not preempted-before-step-3, not resumed; excl. preempted now
        for (int i = threadIdx.x; i < n; i += blockDim.x) s.flag[i] &= ~8;
        __syncthreads();
        // "active" was fixed before this step: recompute membership from snapshot
        // flags: members preempted in step 3 are excluded by bit0 anyway.
        for (int i = threadIdx.x; i < n; i += blockDim.x)
          if (!mem[i].pinned && mem[i].running && !(s.flag[i] & 3)) s.flag[i] |= 8;
        __syncthreads();
        const int nu = rank_sort(s, n, s.ord, [&](int j, int i) {
          if (s.brem[j] != s.brem[i]) return s.brem[j] > s.brem[i];
          if (mem[j].ctx_tokens != mem[i].ctx_tokens) return mem[j].ctx_tokens > mem[i].ctx_tokens;
          return mem[j].request_id < mem[i].request_id;
        });
        const double floor_ = (double)p.h2d_blocked_tokens + (double)(n_active / 2 > 1 ? n_active / 2 : 1);
        for (int k = 0; k < nu; ++k) {
          if (s.mem >= floor_) break;
          emit_preempt(s, o, mem, s.ord[k]);
        }
      }
      for (int i = threadIdx.x; i < n; i += blockDim.x) s.flag[i] &= ~8;
      __syncthreads();
    }
  }

  // ---- step 4: utility rebalance (scheduler.py:654-718)
  {
    const double horizon = __dadd_rn(crit, p.schedule_interval);
    __shared__ int n_run4, n_needy;
    if (threadIdx.x == 0) {
      int nr = 0, nn = 0;
      for (int i = 0; i < n; ++i)
        if (!mem[i].pinned && mem[i].running && !(s.flag[i] & 3)) s.cand[nr++] = (int16_t)i;
      for (int i = 0; i < n; ++i)
        if (!mem[i].pinned && !mem[i].running && !(s.flag[i] & 2) && s.drain[i] < horizon) {
          s.cand[nr + nn] = (int16_t)i;
          ++nn;
        }
      n_run4 = nr;
      n_needy = nn;
    }
    __syncthreads();
    const int nr = n_run4, nn = n_needy;
    if (nn > 0) {
      __shared__ double mem_budget;
      __shared__ int batch_budget;
      __shared__ long long lens[kMaxN];
      __shared__ double rates[kMaxN];
      __shared__ int32_t ids[kMaxN];
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        lens[i] = mem[i].ctx_tokens;
        rates[i] = mem[i].rate;
        ids[i] = mem[i].request_id;
        s.flag[i] &= ~4;
      }
      if (threadIdx.x == 0) {
        long long acc = 0;
        for (int k = 0; k < nr; ++k) acc += mem[s.cand[k]].ctx_tokens;
        const int bb = nr + s.slots;
        batch_budget = bb > 0 ? bb : 0;
        mem_budget = pmax(0.0, __dadd_rn(s.mem, (double)acc));
      }
      __syncthreads();
      select_batch_dev(s, nr + nn, rates, ids, lens, mem_budget, batch_budget);
      // incoming: needy in proposal by (drain, id)
      for (int i = threadIdx.x; i < n; i += blockDim.x) s.flag[i] &= ~8;
      __syncthreads();
      for (int k = nr + threadIdx.x; k < nr + nn; k += blockDim.x)
        if (s.flag[s.cand[k]] & 4) s.flag[s.cand[k]] |= 8;
      __syncthreads();
      const int ninc = rank_sort(s, n, s.ord2, [&](int j, int i) {
        return s.drain[j] != s.drain[i] ? s.drain[j] < s.drain[i] : mem[j].request_id < mem[i].request_id;
      });
      for (int i = threadIdx.x; i < n; i += blockDim.x) s.flag[i] &= ~8;
      __syncthreads();
      // outgoing: runners not in proposal & safe; fallback: runners in proposal & safe; by (-b_rem, id)
      for (int k = threadIdx.x; k < nr; k += blockDim.x) {
        const int i = s.cand[k];
        if (s.safe[i] && !(s.flag[i] & 4)) s.flag[i] |= 8;
      }
      __syncthreads();
      const int nout = rank_sort(s, n, s.ord, [&](int j, int i) {
        return s.brem[j] != s.brem[i] ? s.brem[j] > s.brem[i] : mem[j].request_id < mem[i].request_id;
      });
      for (int i = threadIdx.x; i < n; i += blockDim.x) s.flag[i] &= ~8;
      __syncthreads();
      __shared__ int16_t fb[kMaxN];
      for (int k = threadIdx.x; k < nr; k += blockDim.x) {
        const int i = s.cand[k];
        if (s.safe[i] && (s.flag[i] & 4)) s.flag[i] |= 8;
      }
      __syncthreads();
      const int nfb = rank_sort(s, n, fb, [&](int j, int i) {
        return s.brem[j] != s.brem[i] ? s.brem[j] > s.brem[i] : mem[j].request_id < mem[i].request_id;
      });
      for (int i = threadIdx.x; i < n; i += blockDim.x) s.flag[i] &= ~8;
      __syncthreads();
      if (threadIdx.x == 0) {
        int po = 0, pf = 0;
        for (int k = 0; k < ninc; ++k) {
          const int m = s.ord2[k];
          if (s.slots > 0 && (double)mem[m].ctx_tokens <= s.mem) {
            const int how = restore_how(mem[m], p.offload_enabled);
            o.resume_ids[s.n_res] = mem[m].request_id;
            o.resume_how[s.n_res] = how;
            s.n_res++;
            if (how == 1) o.recomputed[s.n_rc++] = mem[m].request_id;
            s.flag[m] |= 2;
            s.slots -= 1;
            s.mem = __dsub_rn(s.mem, (double)mem[m].ctx_tokens);
            continue;
          }
          const double bar = __dadd_rn(s.drain[m], p.schedule_interval);
          int victim = -1;
          while (po < nout) {
            const int c = s.ord[po++];
            if (s.drain[c] > bar) {
              victim = c;
              break;
            }
          }
          if (victim < 0) {
            while (pf < nfb) {
              const int c = fb[pf++];
              if (s.flag[c] & 1) continue;
              if (s.drain[c] > bar) {
                victim = c;
                break;
              }
            }
          }
          if (victim < 0) break;
          o.preempt[s.n_pre++] = mem[victim].request_id;
          s.flag[victim] |= 1;
          s.slots += 1;
          s.mem = __dadd_rn(s.mem, (double)mem[victim].gpu_resident);
          const int how = restore_how(mem[m], p.offload_enabled);
          o.resume_ids[s.n_res] = mem[m].request_id;
          o.resume_how[s.n_res] = how;
          s.n_res++;
          if (how == 1) o.recomputed[s.n_rc++] = mem[m].request_id;
          s.flag[m] |= 2;
          s.slots -= 1;
          s.mem = __dsub_rn(s.mem, (double)mem[m].ctx_tokens);
        }
      }
      __syncthreads();
    }
  }

  // ---- step 5: prefill partition (scheduler.py:720-727, :292-325)
  if (threadIdx.x == 0) {
    const int na = s.n_adm;
    long long acc = 0;
    for (int k = 0; k < na; ++k) acc += wait[o.admitted[k]].prompt_len + 1;
    const double budget = __dadd_rn(pmax(s.mem, 0.0), (double)acc);
    int nb = 0, nid = 0;
    if (na > 0) {
      for (int k = 0; k < na; ++k) {
        const tf_waiter& w = wait[o.admitted[k]];
        if (w.waited_s > 1.3 && (double)(w.prompt_len + 1) <= budget) {
          o.batch_ids[nid++] = w.request_id;
          o.batch_sizes[nb++] = 1;
        }
      }
      int cur = 0;
      double used = 0.0;
      for (int k = 0; k < na; ++k) {
        const tf_waiter& w = wait[o.admitted[k]];
        if (w.waited_s > 1.3) continue;
        const double tok = (double)(w.prompt_len + 1);
        if (tok > budget) continue;
        if (cur > 0 && __dadd_rn(used, tok) > budget) {
          o.batch_sizes[nb++] = cur;
          cur = 0;
          used = 0.0;
        }
        o.batch_ids[nid++] = w.request_id;
        ++cur;
        used = __dadd_rn(used, tok);
      }
      if (cur > 0) o.batch_sizes[nb++] = cur;
    }
    for (int k = 0; k < na; ++k) o.admitted[k] = wait[o.admitted[k]].request_id;
    o.counts[0] = 0;
    o.counts[1] = s.n_pre;
    o.counts[2] = s.n_res;
    o.counts[3] = na;
    o.counts[4] = s.n_rc;
    o.counts[5] = nb;
  }
}

// Order-preserving pacing filter (scheduler.py:811-823): keep member i iff
// b_rem[i] <= rates[i] * lim.  The inputs are read ONCE (coalesced; they may
// live in mapped host memory) into shared memory, then warp 0 compacts the
// kept ids in order with ballots.
__global__ void iteration_kernel(const int32_t* ids, const long long* brem, const double* rates, int n, double lim,
                                 int32_t* out, int32_t* n_out) {
  __shared__ uint8_t keep_sh[kMaxN];
  __shared__ int32_t id_sh[kMaxN];
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    keep_sh[i] = ((double)brem[i] <= __dmul_rn(rates[i], lim)) ? 1 : 0;
    id_sh[i] = ids[i];
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    int base = 0;
    for (int c = 0; c < n; c += 32) {
      const int i = c + lane;
      const bool k = i < n && keep_sh[i];
      const unsigned bal = __ballot_sync(0xffffffffu, k);
      if (k) out[base + __popc(bal & ((1u << lane) - 1))] = id_sh[i];
      base += __popc(bal);
    }
    if (lane == 0) *n_out = base;
  }
}

__global__ void __launch_bounds__(kSelThreads) select_kernel(const tf_prio* v, int n, double gpu_mem, int max_batch,
                                                              uint8_t* chosen) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>(smem_raw);
  __shared__ long long lens[kMaxN];
  __shared__ double rates[kMaxN];
  __shared__ int32_t ids[kMaxN];
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    s.phi[i] = v[i].phi;
    s.vt[i] = __dmul_rn(v[i].value, v[i].t_prime);
    s.util[i] = v[i].utility;
    lens[i] = v[i].length;
    rates[i] = v[i].rate;
    ids[i] = v[i].request_id;
    s.cand[i] = (int16_t)i;
    s.flag[i] = 0;
  }
  __syncthreads();
  select_batch_dev(s, n, rates, ids, lens, gpu_mem, max_batch);
  for (int i = threadIdx.x; i < n; i += blockDim.x) chosen[i] = (s.flag[i] & 4) ? 1 : 0;
}

// ----------------------------------------------------------- host wrapper
struct Selector {
  char* dev;
  int64_t dev_bytes;
  char* host;
  int64_t host_bytes;
  int32_t max_n, max_w;
  char* host_dev;  // device-visible alias of the pinned host workspace (zero-copy I/O)
};

static std::vector<Selector*> g_sel;

static int64_t align_up(int64_t x) { return (x + 255) & ~(int64_t)255; }

struct Layout {
  int64_t params, members, waiters, rows, globals, counts, preempt, resume_ids, resume_how, admitted, recomputed,
      batch_sizes, batch_ids, tprime_out, tprime_set, member_ids, aux, total;
};

static Layout layout(int32_t max_n, int32_t max_w) {
  Layout L;
  int64_t o = 0;
  auto take = [&](int64_t bytes) {
    int64_t r = o;
    o += align_up(bytes);
    return r;
  };
  L.params = take(sizeof(tf_tick_params));
  L.members = take((int64_t)max_n * sizeof(tf_member));
  L.waiters = take((int64_t)max_w * sizeof(tf_waiter));
  L.rows = take((int64_t)max_n * sizeof(tf_req_row));
  L.globals = take(sizeof(tf_snap_globals));
  L.counts = take(8 * sizeof(int32_t));
  L.preempt = take((int64_t)max_n * 4);
  L.resume_ids = take((int64_t)max_n * 4);
  L.resume_how = take((int64_t)max_n * 4);
  L.admitted = take((int64_t)max_w * 4);
  L.recomputed = take((int64_t)max_n * 4);
  L.batch_sizes = take((int64_t)max_w * 4);
  L.batch_ids = take((int64_t)max_w * 4);
  L.tprime_out = take((int64_t)max_n * 8);
  L.tprime_set = take((int64_t)max_n * 4);
  L.member_ids = take((int64_t)max_n * 4);
  L.aux = take((int64_t)max_n * 24 + 64);
  L.total = o;
  return L;
}

static Selector* get_sel(int64_t h) {
  if (h <= 0 || h > (int64_t)g_sel.size()) return nullptr;
  return g_sel[h - 1];
}


// ------------------------------------------------------------------------
// On-device snapshot builder (tokensim/engine.py:993-1061 restated): one CTA
// compacts the in-service, not generation-complete requests in id order and
// derives their member fields in the reference's float64 operation order
// (this unit is compiled with -fmad=false, so the four-term t_io sum rounds
// exactly like CPython).  Writes params.n_members for the tick kernel.
__device__ __forceinline__ bool st_in_service(int st) { return st >= TF_ST_PREFILL_WAIT && st <= TF_ST_RECOMPUTING; }
__device__ __forceinline__ bool st_pinned(int st) {
  return st == TF_ST_PREFILL_WAIT || st == TF_ST_PREFILLING || st == TF_ST_LOADING || st == TF_ST_RECOMPUTING;
}

__global__ void __launch_bounds__(kSelThreads) snapshot_kernel(const tf_req_row* __restrict__ rows, int n_rows,
                                                               const tf_snap_globals* __restrict__ g,
                                                               tf_tick_params* p, tf_member* mem, int32_t* ids,
                                                               int32_t* counts) {
  __shared__ int warp_tot[kSelThreads / 32];
  __shared__ int base;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  const double d2h_rate = g->d2h_rate, h2d_rate = g->h2d_rate, pf = g->prefill_s_per_token;
  const double qd = (double)g->q_d2h_tokens / d2h_rate, qh = (double)g->q_h2d_tokens / h2d_rate;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int off = 0; off < n_rows; off += kSelThreads) {
    const int i = off + threadIdx.x;
    bool take = false;
    if (i < n_rows) {
      const tf_req_row& r = rows[i];
      take = st_in_service(r.status) && !(r.generated >= r.output_len);
    }
    // block-wide exclusive scan of the take flags (keeps id order)
    const unsigned bal = __ballot_sync(0xffffffffu, take);
    const int in_warp = __popc(bal & ((1u << lane) - 1));
    if (lane == 0) warp_tot[warp] = __popc(bal);
    __syncthreads();
    int before = base;
    for (int w = 0; w < warp; ++w) before += warp_tot[w];
    if (take) {
      const tf_req_row& r = rows[i];
      tf_member& m = mem[before + in_warp];
      m.request_id = r.request_id;
      m.prompt_len = r.prompt_len;
      m.output_len = r.output_len;
      m.running = r.status == TF_ST_RUNNING;
      m.pinned = st_pinned(r.status);
      m.has_tprime = r.has_tprime;
      m.generated = r.generated;
      m.consumed = r.consumed;
      m.ctx_tokens = r.total_kv;
      m.gpu_resident = r.gpu_resident;
      m.arrival_time = r.arrival_time;
      m.rate = r.rate;
      m.busy_since_tick = r.busy_since_tick;
      long long tail, load;
      if (r.gpu_resident >= r.total_kv) {
        tail = load = 0;
      } else {
        tail = r.total_kv - r.cpu_synced > 0 ? r.total_kv - r.cpu_synced : 0;
        load = r.total_kv - r.gpu_resident > 0 ? r.total_kv - r.gpu_resident : 0;
      }
      // q_d2h/d2h_rate + tail/d2h_rate + q_h2d/h2d_rate + load/h2d_rate, left to right
      m.t_io = ((qd + (double)tail / d2h_rate) + qh) + (double)load / h2d_rate;
      m.t_recompute = pf * (double)r.total_kv;
      m.last_iter_time = r.last_iter_time;
      m.t_prime = r.t_prime;
      ids[before + in_warp] = r.request_id;
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int w = 0; w < kSelThreads / 32; ++w) base += warp_tot[w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    p->n_members = base;
    counts[7] = base;
  }
}

static int run_tick(int64_t sel, const tf_tick_params* p, const tf_member* members, const tf_waiter* waiting,
                    tf_tick_result* out, void* stream, int fastpath, const tf_req_row* rows = nullptr,
                    int32_t n_rows = 0, const tf_snap_globals* g = nullptr, int32_t* member_ids = nullptr,
                    int32_t* n_members_out = nullptr) {
  Selector* S = get_sel(sel);
  TF_CHECK_ARG(S, "selector: unknown handle");
  TF_CHECK_ARG(p && out && out->counts, "selector: NULL params/result");
  TF_CHECK_ARG(p->n_members >= 0 && p->n_members <= S->max_n, "selector: n_members %d exceeds capacity %d",
               p->n_members, S->max_n);
  TF_CHECK_ARG(p->n_waiting >= 0 && p->n_waiting <= S->max_w, "selector: n_waiting %d exceeds capacity %d",
               p->n_waiting, S->max_w);
  TF_CHECK_ARG(p->per_request_mem_estimate > 0, "per_request_estimate must be > 0");
  TF_CHECK_ARG(p->gpu_mem_total + p->cpu_mem_total >= p->per_request_mem_estimate,
               "total_mem must cover at least one request");
  int n = p->n_members;
  const int w = p->n_waiting;
  Layout L = layout(S->max_n, S->max_w);
  cudaStream_t st = (cudaStream_t)stream;
  // stage inputs in the pinned host workspace, one H2D copy
  memcpy(S->host + L.params, p, sizeof(*p));
  if (rows) {
    TF_CHECK_ARG(n_rows >= 0 && n_rows <= S->max_n, "selector: n_rows %d exceeds capacity %d", n_rows, S->max_n);
    TF_CHECK_ARG(g && member_ids && n_members_out, "selector: NULL rows-path argument");
    if (n_rows) memcpy(S->host + L.rows, rows, (size_t)n_rows * sizeof(tf_req_row));
    memcpy(S->host + L.globals, g, sizeof(*g));
  } else if (n) {
    memcpy(S->host + L.members, members, (size_t)n * sizeof(tf_member));
  }
  if (w) memcpy(S->host + L.waiters, waiting, (size_t)w * sizeof(tf_waiter));
  TF_CUDA(cudaMemcpyAsync(S->dev, S->host, L.counts, cudaMemcpyHostToDevice, st));
  if (rows) {
    snapshot_kernel<<<1, kSelThreads, 0, st>>>((const tf_req_row*)(S->dev + L.rows), n_rows,
                                               (const tf_snap_globals*)(S->dev + L.globals),
                                               (tf_tick_params*)(S->dev + L.params), (tf_member*)(S->dev + L.members),
                                               (int32_t*)(S->dev + L.member_ids), (int32_t*)(S->dev + L.counts));
    TF_LAUNCH_CHECK();
  }
  TickArgs a;
  a.p = (const tf_tick_params*)(S->dev + L.params);
  a.mem = (const tf_member*)(S->dev + L.members);
  a.wait = (const tf_waiter*)(S->dev + L.waiters);
  a.o.counts = (int32_t*)(S->dev + L.counts);
  a.o.preempt = (int32_t*)(S->dev + L.preempt);
  a.o.resume_ids = (int32_t*)(S->dev + L.resume_ids);
  a.o.resume_how = (int32_t*)(S->dev + L.resume_how);
  a.o.admitted = (int32_t*)(S->dev + L.admitted);
  a.o.recomputed = (int32_t*)(S->dev + L.recomputed);
  a.o.batch_sizes = (int32_t*)(S->dev + L.batch_sizes);
  a.o.batch_ids = (int32_t*)(S->dev + L.batch_ids);
  a.o.tprime_out = (double*)(S->dev + L.tprime_out);
  a.o.tprime_set = (int32_t*)(S->dev + L.tprime_set);
  a.fastpath = fastpath;
  tick_kernel<<<1, kSelThreads, sizeof(Smem), st>>>(a);
  TF_LAUNCH_CHECK();
  TF_CUDA(cudaMemcpyAsync(S->host + L.counts, S->dev + L.counts, L.aux - L.counts, cudaMemcpyDeviceToHost, st));
  TF_CUDA(cudaStreamSynchronize(st));
  const int32_t* c = (const int32_t*)(S->host + L.counts);
  memcpy(out->counts, c, 6 * sizeof(int32_t));
  if (rows) {
    n = c[7];
    *n_members_out = n;
    memcpy(member_ids, S->host + L.member_ids, (size_t)n * 4);
  }
  auto cp = [&](void* dst, int64_t off, int64_t bytes) {
    if (dst && bytes > 0) memcpy(dst, S->host + off, (size_t)bytes);
  };
  cp(out->preempt, L.preempt, (int64_t)c[1] * 4);
  cp(out->resume_ids, L.resume_ids, (int64_t)c[2] * 4);
  cp(out->resume_how, L.resume_how, (int64_t)c[2] * 4);
  cp(out->admitted, L.admitted, (int64_t)c[3] * 4);
  cp(out->recomputed, L.recomputed, (int64_t)c[4] * 4);
  int nb = c[5], nid = 0;
  cp(out->batch_sizes, L.batch_sizes, (int64_t)nb * 4);
  for (int k = 0; k < nb; ++k) nid += ((const int32_t*)(S->host + L.batch_sizes))[k];
  cp(out->batch_ids, L.batch_ids, (int64_t)nid * 4);
  if (!fastpath) {
    cp(out->t_prime_out, L.tprime_out, (int64_t)n * 8);
    cp(out->t_prime_set, L.tprime_set, (int64_t)n * 4);
  }
  return TF_OK;
}

}  // namespace tf

using namespace tf;

extern "C" {

double tf_host_glibc_exp(double x) { return tf_glibc_exp(x); }

int64_t tf_selector_workspace_bytes(int32_t max_members, int32_t max_waiting) {
  return layout(max_members, max_waiting).total;
}

int tf_selector_init(void* dev_ws, int64_t dev_bytes, void* host_pinned_ws, int64_t host_bytes, int32_t max_members,
                     int32_t max_waiting, int64_t* out_handle) {
  TF_CHECK_ARG(out_handle, "tf_selector_init: out_handle NULL");
  TF_CHECK_ARG(max_members > 0 && max_members <= kMaxN, "tf_selector_init: max_members must be in [1, %d]", kMaxN);
  TF_CHECK_ARG(max_waiting > 0 && max_waiting <= kMaxW, "tf_selector_init: max_waiting must be in [1, %d]", kMaxW);
  const int64_t need = layout(max_members, max_waiting).total;
  TF_CHECK_ARG(dev_ws && dev_bytes >= need, "tf_selector_init: device workspace too small");
  TF_CHECK_ARG(host_pinned_ws && host_bytes >= need, "tf_selector_init: host workspace too small");
  static bool attr_set = false;
  if (!attr_set) {
    TF_CUDA(cudaFuncSetAttribute(tick_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem)));
    TF_CUDA(cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem)));
    attr_set = true;
  }
  void* hdev = nullptr;
  if (cudaHostGetDevicePointer(&hdev, host_pinned_ws, 0) != cudaSuccess) {
    cudaGetLastError();
    set_error("tf_selector_init: the host workspace is not pinned / mapped host memory");
    return TF_EINVAL;
  }
  Selector* S = new Selector{(char*)dev_ws, dev_bytes, (char*)host_pinned_ws, host_bytes, max_members, max_waiting,
                             (char*)hdev};
  g_sel.push_back(S);
  *out_handle = (int64_t)g_sel.size();
  return TF_OK;
}

int tf_selector_destroy(int64_t sel) {
  Selector* S = get_sel(sel);
  TF_CHECK_ARG(S, "tf_selector_destroy: unknown handle");
  delete S;
  g_sel[sel - 1] = nullptr;
  return TF_OK;
}

int tf_policy_tick(int64_t sel, const tf_tick_params* p, const tf_member* members, const tf_waiter* waiting,
                   tf_tick_result* out, void* stream) {
  return run_tick(sel, p, members, waiting, out, stream, 0);
}

int tf_policy_tick_rows(int64_t sel, const tf_tick_params* p, const tf_req_row* rows, int32_t n_rows,
                        const tf_snap_globals* g, const tf_waiter* waiting, tf_tick_result* out, int32_t* member_ids,
                        int32_t* n_members, void* stream) {
  TF_CHECK_ARG(n_rows == 0 || rows, "tf_policy_tick_rows: NULL rows");
  static const tf_req_row kNone{};
  return run_tick(sel, p, nullptr, waiting, out, stream, 0, rows ? rows : &kNone, n_rows, g, member_ids, n_members);
}

int tf_policy_fastpath(int64_t sel, const tf_tick_params* p, const tf_member* members, const tf_waiter* waiting,
                       tf_tick_result* out, void* stream) {
  return run_tick(sel, p, members, waiting, out, stream, 1);
}

int tf_iteration_batch(int64_t sel, const int32_t* ids, const int64_t* b_rem, const double* rates, int32_t n,
                       int32_t contention, int32_t mode, double pacing_buffer_seconds, int32_t* out_ids,
                       int32_t* n_out, void* stream) {
  Selector* S = get_sel(sel);
  TF_CHECK_ARG(S, "tf_iteration_batch: unknown handle");
  TF_CHECK_ARG(n >= 0 && n <= S->max_n, "tf_iteration_batch: n out of range");
  TF_CHECK_ARG(n_out && (n == 0 || (ids && b_rem && rates && out_ids)), "tf_iteration_batch: NULL pointer");
  if (!contention || mode == 1) {  // work-conserving: everyone decodes (scheduler.py:820-821)
    for (int i = 0; i < n; ++i) out_ids[i] = ids[i];
    *n_out = n;
    return TF_OK;
  }
  if (n == 0) {
    *n_out = 0;
    return TF_OK;
  }
  Layout L = layout(S->max_n, S->max_w);
  cudaStream_t st = (cudaStream_t)stream;
  // Zero-copy: the kernel reads the (ids, b_rem, rates) rows straight out of
  // the pinned host workspace and writes its result back there - this call
  // sits between every decode step's completion and the next dispatch, and
  // three copy-engine transfers (each a DMA setup, possibly queued behind KV
  // swaps) cost several times the kernel itself
  char* h = S->host + L.members;
  char* hd = S->host_dev + L.members;
  memcpy(h, ids, (size_t)n * 4);
  memcpy(h + 4 * S->max_n, b_rem, (size_t)n * 8);
  memcpy(h + 12 * S->max_n, rates, (size_t)n * 8);
  int32_t* dout = (int32_t*)(S->host_dev + L.preempt);
  int32_t* dn = (int32_t*)(S->host_dev + L.counts);
  iteration_kernel<<<1, 256, 0, st>>>((const int32_t*)hd, (const long long*)(hd + 4 * S->max_n),
                                      (const double*)(hd + 12 * S->max_n), n, pacing_buffer_seconds, dout, dn);
  TF_LAUNCH_CHECK();
  TF_CUDA(cudaStreamSynchronize(st));
  *n_out = *(int32_t*)(S->host + L.counts);
  memcpy(out_ids, S->host + L.preempt, (size_t)(*n_out) * 4);
  return TF_OK;
}

int tf_select_batch(int64_t sel, const tf_prio* views, int32_t n, double gpu_mem, int32_t max_batch,
                    uint8_t* out_chosen, void* stream) {
  Selector* S = get_sel(sel);
  TF_CHECK_ARG(S, "tf_select_batch: unknown handle");
  TF_CHECK_ARG(max_batch >= 0 && gpu_mem >= 0, "budgets must be non-negative");
  TF_CHECK_ARG(n >= 0 && n <= S->max_n, "tf_select_batch: n out of range");
  if (n == 0) return TF_OK;
  TF_CHECK_ARG(views && out_chosen, "tf_select_batch: NULL pointer");
  Layout L = layout(S->max_n, S->max_w);
  cudaStream_t st = (cudaStream_t)stream;
  static_assert(sizeof(tf_prio) <= sizeof(tf_member), "tf_prio must fit the member slots");
  memcpy(S->host + L.members, views, (size_t)n * sizeof(tf_prio));
  TF_CUDA(cudaMemcpyAsync(S->dev + L.members, S->host + L.members, (size_t)n * sizeof(tf_prio), cudaMemcpyHostToDevice,
                          st));
  uint8_t* dch = (uint8_t*)(S->dev + L.aux);
  select_kernel<<<1, kSelThreads, sizeof(Smem), st>>>((const tf_prio*)(S->dev + L.members), n, gpu_mem, max_batch,
                                                      dch);
  TF_LAUNCH_CHECK();
  TF_CUDA(cudaMemcpyAsync(S->host + L.aux, dch, n, cudaMemcpyDeviceToHost, st));
  TF_CUDA(cudaStreamSynchronize(st));
  memcpy(out_chosen, S->host + L.aux, n);
  return TF_OK;
}

}  // extern "C"
