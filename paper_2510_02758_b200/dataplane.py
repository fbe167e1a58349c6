"""GPU data plane: paged KV block manager + swap engine + decode step.

Owns the KV pool in HBM, the pinned host store, the device-resident block
tables and the copy streams, and turns every token-count transition of the
engine (engine.py here, tokensim/engine.py in the reference) into real work
through the C ABI (_tf_b200.so):

  transition (reference)                        GPU work
  prefill dispatch        engine.py:669-692     block alloc + KV write
  decode dispatch         engine.py:693-708     block alloc + KV append + paged attention
  write-through / evict   engine.py:781-848     tf_kv_gather_d2h on the evict stream
  load                    engine.py:850-888     tf_kv_scatter_h2d on the load stream
  preempt instant release kvstore.py:144-154    block frees
  recompute / done        engine.py:542-557, :889-917  block frees

Token-range semantics (which positions each count refers to) are the
canonical ones written down in DESIGN.md and restated independently by
oracle/dataplane.py; block tables and bytes must match it bit for bit.

Pool layout (block-major): block[b] = [layer][K|V][kv_head][slot][head_dim]
bf16, identical in HBM and in the pinned host store, so a full block of all
layers moves as one contiguous 2 MiB run (Llama3-8B).

Modes
  replay    one CUDA stream for everything: program order is stream order,
            so every hazard (free-then-reuse, load-after-evict) is ordered
            by construction; used for bit-exact parity runs.
  realtime  compute / evict (d2h) / load (h2d) streams overlapped; block
            frees are fenced by CUDA events before reuse, loads of a range
            wait on the eviction that produced it.
"""
from __future__ import annotations

import ctypes as C
from collections import deque

import os

import numpy as np
import torch

from . import _lib
from ._lib import TIER_GPU, TIER_HOST, TfSeg, TfSpan, check, lib

LIVE, DETACHED, RESERVED, HOSTV = np.uint8(1), np.uint8(2), np.uint8(4), np.uint8(8)
_GROW_BATCH = os.environ.get("TF_GROW_BATCH", "1") != "0"  # A/B switch for the batched decode-growth allocation
CLR_LIVE, CLR_DETACHED, CLR_RESERVED, CLR_HOSTV = np.uint8(0xFE), np.uint8(0xFD), np.uint8(0xFB), np.uint8(0xF7)


def _i32(a) -> C.Array:
    a = np.ascontiguousarray(a, dtype=np.int32)
    return (C.c_int32 * max(1, a.size)).from_buffer_copy(a.tobytes() if a.size else b"\0\0\0\0")


class KvPool:
    """HBM pool + pinned host store + C-ABI pool handle."""

    def __init__(self, n_blocks, n_host_blocks, n_layers, kv_heads, head_dim, block_tokens=16, device="cuda"):
        self.n_blocks, self.n_host_blocks = n_blocks, n_host_blocks
        self.L, self.H, self.D, self.B = n_layers, kv_heads, head_dim, block_tokens
        self.block_elems = n_layers * 2 * kv_heads * block_tokens * head_dim
        self.device = torch.device(device)
        self.gpu = torch.empty(n_blocks * self.block_elems, dtype=torch.int16, device=self.device)
        self.host = torch.empty(max(1, n_host_blocks) * self.block_elems, dtype=torch.int16, pin_memory=True)
        h = C.c_int64()
        check(lib.tf_pool_init(C.c_void_p(self.gpu.data_ptr()), n_blocks, C.c_void_p(self.host.data_ptr()),
                               n_host_blocks, n_layers, block_tokens, kv_heads, head_dim, 0, C.byref(h)),
              "tf_pool_init")
        self.handle = h.value

    @property
    def block_bytes(self) -> int:
        return self.block_elems * 2

    def alloc(self, tier: int, n: int) -> list:
        if n == 0:
            return []
        out = (C.c_int32 * n)()
        check(lib.tf_blocks_alloc(self.handle, tier, n, out), "tf_blocks_alloc")
        return list(out)

    def free(self, tier: int, ids) -> None:
        ids = list(ids)
        if ids:
            check(lib.tf_blocks_free(self.handle, tier, _i32(ids), len(ids)), "tf_blocks_free")

    def free_count(self, tier: int) -> int:
        return lib.tf_blocks_free_count(self.handle, tier)

    def gpu_view(self) -> torch.Tensor:
        """[n_blocks, L, 2, H, B, D] int16 view of the HBM pool (bf16 bits)."""
        return self.gpu.view(self.n_blocks, self.L, 2, self.H, self.B, self.D)

    def host_view(self) -> torch.Tensor:
        return self.host[: self.n_host_blocks * self.block_elems].view(self.n_host_blocks, self.L, 2, self.H, self.B,
                                                                        self.D)

    def close(self):
        if self.handle:
            lib.tf_pool_destroy(self.handle)
            self.handle = 0


class GpuDataPlane:
    """Engine hooks -> block manager bookkeeping + kernel launches."""

    def __init__(self, reqs, pool: KvPool, mode: str = "replay", kv_source: str = "synthetic", seed: int = 0,
                 attention: str = "all", engine: int = _lib.ENGINE_SM, model=None, n_q_heads: int | None = None):
        assert mode in ("replay", "realtime")
        self.pool, self.mode, self.kv_source, self.seed = pool, mode, kv_source, seed
        self.attention = attention  # "all" layers, "none", or an int layer count
        self.swap_engine = engine
        self.model = model
        self.n_q_heads = n_q_heads or 2 * pool.H
        self.B = pool.B
        dev = pool.device
        self.max_len = max(r.prompt_len + r.output_len + 2 for r in reqs)
        self.nlb = (self.max_len + self.B - 1) // self.B
        n_rows = max(r.id for r in reqs) + 1
        # one row per request id (rows are per-request views: flags[rid], gtab[rid]);
        # 2-D so a decode step's per-member updates are single vectorised ops
        n_ids = max(r.id for r in reqs) + 1
        self.flags = np.zeros((n_ids, self.nlb * self.B), np.uint8)
        self.gtab = np.full((n_ids, self.nlb), -1, np.int32)
        self.htab = np.full((n_ids, self.nlb), -1, np.int32)
        self.host_hi = {r.id: 0 for r in reqs}
        # one extra row: padding rows of graph-captured decode steps point there
        self.table = torch.full((n_rows + 1, self.nlb), -1, dtype=torch.int32, device=dev)
        self.scratch_row = n_rows
        self.scratch_block = None
        # fused write-through (realtime): device host-block table read by the
        # decode epilogue; HOSTV flags mark positions mirrored on the host
        self.fused_wt = False
        self.htable = None
        self._pending_htable = []
        if mode == "replay":
            self.s_compute = self.s_evict = self.s_load = torch.cuda.Stream(device=dev)
        else:
            self.s_compute = torch.cuda.Stream(device=dev)
            # copy streams at high priority: the SM swap kernel (partial-block
            # edges of the auto engine) gets SMs as soon as running compute CTAs
            # retire, instead of queueing behind a whole prefill / decode step -
            # otherwise a load's measured rate collapses to the prefill's
            # duration and the policy's t_io estimate (kvstore.py:173-193)
            # tips every restore towards recompute
            self.s_evict = torch.cuda.Stream(device=dev, priority=-1)
            self.s_load = torch.cuda.Stream(device=dev, priority=-1)
        self._pending_table = []  # (row, lb, block) not yet applied on device
        self._appending = {}  # rid -> position reserved by the in-flight decode step
        self._d2h_busy = None  # (rid, lo, hi, kind, event)
        self._last_d2h_event = {}  # rid -> event of its last d2h (loads of that range wait on it)
        self._quarantine: deque = deque()  # (event, [blocks]) realtime frees awaiting their fence
        self._q_blocks = 0  # blocks held in the quarantine
        self.peak_blocks = 0
        self.peak_host_blocks = 0
        self.stats = {"d2h_tokens": 0, "h2d_tokens": 0, "d2h_launches": 0, "h2d_launches": 0, "append_tokens": 0,
                      "fill_tokens": 0, "attn_launches": 0, "decode_steps": 0}
        self._events = []  # (kind, tokens, start_evt, end_evt) for measured transfer rates
        self._seglog = []  # per entry of _events: the chunk's (slot_begin, n_slots) segments (probe replays)
        ws = max(1, int(lib.tf_paged_decode_attn_workspace(pool.handle, max(1, len(reqs)), self.max_len, 64)))
        self._attn_ws = torch.zeros(ws, dtype=torch.uint8, device=dev)
        self.attn_out = None
        # the tables / workspace above were filled on the default stream; the
        # compute / copy streams are non-blocking, so order them explicitly
        torch.cuda.synchronize(dev)

    def enable_fused_write_through(self):
        """Mirror every decoded token to the host inside the decode step
         instead of in separate write-through chunks."""
        if self.mode != "realtime":
            raise ValueError("fused write-through changes the token-count semantics; realtime mode only")
        self.fused_wt = True
        self.htable = torch.full_like(self.table, -1)
        torch.cuda.synchronize(self.pool.device)  # filled on the default stream, read on s_compute

    def enable_scratch(self):
        """Reserve one block for the padding rows of captured decode graphs."""
        if self.scratch_block is None:
            self.scratch_block = self._alloc_blocks(1)[0]
            self.table[self.scratch_row].fill_(self.scratch_block)
            torch.cuda.synchronize()
        return self.scratch_block

    # ------------------------------------------------------------ block table
    def _reconcile(self, rid, blocks):
        f, tab = self.flags[rid], self.gtab[rid]
        blocks = np.unique(np.fromiter(blocks, dtype=np.int64) if not isinstance(blocks, np.ndarray)
                           else blocks.astype(np.int64, copy=False))
        if blocks.size:
            # HBM occupancy = LIVE | DETACHED | RESERVED (HOSTV only marks the host mirror)
            occ = (f.reshape(-1, self.B)[blocks] & 7).any(axis=1)
            mapped = tab[blocks] >= 0
            fr = blocks[~occ & mapped]  # ascending: frees first (LIFO push) ...
            if fr.size:
                freed = tab[fr].tolist()
                tab[fr] = -1
                self._pending_table.extend((rid, j, -1) for j in fr.tolist())
                self._release_blocks(freed)
            need = blocks[occ & ~mapped]  # ... then allocations (pop), ascending
            if need.size:
                ids = self._alloc_blocks(len(need))
                tab[need] = ids
                self._pending_table.extend(zip([rid] * len(ids), need.tolist(), ids))
        used = self.pool.n_blocks - self.pool.free_count(TIER_GPU) - self._q_blocks
        self.peak_blocks = max(self.peak_blocks, used)

    def _release_blocks(self, ids):
        if self.mode == "replay":
            self.pool.free(TIER_GPU, ids)
        else:
            # reusable once every stream has passed its current work
            evs = []
            for s in (self.s_compute, self.s_evict, self.s_load):
                ev = torch.cuda.Event()
                ev.record(s)
                evs.append(ev)
            self._quarantine.append((evs, ids))
            self._q_blocks += len(ids)

    def _alloc_blocks(self, n):
        if self.mode == "realtime":
            while self._quarantine and all(e.query() for e in self._quarantine[0][0]):
                ids = self._quarantine.popleft()[1]
                self._q_blocks -= len(ids)
                self.pool.free(TIER_GPU, ids)
            while self._quarantine and self.pool.free_count(TIER_GPU) < n:
                evs, ids = self._quarantine.popleft()
                self._q_blocks -= len(ids)
                for e in evs:
                    e.synchronize()
                self.pool.free(TIER_GPU, ids)
        return self.pool.alloc(TIER_GPU, n)

    def _flush_table(self, stream):
        if not self._pending_table:
            return
        # last write per (row, lb) wins: the kernel applies triples in parallel
        last = {}
        for row, lb, blk in self._pending_table:
            last[(row, lb)] = blk
        self._pending_table = []
        t = np.asarray([(r, j, b) for (r, j), b in last.items()], np.int32).reshape(-1)
        check(lib.tf_table_apply(C.c_void_p(self.table.data_ptr()), self.nlb, _i32(t), len(t) // 3,
                                 C.c_void_p(stream.cuda_stream)), "tf_table_apply")

    def _segments(self, rid, positions, host=True):
        """Group sorted positions into per-block slot runs -> TfSeg array."""
        segs = []
        if len(positions) == 0:
            return segs
        p = np.asarray(positions)
        br = np.nonzero(np.diff(p) != 1)[0] + 1
        for run in np.split(p, br):
            lo, hi = int(run[0]), int(run[-1]) + 1
            while lo < hi:
                j = lo // self.B
                e = min(hi, (j + 1) * self.B)
                segs.append((int(self.gtab[rid][j]), int(self.htab[rid][j]) if host else -1, lo - j * self.B, e - lo))
                lo = e
        return segs

    @staticmethod
    def _seg_array(segs):
        arr = (TfSeg * max(1, len(segs)))()
        for i, (g, h, s, n) in enumerate(segs):
            arr[i].gpu_block, arr[i].host_block, arr[i].slot_begin, arr[i].n_slots = g, h, s, n
        return arr

    # ------------------------------------------------------------ KV writes
    def _write_kv(self, spans, stream):
        """spans: (rid, lo, hi) positions whose KV is produced now."""
        if not spans:
            return
        self._flush_table(stream)
        if self.kv_source == "synthetic":
            stream = self.s_compute
            arr = (TfSpan * len(spans))()
            for i, (rid, lo, hi) in enumerate(spans):
                arr[i].row, arr[i].rid, arr[i].pos_begin, arr[i].pos_end = rid, rid, lo, hi
            check(lib.tf_kv_fill_synthetic(self.pool.handle, C.c_void_p(self.table.data_ptr()), self.nlb, arr,
                                           len(spans), self.seed, C.c_void_p(stream.cuda_stream)),
                  "tf_kv_fill_synthetic")

    # ------------------------------------------------------------ engine hooks
    def fill_start(self, job, eng):
        spans = []
        for rid in job.members:
            tot = eng.state[rid].kv.total_kv
            lo = 0 if job.kind == "recompute" else tot
            hi = lo + job.reserve[rid]
            f = self.flags[rid]
            if (f[lo:hi] & (LIVE | RESERVED)).any():
                raise _lib.InvariantError(f"prefill of {rid} overlaps resident KV")
            f[lo:hi] |= RESERVED
            self._reconcile(rid, range(lo // self.B, (hi - 1) // self.B + 1))
            if self.fused_wt:
                htab = self.htab[rid]
                for j in range(lo // self.B, (hi - 1) // self.B + 1):
                    if htab[j] < 0:
                        htab[j] = self.pool.alloc(TIER_HOST, 1)[0]
                        self._pending_htable.append((rid, j, int(htab[j])))
            spans.append((rid, lo, hi))
            self.stats["fill_tokens"] += hi - lo
        self._wait_d2h_of(spans, self.s_compute)
        if self.model is not None and self.kv_source == "model":
            self._flush_table(self.s_compute)
            if self.fused_wt:
                self._flush_htable(self.s_compute)
            self.model.prefill(self, job, spans, eng)
        else:
            self._write_kv(spans, self.s_compute)

    def fill_done(self, rid):
        f = self.flags[rid]
        m = (f & RESERVED) != 0
        if self.fused_wt:
            idx = np.nonzero(m)[0]
            f[m] = (f[m] & CLR_RESERVED) | LIVE | HOSTV
            if len(idx):
                self.host_hi[rid] = max(self.host_hi[rid], int(idx[-1]) + 1)
        else:
            f[m] = (f[m] & CLR_RESERVED) | LIVE
        if self.model is not None and self.kv_source == "model":
            self.model.fill_commit(rid)

    def decode_start(self, batch, eng):
        n = len(batch)
        rids = np.fromiter(batch, np.int64, n)
        pos = np.fromiter((eng.state[r].kv.total_kv for r in batch), np.int64, n)
        if eng.debug_checks:
            for rid, p in zip(batch, pos.tolist()):
                if not (self.flags[rid][:p] & LIVE).all():
                    raise _lib.InvariantError(f"decode of {rid} reads non-resident KV")
        self.flags[rids, pos] |= RESERVED
        self._appending.update(zip(batch, pos.tolist()))
        j = pos // self.B
        # a member whose new position opens an unmapped logical block gets a
        # fresh block: one allocator call for all of them, handed out in batch
        # order - exactly the blocks per-member reconciles would pop from the
        # LIFO stack (nothing is freed here: the block was unmapped), at a
        # fraction of the host time (every 16th step all B members grow)
        grow = self.gtab[rids, j] < 0
        if grow.any() and not _GROW_BATCH:
            for rid, jj in zip(rids[grow].tolist(), j[grow].tolist()):
                self._reconcile(rid, [jj])
        elif grow.any():
            r_g, j_g = rids[grow], j[grow]
            ids = self._alloc_blocks(int(grow.sum()))
            self.gtab[r_g, j_g] = ids
            self._pending_table.extend(zip(r_g.tolist(), j_g.tolist(), ids))
            used = self.pool.n_blocks - self.pool.free_count(TIER_GPU) - self._q_blocks
            self.peak_blocks = max(self.peak_blocks, used)
        if self.fused_wt:
            for rid, jj in zip(batch, j.tolist()):
                if self.htab[rid][jj] < 0:
                    self.htab[rid][jj] = self.pool.alloc(TIER_HOST, 1)[0]
                    self._pending_htable.append((rid, jj, int(self.htab[rid][jj])))
        self.stats["append_tokens"] += len(batch)
        self.stats["decode_steps"] += 1
        busy = self._d2h_busy
        if self.mode == "realtime" and busy is not None and busy[0] in batch:
            self.s_compute.wait_event(busy[4])
        if self.model is not None and self.kv_source == "model":
            self._flush_table(self.s_compute)
            if self.fused_wt:
                self._flush_htable(self.s_compute)
            self.model.decode(self, batch, eng)
        else:
            self._write_kv([(rid, p, p + 1) for rid, p in zip(batch, pos.tolist())], self.s_compute)
            self._synthetic_attention(batch, eng)

    def decode_done(self, batch, made):
        made = set(made)
        if self.model is not None and self.kv_source == "model":
            self.model.decode_commit(made)
        n = len(batch)
        rids = np.fromiter(batch, np.int64, n)
        pos = np.fromiter((self._appending.pop(r) for r in batch), np.int64, n)  # the slot each reserved
        ok = np.fromiter((r in made for r in batch), bool, n)
        F = self.flags
        if ok.any():
            r1, p1 = rids[ok], pos[ok]
            if self.fused_wt:
                F[r1, p1] |= HOSTV  # mirrored to the host by the fused epilogue
                for rid, p in zip(r1.tolist(), p1.tolist()):
                    self.host_hi[rid] = max(self.host_hi[rid], p + 1)
            F[r1, p1] = (F[r1, p1] & CLR_RESERVED) | LIVE
        if not ok.all():
            r0, p0 = rids[~ok], pos[~ok]
            F[r0, p0] &= CLR_RESERVED
            for rid, p in zip(r0.tolist(), p0.tolist()):
                self._reconcile(rid, (p // self.B,))

    def d2h_start(self, ch, eng):
        rid = ch.owner
        cs = eng.state[rid].kv.cpu_synced
        lo, hi = cs, cs + ch.tokens
        f = self.flags[rid]
        if not (f[lo:hi] & LIVE).all():
            raise _lib.InvariantError(f"d2h of {rid} [{lo},{hi}) reads non-resident KV")
        htab = self.htab[rid]
        need = [j for j in range(lo // self.B, (hi - 1) // self.B + 1) if htab[j] < 0]
        for j, b in zip(need, self.pool.alloc(TIER_HOST, len(need))):
            htab[j] = b
        self.peak_host_blocks = max(self.peak_host_blocks, self.pool.n_host_blocks - self.pool.free_count(TIER_HOST))
        self.host_hi[rid] = max(self.host_hi[rid], hi)
        segs = self._segments(rid, np.arange(lo, hi))
        # realtime: [cs, cs+n) was appended by decode steps whose completion the
        # engine already observed, so the gather needs no wait on the compute stream
        st = self.s_evict
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(st)
        check(lib.tf_kv_gather_d2h(self.pool.handle, self._seg_array(segs), len(segs), 0, self.pool.L,
                                   self.swap_engine, C.c_void_p(st.cuda_stream)), "tf_kv_gather_d2h")
        t1.record(st)
        self._events.append(("d2h", ch.tokens, t0, t1))
        self._seglog.append([(s0, n) for _, _, s0, n in segs])
        if ch.kind == "evict":
            f[lo:hi] = (f[lo:hi] & CLR_LIVE) | DETACHED
        self._d2h_busy = (rid, lo, hi, ch.kind, t1)
        self._last_d2h_event[rid] = t1
        self.stats["d2h_tokens"] += ch.tokens
        self.stats["d2h_launches"] += 1
        return t0, t1

    def d2h_done(self, ch, alive):
        rid, lo, hi, kind, ev = self._d2h_busy
        self._d2h_busy = None
        if self.fused_wt and alive:
            self.flags[rid][lo:hi] |= HOSTV
        if kind == "evict":
            self.flags[rid][lo:hi] &= CLR_DETACHED
            if self.mode == "realtime":
                ev.synchronize()
            self._reconcile(rid, range(lo // self.B, (hi - 1) // self.B + 1))

    def h2d_start(self, ch, eng):
        rid = ch.owner
        tot = eng.state[rid].kv.total_kv
        f = self.flags[rid]
        miss = np.nonzero((f[:tot] & LIVE) == 0)[0][: ch.tokens]
        if len(miss) != ch.tokens or (len(miss) and miss[-1] >= self.host_hi[rid]):
            raise _lib.InvariantError(f"load of {rid} needs positions missing from the host store")
        f[miss] |= LIVE
        self._reconcile(rid, miss // self.B)
        st = self.s_load
        ev = self._last_d2h_event.get(rid)
        if self.mode == "realtime" and ev is not None:
            st.wait_event(ev)
        segs = self._segments(rid, miss)
        if self.swap_engine == _lib.ENGINE_CE:
            segs = self._widen_loads(rid, segs, miss)
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(st)
        check(lib.tf_kv_scatter_h2d(self.pool.handle, self._seg_array(segs), len(segs), 0, self.pool.L,
                                    self.swap_engine, C.c_void_p(st.cuda_stream)), "tf_kv_scatter_h2d")
        t1.record(st)
        self._events.append(("h2d", ch.tokens, t0, t1))
        self._seglog.append([(s0, n) for _, _, s0, n in segs])
        self.stats["h2d_tokens"] += ch.tokens
        self.stats["h2d_launches"] += 1
        # realtime: the request turns RUNNING only after the engine observed
        # every load chunk complete, so decode needs no wait on this stream
        return t0, t1

    def _widen_loads(self, rid, segs, miss):
        """(1-D copy-engine mode only) A partial-block load whose block holds
        nothing else (no other slot LIVE / RESERVED / DETACHED) is issued as
        the whole block: one contiguous run instead of 2*kv_heads*layers short
        runs.  The default engine moves a partial block as one 2-D copy.  The extra slots carry host bytes no one reads (they
        lie beyond the request's context, or are refilled before use)."""
        f, tab = self.flags[rid], self.gtab[rid]
        loading = np.zeros(len(f), bool)
        loading[miss] = True
        out = []
        for g, h, s0, n in segs:
            if n < self.B:
                j = int(np.nonzero(tab == g)[0][0])
                lo, hi = j * self.B, (j + 1) * self.B
                others = (f[lo:hi] & (LIVE | RESERVED | DETACHED)).astype(bool) & ~loading[lo:hi]
                if not others.any():
                    s0, n = 0, self.B
            out.append((g, h, s0, n))
        return out

    def release_prefix(self, rid, n):
        f = self.flags[rid]
        idx = np.nonzero(f & LIVE)[0][:n]
        if len(idx) != n:
            raise _lib.InvariantError(f"instant release of {n} tokens but {len(idx)} resident")
        f[idx] &= CLR_LIVE
        self._reconcile(rid, idx // self.B)

    def cancel_evicts(self, rid):
        pass

    def drop_gpu(self, rid):
        f = self.flags[rid]
        idx = np.nonzero(f & LIVE)[0]
        f[idx] &= CLR_LIVE
        self._reconcile(rid, idx // self.B)

    def drop_host(self, rid):
        tab = self.htab[rid]
        ids = [int(b) for b in tab if b >= 0]
        if self.fused_wt:
            for j in np.nonzero(tab >= 0)[0]:
                self._pending_htable.append((rid, int(j), -1))
            self.flags[rid] &= CLR_HOSTV
        tab[:] = -1
        self.pool.free(TIER_HOST, ids)
        self.host_hi[rid] = 0

    def host_frontier(self, rid, cs, total):
        """Fused write-through: the host prefix extends over every position the
        decode epilogue (or a landed chunk) already mirrored."""
        f = self.flags[rid]
        while cs < total and f[cs] & HOSTV:
            cs += 1
        return cs

    def _flush_htable(self, stream):
        if not self._pending_htable:
            return
        last = {}
        for row, lb, blk in self._pending_htable:
            last[(row, lb)] = blk
        self._pending_htable = []
        t = np.asarray([(r, j, b) for (r, j), b in last.items()], np.int32).reshape(-1)
        check(lib.tf_table_apply(C.c_void_p(self.htable.data_ptr()), self.nlb, _i32(t), len(t) // 3,
                                 C.c_void_p(stream.cuda_stream)), "tf_table_apply(host)")

    def finish(self, rid):
        f = self.flags[rid]
        idx = np.nonzero(f)[0]
        f[:] = 0
        self._reconcile(rid, idx // self.B)
        self.drop_host(rid)

    def audit(self, eng):
        for rid, s in eng.state.items():
            if s.status in ("gen_done", "done"):
                continue
            f = self.flags[rid]
            fly = eng.h2d.in_service.tokens if (eng.h2d.in_service is not None and eng.h2d.in_service.owner == rid) else 0
            n = int(np.count_nonzero(f & LIVE)) + int(np.count_nonzero(f & DETACHED))
            if n != s.kv.gpu_resident + fly:
                raise _lib.InvariantError(f"request {rid}: {n} resident positions vs ledger {s.kv.gpu_resident}+{fly}")

    def _wait_d2h_of(self, spans, stream):
        if self.mode != "realtime":
            return
        for rid, _, _ in spans:
            busy = self._d2h_busy
            if busy is not None and busy[0] == rid:
                stream.wait_event(busy[4])

    # ------------------------------------------------------------ attention
    def _synthetic_attention(self, batch, eng):
        """Decode attention over each member's paged KV (synthetic q)."""
        if self.attention == "none" or not batch:
            return
        n_layers = self.pool.L if self.attention == "all" else int(self.attention)
        st = self.s_compute
        B = len(batch)
        pos = [eng.state[r].kv.total_kv for r in batch]
        hq = self.n_q_heads
        scale = 1.0 / float(self.pool.D) ** 0.5
        # every input is uploaded / allocated ON the launching stream: the
        # kernels are stream-ordered after their copies, and the caching
        # allocator only recycles these blocks once st has passed them
        with torch.cuda.stream(st):
            rows = torch.tensor(list(batch), dtype=torch.int32).pin_memory().to(self.pool.device, non_blocking=True)
            ctx = torch.tensor([p + 1 for p in pos], dtype=torch.int32).pin_memory().to(self.pool.device,
                                                                                          non_blocking=True)
            posd = torch.tensor(pos, dtype=torch.int32).pin_memory().to(self.pool.device, non_blocking=True)
            q = torch.empty((B, hq, self.pool.D), dtype=torch.int16, device=self.pool.device)
            out = torch.empty_like(q)
            ws_need = int(lib.tf_paged_decode_attn_workspace(self.pool.handle, B, max(pos) + 1, hq))
            if ws_need > self._attn_ws.numel():
                self._attn_ws = torch.zeros(ws_need, dtype=torch.uint8, device=self.pool.device)
            for layer in range(n_layers):
                check(lib.tf_q_fill_synthetic(C.c_void_p(q.data_ptr()), C.c_void_p(rows.data_ptr()),
                                              C.c_void_p(posd.data_ptr()), B, layer, hq, self.pool.D, self.seed,
                                              C.c_void_p(st.cuda_stream)), "tf_q_fill_synthetic")
                check(lib.tf_paged_decode_attn(self.pool.handle, C.c_void_p(q.data_ptr()),
                                               C.c_void_p(self.table.data_ptr()), self.nlb,
                                               C.c_void_p(rows.data_ptr()), C.c_void_p(ctx.data_ptr()), B,
                                               max(pos) + 1, layer, hq, scale, C.c_void_p(out.data_ptr()),
                                               C.c_void_p(self._attn_ws.data_ptr()), self._attn_ws.numel(),
                                               C.c_void_p(st.cuda_stream)), "tf_paged_decode_attn")
                self.stats["attn_launches"] += 1
        self.attn_out = (list(batch), pos, out)

    # ------------------------------------------------------------ inspection
    def record_event(self):
        """Timing event at the current tail of the compute stream (the
        real-time engine's completion / clock-anchor events)."""
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(self.s_compute)
        return ev

    def synchronize(self):
        for s in {self.s_compute, self.s_evict, self.s_load}:
            s.synchronize()

    def block_table(self, rid):
        return self.gtab[rid].copy()

    def host_table(self, rid):
        return self.htab[rid].copy()

    def device_table(self) -> np.ndarray:
        self.synchronize()
        return self.table.cpu().numpy()

    def transfer_log(self):
        """(direction, tokens, ms) of every launched chunk (synchronises)."""
        self.synchronize()
        return [(k, n, a.elapsed_time(b)) for k, n, a, b in self._events]


def profile_hooks(dp):
    """Debug aid: accumulate the host wall time of every engine hook of ``dp``
    (dp.hook_time[name] = [calls, seconds])."""
    import functools
    import time as _time

    dp.hook_time = {}
    for name in ("fill_start", "fill_done", "decode_start", "decode_done", "d2h_start", "d2h_done", "h2d_start",
                 "release_prefix", "drop_gpu", "drop_host", "finish"):
        fn = getattr(dp, name)

        def wrap(*a, _fn=fn, _name=name, **k):
            t = _time.perf_counter()
            try:
                return _fn(*a, **k)
            finally:
                rec = dp.hook_time.setdefault(_name, [0, 0.0])
                rec[0] += 1
                rec[1] += _time.perf_counter() - t

        setattr(dp, name, functools.wraps(fn)(wrap))
    return dp
