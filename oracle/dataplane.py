"""CPU restatement of the unpinned data plane (TEST ORACLE).

The reference counts KV in tokens and never materialises block tables, bytes
or attention (kvstore.py:35-59).  This module fixes the
token-range meaning of every count transition and
executes it on plain numpy arrays, one flag per token position, so it is
obviously correct rather than fast.  It is driven through the hook calls of
``oracle.refsim.sim.Sim``; the GPU data plane (paper_2510_02758_b200) must
produce bit-identical block tables and pool / host-store bytes.

Canonical semantics:

* positions of request r are 0..total_kv-1; logical block j = p // B.
* a position is LIVE (in the resident copy), DETACHED (being evicted by the
  in-service d2h chunk) or RESERVED (written by an in-flight prefill /
  decode append); LIVE and DETACHED may coexist (reloaded before the old
  eviction landed - the two copies share one slot).
* logical block j of r is mapped to a physical block iff any of its
  positions has a flag.  After each hook the affected blocks are reconciled
  in ascending j: frees first (pushed on a LIFO free stack), then
  allocations (popped).  The stack starts as [N-1, ..., 0] (block 0 first).
* d2h chunk at service start copies [cpu_synced, cpu_synced+n) pool->host
  (engine.py:571-617 lands it; FIFO per channel makes the range a prefix
  extension); an evict chunk additionally moves those positions
  LIVE -> DETACHED and frees them when it lands.
* preemption releases the synced prefix L & [0, cpu_synced)
  (kvstore.py:144-154, engine.py:839-841).
* an h2d load chunk at service start refills the n lowest non-LIVE
  positions of [0, total_kv) from the host store (engine.py:880-888).
* recompute / baseline eviction drop every LIVE position
  (engine.py:827-833, :889-904, :717-731).
* host blocks are allocated at d2h start (ascending j, own LIFO stack) and
  freed when the request finishes or its host copy is discarded.

KV contents are synthetic and position-determined (``kv_bits``), so the
expected pool and host bytes are computable without a model.
"""
from __future__ import annotations

import numpy as np

LIVE, DETACHED, RESERVED = np.uint8(1), np.uint8(2), np.uint8(4)
NOT_LIVE, NOT_DETACHED, NOT_RESERVED = np.uint8(0xFE), np.uint8(0xFD), np.uint8(0xFB)
M32 = 0xFFFFFFFF


def fmix32(x: np.ndarray) -> np.ndarray:
    x = x.astype(np.uint64) & M32
    x ^= x >> 16
    x = (x * 0x85EBCA6B) & M32
    x ^= x >> 13
    x = (x * 0xC2B2AE35) & M32
    x ^= x >> 16
    return x


def kv_bits(rid, pos, layer, kv, head, dim, seed: int = 0) -> np.ndarray:
    """Synthetic bf16 bit pattern for one KV element (broadcasting numpy).

    value = +-[0.5, 1): sign and 7 mantissa bits from a 32-bit mix of the
    coordinates.  Identical formula in csrc/tf_common.cuh (tf_kv_bits).
    """
    u = lambda v: np.asarray(v, dtype=np.uint64)
    x = (u(rid) * 0x9E3779B1 + u(pos) * 0x85EBCA77 + u(layer) * 0xC2B2AE3D
         + u(kv) * 0x27D4EB2F + u(head) * 0x165667B1 + u(dim) * 0x61C88647 + u(seed) * 0x2545F491) & M32
    x = fmix32(x)
    return ((x & 0x807F) | 0x3F00).astype(np.uint16)


def q_bits(rid, pos, layer, qhead, dim, seed: int = 0) -> np.ndarray:
    """Synthetic query (bf16 bits) for the decode at position ``pos``."""
    return kv_bits(rid + 0x5000, pos, layer, 2, qhead, dim, seed)


def bf16_to_f32(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << 16).view(np.float32)


class CpuDataPlane:
    def __init__(self, reqs, n_blocks, n_host_blocks, n_layers, n_kv_heads, head_dim, block=16, seed=0,
                 store_bytes=True):
        self.B = block
        self.L, self.H, self.D = n_layers, n_kv_heads, head_dim
        self.seed = seed
        self.flags = {r.id: np.zeros(r.prompt_len + r.output_len + 2, np.uint8) for r in reqs}
        nlb = {r.id: (r.prompt_len + r.output_len + 2 + block - 1) // block for r in reqs}
        self.gtab = {rid: np.full(n, -1, np.int32) for rid, n in nlb.items()}
        self.htab = {rid: np.full(n, -1, np.int32) for rid, n in nlb.items()}
        self.host_hi = {rid: 0 for rid in nlb}  # host copy valid for [0, host_hi)
        self.free = list(range(n_blocks - 1, -1, -1))
        self.hfree = list(range(n_host_blocks - 1, -1, -1))
        self.n_blocks, self.n_host = n_blocks, n_host_blocks
        self.store = store_bytes
        shape = (block, n_layers, 2, n_kv_heads, head_dim)
        # pool[block][layer][kv][head][slot][dim] (block-major)
        if store_bytes:
            self.pool = np.zeros((n_blocks, n_layers, 2, n_kv_heads, block, head_dim), np.uint16)
            self.host = np.zeros((n_host_blocks, n_layers, 2, n_kv_heads, block, head_dim), np.uint16)
        self.d2h_busy = None  # (rid, lo, hi, kind)
        self.peak_blocks = 0
        self.peak_host_blocks = 0
        self.ops = {"d2h_tokens": 0, "h2d_tokens": 0, "append_tokens": 0, "fill_tokens": 0}
        self._coords = np.meshgrid(np.arange(n_layers), np.arange(2), np.arange(n_kv_heads),
                                   np.arange(head_dim), indexing="ij")

    # ---- helpers
    def _values(self, rid, positions):
        """KV bits for (positions) -> [n][L][2][H][D]."""
        l, k, h, d = self._coords
        p = np.asarray(positions, np.uint64)[:, None, None, None, None]
        return kv_bits(rid, p, l[None], k[None], h[None], d[None], self.seed)

    def _reconcile(self, rid, blocks):
        f, tab = self.flags[rid], self.gtab[rid]
        blocks = sorted(set(int(j) for j in blocks))
        occ = {j: bool(f[j * self.B:(j + 1) * self.B].any()) for j in blocks}
        for j in blocks:
            if not occ[j] and tab[j] >= 0:
                self.free.append(int(tab[j]))
                tab[j] = -1
        for j in blocks:
            if occ[j] and tab[j] < 0:
                if not self.free:
                    raise MemoryError("GPU block pool exhausted")
                tab[j] = self.free.pop()
        self.peak_blocks = max(self.peak_blocks, self.n_blocks - len(self.free))

    def _slots(self, rid, positions):
        positions = np.asarray(positions)
        blk = self.gtab[rid][positions // self.B]
        assert (blk >= 0).all(), "unmapped position"
        return blk, positions % self.B

    def _write_pool(self, rid, positions):
        if not self.store or len(positions) == 0:
            return
        blk, slot = self._slots(rid, positions)
        vals = self._values(rid, positions)  # [n][L][2][H][D]
        self.pool[blk, :, :, :, slot] = vals

    def _blocks_of(self, positions):
        return {int(p) // self.B for p in positions}

    # ---- hooks (called by oracle.refsim.sim.Sim)
    def fill_start(self, job, sim):
        for rid in job.members:
            tot = sim.R[rid].kv.total_kv
            lo = 0 if job.kind == "recompute" else tot
            hi = lo + job.reserve[rid]
            pos = np.arange(lo, hi)
            assert not (self.flags[rid][pos] & (LIVE | RESERVED)).any()
            self.flags[rid][pos] |= RESERVED
            self._reconcile(rid, self._blocks_of(pos))
            self._write_pool(rid, pos)
            self.ops["fill_tokens"] += len(pos)

    def fill_done(self, rid):
        f = self.flags[rid]
        res = (f & RESERVED) != 0
        f[res] = (f[res] & NOT_RESERVED) | LIVE

    def decode_start(self, batch, sim):
        for rid in batch:
            s = sim.R[rid]
            p = s.kv.total_kv
            f = self.flags[rid]
            assert (f[:p] & LIVE).all(), f"decode of {rid} reads non-resident KV"
            f[p] |= RESERVED
            self._reconcile(rid, [p // self.B])
            self._write_pool(rid, [p])
            self.ops["append_tokens"] += 1

    def decode_done(self, batch, made):
        made = set(made)
        for rid in batch:
            f = self.flags[rid]
            idx = np.nonzero(f & RESERVED)[0]
            if rid in made:
                f[idx] = (f[idx] & NOT_RESERVED) | LIVE
            else:
                f[idx] &= NOT_RESERVED
                self._reconcile(rid, self._blocks_of(idx))

    def d2h_start(self, ch, sim):
        rid = ch.owner
        cs = sim.R[rid].kv.cpu_synced
        pos = np.arange(cs, cs + ch.tokens)
        f = self.flags[rid]
        assert (f[pos] & LIVE).all(), "d2h reads non-resident KV"
        htab = self.htab[rid]
        for j in sorted(self._blocks_of(pos)):
            if htab[j] < 0:
                if not self.hfree:
                    raise MemoryError("host store exhausted")
                htab[j] = self.hfree.pop()
        self.peak_host_blocks = max(self.peak_host_blocks, self.n_host - len(self.hfree))
        if self.store:
            blk, slot = self._slots(rid, pos)
            hb = htab[pos // self.B]
            self.host[hb, :, :, :, slot] = self.pool[blk, :, :, :, slot]
        self.host_hi[rid] = max(self.host_hi[rid], cs + ch.tokens)
        if ch.kind == "evict":
            f[pos] = (f[pos] & NOT_LIVE) | DETACHED
        self.d2h_busy = (rid, cs, cs + ch.tokens, ch.kind)
        self.ops["d2h_tokens"] += ch.tokens

    def d2h_done(self, ch, alive):
        rid, lo, hi, kind = self.d2h_busy
        self.d2h_busy = None
        assert rid == ch.owner
        if kind == "evict":
            pos = np.arange(lo, hi)
            self.flags[rid][pos] &= NOT_DETACHED
            self._reconcile(rid, self._blocks_of(pos))

    def h2d_start(self, ch, sim):
        rid = ch.owner
        tot = sim.R[rid].kv.total_kv
        f = self.flags[rid]
        miss = np.nonzero((f[:tot] & LIVE) == 0)[0][: ch.tokens]
        assert len(miss) == ch.tokens, "load larger than the missing set"
        assert (miss < self.host_hi[rid]).all(), "load of a position never written to host"
        f[miss] |= LIVE
        self._reconcile(rid, self._blocks_of(miss))
        if self.store:
            blk, slot = self._slots(rid, miss)
            hb = self.htab[rid][miss // self.B]
            assert (hb >= 0).all()
            self.pool[blk, :, :, :, slot] = self.host[hb, :, :, :, slot]
        self.ops["h2d_tokens"] += ch.tokens

    def release_prefix(self, rid, n):
        f = self.flags[rid]
        cs = None
        idx = np.nonzero(f & LIVE)[0]
        rel = idx[:n]
        assert len(rel) == n
        f[rel] &= NOT_LIVE
        self._reconcile(rid, self._blocks_of(rel))
        del cs

    def cancel_evicts(self, rid):
        pass

    def drop_gpu(self, rid):
        f = self.flags[rid]
        idx = np.nonzero(f & LIVE)[0]
        f[idx] &= NOT_LIVE
        self._reconcile(rid, self._blocks_of(idx))

    def drop_host(self, rid):
        tab = self.htab[rid]
        for j in range(len(tab)):
            if tab[j] >= 0:
                self.hfree.append(int(tab[j]))
                tab[j] = -1
        self.host_hi[rid] = 0

    def finish(self, rid):
        f = self.flags[rid]
        idx = np.nonzero(f)[0]
        f[:] = 0
        self._reconcile(rid, self._blocks_of(idx))
        self.drop_host(rid)

    def audit(self, sim):
        for rid, s in sim.R.items():
            f = self.flags[rid]
            n_live = int(np.count_nonzero(f & LIVE))
            n_det = int(np.count_nonzero(f & DETACHED))
            fly = sim.h2d.busy.tokens if (sim.h2d.busy is not None and sim.h2d.busy.owner == rid) else 0
            if s.state in ("gen_done", "done"):
                continue
            assert n_live + n_det == s.kv.gpu_resident + fly, (rid, n_live, n_det, s.kv.gpu_resident, fly)
            if s.state == "running":
                assert (f[: s.kv.total_kv] & LIVE).all()
            assert s.kv.cpu_synced <= self.host_hi[rid] or s.kv.cpu_synced == 0

    # ---- views for comparisons
    def block_table(self, rid):
        return self.gtab[rid].copy()

    def host_table(self, rid):
        return self.htab[rid].copy()

    def live_positions(self, rid):
        return np.nonzero(self.flags[rid] & LIVE)[0]


def attention_ref(q: np.ndarray, k: np.ndarray, v: np.ndarray, scale: float) -> np.ndarray:
    """fp32 GQA decode attention for one request and one layer.

    q [Hq][D], k/v [T][Hkv][D] (float32) -> out [Hq][D]; q head h reads kv
    head h // (Hq/Hkv).  The tolerance the GPU kernel is held to is stated in
    tests/test_attention_gpu.py.
    """
    hq, d = q.shape
    hkv = k.shape[1]
    g = hq // hkv
    out = np.empty((hq, d), np.float32)
    for h in range(hq):
        kh = k[:, h // g, :].astype(np.float64)
        s = kh @ q[h].astype(np.float64) * scale
        s -= s.max()
        p = np.exp(s)
        p /= p.sum()
        out[h] = (p @ v[:, h // g, :].astype(np.float64)).astype(np.float32)
    return out
