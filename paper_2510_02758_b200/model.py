"""Llama-style decoder on the paged KV pool (random-init weights).

Used for the C1 tiny decoder and the C2 Llama3-8B configuration.  The hot
path ops are this package's kernels: K/V rows are appended into the paged
block pool (tf_kv_append) and decode attention reads the block tables
directly (tf_paged_decode_attn).  Projections / MLP / logits are plain
cuBLAS GEMMs via torch.matmul (library GEMMs); prefill
attention over a fresh prompt uses torch SDPA.

Token pipeline (matches the reference's counts, engine.py:484-540): a
prefill of a P-token prompt writes KV for P+1 positions - the prompt, then
its first output token t0 at position P - and keeps t1 pending; every
decode step emits the pending token of each member, appends its KV at
position total_kv and computes the next pending token.  A recompute
re-runs the prompt plus the generated tokens (positions [0, total_kv)).
"""
from __future__ import annotations

import ctypes as C
import math
import os
import time

import numpy as np
import torch
from torch.nn.attention.varlen import varlen_attn

from . import _lib
from ._lib import check, lib

_DEBUG_GRAPHS = os.environ.get("TF_DEBUG_GRAPHS") == "1"  # sync + range-check every graph replay (debug)
# Prompt prefills replayed from the token-bucket graphs (default) or launched
# eagerly (TF_PROMPT_GRAPHS=0).  The graphs cut the host time of a prompt
# prefill from ~10 ms to ~0.7 ms, and an eager prefill holds the GPU for its
# host-bound launch sequence: in bench.py's serving window (20 schedule
# intervals of the C2 burst) prefills take 0.22 s of device time with graphs
# and 1.1-1.15 s eager, 14.2-14.7K vs 10.9K effective tok/s.  Over the
# whole burst the eager path's slower measured prefills make the reference
# policy recompute and preempt less (1,644 vs 1,537 effective tok/s, P99 TTFT
# 101.6 vs 124.6 s: profiles/r2_full_run_prompt_graphs_ab.json).  Recompute
# prefills always replay graphs.
_PROMPT_GRAPHS = os.environ.get("TF_PROMPT_GRAPHS", "1") == "1"


class _Staging:
    """Grow-only pinned host + device buffer for a host -> device input:
    one zero-copy transfer (tf_copy_small) on the compute stream, no pinned
    allocation per call (cudaHostAlloc is slow) and no copy-engine queueing
    behind KV loads.  Reused call after call: the engine runs one GPU job at a
    time and the next call comes after the previous job completed."""

    def __init__(self, device):
        self.device = device
        self.h = self.d = None

    def to_device(self, t: torch.Tensor, stream) -> torch.Tensor:
        t = t.contiguous()
        nb = t.numel() * t.element_size()
        if self.h is None or self.h.numel() < nb:
            cap = max(nb, 2 * (self.h.numel() if self.h is not None else 0), 4096)
            self.h = torch.empty(cap, dtype=torch.uint8, pin_memory=True)
            self.d = torch.empty(cap, dtype=torch.uint8, device=self.device)
        self.h[:nb].copy_(t.view(-1).view(torch.uint8))
        check(lib.tf_copy_small(C.c_void_p(self.d.data_ptr()), C.c_void_p(self.h.data_ptr()), nb,
                                C.c_void_p(stream.cuda_stream)), "tf_copy_small")
        return self.d[:nb].view(t.dtype).view(t.shape)


class PagedDecoder:
    def __init__(self, shape, device="cuda", seed=0, dtype=torch.bfloat16, max_batch=256, tp=None):
        """``tp`` (tp.TpGroup): keep this rank's 1/TP of the heads / MLP columns
        (C4).  Each weight is drawn in full with the same generator stream as
        TP=1 and sliced, so a TP model is the TP=1 model partitioned."""
        self.s = shape
        self.tp = tp
        self.device = torch.device(device)
        g = torch.Generator(device=self.device).manual_seed(seed)
        d, hq, hkv, hd, ffn = shape.hidden, shape.n_q_heads, shape.n_kv_heads, shape.head_dim, shape.ffn
        rank, size = (tp.rank, tp.size) if tp is not None else (0, 1)
        if hkv % size or ffn % size:
            raise ValueError(f"TP={size} does not divide {hkv} kv heads / ffn {ffn}")
        self.hq, self.hkv, self.ffn = hq // size, hkv // size, ffn // size
        qc = slice(rank * self.hq * hd, (rank + 1) * self.hq * hd)
        kc = slice(hq * hd + rank * self.hkv * hd, hq * hd + (rank + 1) * self.hkv * hd)
        vc = slice((hq + hkv) * hd + rank * self.hkv * hd, (hq + hkv) * hd + (rank + 1) * self.hkv * hd)
        fc = slice(rank * self.ffn, (rank + 1) * self.ffn)

        def w(*dims):
            t = torch.empty(*dims, device=self.device, dtype=dtype)
            t.normal_(0.0, 0.02, generator=g)
            return t

        def shard_qkv(t):  # [.., (hq + 2 hkv) hd] -> [.., (hq + 2 hkv)/TP hd] as [q | k | v]
            return t if size == 1 else torch.cat([t[..., qc], t[..., kc], t[..., vc]], -1).contiguous()

        def shard_gu(t):  # [d, 2 ffn] -> [d, 2 ffn/TP] as [gate | up]
            return t if size == 1 else torch.cat([t[:, fc], t[:, ffn:][:, fc]], -1).contiguous()

        self.embed = w(shape.vocab, d)
        self.layers = []
        for _ in range(shape.n_layers):
            L = {"ln1": torch.ones(d, device=self.device, dtype=dtype),
                 "wqkv": shard_qkv(w(d, (hq + 2 * hkv) * hd))}
            if shape.qkv_bias:
                L["bqkv"] = shard_qkv(w((hq + 2 * hkv) * hd))
            wo = w(hq * hd, d)
            L["wo"] = wo if size == 1 else wo[qc].contiguous()
            L["ln2"] = torch.ones(d, device=self.device, dtype=dtype)
            L["wgu"] = shard_gu(w(d, 2 * ffn))
            wd = w(ffn, d)
            L["wd"] = wd if size == 1 else wd[fc].contiguous()
            del wo, wd
            self.layers.append(L)
        self.ln_f = torch.ones(d, device=self.device, dtype=dtype)
        self.lm_head = w(d, shape.vocab)
        inv = 1.0 / (shape.rope_theta ** (torch.arange(0, hd, 2, device=self.device, dtype=torch.float32) / hd))
        self._inv_freq = inv
        self.pending = {}  # rid -> next token to emit
        self.history = {}  # rid -> generated tokens (for recompute)
        self.keep_logits, self.last_logits, self.graph_logits = False, None, {}
        self._stage_ev, self.stage_waits = {}, 0
        self.attn_graph_ms = None  # measure_attention(graph_reps=...): avg launch inside a CUDA graph
        self.lpt_order = os.environ.get("TF_LPT", "0") == "1"  # decode rows longest-context first
        self.prompts = {}
        self._unresolved = {}  # rid -> (pinned buffer, column) of an in-flight prefill's t0/t1
        self.scale = 1.0 / math.sqrt(hd)
        self._ws = torch.zeros(1, dtype=torch.uint8, device=self.device)
        self.steps = 0
        self.attn_timing = None  # list -> (algorithmic bytes, start event, end event) per attention launch
        self._st_tok, self._st_meta, self._st_rows = (_Staging(self.device) for _ in range(3))
        self.host_s = {}  # host-side launch time per phase: name -> [calls, seconds, tokens]
        if self.device.type == "cuda":  # (a CPU-constructed model only serves weight-layout tests)
            self._pf_out = torch.zeros(2 * 4096, dtype=torch.long, pin_memory=True)  # prefill t0 / t1 readback
            self._dec_out = torch.zeros(4096, dtype=torch.long, pin_memory=True)  # sampled ids readback
        self._graphs = {}
        self._pgraphs = {}  # recompute prefill graphs per token bucket
        self._graph_launches = {}  # this library's kernels captured per graph
        self.replayed_launches = 0  # ... and re-run by graph replays so far
        if self.device.type == "cuda":
            # weights and buffers were generated on the default stream; every
            # later use is on the data plane's non-blocking streams
            torch.cuda.synchronize(self.device)

    def launch_count(self) -> int:
        """This library's kernel launches so far: direct C-ABI launches plus
        the captured ones every graph replay re-ran."""
        return int(lib.tf_launch_count()) + self.replayed_launches

    # ------------------------------------------------------------ pieces
    def prompt_tokens(self, rid: int, n: int) -> torch.Tensor:
        if rid not in self.prompts:
            g = torch.Generator().manual_seed(1000003 * (rid + 1))
            self.prompts[rid] = torch.randint(0, self.s.vocab, (n,), generator=g)
        return self.prompts[rid]

    def _rms(self, x, w):
        x = x.contiguous()
        y = torch.empty_like(x)
        check(lib.tf_rmsnorm(C.c_void_p(x.data_ptr()), C.c_void_p(w.data_ptr()), C.c_void_p(y.data_ptr()),
                             x.numel() // x.shape[-1], x.shape[-1], self.s.rms_eps,
                             C.c_void_p(torch.cuda.current_stream().cuda_stream)), "tf_rmsnorm")
        return y

    def _sample_normed(self, h):
        """Greedy next token from the final-normed hidden states; with
        ``keep_logits`` set (tests, eager only) the logits stay in ``last_logits``."""
        lg = h @ self.lm_head
        if self.keep_logits:
            self.last_logits = lg
        return lg.argmax(-1)

    def _rope(self, x, pos):
        # x [n, heads, hd], pos [n] (int64)
        ang = pos.float()[:, None] * self._inv_freq[None, :]
        cos, sin = ang.cos()[:, None, :], ang.sin()[:, None, :]
        x1, x2 = x[..., 0::2].float(), x[..., 1::2].float()
        out = torch.empty_like(x)
        out[..., 0::2] = (x1 * cos - x2 * sin).to(x.dtype)
        out[..., 1::2] = (x1 * sin + x2 * cos).to(x.dtype)
        return out

    def _append(self, dp, rows, pos, layer, k, v, stream):
        n = rows.numel()
        check(lib.tf_kv_append(dp.pool.handle, C.c_void_p(dp.table.data_ptr()), dp.nlb, C.c_void_p(rows.data_ptr()),
                               C.c_void_p(pos.data_ptr()), n, layer, C.c_void_p(k.data_ptr()),
                               C.c_void_p(v.data_ptr()), k.stride(0), C.c_void_p(stream.cuda_stream)), "tf_kv_append")

    def _proj_residual(self, x, a, w):
        """x + a @ w; under TP each rank holds a row slice of w, rank 0 adds the
        residual and one all-reduce (sum) completes both."""
        if self.tp is None or self.tp.size == 1:
            return torch.addmm(x, a, w)
        y = torch.addmm(x, a, w) if self.tp.rank == 0 else a @ w
        return self.tp.all_reduce(y)

    def _qkv(self, h, L):
        return torch.addmm(L["bqkv"], h, L["wqkv"]) if "bqkv" in L else h @ L["wqkv"]

    def _proj_residual_norm(self, x, a, w, gamma):
        """(x + a @ w, rmsnorm(x + a @ w) * gamma): a sub-layer's output
        projection, its residual and the next sub-layer's input norm.  Under
        TP with a peer-memory communicator (tp.PeerAllReduce) the rank's GEMM
        writes its partial into its registered buffer and ONE kernel
        (tf_ar_residual_rmsnorm) does the all-reduce over NVLink, the residual
        add and the norm; otherwise addmm (+ NCCL all-reduce) and tf_rmsnorm."""
        ar = getattr(self.tp, "ar", None) if self.tp is not None and self.tp.size > 1 else None
        if self.tp is None or self.tp.size == 1:
            # plain GEMM (faster than addmm with the residual in the epilogue at
            # decode shapes) + one fused residual-add / RMSNorm kernel
            y = a @ w
            h = torch.empty_like(x)
            check(lib.tf_residual_rmsnorm(C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()),
                                          C.c_void_p(gamma.data_ptr()), C.c_void_p(h.data_ptr()), x.shape[0],
                                          x.shape[1], self.s.rms_eps,
                                          C.c_void_p(torch.cuda.current_stream().cuda_stream)), "tf_residual_rmsnorm")
            return x, h
        if ar is None or not ar.fits(x.shape[0], x.shape[1]):
            x = self._proj_residual(x, a, w)
            return x, self._rms(x, gamma)
        part = ar.partial(x.shape[0], x.shape[1])
        torch.mm(a, w, out=part)
        h = torch.empty_like(x)
        ar.residual_rmsnorm(x, gamma, h, self.s.rms_eps, torch.cuda.current_stream())
        return x, h

    def _mlp_act(self, h, L):
        gu = h @ L["wgu"]
        act = torch.empty((gu.shape[0], self.ffn), device=gu.device, dtype=gu.dtype)
        check(lib.tf_silu_mul(C.c_void_p(gu.data_ptr()), C.c_void_p(act.data_ptr()), gu.shape[0], self.ffn,
                              C.c_void_p(torch.cuda.current_stream().cuda_stream)), "tf_silu_mul")
        return act

    def _next_norm(self, li):
        return self.layers[li + 1]["ln1"] if li + 1 < len(self.layers) else self.ln_f

    # ------------------------------------------------------------ forward passes
    @torch.no_grad()
    def _prefill_batch(self, dp, seqs, st):
        """One causal forward over several fresh sequences (tokens concatenated
        for the GEMMs, attention per sequence with the flash backend), writing
        their KV into the paged pool.  seqs: [(rid, tokens[int64 cpu], pos0)].
        Returns the argmax token after each sequence's last position (device)."""
        s = self.s
        lens = [t.numel() for _, t, _ in seqs]
        # every host->device input goes through pinned memory, non-blocking: a
        # pageable copy would block the host until the compute stream drains
        toks = self._st_tok.to_device(torch.cat([t for _, t, _ in seqs]), st)
        rows_h = torch.repeat_interleave(torch.tensor([rid for rid, _, _ in seqs], dtype=torch.int32),
                                         torch.tensor(lens))
        pos_h = torch.cat([torch.arange(p0, p0 + t.numel(), dtype=torch.int32) for _, t, p0 in seqs])
        cu_h = torch.zeros(len(lens) + 1, dtype=torch.int32)
        cu_h[1:] = torch.cumsum(torch.tensor(lens, dtype=torch.int32), 0)
        meta = self._st_meta.to_device(torch.cat([rows_h, pos_h, cu_h]), st)
        n = toks.numel()
        rows, pos32, cu = meta[:n], meta[n:2 * n], meta[2 * n:]
        return self._prefill_core(dp, toks, rows, pos32, cu, max(lens), (cu[1:] - 1).long(), st)

    def _prefill_core(self, dp, toks, rows, pos32, cu, max_len, last, st):
        """Causal forward of the concatenated sequences ``toks`` (device) whose
        tokens go to (rows, pos32) of the paged pool; cu = cumulative sequence
        starts (int32, device); returns the argmax after token ``last``."""
        s = self.s
        n = toks.numel()
        G = self.hq // self.hkv
        x = self.embed[toks]
        q = torch.empty((n, self.hq, s.head_dim), device=self.device, dtype=x.dtype)
        kvb = torch.empty((2, n, self.hkv, s.head_dim), device=self.device, dtype=x.dtype)
        k, v = kvb[0], kvb[1]
        h = self._rms(x, self.layers[0]["ln1"])
        for li, L in enumerate(self.layers):
            qkv = self._qkv(h, L)
            # rotary q/k + paged K/V append (+ host mirror when write-through is
            # fused) + contiguous k/v for the prompt attention
            if getattr(dp, "fused_wt", False):
                check(lib.tf_rope_kv_append_wt(dp.pool.handle, C.c_void_p(dp.table.data_ptr()),
                                               C.c_void_p(dp.htable.data_ptr()), dp.nlb, C.c_void_p(rows.data_ptr()),
                                               C.c_void_p(pos32.data_ptr()), n, li, C.c_void_p(qkv.data_ptr()),
                                               self.hq, C.c_void_p(self._inv_freq.data_ptr()),
                                               C.c_void_p(q.data_ptr()), C.c_void_p(kvb.data_ptr()),
                                               C.c_void_p(st.cuda_stream)), "tf_rope_kv_append_wt")
            else:
                check(lib.tf_rope_kv_append(dp.pool.handle, C.c_void_p(dp.table.data_ptr()), dp.nlb,
                                            C.c_void_p(rows.data_ptr()), C.c_void_p(pos32.data_ptr()), n, li,
                                            C.c_void_p(qkv.data_ptr()), self.hq,
                                            C.c_void_p(self._inv_freq.data_ptr()), C.c_void_p(q.data_ptr()),
                                            C.c_void_p(kvb.data_ptr()), C.c_void_p(st.cuda_stream)),
                      "tf_rope_kv_append")
            # causal attention over every sequence of the batch in ONE varlen
            # flash-attention call (library kernel; per-sequence launches made
            # the host the bottleneck of recompute-heavy phases)
            kx = k.repeat_interleave(G, dim=1) if G > 1 else k
            vx = v.repeat_interleave(G, dim=1) if G > 1 else v
            a = varlen_attn(q, kx, vx, cu, cu, max_len, max_len, window_size=(-1, 0)).reshape(n, -1)
            x, h = self._proj_residual_norm(x, a, L["wo"], L["ln2"])
            x, h = self._proj_residual_norm(x, self._mlp_act(h, L), L["wd"], self._next_norm(li))
        return self._sample_normed(h[last])

    @torch.no_grad()
    def prefill(self, dp, job, spans, eng):
        """A prefill job: prompts (+ t0 decode) or recomputes; no host syncs."""
        t_host = time.perf_counter()
        try:
            self._prefill_job(dp, job, spans, eng)
        finally:
            h = self.host_s.setdefault("prefill", [0, 0.0, 0])
            h[0] += 1
            h[1] += time.perf_counter() - t_host
            h[2] += sum(hi - lo for _, lo, hi in spans)

    def _prefill_job(self, dp, job, spans, eng):
        st = dp.s_compute
        with torch.cuda.stream(st):
            seqs = []
            for rid, lo, hi in spans:
                spec = eng.state[rid].spec
                prompt = self.prompt_tokens(rid, spec.prompt_len)
                if job.kind == "recompute":
                    hist = torch.tensor(self.history.get(rid, []), dtype=torch.long)
                    toks = torch.cat([prompt, hist])[: hi - lo]
                    if len(spans) == 1 and self._prefill_fits_graph([(rid, toks, 0)]):
                        self._recompute_graph(dp, rid, toks, st)
                        return
                    seqs.append((rid, toks, 0))
                elif job.kind == "chunk":
                    raise NotImplementedError("chunked prefill (baseline 'chunked' policy) needs prefix attention; "
                                              "use the synthetic KV source for that baseline")
                else:
                    seqs.append((rid, prompt[lo: hi - 1], lo))
            if job.kind != "recompute" and _PROMPT_GRAPHS and self._prefill_fits_graph(seqs) and self.attn_timing is None:
                t0 = self._prefill_graph(dp, seqs, st)
            else:
                t0 = self._prefill_batch(dp, seqs, st)
            if job.kind == "recompute":
                return
            rids = [r for r, _, _ in seqs]
            pos1 = [hi - 1 for _, _, hi in spans]
            if self._graphs and len(rids) <= max(self._graphs) and self.attn_timing is None:
                t1 = self._decode_graph(dp, rids, pos1, st, tokens_dev=t0)  # 3 launches instead of ~320
            else:
                t1 = self._decode_rows(dp, rids, t0, pos1, st)
            t01 = torch.stack([t0, t1]).contiguous()
            buf = self._pf_out[: 2 * len(rids)].view(2, len(rids))
            # zero-copy D2H: the prefill's end event must not wait behind evict copies
            check(lib.tf_copy_small(C.c_void_p(buf.data_ptr()), C.c_void_p(t01.data_ptr()), buf.numel() * 8,
                                    C.c_void_p(st.cuda_stream)), "tf_copy_small")
            for i, rid in enumerate(rids):
                self._unresolved[rid] = (buf, i)

    def fill_commit(self, rid):
        """Prefill job finished (its end event fired): t0 emitted, t1 pending."""
        if rid in self._unresolved:
            buf, i = self._unresolved.pop(rid)
            self.history[rid] = [int(buf[0, i])]
            self.pending[rid] = int(buf[1, i])

    @torch.no_grad()
    def decode(self, dp, batch, eng):
        st = dp.s_compute
        if self.lpt_order:
            # longest context first: attention CTAs are dispatched in row order,
            # so the long (request, head) items start in the first wave and the
            # tail wave holds the short ones (LPT); tokens map back by rid
            batch = sorted(batch, key=lambda r: -eng.state[r].kv.total_kv)
        pos = [eng.state[r].kv.total_kv for r in batch]
        with torch.cuda.stream(st):
            if self._graphs and len(batch) <= max(self._graphs) and self.attn_timing is None:
                nxt = self._decode_graph(dp, list(batch), pos, st)
            else:
                toks = torch.tensor([self.pending[r] for r in batch], dtype=torch.long)
                nxt = self._decode_rows(dp, list(batch), self._st_tok.to_device(toks, st), pos, st)
            dp.stats["attn_launches"] += self.s.n_layers
            host = self._dec_out[: len(batch)]
            nxt = nxt.contiguous()
            # sampled ids -> client (D2H of the step's result), zero-copy so the
            # step's end event does not wait behind evict / write-through copies
            check(lib.tf_copy_small(C.c_void_p(host.data_ptr()), C.c_void_p(nxt.data_ptr()), host.numel() * 8,
                                    C.c_void_p(st.cuda_stream)), "tf_copy_small")
            self._last = (list(batch), host)
        self.steps += 1

    def decode_commit(self, made):
        """Host side of a finished decode step: emit pending tokens of members that produced."""
        batch, host = self._last
        vals = host.tolist()
        for rid, t in zip(batch, vals):
            if rid in made:
                self.history.setdefault(rid, []).append(self.pending[rid])
                self.pending[rid] = t

    @torch.no_grad()
    def measure_attention(self, dp, rids, positions, reps=3, plan="exact", graph_reps=0):
        """Time the paged-attention kernel on a live batch (all layers, CUDA
        events on the launching stream) -> [(algorithmic bytes, ms)] per launch.

        plan="graph" launches it exactly as the captured decode graphs do: the
        batch padded to its bucket with scratch rows (ctx 1) and max_ctx = the
        pool's maximum context; plan="exact" uses B and max(ctx).  The
        algorithmic bytes count the real rows only.  With
        ``graph_reps`` the layers are also captured into one CUDA graph and
        replayed: the average launch duration as in the decode graphs is left
        in ``self.attn_graph_ms``."""
        s = self.s
        st = dp.s_compute
        B = len(rids)
        rows_l, pos_l = list(rids), list(positions)
        if self.lpt_order:  # the row order decode() launches with
            order = sorted(range(B), key=lambda i: -pos_l[i])
            rows_l, pos_l = [rows_l[i] for i in order], [pos_l[i] for i in order]
        max_ctx = max(positions) + 1
        if plan == "graph" and self._graphs:
            Bp = next(b for b in sorted(self._graphs) if b >= B)
            rows_l += [dp.scratch_row] * (Bp - B)
            pos_l += [0] * (Bp - B)
            max_ctx = self._gmax_ctx
        Bl = len(rows_l)
        with torch.cuda.stream(st):
            rows = torch.tensor(rows_l, dtype=torch.int32, device=self.device)
            ctx = torch.tensor([p + 1 for p in pos_l], dtype=torch.int32, device=self.device)
            q = torch.randn((Bl, self.hq, s.head_dim), device=self.device).to(torch.bfloat16)
            out = torch.empty_like(q)
            ws_n = max(1, int(lib.tf_paged_decode_attn_workspace(dp.pool.handle, Bl, max_ctx, self.hq)))
            ws = torch.zeros(ws_n, dtype=torch.uint8, device=self.device)
            abytes = (sum(positions) + B) * 2 * self.hkv * s.head_dim * 2 + 2 * B * self.hq * s.head_dim * 2 \
                + sum((p + 16) // 16 for p in positions) * 4
            res = []
            for r in range(reps + 1):
                for li in range(s.n_layers):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(st)
                    check(lib.tf_paged_decode_attn(dp.pool.handle, C.c_void_p(q.data_ptr()),
                                                   C.c_void_p(dp.table.data_ptr()), dp.nlb,
                                                   C.c_void_p(rows.data_ptr()), C.c_void_p(ctx.data_ptr()), Bl,
                                                   max_ctx, li, self.hq, self.scale, C.c_void_p(out.data_ptr()),
                                                   C.c_void_p(ws.data_ptr()), ws_n, C.c_void_p(st.cuda_stream)),
                          "tf_paged_decode_attn")
                    e1.record(st)
                    if r > 0:  # first pass is warm-up
                        res.append((abytes, e0, e1))
            per_launch = None
            if graph_reps:
                # the same launches as they run inside the decode graphs: all
                # layers back to back in one CUDA graph, one event pair around
                # graph_reps replays (no host, no per-launch event in between)
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=st):
                    for li in range(s.n_layers):
                        check(lib.tf_paged_decode_attn(dp.pool.handle, C.c_void_p(q.data_ptr()),
                                                       C.c_void_p(dp.table.data_ptr()), dp.nlb,
                                                       C.c_void_p(rows.data_ptr()), C.c_void_p(ctx.data_ptr()), Bl,
                                                       max_ctx, li, self.hq, self.scale, C.c_void_p(out.data_ptr()),
                                                       C.c_void_p(ws.data_ptr()), ws_n,
                                                       C.c_void_p(torch.cuda.current_stream().cuda_stream)),
                              "tf_paged_decode_attn")
                g.replay()
                g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                g0.record(st)
                for _ in range(graph_reps):
                    g.replay()
                g1.record(st)
        st.synchronize()
        if graph_reps:
            per_launch = g0.elapsed_time(g1) / (graph_reps * s.n_layers)
            self.attn_graph_ms = per_launch
        return [(b, e0.elapsed_time(e1)) for b, e0, e1 in res]

    # ------------------------------------------------------------ CUDA graphs
    def enable_graphs(self, dp, buckets=(8, 16, 24, 32, 48, 64, 80, 96, 112, 128), prefill_buckets=128):
        """Capture the decode forward once per batch-size bucket.

        Shapes are static per bucket: padded rows point at a scratch table row
        (one reserved block), attention is planned for the pool's maximum
        context (rows shorter than that exit their empty split CTAs early).
        A step then costs one H2D of [tokens, rows, positions], one graph
        launch and one D2H of the sampled ids.
        """
        s = self.s
        self._gdp = dp
        self._gmax_ctx = dp.nlb * dp.B
        self._graphs = {}
        mempool = torch.cuda.graph_pool_handle()
        st = dp.s_compute
        for Bp in buckets:
            io = torch.zeros((3, Bp), dtype=torch.int64, device=self.device)
            io[1].fill_(dp.scratch_row)
            stage = torch.zeros((3, Bp), dtype=torch.int64, pin_memory=True)
            ws_n = max(1, int(lib.tf_paged_decode_attn_workspace(dp.pool.handle, Bp, self._gmax_ctx, self.hq)))
            ws = torch.zeros(ws_n, dtype=torch.uint8, device=self.device)
            # io / ws were initialised on the default stream and st is a
            # non-blocking stream: without this the warm-up can read them
            # before the fills ran (garbage token ids / rows -> an illegal
            # address, seen with two processes time-slicing one GPU)
            st.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(st):
                self._forward_graphable(dp, io, Bp, ws, st)  # warm-up (kernel attributes, cuBLAS handles)
            st.synchronize()
            g = torch.cuda.CUDAGraph()
            c0 = lib.tf_launch_count()
            with torch.cuda.graph(g, pool=mempool, stream=st):
                out = self._forward_graphable(dp, io, Bp, ws, torch.cuda.current_stream())
            self._graph_launches[("decode", Bp)] = lib.tf_launch_count() - c0
            self._graphs[Bp] = (g, io, stage, out, ws)
            if self.keep_logits:  # the bucket's static logits (tests)
                self.graph_logits[Bp] = self.last_logits
        st.synchronize()
        if prefill_buckets:
            self._capture_recompute_graphs(dp, mempool, st, prefill_buckets)

    PF_SEQS = 8  # real sequences per captured prefill graph

    @staticmethod
    def _prefill_bucket_sizes(top, step):
        """Token buckets of the prefill graphs: ``step``-token steps up to 1024,
        2 x step up to 2048, 4 x step above (a 533-token prompt pads to 640,
        not to 1024), capped at ``top``."""
        out, T = [], 0
        while T < top:
            T += step if T < 1024 else (2 * step if T < 2048 else 4 * step)
            out.append(min(T, top))
        return sorted(set(out))

    def _capture_recompute_graphs(self, dp, mempool, st, step):
        """Prefills (prompt prefills of up to PF_SEQS requests, and recomputes:
        one request re-prefilling its whole context, engine.py:889-917) as CUDA
        graphs per token bucket: the host launches one graph instead of ~400
        kernels (an eager 32-layer prefill costs ~10 ms of host time, longer
        than the GPU needs for a 512-token prompt), so the serving loop stays
        responsive.  Layout of a bucket of T tokens: the real sequences, then
        one padding sequence on the scratch row up to T; cu_seqlens has a
        fixed PF_SEQS + 2 entries (unused real slots are zero-length), and the
        argmax is taken after each real sequence's last token."""
        self._pgraphs = {}
        NS = self.PF_SEQS
        top = min(dp.max_len + NS, dp.nlb * dp.B)
        for T in self._prefill_bucket_sizes(top, step):
            tok = torch.zeros(T, dtype=torch.int64, device=self.device)
            meta = torch.zeros(2 * T + NS + 2, dtype=torch.int32, device=self.device)
            last = torch.zeros(NS, dtype=torch.int64, device=self.device)
            meta[:T] = dp.scratch_row
            meta[T:2 * T] = torch.arange(T, dtype=torch.int32, device=self.device)
            meta[2 * T + NS + 1] = T  # all real slots empty, padding = [0, T)
            rows, pos32, cu = meta[:T], meta[T:2 * T], meta[2 * T:]
            st.wait_stream(torch.cuda.current_stream())  # the fills above ran on the default stream
            with torch.cuda.stream(st):
                self._prefill_core(dp, tok, rows, pos32, cu, T, last, st)  # warm-up
            st.synchronize()
            g = torch.cuda.CUDAGraph()
            c0 = lib.tf_launch_count()
            with torch.cuda.graph(g, pool=mempool, stream=st):
                out = self._prefill_core(dp, tok, rows, pos32, cu, T, last, torch.cuda.current_stream())
            self._graph_launches[("recompute", T)] = lib.tf_launch_count() - c0
            stage_tok = torch.zeros(T, dtype=torch.int64, pin_memory=True)
            stage_meta = torch.zeros(2 * T + NS + 2, dtype=torch.int32, pin_memory=True)
            stage_last = torch.zeros(NS, dtype=torch.int64, pin_memory=True)
            self._pgraphs[T] = (g, tok, meta, last, stage_tok, stage_meta, stage_last, out)
        st.synchronize()

    def _prefill_fits_graph(self, seqs) -> bool:
        if not self._pgraphs or len(seqs) > self.PF_SEQS or any(p0 != 0 for _, _, p0 in seqs):
            return False
        return sum(t.numel() for _, t, _ in seqs) <= max(self._pgraphs)

    def _prefill_graph(self, dp, seqs, st):
        """Replay the prefill graph of the smallest bucket that holds ``seqs``
        = [(rid, tokens[int64 cpu], 0)]; returns the argmax after each
        sequence's last token (copied out of the graph's static output)."""
        NS = self.PF_SEQS
        lens = [t.numel() for _, t, _ in seqs]
        n = sum(lens)
        T = next(b for b in sorted(self._pgraphs) if b >= n)
        g, tok, meta, last, stage_tok, stage_meta, stage_last, out = self._pgraphs[T]
        self._stage_guard(("p", T))
        st_tok, st_meta, st_last = stage_tok.numpy(), stage_meta.numpy(), stage_last.numpy()
        st_tok[:n] = torch.cat([t for _, t, _ in seqs]).numpy()
        st_tok[n:] = 0
        st_meta[:], st_last[:] = self.prefill_layout([r for r, _, _ in seqs], lens, T, NS, dp.scratch_row)
        with torch.cuda.stream(st):
            for dst, src in ((tok, stage_tok), (meta, stage_meta), (last, stage_last)):
                check(lib.tf_copy_small(C.c_void_p(dst.data_ptr()), C.c_void_p(src.data_ptr()),
                                        dst.numel() * dst.element_size(), C.c_void_p(st.cuda_stream)),
                      "tf_copy_small")
            self._stage_mark(("p", T), st)
            g.replay()
            self.replayed_launches += self._graph_launches.get(("recompute", T), 0)
        if _DEBUG_GRAPHS:
            st.synchronize()
            tv, lv, mv = tok.cpu(), last.cpu(), meta.cpu()
            assert 0 <= int(tv.min()) and int(tv.max()) < self.s.vocab, ("prefill tok", T, n, tv.tolist()[:n + 4])
            assert 0 <= int(lv.min()) and int(lv.max()) < T, ("prefill last", T, lv.tolist())
            assert torch.equal(tv[:n], stage_tok[:n]) and torch.equal(mv, stage_meta), ("prefill stage", T, n)
            ov = out[: len(seqs)].cpu()
            assert 0 <= int(ov.min()) and int(ov.max()) < self.s.vocab, ("prefill out", ov.tolist())
        # copied out of the graph pool before any other graph replays: all graphs
        # share one memory pool, and a graph captured EARLIER (the decode graph
        # that samples t1 next) may reuse this output's addresses for its own
        # intermediates
        with torch.cuda.stream(st):
            return out[: len(seqs)].clone()

    @staticmethod
    def prefill_layout(rids, lens, T, NS, scratch_row):
        """Device inputs of a prefill graph of T tokens for sequences of
        ``lens`` tokens (request ``rids``): meta = [row of every token | its
        position | cu_seqlens (NS + 2 entries)] and the index of each
        sequence's last token (NS entries).  The real sequences come first,
        unused sequence slots are zero-length, and the padding sequence
        [sum(lens), T) sits on the scratch row."""
        n = sum(lens)
        if len(lens) > NS or n > T:
            raise ValueError(f"{len(lens)} sequences / {n} tokens do not fit a {T}-token graph with {NS} slots")
        meta = np.empty(2 * T + NS + 2, np.int32)
        last = np.zeros(NS, np.int64)
        cu = meta[2 * T:]
        cu[0] = 0
        o = 0
        for i, (rid, ln) in enumerate(zip(rids, lens)):
            meta[o:o + ln] = rid
            meta[T + o:T + o + ln] = np.arange(ln, dtype=np.int32)
            o += ln
            cu[i + 1] = o
            last[i] = o - 1
        cu[len(lens) + 1:NS + 1] = o  # unused real slots: zero-length
        cu[NS + 1] = T                # the padding sequence [n, T) on the scratch row
        meta[n:T] = scratch_row
        meta[T + n:2 * T] = np.arange(T - n, dtype=np.int32)
        return meta, last

    def _recompute_graph(self, dp, rid, toks, st):
        self._prefill_graph(dp, [(rid, toks, 0)], st)

    def _stage_guard(self, key):
        """A pinned staging buffer is rewritten only after the GPU read its
        previous contents (the zero-copy tf_copy_small of the last replay that
        used it); counts the times the host actually had to wait."""
        ev = self._stage_ev.get(key)
        if ev is not None and not ev.query():
            self.stage_waits += 1
            ev.synchronize()

    def _stage_mark(self, key, st):
        ev = self._stage_ev.get(key)
        if ev is None:
            ev = self._stage_ev[key] = torch.cuda.Event()
        ev.record(st)

    def _forward_graphable(self, dp, io, Bp, ws, st):
        rows = io[1].to(torch.int32)
        pos32 = io[2].to(torch.int32)
        ctx = pos32 + 1
        return self._layers_decode(dp, io[0], rows, pos32, ctx, Bp, self._gmax_ctx, ws, st, timing=None)

    def _decode_graph(self, dp, rids, positions, st, tokens_dev=None):
        """Replay the captured decode forward of the batch's bucket.  Token ids
        come from the pending table, or from ``tokens_dev`` (a device tensor,
        e.g. the prefill's first sampled tokens) without a host round trip."""
        B = len(rids)
        Bp = next(b for b in sorted(self._graphs) if b >= B)
        g, io, stage, out, _ = self._graphs[Bp]
        self._stage_guard(("d", Bp))
        # numpy view of the pinned staging rows: list -> int64 row writes cost a
        # few us each, torch.tensor(list) + slice copies ~4x that (host time
        # here sits between a step's completion and the next step's launch)
        sn = stage.numpy()
        if tokens_dev is not None:
            sn[0, :B] = 0
        else:
            pend = self.pending
            sn[0, :B] = [pend[r] for r in rids]
        sn[0, B:] = 0
        sn[1, :B] = rids
        sn[1, B:] = dp.scratch_row
        sn[2, :B] = positions
        sn[2, B:] = 0
        with torch.cuda.stream(st):
            # zero-copy read of the pinned staging row (not a copy-engine H2D:
            # those queue behind KV loads on the same engine)
            check(lib.tf_copy_small(C.c_void_p(io.data_ptr()), C.c_void_p(stage.data_ptr()),
                                    io.numel() * io.element_size(), C.c_void_p(st.cuda_stream)), "tf_copy_small")
            self._stage_mark(("d", Bp), st)
            if tokens_dev is not None:
                io[0, :B].copy_(tokens_dev)
            g.replay()
            self.replayed_launches += self._graph_launches.get(("decode", Bp), 0)
        if _DEBUG_GRAPHS:
            st.synchronize()
            iv = io.cpu()
            assert 0 <= int(iv[0].min()) and int(iv[0].max()) < self.s.vocab, ("decode tokens", Bp, B, iv[0].tolist(),
                                                                            tokens_dev is not None)
            assert torch.equal(iv[1:], stage[1:]), ("decode stage rows/pos", Bp, B)
        # the staging buffer is reused next step only after this step completed
        return out[:B]

    def _decode_rows(self, dp, rids, tokens, positions, st):
        s = self.s
        B = len(rids)
        rp = self._st_rows.to_device(torch.tensor([rids, positions], dtype=torch.int32), st)
        rows, pos32 = rp[0], rp[1]
        ctx = pos32 + 1
        max_ctx = max(positions) + 1
        need = int(lib.tf_paged_decode_attn_workspace(dp.pool.handle, B, max_ctx, self.hq))
        if need > self._ws.numel():
            self._ws = torch.zeros(need, dtype=torch.uint8, device=self.device)
        return self._layers_decode(dp, tokens, rows, pos32, ctx, B, max_ctx, self._ws, st, self.attn_timing,
                                   positions)

    def _layers_decode(self, dp, tokens, rows, pos32, ctx, B, max_ctx, ws, st, timing, positions=None):
        s = self.s
        x = self.embed[tokens]
        attn = torch.empty((B, self.hq, s.head_dim), device=self.device, dtype=x.dtype)
        if timing is not None:
            # algorithmic bytes of one launch: K+V of every context token, q in,
            # out, block-table entries
            abytes = (sum(positions) + B) * 2 * self.hkv * s.head_dim * 2 + 2 * B * self.hq * s.head_dim * 2 \
                + sum((p + 16) // 16 for p in positions) * 4
        q = torch.empty((B, self.hq, s.head_dim), device=self.device, dtype=x.dtype)
        h = self._rms(x, self.layers[0]["ln1"])
        for li, L in enumerate(self.layers):
            qkv = self._qkv(h, L)
            # fused rotary embedding + paged K/V append + q layout (one launch)
            if getattr(dp, "fused_wt", False):
                # write-through fused into the append epilogue (host mirror in the same step)
                check(lib.tf_rope_kv_append_wt(dp.pool.handle, C.c_void_p(dp.table.data_ptr()),
                                               C.c_void_p(dp.htable.data_ptr()), dp.nlb, C.c_void_p(rows.data_ptr()),
                                               C.c_void_p(pos32.data_ptr()), B, li, C.c_void_p(qkv.data_ptr()),
                                               self.hq, C.c_void_p(self._inv_freq.data_ptr()),
                                               C.c_void_p(q.data_ptr()), None, C.c_void_p(st.cuda_stream)),
                      "tf_rope_kv_append_wt")
            else:
                check(lib.tf_rope_kv_append(dp.pool.handle, C.c_void_p(dp.table.data_ptr()), dp.nlb,
                                            C.c_void_p(rows.data_ptr()), C.c_void_p(pos32.data_ptr()), B, li,
                                            C.c_void_p(qkv.data_ptr()), self.hq,
                                            C.c_void_p(self._inv_freq.data_ptr()), C.c_void_p(q.data_ptr()), None,
                                            C.c_void_p(st.cuda_stream)), "tf_rope_kv_append")
            if timing is not None:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
            check(lib.tf_paged_decode_attn(dp.pool.handle, C.c_void_p(q.data_ptr()), C.c_void_p(dp.table.data_ptr()),
                                           dp.nlb, C.c_void_p(rows.data_ptr()), C.c_void_p(ctx.data_ptr()), B, max_ctx,
                                           li, self.hq, self.scale, C.c_void_p(attn.data_ptr()),
                                           C.c_void_p(ws.data_ptr()), ws.numel(),
                                           C.c_void_p(st.cuda_stream)), "tf_paged_decode_attn")
            if timing is not None:
                e1.record(st)
                timing.append((abytes, e0, e1))
            x, h = self._proj_residual_norm(x, attn.view(B, -1), L["wo"], L["ln2"])
            x, h = self._proj_residual_norm(x, self._mlp_act(h, L), L["wd"], self._next_norm(li))
        return self._sample_normed(h)
