"""GPU batch-priority selector (host side of csrc/tf_select.cu).

Packs a ``SystemSnapshot`` into the C structs of include/tokenflow_b200.h,
runs the single-CTA decision kernel and unpacks a ``TickDecision``.  The
workspace (device + pinned host) is allocated once through torch and only
borrowed by the library.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from ._lib import TfMember, TfPrio, TfReqRow, TfSnapGlobals, TfTickParams, TfTickResult, TfWaiter, check, lib

MODE_CODES = {"buffer_aware": 0, "fcfs_fallback": 1}
MODE_NAMES = {v: k for k, v in MODE_CODES.items()}


class GpuSelector:
    def __init__(self, max_members: int = 1024, max_waiting: int = 2048, device=None):
        if not torch.cuda.is_available():
            raise RuntimeError("GpuSelector needs a CUDA device (no CPU fallback)")
        self.device = torch.device(device or "cuda")
        self.max_n, self.max_w = max_members, max_waiting
        nbytes = int(lib.tf_selector_workspace_bytes(max_members, max_waiting))
        self._dev = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        self._host = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
        h = C.c_int64()
        check(lib.tf_selector_init(C.c_void_p(self._dev.data_ptr()), nbytes, C.c_void_p(self._host.data_ptr()),
                                   nbytes, max_members, max_waiting, C.byref(h)), "tf_selector_init")
        self.handle = h.value
        self.stream = torch.cuda.Stream(device=self.device)
        self._res = {k: (C.c_int32 * max(1, n))() for k, n in (
            ("counts", 8), ("preempt", max_members), ("resume_ids", max_members), ("resume_how", max_members),
            ("admitted", max_waiting), ("recomputed", max_members), ("batch_sizes", max_waiting),
            ("batch_ids", max_waiting), ("t_prime_set", max_members))}
        self._tp = (C.c_double * max_members)()
        self._members = (TfMember * max_members)()
        self._waiters = (TfWaiter * max_waiting)()
        self.calls = 0

    # ------------------------------------------------------------------ packing
    def _params(self, snap, cfg, mode_code: int) -> TfTickParams:
        p = TfTickParams()
        p.n_members = 0 if hasattr(snap, "rows") else len(snap.members)
        p.n_waiting = len(snap.waiting)
        if p.n_members > self.max_n or p.n_waiting > self.max_w:
            raise ValueError("snapshot exceeds selector capacity")
        p.free_slots, p.max_batch = snap.free_slots, snap.max_batch
        p.offload_enabled, p.mode = int(bool(snap.offload_enabled)), mode_code
        p.h2d_blocked_tokens = int(snap.h2d_blocked_tokens)
        p.now, p.gpu_mem_free = snap.now, float(snap.gpu_mem_free)
        p.gpu_mem_total, p.cpu_mem_total, p.gamma = float(snap.gpu_mem_total), float(snap.cpu_mem_total), snap.gamma
        for name in ("schedule_interval", "per_request_mem_estimate", "workingset_adjust_rate", "buffer_safety_factor",
                     "penalty_weight", "tau_schedule", "critical_buffer_seconds", "value_threshold_frac",
                     "value_decay_alpha", "pacing_buffer_seconds", "ema_factor"):
            setattr(p, name, float(getattr(cfg, name)))
        return p

    def _pack(self, snap, t_prime: dict):
        for i, m in enumerate(snap.members):
            d = self._members[i]
            d.request_id, d.prompt_len, d.output_len = m.request_id, m.prompt_len, m.output_len
            d.running, d.pinned = int(m.running), int(m.pinned)
            d.generated, d.consumed, d.ctx_tokens, d.gpu_resident = m.generated, m.consumed, m.ctx_tokens, m.gpu_resident
            d.arrival_time, d.rate, d.busy_since_tick = m.arrival_time, m.rate, m.busy_since_tick
            d.t_io, d.t_recompute = m.t_io, m.t_recompute
            d.last_iter_time = m.last_iter_time or 0.0
            tp = t_prime.get(m.request_id)
            d.has_tprime = int(tp is not None)
            d.t_prime = tp if tp is not None else 0.0
        for i, w in enumerate(snap.waiting):
            d = self._waiters[i]
            d.request_id, d.prompt_len, d.waited_s = w.request_id, w.prompt_len, w.waited_s

    def _result(self) -> TfTickResult:
        r = TfTickResult()
        for k, arr in self._res.items():
            setattr(r, k, C.cast(arr, C.POINTER(C.c_int32)))
        r.t_prime_out = C.cast(self._tp, C.POINTER(C.c_double))
        return r

    # -------------------------------------------------------------- decisions
    def tick(self, snap, cfg, t_prime: dict, mode: str):
        """on_tick -> (mode, preempt, resume[(id, how)], admitted, recomputed, batches); updates t_prime."""
        self._pack(snap, t_prime)
        p = self._params(snap, cfg, MODE_CODES[mode])
        r = self._result()
        check(lib.tf_policy_tick(self.handle, C.byref(p), self._members, self._waiters, C.byref(r),
                                 C.c_void_p(_lib.stream_ptr(self.stream))), "tf_policy_tick")
        self.calls += 1
        for i, m in enumerate(snap.members):
            if self._res["t_prime_set"][i]:
                t_prime[m.request_id] = self._tp[i]
        return self._unpack()

    def tick_rows(self, snap, cfg, t_prime: dict, mode: str):
        """on_tick from a RowsSnapshot: the member view is built on the device
        (tf_policy_tick_rows); t_prime is filled into the rows here."""
        rows = snap.rows
        for i in range(snap.n_rows):
            r = rows[i]
            tp = t_prime.get(r.request_id)
            r.has_tprime = int(tp is not None)
            r.t_prime = tp if tp is not None else 0.0
        for i, w in enumerate(snap.waiting):
            d = self._waiters[i]
            d.request_id, d.prompt_len, d.waited_s = w.request_id, w.prompt_len, w.waited_s
        p = self._params(snap, cfg, MODE_CODES[mode])
        p.n_members = 0
        r = self._result()
        ids = (C.c_int32 * max(1, snap.n_rows))()
        nm = C.c_int32()
        check(lib.tf_policy_tick_rows(self.handle, C.byref(p), rows, snap.n_rows, C.byref(snap.globals),
                                      self._waiters, C.byref(r), ids, C.byref(nm),
                                      C.c_void_p(_lib.stream_ptr(self.stream))), "tf_policy_tick_rows")
        self.calls += 1
        for i in range(nm.value):
            if self._res["t_prime_set"][i]:
                t_prime[ids[i]] = self._tp[i]
        return self._unpack()

    def fastpath(self, snap, cfg, mode: str):
        self._pack(snap, {})
        p = self._params(snap, cfg, MODE_CODES[mode])
        r = self._result()
        check(lib.tf_policy_fastpath(self.handle, C.byref(p), self._members, self._waiters, C.byref(r),
                                     C.c_void_p(_lib.stream_ptr(self.stream))), "tf_policy_fastpath")
        self.calls += 1
        return self._unpack()

    def _unpack(self):
        c = self._res["counts"]
        mode, npre, nres, nadm, nrc, nbat = c[0], c[1], c[2], c[3], c[4], c[5]
        pre = list(self._res["preempt"][:npre])
        ids, how = self._res["resume_ids"][:nres], self._res["resume_how"][:nres]
        resume = [(i, "recompute" if h else "load") for i, h in zip(ids, how)]
        adm = list(self._res["admitted"][:nadm])
        rc = list(self._res["recomputed"][:nrc])
        batches, k = [], 0
        for s in self._res["batch_sizes"][:nbat]:
            batches.append(list(self._res["batch_ids"][k:k + s]))
            k += s
        return MODE_NAMES[mode], pre, resume, adm, rc, batches

    def iteration_batch(self, running, contention: bool, mode: str, pacing: float) -> list:
        # called before every decode dispatch: pack through numpy (ctypes
        # varargs construction cost ~0.1 us per element and dominated the call)
        n = len(running)
        if n == 0:
            return []
        ids = np.fromiter((t[0] for t in running), np.int32, n)
        br = np.fromiter((t[1] for t in running), np.int64, n)
        rt = np.fromiter((t[2] for t in running), np.float64, n)
        out = self._res["preempt"]
        nout = C.c_int32()
        check(lib.tf_iteration_batch(self.handle, ids.ctypes.data_as(C.POINTER(C.c_int32)),
                                     br.ctypes.data_as(C.POINTER(C.c_int64)),
                                     rt.ctypes.data_as(C.POINTER(C.c_double)), n, int(bool(contention)),
                                     MODE_CODES[mode], pacing, out, C.byref(nout),
                                     C.c_void_p(_lib.stream_ptr(self.stream))), "tf_iteration_batch")
        return out[:nout.value]

    def select_batch(self, views, gpu_mem, max_batch, lengths) -> set:
        n = len(views)
        arr = (TfPrio * max(1, n))()
        for i, v in enumerate(views):
            d = arr[i]
            d.request_id, d.length = v.request_id, int(lengths[v.request_id])
            d.phi, d.value, d.t_prime, d.rate, d.utility = v.phi, v.value, v.t_prime, v.rate, v.utility
        chosen = (C.c_uint8 * max(1, n))()
        check(lib.tf_select_batch(self.handle, arr, n, float(gpu_mem), int(max_batch), chosen,
                                  C.c_void_p(_lib.stream_ptr(self.stream))), "tf_select_batch")
        return {views[i].request_id for i in range(n) if chosen[i]}


_default = None


def default_selector() -> GpuSelector:
    global _default
    if _default is None:
        _default = GpuSelector()
    return _default
