"""Tensor parallelism for the C4 configuration (Qwen2.5-32B over NVLink).

SURVEY 8(e): TP is the one configuration with a real exchange step.  Each TP
rank holds 1/TP of every layer's attention heads and MLP columns, and its own
shard of the paged KV pool (n_kv_heads/TP heads per block), which it swaps
over its OWN host link - so swap bytes per rank are bytes/TP, in lockstep.

Two collectives, nothing else:

* data path: one all-reduce (sum) after o_proj and one after down_proj per
  layer (B x hidden bf16 each), on the compute stream (``model.PagedDecoder``
  with ``tp=TpGroup(...)``).  With a ``PeerAllReduce`` attached (the default
  of ``bench.py --config c4``) each rank's GEMM writes its partial into a
  registered buffer and one kernel (``tf_ar_residual_rmsnorm``) reads the
  peers' partials over NVLink, adds the residual and applies the next RMSNorm
  - graph-capturable, no NCCL on the data path; without it, NCCL;
* control path: ``Lockstep.agree`` - one 10-double all-reduce (max) per loop
  iteration of the real-time engine over a CPU (gloo) group.  Instead of
  broadcasting rank 0's decisions, every rank runs the same deterministic
  engine and bit-exact GPU selector on the same agreed event sequence: a
  completion (decode step, prefill, d2h / h2d chunk) is taken once it fired on
  every rank, at the latest rank's device time, and the clock is the earliest
  rank's.  Identical inputs -> identical decisions, block tables and chunk
  sequences on every rank (checked at the end with ``Lockstep.same``).
"""
from __future__ import annotations

import hashlib
import math

import numpy as np
import torch
import torch.distributed as dist


class Lockstep:
    """Completion / clock consensus of the TP ranks' real-time engines."""

    def __init__(self, group=None):
        self.group = group
        self.world = dist.get_world_size(group)
        self.calls = 0

    def agree(self, clock: float, flags, ends, starts):
        """-> (clock, flags, ends, starts) agreed over the ranks: an item is
        done iff done on every rank; its end / start is the latest rank's; the
        clock is the EARLIEST rank's (each rank read it before querying its
        events, so an item not yet done on some rank ends after that rank's
        clock, hence after the agreed one - events up to the agreed clock can
        be drained before any completion still to come)."""
        k = len(flags)
        v = np.empty(1 + 3 * k, dtype=np.float64)
        v[0] = -clock  # max of -clock = min clock
        for i in range(k):
            # max-reduction of (1 - done): an item is done only if done everywhere
            v[1 + i] = 0.0 if flags[i] else 1.0
            v[1 + k + i] = ends[i] if flags[i] else -math.inf
            v[1 + 2 * k + i] = starts[i] if flags[i] else -math.inf
        t = torch.from_numpy(v)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        self.calls += 1
        return (-float(v[0]), [v[1 + i] == 0.0 for i in range(k)], [float(v[1 + k + i]) for i in range(k)],
                [float(v[1 + 2 * k + i]) for i in range(k)])

    def same(self, text: str) -> bool:
        """True iff every rank holds the same ``text`` (e.g. the event hash)."""
        h = hashlib.sha256(text.encode()).digest()
        mine = torch.tensor(list(h), dtype=torch.float64)
        lo, hi = mine.clone(), mine.clone()
        dist.all_reduce(lo, op=dist.ReduceOp.MIN, group=self.group)
        dist.all_reduce(hi, op=dist.ReduceOp.MAX, group=self.group)
        return bool(torch.equal(lo, hi))


class TpGroup:
    """This rank's slice of a TP model: rank, size and the NCCL group of the
    data-path all-reduces."""

    def __init__(self, rank: int, size: int, group=None, ar: "PeerAllReduce | None" = None):
        self.rank, self.size, self.group = rank, size, group
        self.ar = ar  # peer-memory data path (None: NCCL all-reduce)

    def heads(self, n: int) -> range:
        if n % self.size:
            raise ValueError(f"{n} heads do not split over TP={self.size}")
        k = n // self.size
        return range(self.rank * k, (self.rank + 1) * k)

    def cols(self, n: int) -> slice:
        if n % self.size:
            raise ValueError(f"{n} columns do not split over TP={self.size}")
        k = n // self.size
        return slice(self.rank * k, (self.rank + 1) * k)

    def all_reduce(self, x: torch.Tensor) -> torch.Tensor:
        if self.size > 1:
            dist.all_reduce(x, group=self.group)
        return x


class PeerAllReduce:
    """This rank's peer-memory all-reduce communicator (csrc/tf_ar.cu).

    Buffers are cudaMalloc'ed by the library and mapped into every peer with
    CUDA IPC handles exchanged once over ``group`` (any torch.distributed
    backend; gloo works).  Ranks living in one process (tests) are linked
    with ``PeerAllReduce.link`` instead."""

    def __init__(self, rank: int, world: int, capacity_bytes: int, device=None, max_ctas: int = 0):
        from . import _lib

        self._lib = _lib
        self.rank, self.world, self.capacity = rank, world, int(capacity_bytes)
        h = _lib.C.c_int64()
        _lib.check(_lib.lib.tf_ar_create(rank, world, self.capacity, max_ctas, _lib.C.byref(h)), "tf_ar_create")
        self.handle = h.value
        ptr = _lib.lib.tf_ar_buffer(self.handle)

        class _Cai:  # zero-copy torch view of the library-owned buffer
            __cuda_array_interface__ = {"shape": (self.capacity // 2,), "typestr": "<i2", "data": (ptr, False),
                                        "version": 2}

        self._buf = torch.as_tensor(_Cai(), device=device or torch.device("cuda", torch.cuda.current_device()))
        self._buf = self._buf.view(torch.bfloat16)

    @classmethod
    def from_group(cls, rank: int, world: int, capacity_bytes: int, group=None, device=None,
                   max_ctas: int = 0) -> "PeerAllReduce":
        self = cls(rank, world, capacity_bytes, device, max_ctas)
        C = self._lib.C
        mine = (C.c_uint8 * 128)()
        self._lib.check(self._lib.lib.tf_ar_export(self.handle, mine), "tf_ar_export")
        every = [None] * world
        dist.all_gather_object(every, bytes(mine), group=group)
        allh = (C.c_uint8 * (128 * world)).from_buffer_copy(b"".join(every))
        self._lib.check(self._lib.lib.tf_ar_open(self.handle, allh), "tf_ar_open")
        return self

    @staticmethod
    def link(ranks) -> None:
        """Same-process ranks (one per thread / stream): every rank sees the
        others' buffers directly."""
        from . import _lib

        n = len(ranks)
        data = (_lib.C.c_void_p * n)(*[_lib.lib.tf_ar_buffer(r.handle) for r in ranks])
        ctl = (_lib.C.c_void_p * n)(*[_lib.lib.tf_ar_ctl(r.handle) for r in ranks])
        for r in ranks:
            _lib.check(_lib.lib.tf_ar_set_peers(r.handle, data, ctl), "tf_ar_set_peers")

    def fits(self, rows: int, dim: int) -> bool:
        return rows * dim * 2 <= self.capacity

    def partial(self, rows: int, dim: int) -> torch.Tensor:
        """[rows, dim] bf16 view of this rank's registered buffer (GEMM output)."""
        return self._buf[: rows * dim].view(rows, dim)

    def residual_rmsnorm(self, x, gamma, h_out, eps, stream=None) -> None:
        """x += sum over ranks of partial(x.shape); h_out = rmsnorm(x) * gamma."""
        C = self._lib.C
        rows, dim = x.shape
        st = stream if stream is not None else torch.cuda.current_stream()
        self._lib.check(self._lib.lib.tf_ar_residual_rmsnorm(
            self.handle, C.c_void_p(x.data_ptr()), C.c_void_p(gamma.data_ptr()) if gamma is not None else None,
            C.c_void_p(h_out.data_ptr()) if h_out is not None else None, rows, dim, eps,
            C.c_void_p(st.cuda_stream)), "tf_ar_residual_rmsnorm")

    def status(self) -> int:
        return int(self._lib.lib.tf_ar_status(self.handle))

    def close(self) -> None:
        if self.handle:
            self._buf = None
            self._lib.lib.tf_ar_destroy(self.handle)
            self.handle = 0
