"""Tensor parallelism for the C4 configuration (Qwen2.5-32B over NVLink).

SURVEY 8(e): TP is the one configuration with a real exchange step.  Each TP
rank holds 1/TP of every layer's attention heads and MLP columns, and its own
shard of the paged KV pool (n_kv_heads/TP heads per block), which it swaps
over its OWN host link - so swap bytes per rank are bytes/TP, in lockstep.

Two collectives, nothing else:

* data path: one NCCL all-reduce (sum) after o_proj and one after down_proj
  per layer (B x hidden bf16 each), on the compute stream
  (``model.PagedDecoder`` with ``tp=TpGroup(...)``);
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

    def __init__(self, rank: int, size: int, group=None):
        self.rank, self.size, self.group = rank, size, group

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
