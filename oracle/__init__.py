"""CPU oracle for the TokenFlow KV-movement hot path.

TEST INFRASTRUCTURE ONLY.  Nothing under ``oracle/`` is part of the product:
only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import it, and only as the
checker (or as the timed CPU reference arm), never as the thing measured or
shipped.  The product path (``paper_2510_02758_b200``) never imports it and
fails loudly when its CUDA library is missing.

Contents (each function cites the reference file:line it restates; paths
are relative to /root/reference/pkg/src):

* ``refsim``    - a restatement of the reference simulator (tokensim):
                  planner (kvstore.py), policies (scheduler.py), the
                  discrete-event engine (engine.py), cost model (costs.py),
                  metrics (metrics.py) and the trace CSV loader
                  (workload.py).  Pinned against golden fixtures produced by
                  the unmodified reference (tests/golden/, made by
                  tools/make_golden.py): event hashes, decision logs,
                  chunk-transfer rows, per-request records.
* ``dataplane`` - the CPU restatement of what the reference leaves unpinned
                  (SURVEY.md 8c): a deterministic paged block allocator and
                  block tables, token-range residency, byte movement between
                  a CPU "HBM pool" and a CPU "host store", synthetic KV
                  contents, and fp32 paged decode attention.
* ``cpu_baseline`` - the CPU restatement of one C2 decode step (model
                  forward, fp32 attention, swap gather, on_tick), timed on
                  the host cores for bench.py's ``cpu_baseline`` and
                  ``--impl reference`` legs.

Parity pin: decisions/schedules are pinned by the reference's own outputs
(golden fixtures).  Block tables, swapped bytes and attention are pinned by
construction rules derived from the reference's token-count semantics
(engine.py:571-617, :817-917, :510-540; kvstore.py:144-170) - the reference
has no tensors, so those rows are "restated, not reference-executed".
"""
