"""Real-time serving loop over the GPU data plane (measured clock).

Same handlers and policy as the replay engine (engine.py), but time is the
wall clock and every duration comes from the hardware:

* a decode iteration / prefill is launched on the compute stream and
  completes when its CUDA end event fires; the engine time of completion is
  the event's device timestamp (cudaEventElapsedTime from an anchor event),
  so the reported ``iter_time`` is the kernels' real duration;
* write-through / evict chunks run on the evict stream and loads on the
  load stream concurrently with decode (the reference's full-duplex PCIe
  pair, engine.py:235-247); their measured token rates feed
  ``update_rate_ema`` exactly like the reference's simulated ones;
* readers consume on the same clock at their configured rates.

``lockstep`` (tensor parallelism, C4): every TP rank runs this same engine
on its own shard; completions are agreed with one small collective per
loop iteration (``Lockstep.agree``: a completion counts once it fired on
EVERY rank, at the LATEST rank's time; the clock is the earliest rank's), so
all ranks see the same event sequence at the same times and the
deterministic engine + bit-exact selector take identical decisions with no
decision broadcast.

``skip_idle``: when the GPU and both copy streams are idle and the next
event is a reader / arrival / tick in the future, the clock jumps to it
instead of sleeping (nothing is in flight, so no measured duration spans a
jump).  Busy periods run at true wall-clock speed, so copy/compute overlap
is real; only idle gaps are compressed.  A run therefore takes about the
GPU's busy time instead of the readers' reading time.
"""
from __future__ import annotations

import heapq
import math
import time

from .engine import (
    _ORDER,
    CHUNK_TRANSFER_DONE,
    DECODE_ITER_DONE,
    PREFILL_DONE,
    PREFILL_WAIT,
    PREFILLING,
    DeadlockError,
    Engine,
    _Job,
)


class RealtimeEngine(Engine):
    def __init__(self, trace, policy, cm, sim, dataplane, skip_idle: bool = True, on_step=None, max_steps=None,
                 lockstep=None, max_wall_s=None):
        super().__init__(trace, policy, cm, sim, dataplane)
        self.lockstep = lockstep
        self.max_wall_s = max_wall_s  # stop (truncated) after this much wall time
        self.truncated = False
        assert dataplane is not None and dataplane.mode == "realtime"
        self.skip_idle = skip_idle
        self.on_step = on_step  # callback(record dict) after every decode iteration
        self.max_steps = max_steps
        self.steps = []  # per decode iteration: start, end, batch size, produced, effective weight
        self.jobs = []  # every GPU job (decode and prefill): (kind, start, end, device seconds)
        self._gpu = None  # (kind, payload, start_time, end_event)
        self._lanes = {"d2h": None, "h2d": None}  # (start_time, end_event)
        self._anchor = None
        self.skipped_s = 0.0
        self.wall_s = 0.0
        self._stop = False
        self._defer_wt, self._wt_deferred = False, None

    # ------------------------------------------ write-through after dispatch
    # The reference plans the next write-through chunks and then dispatches the
    # next GPU job at the same instant (engine.py _on_decode_iter_done /
    # _on_prefill_done).  Nothing in the dispatch depends on the plan (d2h
    # chunks change no HBM accounting), so in real time the dispatch goes
    # first: the host work of planning and starting a copy (a selector call
    # and a d2h launch, ~0.1 ms) no longer sits between a decode step's end
    # and the next step's launch.
    def _on_decode_iter_done(self, time, subject, batch, iter_time):
        self._defer_wt = True
        try:
            super()._on_decode_iter_done(time, subject, batch, iter_time)
        finally:
            self._defer_wt = False
        self._flush_deferred_wt()

    def _on_prefill_done(self, time, subject, job, duration):
        self._defer_wt = True
        try:
            super()._on_prefill_done(time, subject, job, duration)
        finally:
            self._defer_wt = False
        self._flush_deferred_wt()

    def _plan_write_through(self, time):
        if self._defer_wt:
            self._wt_deferred = time
            return
        super()._plan_write_through(time)

    def _flush_deferred_wt(self):
        if self._wt_deferred is not None:
            t, self._wt_deferred = self._wt_deferred, None
            super()._plan_write_through(t)

    # ------------------------------------------------- fused write-through
    def _after_decode_commit(self, produced):
        if not self.dp.fused_wt:
            return
        for rid in produced:
            kv = self.state[rid].kv
            kv.cpu_synced = self.dp.host_frontier(rid, kv.cpu_synced, kv.total_kv)

    def _after_d2h_land(self, rid):
        if self.dp.fused_wt:
            kv = self.state[rid].kv
            kv.cpu_synced = self.dp.host_frontier(rid, kv.cpu_synced, kv.total_kv)

    # ------------------------------------------------------------------ clock
    def _clock(self) -> float:
        return time.perf_counter() - self._t0 + self.skipped_s

    def shift_clock(self, dt: float):
        """Exclude ``dt`` seconds of wall time (e.g. a measurement pause) from the
        serving clock."""
        self._t0 += dt
        self._reanchor()

    def _reanchor(self):
        ev = self.dp.record_event()
        ev.synchronize()
        self._anchor = (ev, self._clock())

    def _event_time(self, ev) -> float:
        a, t = self._anchor
        return t + a.elapsed_time(ev) / 1e3

    # ------------------------------------------------------------ dispatching
    def _dispatch_gpu(self, time_):
        if self.gpu_job is not None:
            return
        start = time_
        prefer_decode = (self.policy.interleave_prefill_chunks and self._last_gpu_kind == "prefill"
                         and bool(self._decode_candidates()))
        if self.prefill_queue and not prefer_decode:
            job = self.prefill_queue[0]
            need = sum(job.reserve.values())
            if need <= self._mem_free():
                self.prefill_queue.popleft()
                for rid in job.members:
                    self._uncommit(rid, job.reserve[rid])
                    if self.state[rid].status == PREFILL_WAIT:
                        self.state[rid].status = PREFILLING
                self._mem_acquire(need)
                ev0 = self.dp.record_event()
                self.dp.fill_start(job, self)
                self.gpu_job = job
                self._gpu = ("prefill", job, start, self._end_event(), ev0)
                return
        chosen = self._decode_candidates()
        if not chosen:
            return
        free = max(0, self._growth_budget())
        if len(chosen) > free:
            chosen = self._shed_for_memory(time_, chosen, free)
        if not chosen:
            return
        batch = tuple(chosen)
        ev0 = self.dp.record_event()
        self.dp.decode_start(batch, self)
        self.gpu_job = ("decode", batch)
        self._gpu = ("decode", batch, start, self._end_event(), ev0)

    def _end_event(self):
        return self.dp.record_event()

    def _start_channel(self, time_, ch_):
        if ch_.in_service is not None or not ch_.queue:
            return
        head = ch_.queue[0]
        if ch_.direction == "h2d":
            if not self.sim.overlap and self.d2h.carries("evict"):
                return
            if head.tokens > self._mem_free() - self.mem_committed:
                return
            self._mem_acquire(head.tokens)
        ch_.queue.popleft()
        ch_.in_service = head
        ch_.started = time_
        ev0, ev1 = (self.dp.d2h_start if ch_.direction == "d2h" else self.dp.h2d_start)(head, self)
        self._lanes[ch_.direction] = (time_, ev1, ev0)

    # ------------------------------------------------------------------- loop
    def _poll_completions(self):
        """-> (progressed, clock).  A job's duration is its DEVICE span (start
        event recorded just before its launch .. end event), so host lag in
        issuing it (e.g. while Python enqueues a long prefill) is not charged to
        the job - the measured rates that feed update_rate_ema / the policy's
        t_io (kvstore.py:173-193, :255-259) see only the transfer itself.
        Lockstep: done flags, end and start times and the clock are agreed
        over the TP ranks."""
        slots = (("gpu", self._gpu, 0), ("d2h", self._lanes["d2h"], 1), ("h2d", self._lanes["h2d"], 1))
        # the clock is read BEFORE the events are queried: a job not observed
        # done below finishes after `clock`, so draining the heap up to `clock`
        # can never run an event that a still-unobserved completion precedes
        clock = self._clock()
        flags, ends, starts = [], [], []
        for what, v, _ in slots:
            # v = (host start time, end event, start event)
            ok = v is not None and v[1 if what != "gpu" else 3].query()
            flags.append(ok)
            if ok:
                e_end, e_start = (v[3], v[4]) if what == "gpu" else (v[1], v[2])
                st = max(v[2] if what == "gpu" else v[0], self._event_time(e_start))
                starts.append(st)
                ends.append(max(self._event_time(e_end), st))
            else:
                starts.append(0.0)
                ends.append(0.0)
        if self.lockstep is not None:
            clock, flags, ends, starts = self.lockstep.agree(clock, flags, ends, starts)
        done = [(t, order, what, s0) for (what, _, order), ok, t, s0 in zip(slots, flags, ends, starts) if ok]
        if not done:
            return False, clock
        done.sort()
        for t, _, what, s0 in done:
            kind_done = (PREFILL_DONE if self._gpu[0] == "prefill" else DECODE_ITER_DONE) if what == "gpu" \
                else CHUNK_TRANSFER_DONE
            self._drain_heap((t, _ORDER[kind_done]))
            self.now = max(self.now, t)
            if what == "gpu":
                kind, payload = self._gpu[0], self._gpu[1]
                self._gpu = None
                dur = max(t - s0, 1e-9)
                self.jobs.append((kind, s0, t, dur))
                if kind == "prefill":
                    self._on_prefill_done(t, min(payload.members), payload, dur)
                else:
                    n_before = len(self.steps)
                    self._record_step(payload, s0, t, dur)
                    self._on_decode_iter_done(t, min(payload), payload, dur)
                    self._finish_step(n_before)
            else:
                self._lanes[what] = None
                ch_ = self.d2h if what == "d2h" else self.h2d
                ch_.started = max(ch_.started, s0)
                self._on_chunk_transfer_done(t, -1, what)
        return True, clock

    def _record_step(self, batch, start, end, dur):
        self._step_pre = {r: (self.state[r].status, self.state[r].generated) for r in batch}
        self.steps.append({"start": start, "end": end, "dur": dur, "batch": len(batch), "rids": list(batch)})

    def _finish_step(self, idx):
        rec = self.steps[idx]
        made, eff = 0, 0.0
        for rid, (_, g0) in self._step_pre.items():
            st = self.state[rid]
            if st.generated > g0:
                made += 1
                b = st.record.buffer_at_gen[-1]
                lo, hi = 0.10 * st.spec.output_len, 0.20 * st.spec.output_len
                eff += 1.0 if b < lo else (0.0 if b >= hi else (hi - b) / (hi - lo))
        rec["tokens"], rec["effective"] = made, eff
        if self.on_step is not None:
            self.on_step(rec, self)
        if self.max_steps is not None and len(self.steps) >= self.max_steps:
            self._stop = True

    def _drain_heap(self, until) -> bool:
        """Process queued events strictly before ``until`` = (time, kind order):
        a completion observed late is handled only after every event that
        precedes it (discrete-event order of the reference, engine.py _ORDER)."""
        ran = False
        while self._heap and self._heap[0][:2] < until:
            t, _, subject, seq = heapq.heappop(self._heap)
            kind, payload = self._payload.pop(seq)
            self.now = max(self.now, t)
            self._last_event_time = self.now
            self._handlers[kind](t, subject, *payload)
            ran = True
            if self.live == 0 or self._stop:
                break
        return ran

    def run(self):
        for r in self.trace.requests:
            self._push(r.arrival_time, "arrival", r.id)
        self._push(0.0, "schedule_tick", -1)
        self._handlers = {"arrival": self._on_arrival, "schedule_tick": self._on_schedule_tick,
                          "request_done": self._on_request_done, "consume": self._on_consume}
        self._t0 = time.perf_counter()
        self._reanchor()
        wall0 = time.perf_counter()
        idle_spins = 0
        while self.live > 0 and not self._stop:
            if self.max_wall_s is not None and time.perf_counter() - wall0 > self.max_wall_s:
                self.truncated = True
                break
            progressed, now = self._poll_completions()
            if self.live > 0 and not self._stop and self._drain_heap((now, math.inf)):
                progressed = True
            if progressed:
                idle_spins = 0
                continue
            busy = self._gpu is not None or any(v is not None for v in self._lanes.values())
            if not busy:
                if not self._heap:
                    raise DeadlockError(f"{self.live} requests incomplete but nothing is scheduled")
                gap = self._heap[0][0] - now
                if gap > 0:
                    if self.skip_idle:
                        self.skipped_s += gap
                        self._reanchor()
                    else:
                        time.sleep(min(gap, 0.01))
            else:
                # waiting on the device: keep polling (a timed sleep oversleeps by
                # ~50 us, which would sit between every job and the next
                # dispatch); yield the GIL now and then for the clock sampler
                idle_spins += 1
                if idle_spins % 256 == 0:
                    time.sleep(0)
        self.dp.synchronize()
        self.wall_s = time.perf_counter() - wall0
        self._last_event_time = max(self._last_event_time, self.now)
        return self._result()

    def _result(self):
        from .engine import SimResult

        records = [self.state[r.id].record for r in self.trace.requests]
        return SimResult(self.policy.name, records, self.event_log, self.decision_log, self._last_event_time,
                         self.total_preemptions, self.total_recomputes,
                         list(getattr(self.policy, "mode_changes", [])), dict(self.dp.stats))
