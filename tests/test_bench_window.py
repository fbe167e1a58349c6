"""bench.py's window bookkeeping on the CPU: where the timed window sits on
the serving clock (`window_clock`: the ticks that moved requests) and the
window's device-time accounting (every GPU job inside it, prefills included)."""
import sys
from types import SimpleNamespace

from conftest import ROOT

sys.path.insert(0, str(ROOT))
import bench  # noqa: E402


def _eng(ticks, steps, jobs=()):
    return SimpleNamespace(decision_log=ticks, steps=steps, jobs=list(jobs),
                           policy=SimpleNamespace(cfg=SimpleNamespace(schedule_interval=0.5)))


def test_window_clock_lists_only_ticks_that_moved_requests():
    ticks = [{"time": 0.5, "mode": "buffer_aware", "preempted": [], "admitted": []},
             {"time": 2.0, "mode": "buffer_aware", "preempted": list(range(53)), "admitted": list(range(53, 106)),
              "resumed": [], "recomputed": []},
             {"time": 2.5, "mode": "buffer_aware", "preempted": [], "admitted": [], "resumed": [7]},
             {"time": 9.0, "mode": "buffer_aware", "preempted": [1], "admitted": []}]
    steps = [{"start": 1.9, "end": 1.906}, {"start": 1.95, "end": 2.1}]
    w = bench._window_clock(_eng(ticks, steps), steps)
    assert (w["start_s"], w["end_s"], w["first_decode_s"]) == (1.9, 2.1, 1.9)
    assert w["ticks_fired"] == 3  # up to one interval past the window's end
    moved = w["ticks_that_moved_requests"]
    assert [m["t"] for m in moved] == [2.0, 2.5]
    assert (moved[0]["preempted"], moved[0]["admitted"], moved[1]["resumed"]) == (53, 53, 1)


def test_window_stats_count_prefills_inside_the_window():
    steps = [{"start": 1.0, "end": 1.005, "effective": 100.0, "tokens": 128, "batch": 128},
             {"start": 1.2, "end": 1.205, "effective": 90.0, "tokens": 128, "batch": 128}]
    jobs = [("decode", 1.0, 1.005, 0.005), ("prefill", 1.01, 1.19, 0.18), ("decode", 1.2, 1.205, 0.005),
            ("prefill", 1.3, 1.4, 0.1)]  # the last one is after the window
    dp = SimpleNamespace(transfer_log=lambda: [("d2h", 16, 0.5), ("h2d", 32, 1.0)])
    st = bench._window_stats(_eng([], steps, jobs), dp, steps, 0, 2, 131072)
    assert st["dev_s"] == 0.19 and st["prefill_s"] == 0.18
    assert (st["eff"], st["toks"], st["batch_sum"]) == (190.0, 256, 256)
    assert (st["d2h_tok"], st["h2d_tok"], st["chunks"]) == (16, 32, 2)
