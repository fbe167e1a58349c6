"""CPython 3.12 ``sum()`` semantics (TEST ORACLE).

Since CPython 3.12 the builtin ``sum`` adds floats with Neumaier's
compensated algorithm (Objects/bltinmodule.c builtin_sum_impl); the
reference's float sums (scheduler.py:191-193, :249-250; engine.py:1066-1067;
metrics.py:122-124, :152) therefore are NOT plain left-to-right adds.  This
restates that loop so the oracle (and the CUDA selector) reproduce them bit
for bit.
"""
from __future__ import annotations

import math


def pysum(values):
    it = iter(values)
    acc = 0
    for x in it:
        if isinstance(x, float):
            f = acc + x
            c = 0.0
            for y in it:
                y = float(y)
                t = f + y
                if abs(f) >= abs(y):
                    c += (f - t) + y
                else:
                    c += (y - t) + f
                f = t
            if c and math.isfinite(c):
                f += c
            return f
        acc += x
    return acc
