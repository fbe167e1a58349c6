"""Trace CSV loading (restates workload.py:251-281 load_trace; TEST ORACLE)."""
from __future__ import annotations

import csv

from .sim import Req

HEADER = ["id", "arrival_s", "prompt_tokens", "output_tokens", "rate_tps"]


def read_trace(path) -> list:
    rows = []
    with open(path, newline="", encoding="utf-8") as f:
        for i, row in enumerate(csv.reader(f), start=1):
            if not row or (len(row) == 1 and not row[0].strip()):
                continue
            if i == 1 and [c.strip() for c in row] == HEADER:
                continue
            if len(row) != 5:
                raise ValueError(f"line {i}: expected 5 fields")
            rows.append(Req(int(row[0]), float(row[1]), int(row[2]), int(row[3]), float(row[4])))
    rows.sort(key=lambda r: (r.arrival_time, r.id))
    return rows
