import gzip
import json
import math
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running")


def load_golden(kind: str, name: str) -> dict:
    with gzip.open(GOLDEN / kind / f"{name}.json.gz") as f:
        return json.load(f)


def golden_names(kind: str) -> list:
    return sorted(p.name[: -len(".json.gz")] for p in (GOLDEN / kind).glob("*.json.gz"))


def trace_path(name: str) -> str:
    return str(GOLDEN / "traces" / f"{name}.csv")


def pool_blocks(sim: dict, n_requests: int) -> int:
    """Physical HBM blocks for a run: ledger capacity + per-request edge slack."""
    return math.ceil(sim["gpu_mem_tokens"] / 16) + 4 * n_requests + sim["max_batch"]


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda")
