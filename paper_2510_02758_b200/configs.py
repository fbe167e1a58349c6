"""Named workload configurations (BASELINE.json ``configs``).

C1  reference CPU workload: 32-request burst on a tiny random-init decoder
    (2 layers, d=256, 4 q / 2 kv heads, hd 64, paged KV block 16).  The
    scheduler/cost parameters are SURVEY.md 8(d)'s oracle config.
C2  Llama3-8B bf16, 1xB200, 256-request Poisson burst (lambda=10, first 256
    arrivals of a 30 s trace, seed 1) with the KV pool capped at 163,840
    tokens (20 GiB, 10,240 blocks) so that about 25% of the burst's peak
    footprint fits (the paper's mem-frac=0.3).
C3  C2 request-sharded over G replicas (request i -> replica i mod G).
C4  Qwen2.5-32B bf16, tensor-parallel over TP = 1/2/4/8 B200s (NCCL), the C2
    request population and ledger (163,840 tokens; 256 KiB of KV per token,
    split over the TP ranks' pools and host links).
C5  KV swap sweep (block counts 1..64K) - see bench_swap.py.

Each config can build the reference-shaped dataclasses from *any* module
that defines ``SimConfig``/``CostModel``/``SchedulerConfig`` with the
reference's field names, so the same numbers feed the golden-fixture
generator (reference classes) and this package (mirror classes).
"""
from __future__ import annotations

from dataclasses import dataclass, field


@dataclass(frozen=True)
class ModelShape:
    name: str
    n_layers: int
    hidden: int
    n_q_heads: int
    n_kv_heads: int
    head_dim: int
    ffn: int
    vocab: int
    rope_theta: float = 500000.0
    rms_eps: float = 1e-5
    qkv_bias: bool = False  # Qwen2 family: bias on the q/k/v projections

    @property
    def kv_bytes_per_token_layer(self) -> int:
        # K and V, bf16
        return 2 * self.n_kv_heads * self.head_dim * 2

    @property
    def kv_bytes_per_token(self) -> int:
        return self.kv_bytes_per_token_layer * self.n_layers


TINY = ModelShape("tiny-decoder", n_layers=2, hidden=256, n_q_heads=4, n_kv_heads=2,
                  head_dim=64, ffn=688, vocab=4096, rope_theta=10000.0)
LLAMA3_8B = ModelShape("llama3-8b", n_layers=32, hidden=4096, n_q_heads=32, n_kv_heads=8,
                       head_dim=128, ffn=14336, vocab=128256)
QWEN25_32B = ModelShape("qwen2.5-32b", n_layers=64, hidden=5120, n_q_heads=40, n_kv_heads=8,
                        head_dim=128, ffn=27648, vocab=152064, rope_theta=1000000.0, rms_eps=1e-6,
                        qkv_bias=True)


@dataclass(frozen=True)
class ServingConfig:
    name: str
    model: ModelShape
    n_requests: int
    seed: int
    prompt_len_dist: tuple
    output_len_dist: tuple
    rate_profile: tuple  # ((rate, weight), ...)
    # SimConfig
    gpu_mem_tokens: int
    max_batch: int
    cpu_mem_tokens: int
    chunk_tokens: int
    write_through_min_tokens: int
    # CostModel (virtual-time replay; seconds / tokens-per-second)
    cost: dict = field(default_factory=dict)
    # SchedulerConfig
    sched: dict = field(default_factory=dict)
    arrivals: str = "burst"
    poisson_rate: float | None = None
    duration: float | None = None
    block_tokens: int = 16

    def sim_cfg(self, cls, **kw):
        base = dict(
            gpu_mem_tokens=self.gpu_mem_tokens,
            max_batch=self.max_batch,
            cpu_mem_tokens=self.cpu_mem_tokens,
            chunk_tokens=self.chunk_tokens,
            write_through_min_tokens=self.write_through_min_tokens,
        )
        base.update(kw)
        return cls(**base)

    def cost_model(self, cls, **kw):
        base = dict(self.cost)
        base.update(kw)
        return cls(**base)

    def sched_cfg(self, cls, **kw):
        base = dict(self.sched)
        base.update(kw)
        return cls(**base)


C1 = ServingConfig(
    name="c1-burst32-tiny",
    model=TINY,
    n_requests=32,
    seed=7,
    prompt_len_dist=(128.0, 32.0),
    output_len_dist=(512.0, 128.0),
    rate_profile=((15.0, 0.4), (20.0, 0.6)),
    gpu_mem_tokens=4096,
    max_batch=8,
    cpu_mem_tokens=32768,
    chunk_tokens=128,
    write_through_min_tokens=16,
    cost=dict(prefill_per_token=4e-5, decode_base=8e-4, decode_per_request=8e-5,
              decode_per_ctx_token=2e-8, h2d_bandwidth=150000, d2h_bandwidth=150000),
    sched=dict(schedule_interval=0.5, per_request_mem_estimate=640.0, buffer_safety_factor=2.0,
               tau_schedule=0.5, critical_buffer_seconds=1.0, pacing_buffer_seconds=8.0),
)

# B200 cost-model priors for Llama3-8B (virtual-time replay and the policy's
# estimates before the first measured sample):
#   prefill  ~16 GFLOP/token at ~0.8 PFLOP/s                 -> 2e-5 s/token
#   decode   16 GB of weights at ~6.5 TB/s + launch overhead -> 3e-3 s/iteration
#   per ctx  128 KiB of KV per token at ~6.5 TB/s            -> 2e-8 s/token
#   PCIe     ~55 GB/s per direction / 128 KiB per token       -> 420,000 tokens/s
C2 = ServingConfig(
    name="c2-llama3-8b-poisson256",
    model=LLAMA3_8B,
    n_requests=256,
    seed=1,
    prompt_len_dist=(512.0, 128.0),
    output_len_dist=(2048.0, 512.0),
    rate_profile=((15.0, 0.4), (20.0, 0.6)),
    gpu_mem_tokens=163840,
    max_batch=128,
    cpu_mem_tokens=655360,
    chunk_tokens=512,
    write_through_min_tokens=16,
    cost=dict(prefill_per_token=2e-5, decode_base=3e-3, decode_per_request=2e-5,
              decode_per_ctx_token=2e-8, h2d_bandwidth=420000, d2h_bandwidth=420000),
    sched=dict(schedule_interval=0.5, per_request_mem_estimate=3100.0, buffer_safety_factor=2.0,
               tau_schedule=0.5, critical_buffer_seconds=1.0, pacing_buffer_seconds=8.0),
    arrivals="poisson",
    poisson_rate=10.0,
    duration=30.0,
)



def c4(tp: int = 1) -> ServingConfig:
    """C4 at tensor-parallel degree ``tp``.  Cost-model priors per rank:
    decode 65.5 GB / TP of weights at ~6.5 TB/s + launch overhead; 256 KiB / TP
    of KV per context token; prefill ~64 GFLOP/token / TP at ~0.8 PFLOP/s;
    PCIe ~55 GB/s per rank link / (256 KiB / TP) per token."""
    from dataclasses import replace

    return replace(
        C2, name=f"c4-qwen2.5-32b-tp{tp}", model=QWEN25_32B,
        cost=dict(prefill_per_token=8e-5 / tp, decode_base=10.5e-3 / tp, decode_per_request=4e-5 / tp,
                  decode_per_ctx_token=4e-8 / tp, h2d_bandwidth=210000 * tp, d2h_bandwidth=210000 * tp),
        sched=dict(C2.sched, per_request_mem_estimate=3100.0))


CONFIGS = {"c1": C1, "c2": C2, "c4": c4(1)}
