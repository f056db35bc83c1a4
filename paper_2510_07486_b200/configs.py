"""The workloads of BASELINE.json `configs`."""
from __future__ import annotations

from dataclasses import dataclass, replace


@dataclass(frozen=True)
class Config:
    name: str
    index: int          # position in BASELINE.json configs (seed = 20251008 + 1000 * index)
    batch: int
    n_q_heads: int
    n_kv_heads: int
    head_dim: int
    seq_len: int
    top_k: int
    window: int
    v_head_dim: int = 0   # 0: head_dim.  Absorbed MLA: keys are the 576-dim latent
                          # (+ rope), values its first 512 dims

    @property
    def group(self) -> int:
        return self.n_q_heads // self.n_kv_heads

    def core_bytes(self, kv_heads: int | None = None) -> int:
        """North-star headline bytes: full-K read + selected K and V reads."""
        h = self.n_kv_heads if kv_heads is None else kv_heads
        D2 = self.head_dim * 2
        return self.batch * h * self.seq_len * D2 + 2 * self.batch * h * self.top_k * D2

    def with_(self, **kw) -> "Config":
        return replace(self, **kw)


TINY = Config("tiny", 0, 1, 2, 1, 64, 256, 32, 4)
QWEN3_8B = Config("qwen3-8b_b32_ctx32k", 1, 32, 32, 8, 128, 32768, 2048, 16)
QWEN3_32B = Config("qwen3-32b_b64_ctx32k", 2, 64, 64, 8, 128, 32768, 2048, 16)


# NEXT-3 attention variants: absorbed MLA as MQA over the latent
# (DeepSeek-V2-Lite: 16 heads; 576 = 512 latent + 64 rope dims, values = the
# latent), and multi-query attention with 64 query heads on one KV head
MLA_16 = Config("mla16_b16_ctx32k", 0, 16, 16, 1, 576, 32768, 2048, 16, v_head_dim=512)
MQA_64 = Config("mqa64_b32_ctx32k", 0, 32, 64, 1, 128, 32768, 2048, 16)


def long_cot(seq_len: int) -> Config:
    return Config(f"long-cot_b8_ctx{seq_len}", 3, 8, 64, 8, 128, seq_len, seq_len // 16, 16)


def high_concurrency(batch: int) -> Config:
    return Config(f"high-conc_b{batch}_ctx4k", 4, batch, 32, 8, 128, 4096, 256, 16)


BY_NAME = {c.name: c for c in (TINY, QWEN3_8B, QWEN3_32B, MLA_16, MQA_64)}


def by_name(name: str) -> Config:
    """A config by name: the three fixed ones, or a sweep point such as
    'long-cot_b8_ctx524288' / 'high-conc_b512_ctx4k' (configs [3], [4])."""
    if name in BY_NAME:
        return BY_NAME[name]
    if name.startswith("long-cot_b8_ctx"):
        return long_cot(int(name.rsplit("ctx", 1)[1]))
    if name.startswith("high-conc_b") and name.endswith("_ctx4k"):
        return high_concurrency(int(name[len("high-conc_b"):-len("_ctx4k")]))
    raise KeyError(f"unknown config {name!r}")
