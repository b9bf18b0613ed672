"""Model shapes (reading R1).

PAPER.md l.380 names only "Qwen3 ... 1.7B and 8B"; the shapes below are the
public Qwen3 config.json values (SURVEY.md §8 shape table).  The tiny shape is
BASELINE.json configs[0] ("2 layers, d=64, 4 heads, vocab 256") with head_dim
128 and 2 KV heads (reading R1 / SURVEY C1), so one kernel specialisation
(head_dim = 128) serves every shape.
"""
from dataclasses import dataclass


@dataclass(frozen=True)
class ModelShape:
    name: str
    layers: int
    hidden: int
    n_q_heads: int
    n_kv_heads: int
    head_dim: int
    ffn: int
    vocab: int
    rms_eps: float = 1e-6
    rope_theta: float = 1e6

    @property
    def q_dim(self):
        return self.n_q_heads * self.head_dim

    @property
    def kv_dim(self):
        return self.n_kv_heads * self.head_dim


SHAPES = {
    "tiny": ModelShape("tiny", 2, 64, 4, 2, 128, 192, 256),
    "qwen3-0.6b": ModelShape("qwen3-0.6b", 28, 1024, 16, 8, 128, 3072, 151936),
    "qwen3-1.7b": ModelShape("qwen3-1.7b", 28, 2048, 16, 8, 128, 6144, 151936),
    "qwen3-4b": ModelShape("qwen3-4b", 36, 2560, 32, 8, 128, 9728, 151936),
}
