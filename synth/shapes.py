"""Model shape presets.

The paper names its models only ("LLaMA-2 ... LLaMA-3 variants", PAPER.md
§4.1; Tab.2).  Shapes, RoPE constants and eps are taken from
the public HF configs of those model names (reading R19, SURVEY.md
§8(d) table).  The two toy shapes are BASELINE.json configs[0].
"""
from __future__ import annotations

from dataclasses import dataclass, replace


@dataclass(frozen=True)
class ModelShape:
    name: str
    vocab: int
    d_model: int
    n_layers: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    d_ffn: int
    rms_eps: float = 1e-5
    rope_theta: float = 10000.0
    rope_kind: int = 0          # 0 = plain rotate-half, 1 = llama3 frequency scaling
    rope_factor: float = 1.0
    lo_ff: float = 1.0          # llama3 low_freq_factor
    hi_ff: float = 4.0          # llama3 high_freq_factor
    rope_orig_max: int = 8192   # llama3 original_max_position_embeddings
    tied: bool = False

    @property
    def q_dim(self) -> int:
        return self.n_heads * self.head_dim

    @property
    def kv_dim(self) -> int:
        return self.n_kv_heads * self.head_dim

    def n_params(self) -> int:
        per_layer = (self.d_model * (self.q_dim + 2 * self.kv_dim) + self.q_dim * self.d_model
                     + 3 * self.d_model * self.d_ffn + 2 * self.d_model)
        emb = self.vocab * self.d_model
        return self.n_layers * per_layer + emb * (1 if self.tied else 2) + self.d_model

    def streamed_bytes_per_pass(self, rows: int = 1) -> int:
        """bf16 bytes every forward pass must read from HBM for the weights:
        all linear layers + lm_head + norms + `rows` embedding rows."""
        per_layer = 2 * (self.d_model * (self.q_dim + 2 * self.kv_dim) + self.q_dim * self.d_model
                         + 3 * self.d_model * self.d_ffn + 2 * self.d_model)
        return self.n_layers * per_layer + 2 * self.vocab * self.d_model + 2 * self.d_model \
            + rows * 2 * self.d_model

    def kv_bytes_per_token_bf16(self) -> int:
        """KV-cache bytes per token of a plain bf16 cache."""
        return self.n_layers * 2 * self.kv_dim * 2

    def kv_bytes_per_token(self) -> int:
        """KV-cache bytes per token as stored by the CUDA path: K and V, each a
        split-bf16 pair (hi + lo planes, reading R28), i.e. 4 bytes
        per element."""
        return self.n_layers * 2 * self.kv_dim * 4


PRESETS = {
    # BASELINE.json configs[0]
    "toy-drafter": ModelShape("toy-drafter", 256, 64, 2, 1, 1, 64, 256, 1e-5, 1e4),
    "toy-verifier": ModelShape("toy-verifier", 256, 128, 4, 2, 1, 64, 512, 1e-5, 1e4),
    # tensor-parallel toy (heads, KV heads, vocab divisible by 1, 2 and 4; d_ffn by 64*4)
    "toy-tp": ModelShape("toy-tp", 1024, 512, 2, 8, 4, 64, 1024, 1e-5, 1e4),
    # paper-style LLaMA-2 hierarchy (Tab.2)
    "llama-68m": ModelShape("llama-68m", 32000, 768, 2, 12, 12, 64, 3072, 1e-6, 1e4),
    "llama2-7b": ModelShape("llama2-7b", 32000, 4096, 32, 32, 32, 128, 11008, 1e-5, 1e4),
    "llama2-13b": ModelShape("llama2-13b", 32000, 5120, 40, 40, 40, 128, 13824, 1e-5, 1e4),
    # LLaMA-3.x hierarchy (Tab.2)
    "llama3.2-1b": ModelShape("llama3.2-1b", 128256, 2048, 16, 32, 8, 64, 8192, 1e-5, 5e5,
                              1, 32.0, 1.0, 4.0, 8192, True),
    "llama3.1-8b": ModelShape("llama3.1-8b", 128256, 4096, 32, 32, 8, 128, 14336, 1e-5, 5e5,
                              1, 8.0, 1.0, 4.0, 8192, False),
    "llama3.1-70b": ModelShape("llama3.1-70b", 128256, 8192, 80, 64, 8, 128, 28672, 1e-5, 5e5,
                               1, 8.0, 1.0, 4.0, 8192, False),
}


def preset(name: str) -> ModelShape:
    return PRESETS[name]


def reduced_depth(shape: ModelShape, n_layers: int) -> ModelShape:
    """Same widths, fewer layers (oracle parity at full width)."""
    return replace(shape, name=f"{shape.name}-L{n_layers}", n_layers=n_layers)
