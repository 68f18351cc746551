"""Seeded random-init bf16 weights.

Every matrix is N(0, std^2) (std = 0.02, the HF default init; SURVEY.md
§8(c) c.1 #9 / reading R20), drawn in fp32 by torch's seeded generator on the
requested device and rounded to bf16.  Norm gains are 1 + gain_std * N(0,1)
rounded to bf16 (gain_std = 0.1 by default, so a swapped or dropped gain is
visible to the parity tests; gain_std = 0 gives HF's all-ones init).

Each tensor has its own generator seeded from (seed, layer, name), so a
reduced-depth model is a prefix of the full one on the same device.  CPU and
CUDA generators produce different streams: tests that compare the oracle with
the GPU path generate once and hand the same bf16 BYTES to both sides.

Layout: PyTorch nn.Linear row-major [out_features, in_features].
"""
from __future__ import annotations

import zlib

import numpy as np
import torch

from .shapes import ModelShape

LAYER_KEYS = ("wq", "wk", "wv", "wo", "wg", "wu", "wd", "n_attn", "n_mlp")


def _seed_of(seed: int, layer: int, name: str) -> int:
    return (zlib.crc32(f"{seed}/{layer}/{name}".encode()) * 2654435761 + seed) % (2 ** 63 - 1)


def _randn(shape, seed, layer, name, device, std):
    g = torch.Generator(device=device)
    g.manual_seed(_seed_of(seed, layer, name))
    t = torch.randn(*shape, generator=g, device=device, dtype=torch.float32)
    return (t * std).to(torch.bfloat16)


def _gain(n, seed, layer, name, device, gain_std):
    if gain_std == 0.0:
        return torch.ones(n, dtype=torch.bfloat16, device=device)
    g = torch.Generator(device=device)
    g.manual_seed(_seed_of(seed, layer, name))
    t = torch.randn(n, generator=g, device=device, dtype=torch.float32)
    return (1.0 + gain_std * t).to(torch.bfloat16)


def make_weights(shape: ModelShape, seed: int, device="cpu", std: float = 0.02,
                 gain_std: float = 0.1) -> dict:
    """Returns {'embed','lm_head','final_norm','layers':[{LAYER_KEYS...}]} of
    contiguous bf16 tensors on `device`.  lm_head is embed when shape.tied."""
    d, hq, hkv, f = shape.d_model, shape.q_dim, shape.kv_dim, shape.d_ffn
    w = {"embed": _randn((shape.vocab, d), seed, -1, "embed", device, std)}
    w["lm_head"] = w["embed"] if shape.tied else _randn((shape.vocab, d), seed, -1, "lm_head",
                                                        device, std)
    w["final_norm"] = _gain(d, seed, -1, "final_norm", device, gain_std)
    layers = []
    for l in range(shape.n_layers):
        layers.append({
            "wq": _randn((hq, d), seed, l, "wq", device, std),
            "wk": _randn((hkv, d), seed, l, "wk", device, std),
            "wv": _randn((hkv, d), seed, l, "wv", device, std),
            "wo": _randn((d, hq), seed, l, "wo", device, std),
            "wg": _randn((f, d), seed, l, "wg", device, std),
            "wu": _randn((f, d), seed, l, "wu", device, std),
            "wd": _randn((d, f), seed, l, "wd", device, std),
            "n_attn": _gain(d, seed, l, "n_attn", device, gain_std),
            "n_mlp": _gain(d, seed, l, "n_mlp", device, gain_std),
        })
    w["layers"] = layers
    return w


def _np64(t: torch.Tensor) -> np.ndarray:
    return t.detach().to("cpu").to(torch.float64).numpy()


def weights_to_numpy(w: dict) -> dict:
    """bf16 torch weights -> float64 numpy (exact: every bf16 is an fp64)."""
    out = {k: _np64(w[k]) for k in ("embed", "lm_head", "final_norm")}
    out["layers"] = [{k: _np64(v) for k, v in lw.items()} for lw in w["layers"]]
    return out


def make_weights_sharded(shape: ModelShape, seed: int, rank: int, tp: int, device="cpu", std: float = 0.02,
                         gain_std: float = 0.1) -> dict:
    """Rank `rank`'s Megatron shard of make_weights(shape, seed) (the layout of
    include/pipespec.h ps_placement: Q/K/V by heads, gate/up by FFN rows, O and
    down by the matching input columns, lm_head by vocabulary rows; embed and
    gains replicated), generated tensor by tensor so the full model is never
    resident (a 70B stage: 141 GB).  Bit-identical to slicing make_weights."""
    T, r = tp, rank
    d, hq, hkv, f = shape.d_model, shape.q_dim, shape.kv_dim, shape.d_ffn
    hd = shape.head_dim
    qh, kh, fr, vr = shape.n_heads // T, shape.n_kv_heads // T, f // T, shape.vocab // T

    def rows(t, a, b):
        return t[a:b].contiguous()

    def cols(t, a, b):
        return t[:, a:b].contiguous()

    embed = _randn((shape.vocab, d), seed, -1, "embed", device, std)
    full_lm = embed if shape.tied else _randn((shape.vocab, d), seed, -1, "lm_head", device, std)
    w = {"embed": embed, "lm_head": rows(full_lm, r * vr, (r + 1) * vr),
         "final_norm": _gain(d, seed, -1, "final_norm", device, gain_std)}
    del full_lm
    layers = []
    for l in range(shape.n_layers):
        layers.append({
            "wq": rows(_randn((hq, d), seed, l, "wq", device, std), r * qh * hd, (r + 1) * qh * hd),
            "wk": rows(_randn((hkv, d), seed, l, "wk", device, std), r * kh * hd, (r + 1) * kh * hd),
            "wv": rows(_randn((hkv, d), seed, l, "wv", device, std), r * kh * hd, (r + 1) * kh * hd),
            "wo": cols(_randn((d, hq), seed, l, "wo", device, std), r * qh * hd, (r + 1) * qh * hd),
            "wg": rows(_randn((f, d), seed, l, "wg", device, std), r * fr, (r + 1) * fr),
            "wu": rows(_randn((f, d), seed, l, "wu", device, std), r * fr, (r + 1) * fr),
            "wd": cols(_randn((d, f), seed, l, "wd", device, std), r * fr, (r + 1) * fr),
            "n_attn": _gain(d, seed, l, "n_attn", device, gain_std),
            "n_mlp": _gain(d, seed, l, "n_mlp", device, gain_std),
        })
    w["layers"] = layers
    return w
