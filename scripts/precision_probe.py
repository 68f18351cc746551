"""Where does the GPU path's logit error come from?  (measurement script)

Runs the LLaMA forward in float64 with torch on the GPU (NOT the oracle: a
probe with optional bf16 rounding at the points where the CUDA path holds a
bf16 value) and compares each variant with the CUDA path's logits for the
bench's verify window (8B shape, 512-token prompt, R = 5).  Prints
max|dlogit| / max|logit| of CUDA vs each variant, per depth.

Rounding points (all in the CUDA path): xg = the RMSNorm operand x*g of the
QKV / gate-up / lm_head GEMMs; att = attention output (O-proj operand);
h = SwiGLU output (down operand); kv = the K/V cache; q = the query operand of
QK^T; p = the softmax probabilities of PV.

Usage: python scripts/precision_probe.py [--layers 2,8,32] [--shape llama3.1-8b]
"""
import argparse
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synth
from oracle.llama import rope_inv_freq

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="llama3.1-8b")
ap.add_argument("--layers", default="0,1,2,8,32")
ap.add_argument("--ctx", type=int, default=512)
ap.add_argument("--variants", default="single", choices=["single", "all-but"])
a = ap.parse_args()


def bf(x, on):
    return x.to(torch.bfloat16).to(torch.float64) if on else x


def forward(s, w, tokens, R, rnd):
    dev = "cuda"
    T = len(tokens)
    H, Hkv, hd = s.n_heads, s.n_kv_heads, s.head_dim
    g = H // Hkv
    inv = torch.tensor(rope_inv_freq(s), dtype=torch.float64, device=dev)
    pos = torch.arange(T, device=dev, dtype=torch.float64)
    ang = pos[:, None] * inv[None, :]
    cos, sin = torch.cat([ang.cos(), ang.cos()], -1), torch.cat([ang.sin(), ang.sin()], -1)

    def rope(x):   # [T, h, hd]
        h2 = hd // 2
        rot = torch.cat([-x[..., h2:], x[..., :h2]], -1)
        return x * cos[:, None, :] + rot * sin[:, None, :]

    def norm(x, gain):
        # CUDA: (x*g) rounded to bf16, scaled by rstd after the GEMM (same value up to rounding)
        r = torch.rsqrt((x * x).mean(-1, keepdim=True) + s.rms_eps)
        return bf(x * gain, "xg" in rnd) * r

    t = torch.tensor(tokens, device=dev)
    x = w["embed"][t].double()
    mask = torch.ones(T, T, device=dev, dtype=torch.bool).tril()
    for lw in w["layers"]:
        W = {k: v.double() for k, v in lw.items()}
        h = norm(x, W["n_attn"])
        q = rope((h @ W["wq"].T).view(T, H, hd))
        k = bf(rope((h @ W["wk"].T).view(T, Hkv, hd)), "kv" in rnd or "k" in rnd)
        v = bf((h @ W["wv"].T).view(T, Hkv, hd), "kv" in rnd or "v" in rnd)
        q = bf(q / math.sqrt(hd), "q" in rnd)
        kk = k.repeat_interleave(g, dim=1)
        vv = v.repeat_interleave(g, dim=1)
        sc = torch.einsum("thd,shd->hts", q, kk).masked_fill(~mask, float("-inf"))
        p = torch.softmax(sc, -1)
        p = bf(p * 1.0, "p" in rnd)
        o = bf(torch.einsum("hts,shd->thd", p, vv).reshape(T, H * hd), "att" in rnd)
        x = x + o @ W["wo"].T
        h = norm(x, W["n_mlp"])
        gt, up = h @ W["wg"].T, h @ W["wu"].T
        x = x + bf(gt / (1 + torch.exp(-gt)) * up, "h" in rnd) @ W["wd"].T
        del W
    xf = norm(x[T - R:], w["final_norm"].double())
    return xf @ w["lm_head"].double().T


def main():
    from paper_2505_01572_b200 import Stage
    base = synth.preset(a.shape)
    full = synth.make_weights(base, seed=1, device="cuda")
    prompt = [int(x) for x in synth.make_prompt(base.vocab, a.ctx, seed=17)]
    ALL = ("xg", "att", "h", "k", "v", "q", "p")
    if a.variants == "all-but":
        variants = [()] + [ALL] + [tuple(x for x in ALL if x not in drop) for drop in
                                   (("k",), ("v",), ("k", "v"), ("p",), ("v", "p"), ("k", "v", "p"), ("q",),
                                    ("q", "p"), ("k", "v", "q", "p"))]
    else:
        variants = [(), ("xg",), ("att",), ("h",), ("kv",), ("q",), ("p",), ("xg", "att", "h"),
                    ("xg", "att", "h", "kv", "q", "p")]
    for L in [int(v) for v in a.layers.split(",")]:
        s = synth.reduced_depth(base, L)
        w = {**full, "layers": full["layers"][:L]}
        st = Stage(s, w, max_seq=a.ctx + 32, max_window=8)
        st.prefill(prompt)
        stream = st.draft(5)
        st.prefill(prompt)
        window = stream[:4]
        _, _, lg = st.verify(window, want_logits=True)
        st.close()
        gpu = torch.tensor(lg, dtype=torch.float64, device="cuda")
        toks = prompt + window
        res = []
        z64 = None
        for rnd in variants:
            z = forward(s, w, toks, 5, set(rnd))
            if z64 is None:
                z64 = z
            m = z64.abs().max().item()
            res.append((",".join(rnd) or "fp64 (oracle)", (gpu - z).abs().max().item() / m,
                        (z - z64).abs().max().item() / m, m))
        for name, e, e64, m in res:
            print(f"L={L:3d}  {name:28s} CUDA-vs-variant {e:.3e}  variant-vs-fp64 {e64:.3e}  (max|logit| {m:.2f})",
                  flush=True)


main()
