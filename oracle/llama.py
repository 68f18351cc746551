"""fp64 reference LLaMA forward, greedy decoding and verification.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

What it follows:
  * The model M_i is a LLaMA-shaped decoder (§4.1 P:181 "LLaMA-2 and
    LLaMA-3 variants"); conventions are HF LlamaForCausalLM's (DESIGN.md
    reading R19): RMSNorm w*x/sqrt(mean(x^2)+eps); rotate-half RoPE with
    inv_freq_i = theta^(-2i/hd) (+ llama3 frequency scaling for 3.x shapes);
    causal GQA attention where KV head j serves query heads j*g .. j*g+g-1;
    SiLU-gated MLP; no biases; scale 1/sqrt(hd); untied or tied lm_head.
  * Greedy decoding, temperature 0: argmax with the LOWEST index among
    equal maxima (np.argmax; reading R12).
  * Verification (Alg.1 P:101-105 "Get draft tokens ... Generate token
    predictions ... Compare against predicted tokens ... Append matching
    tokens"), with the correction / bonus token of Eq.1 P:124-128 (reading R1).

Everything is float64; weights are the bf16 values of `synth.make_weights`
converted exactly.  Pinned by tests/test_oracle_llama.py against HF
LlamaForCausalLM (float64), a brute-force verify, and closed special cases.
"""
from __future__ import annotations

import math

import numpy as np


# ----------------------------------------------------------------------------- RoPE
def rope_inv_freq(shape) -> np.ndarray:
    """inv_freq_i = theta^(-2i/hd), i = 0..hd/2-1; llama3 scaling when rope_kind==1
    (HF `_compute_llama3_parameters`, restated)."""
    hd = shape.head_dim
    inv = 1.0 / (shape.rope_theta ** (np.arange(0, hd, 2, dtype=np.float64) / hd))
    if shape.rope_kind == 1:
        factor, lo, hi, old = shape.rope_factor, shape.lo_ff, shape.hi_ff, shape.rope_orig_max
        low_wavelen = old / lo
        high_wavelen = old / hi
        wavelen = 2.0 * math.pi / inv
        scaled = np.where(wavelen > low_wavelen, inv / factor, inv)
        smooth = (old / wavelen - lo) / (hi - lo)
        smoothed = (1.0 - smooth) * scaled / factor + smooth * scaled
        medium = (wavelen >= high_wavelen) & (wavelen <= low_wavelen)
        inv = np.where(medium, smoothed, scaled)
    return inv


def rotate_half(x: np.ndarray) -> np.ndarray:
    h = x.shape[-1] // 2
    return np.concatenate([-x[..., h:], x[..., :h]], axis=-1)


def apply_rope(x: np.ndarray, pos: np.ndarray, inv_freq: np.ndarray) -> np.ndarray:
    """x: [T, heads, hd]; pos: [T] absolute positions."""
    ang = pos[:, None].astype(np.float64) * inv_freq[None, :]
    emb = np.concatenate([ang, ang], axis=-1)[:, None, :]
    return x * np.cos(emb) + rotate_half(x) * np.sin(emb)


def rms_norm(x: np.ndarray, g: np.ndarray, eps: float) -> np.ndarray:
    return x / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps) * g


def silu(x: np.ndarray) -> np.ndarray:
    return x / (1.0 + np.exp(-x))


# ----------------------------------------------------------------------------- model
class Session:
    """Incremental fp64 forward with a per-layer KV cache.

    `forward(tokens)` appends len(tokens) positions and returns their logits
    [T, V]; `truncate(n)` keeps the KV of the first n positions (the oracle's
    KV rollback, Alg.1).  A fresh Session over the whole sequence is the
    plain full forward; the incremental one is pinned equal to it.
    """

    def __init__(self, weights: dict, shape):
        self.w = weights
        self.s = shape
        self.inv_freq = rope_inv_freq(shape)
        self.k = [np.zeros((0, shape.n_kv_heads, shape.head_dim)) for _ in range(shape.n_layers)]
        self.v = [np.zeros((0, shape.n_kv_heads, shape.head_dim)) for _ in range(shape.n_layers)]

    @property
    def length(self) -> int:
        return self.k[0].shape[0] if self.s.n_layers else self._len0

    _len0 = 0

    def truncate(self, n: int) -> None:
        for l in range(self.s.n_layers):
            self.k[l] = self.k[l][:n]
            self.v[l] = self.v[l][:n]
        if not self.s.n_layers:
            self._len0 = min(self._len0, n)

    def hidden(self, tokens) -> np.ndarray:
        """Final hidden states (before the final norm) for the appended rows."""
        s, w = self.s, self.w
        tokens = np.asarray(tokens, dtype=np.int64)
        T = tokens.shape[0]
        p0 = self.length
        pos = np.arange(p0, p0 + T)
        H, Hkv, hd = s.n_heads, s.n_kv_heads, s.head_dim
        g = H // Hkv
        x = w["embed"][tokens].copy()
        for l, lw in enumerate(w["layers"]):
            h = rms_norm(x, lw["n_attn"], s.rms_eps)
            q = (h @ lw["wq"].T).reshape(T, H, hd)
            k = (h @ lw["wk"].T).reshape(T, Hkv, hd)
            v = (h @ lw["wv"].T).reshape(T, Hkv, hd)
            q = apply_rope(q, pos, self.inv_freq)
            k = apply_rope(k, pos, self.inv_freq)
            self.k[l] = np.concatenate([self.k[l], k], axis=0)
            self.v[l] = np.concatenate([self.v[l], v], axis=0)
            K, V = self.k[l], self.v[l]            # [p0+T, Hkv, hd]
            kpos = np.arange(K.shape[0])
            mask = kpos[None, :] <= pos[:, None]    # causal: key position <= query position
            out = np.empty((T, H, hd))
            for hh in range(H):
                j = hh // g                        # KV head serving query head hh
                sc = (q[:, hh, :] @ K[:, j, :].T) / math.sqrt(hd)
                sc = np.where(mask, sc, -np.inf)
                sc = sc - sc.max(axis=1, keepdims=True)
                p = np.exp(sc)
                p = p / p.sum(axis=1, keepdims=True)
                out[:, hh, :] = p @ V[:, j, :]
            x = x + out.reshape(T, H * hd) @ lw["wo"].T
            h = rms_norm(x, lw["n_mlp"], s.rms_eps)
            x = x + (silu(h @ lw["wg"].T) * (h @ lw["wu"].T)) @ lw["wd"].T
        if not s.n_layers:
            self._len0 = p0 + T
        return x

    def forward(self, tokens) -> np.ndarray:
        x = self.hidden(tokens)
        return rms_norm(x, self.w["final_norm"], self.s.rms_eps) @ self.w["lm_head"].T


def forward_full(weights: dict, shape, tokens) -> np.ndarray:
    """Plain teacher-forced forward of the whole sequence: logits [T, V]."""
    return Session(weights, shape).forward(tokens)


# ----------------------------------------------------------------------------- greedy
def greedy(z: np.ndarray) -> int:
    """argmax over the vocabulary; lowest index among equal maxima (R12)."""
    return int(np.argmax(z))


def top2_gap(z: np.ndarray) -> float:
    """max logit minus second-largest logit (0 on a tie)."""
    part = np.partition(z, -2)
    return float(part[-1] - part[-2])


def ar_decode(weights: dict, shape, prompt, n_new: int, eos: int | None = None):
    """Plain autoregressive greedy decoding of M (§3.1; the lossless target).
    Returns (tokens, gaps) for the generated tokens (prompt excluded)."""
    sess = Session(weights, shape)
    z = sess.forward(prompt)[-1]
    out, gaps = [], []
    for _ in range(n_new):
        t = greedy(z)
        out.append(t)
        gaps.append(top2_gap(z))
        if eos is not None and t == eos:
            break
        z = sess.forward([t])[-1]
    return out, gaps


# ----------------------------------------------------------------------------- verify
def first_mismatch(pred, window) -> int:
    """a = max{ j <= w : pred_t == d_t for all t < j } (Alg.1 P:104 "Compare")."""
    a = 0
    while a < len(window) and pred[a] == window[a]:
        a += 1
    return a


def verify(weights: dict, shape, x, d):
    """One verification step of stage M over draft window d given its committed
    tokens x (len n >= 1).  Teacher-forced: rows j = 0..w are the predictions
    for positions n..n+w given x ++ d[0:j] (causal attention makes one forward
    over x ++ d equal to w+1 separate forwards; pinned by verify_bruteforce).

    Returns dict(a, next, pred, logits[w+1,V], gaps[w+1], appended, rejected, keep)
      appended = d[0:a] + [next]   (matching prefix + correction/bonus, R1)
      rejected = a < w             (signal rejection upstream, Alg.1)
      keep     = n + a + 1         (upstream resync length)
    """
    x = list(map(int, x))
    d = list(map(int, d))
    n, w = len(x), len(d)
    z = forward_full(weights, shape, x + d)[n - 1:n + w]
    pred = [greedy(r) for r in z]
    a = first_mismatch(pred, d)
    nxt = pred[a]
    return dict(a=a, next=nxt, pred=pred, logits=z, gaps=[top2_gap(r) for r in z],
                appended=d[:a] + [nxt], rejected=a < w, keep=n + a + 1)


def verify_bruteforce(weights: dict, shape, x, d):
    """The literal definition: z_j = forward(x ++ d[0:j])[last], j = 0..w."""
    x = list(map(int, x))
    d = list(map(int, d))
    pred = []
    for j in range(len(d) + 1):
        pred.append(greedy(forward_full(weights, shape, x + d[:j])[-1]))
    a = first_mismatch(pred, d)
    return a, pred[a], pred
