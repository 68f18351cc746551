"""Pins for oracle/llama.py: HF LlamaForCausalLM (float64) with identical
weights, closed special cases, and brute-force verification (Alg.1)."""
import math

import numpy as np
import pytest
import torch

import synth
from oracle import llama as L


def hf_model(shape, w):
    from transformers import LlamaConfig, LlamaForCausalLM
    rope = {"rope_theta": shape.rope_theta, "rope_type": "default"}
    if shape.rope_kind == 1:
        rope = {"rope_theta": shape.rope_theta, "rope_type": "llama3", "factor": shape.rope_factor,
                "low_freq_factor": shape.lo_ff, "high_freq_factor": shape.hi_ff,
                "original_max_position_embeddings": shape.rope_orig_max}
    cfg = LlamaConfig(vocab_size=shape.vocab, hidden_size=shape.d_model,
                      intermediate_size=shape.d_ffn, num_hidden_layers=shape.n_layers,
                      num_attention_heads=shape.n_heads, num_key_value_heads=shape.n_kv_heads,
                      head_dim=shape.head_dim, rms_norm_eps=shape.rms_eps, rope_parameters=rope,
                      tie_word_embeddings=shape.tied, max_position_embeddings=4096,
                      attention_bias=False, mlp_bias=False)
    cfg._attn_implementation = "eager"
    m = LlamaForCausalLM(cfg).double().eval()
    sd = {"model.embed_tokens.weight": w["embed"], "model.norm.weight": w["final_norm"],
          "lm_head.weight": w["lm_head"]}
    names = {"wq": "self_attn.q_proj", "wk": "self_attn.k_proj", "wv": "self_attn.v_proj",
             "wo": "self_attn.o_proj", "wg": "mlp.gate_proj", "wu": "mlp.up_proj",
             "wd": "mlp.down_proj", "n_attn": "input_layernorm", "n_mlp": "post_attention_layernorm"}
    for l, lw in enumerate(w["layers"]):
        for k, v in lw.items():
            sd[f"model.layers.{l}.{names[k]}.weight"] = v
    sd = {k: v.to(torch.float64) for k, v in sd.items()}
    m.load_state_dict(sd, strict=False)
    return m


@pytest.mark.parametrize("name", ["toy-verifier", "toy-drafter"])
def test_forward_matches_hf_float64(name):
    s = synth.preset(name)
    w = synth.make_weights(s, seed=3)
    toks = synth.make_prompt(s.vocab, 37, seed=4)
    ours = L.forward_full(synth.weights_to_numpy(w), s, toks)
    with torch.no_grad():
        ref = hf_model(s, w)(torch.tensor(toks[None], dtype=torch.long)).logits[0].numpy()
    # HF builds cos/sin from a float32 inv_freq buffer, so agreement is ~1e-7 relative
    assert np.abs(ours - ref).max() <= 1e-6 * np.abs(ref).max()


def test_llama3_rope_and_gqa_match_hf():
    """llama3 frequency scaling + GQA g=4 at small width (1B-like ratios)."""
    base = synth.preset("llama3.1-8b")
    from dataclasses import replace
    s = replace(base, name="l3-small", vocab=300, d_model=256, n_layers=2, n_heads=8, n_kv_heads=2,
                head_dim=32, d_ffn=512)
    w = synth.make_weights(s, seed=9)
    toks = synth.make_prompt(s.vocab, 50, seed=1)
    ours = L.forward_full(synth.weights_to_numpy(w), s, toks)
    with torch.no_grad():
        ref = hf_model(s, w)(torch.tensor(toks[None], dtype=torch.long)).logits[0].numpy()
    # HF builds cos/sin from a float32 inv_freq buffer, so agreement is ~1e-7 relative
    assert np.abs(ours - ref).max() <= 1e-6 * np.abs(ref).max()


def test_llama3_inv_freq_matches_hf():
    from transformers import LlamaConfig
    from transformers.modeling_rope_utils import ROPE_INIT_FUNCTIONS
    for name in ("llama3.2-1b", "llama3.1-8b"):
        s = synth.preset(name)
        cfg = LlamaConfig(hidden_size=s.d_model, num_attention_heads=s.n_heads, head_dim=s.head_dim,
                          rope_parameters={"rope_theta": s.rope_theta, "rope_type": "llama3",
                                           "factor": s.rope_factor, "low_freq_factor": s.lo_ff,
                                           "high_freq_factor": s.hi_ff,
                                           "original_max_position_embeddings": s.rope_orig_max})
        inv, _ = ROPE_INIT_FUNCTIONS["llama3"](cfg, "cpu")
        assert np.allclose(L.rope_inv_freq(s), inv.double().numpy(), rtol=1e-6, atol=0)


def test_special_cases():
    s = synth.preset("toy-drafter")
    w64 = synth.weights_to_numpy(synth.make_weights(s, seed=5))
    # RoPE at position 0 is the identity
    x = np.random.default_rng(0).standard_normal((1, 2, 64))
    assert np.array_equal(L.apply_rope(x, np.array([0]), L.rope_inv_freq(s)), x)
    # rotation preserves norms pairwise
    y = L.apply_rope(x, np.array([17]), L.rope_inv_freq(s))
    assert np.allclose(np.linalg.norm(y), np.linalg.norm(x))
    # a 0-layer model: logits = rms(E[x]) * g_f @ W_lm^T, the textbook definition
    from dataclasses import replace
    s0 = replace(s, n_layers=0)
    w0 = dict(w64, layers=[])
    tok = [5, 9]
    e = w64["embed"][tok]
    want = (e / np.sqrt((e ** 2).mean(-1, keepdims=True) + s.rms_eps) * w64["final_norm"]) @ w64["lm_head"].T
    assert np.allclose(L.forward_full(w0, s0, tok), want, rtol=1e-13, atol=0)
    # first position attends only to itself: attention output == v (softmax of one score)
    lw = w64["layers"][0]
    h = L.rms_norm(w64["embed"][[7]], lw["n_attn"], s.rms_eps)
    v = h @ lw["wv"].T
    sess = L.Session(dict(w64, layers=[lw]), replace(s, n_layers=1))
    xo = sess.hidden([7])
    # undo the MLP: x_attn = E + v W_o^T, then MLP on top; recompute independently
    xa = w64["embed"][[7]] + v @ lw["wo"].T
    hm = L.rms_norm(xa, lw["n_mlp"], s.rms_eps)
    want = xa + (L.silu(hm @ lw["wg"].T) * (hm @ lw["wu"].T)) @ lw["wd"].T
    assert np.allclose(xo, want, rtol=1e-12, atol=1e-15)


def test_incremental_session_equals_full_forward():
    s = synth.preset("toy-verifier")
    w = synth.weights_to_numpy(synth.make_weights(s, seed=2))
    toks = list(synth.make_prompt(s.vocab, 40, seed=8))
    full = L.forward_full(w, s, toks)
    sess = L.Session(w, s)
    parts = [sess.forward(toks[:20]), sess.forward(toks[20:21]), sess.forward(toks[21:])]
    assert np.allclose(np.concatenate(parts), full, rtol=0, atol=1e-12)
    # truncate == KV rollback: recomputing after truncation reproduces the logits
    sess.truncate(25)
    again = sess.forward(toks[25:])
    assert np.allclose(again, full[25:], rtol=0, atol=1e-12)


def test_greedy_tie_lowest_index():
    z = np.array([0.5, 2.0, -1.0, 2.0])
    assert L.greedy(z) == 1
    assert L.top2_gap(z) == 0.0


def test_ar_decode_matches_hf_generate():
    s = synth.preset("toy-verifier")
    w = synth.make_weights(s, seed=3)
    prompt = synth.make_prompt(s.vocab, 16, seed=6)
    ours, gaps = L.ar_decode(synth.weights_to_numpy(w), s, prompt, 12)
    m = hf_model(s, w)
    with torch.no_grad():
        out = m.generate(torch.tensor(prompt[None], dtype=torch.long), max_new_tokens=12,
                         do_sample=False, min_new_tokens=12)[0, 16:].tolist()
    for t_o, t_h, g in zip(ours, out, gaps):
        if g < 1e-6:
            break                      # near-exact tie: either choice is correct
        assert t_o == t_h


def test_verify_equals_bruteforce_and_definition():
    s = synth.preset("toy-verifier")
    w = synth.weights_to_numpy(synth.make_weights(s, seed=3))
    x = list(synth.make_prompt(s.vocab, 20, seed=1))
    stream, _ = L.ar_decode(w, s, x, 8)
    cases = [
        [],                                   # w = 0: one AR step
        stream[:5],                           # full accept + bonus
        stream[:2] + [(stream[2] + 1) % s.vocab, stream[3]],   # reject at j=2
        [(stream[0] + 7) % s.vocab] + stream[1:4],             # reject at j=0
    ]
    for d in cases:
        r = L.verify(w, s, x, d)
        a, nxt, pred = L.verify_bruteforce(w, s, x, d)
        assert (r["a"], r["next"]) == (a, nxt)
        assert r["pred"] == pred
        assert r["appended"] == list(d[:a]) + [nxt]
        assert r["keep"] == len(x) + a + 1
        assert r["rejected"] == (a < len(d))
    # accepted tokens are exactly the AR stream
    r = L.verify(w, s, x, stream[:5])
    assert r["a"] == 5 and r["appended"] == stream[:6]
    r = L.verify(w, s, x, cases[2])
    assert r["a"] == 2 and r["appended"] == stream[:3]
