"""GPU parity of the bench's verifier at FULL depth (BASELINE configs[1]:
LLaMA-3.1-8B shape, 32 layers, 512-token prompt, the bench's window R = 5)
against the fp64 oracle on the same bf16 weights.

The oracle's weights stream layer by layer (each layer's bf16 tensors are
converted to float64 when the forward reaches it and dropped after), so the
full model never sits in host RAM as float64 at once; the arithmetic is the
unchanged oracle.llama forward (reading R27: fp64 oracle)."""
import numpy as np
import pytest
import torch

import synth
from oracle import llama as L
from tests._parity import check_logits, check_verify

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


class StreamedLayers:
    """A read-once view of bf16 CUDA layers as the oracle's float64 dicts
    (data marshalling only: the same exact bf16 -> fp64 conversion as
    synth.weights_to_numpy, one layer at a time)."""

    def __init__(self, layers):
        self.layers = layers

    def __len__(self):
        return len(self.layers)

    def __iter__(self):
        for lw in self.layers:
            yield {k: v.float().cpu().double().numpy() for k, v in lw.items()}


def test_llama31_8b_full_depth_bench_window():
    from paper_2505_01572_b200 import Stage
    s = synth.preset("llama3.1-8b")
    w = synth.make_weights(s, seed=1, device="cuda")          # bench.py's target weights (seed + 1)
    st = Stage(s, w, max_seq=640, max_window=8)
    prompt = [int(x) for x in synth.make_prompt(s.vocab, 512, seed=17)]
    st.prefill(prompt)
    stream = st.draft(5)
    st.prefill(prompt)
    window = stream[:2] + [(stream[2] + 3) % s.vocab] + stream[3:4]   # w = 4 (R = 5), rejects at 2
    a, nxt, logits = st.verify(window, want_logits=True)
    st.close()
    w64 = {k: w[k].float().cpu().double().numpy() for k in ("embed", "final_norm")}
    w64["lm_head"] = w64["embed"] if s.tied else w["lm_head"].float().cpu().double().numpy()
    w64["layers"] = StreamedLayers(w["layers"])
    ref = L.verify(w64, s, prompt, window)
    rel = check_logits(logits, ref["logits"])
    check_verify((a, nxt), ref, len(window), where="8B full depth")
    print(f"8B full depth: rel logit err {rel:.3e}, a={a}/{ref['a']} next={nxt}/{ref['next']}, "
          f"max|logit| {np.abs(ref['logits']).max():.2f}")
    del w
    torch.cuda.empty_cache()
