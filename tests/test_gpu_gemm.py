"""GPU: the megakernel's tcgen05 GEMM (a10's contraction: the lm_head over
the split-bf16 operand) isolated by a ZERO-layer model, whose logits are
rms(E[tok]) * g_f . W_lm^T -- no attention, no MLP -- against a float64 matmul
of the same bf16 weights (vocabularies spanning ragged tiles, window sizes in
both rows buckets)."""
from dataclasses import replace

import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("vocab,d,rows", [(256, 128, 1), (1000, 4096, 5), (32000, 2048, 17), (128256, 4096, 9),
                                          (300, 192, 32)])
def test_zero_layer_logits_are_the_lm_head_gemm(vocab, d, rows):
    from paper_2505_01572_b200 import Stage
    s = replace(synth.preset("toy-verifier"), name="gemm", vocab=vocab, d_model=d, n_layers=0, n_heads=d // 64,
                n_kv_heads=d // 64, d_ffn=d)
    w = synth.make_weights(s, seed=vocab + d, device="cuda")
    st = Stage(s, w, max_seq=64, max_window=31)
    toks = [int(x) for x in synth.make_prompt(vocab, rows + 1, seed=3)]
    st.prefill(toks[:1])
    a, nxt, logits = st.verify(toks[1:rows], want_logits=True)
    st.close()
    E = w["embed"].double().cpu().numpy()[toks[:rows]]
    xn = E / np.sqrt((E * E).mean(-1, keepdims=True) + s.rms_eps) * w["final_norm"].double().cpu().numpy()
    ref = xn @ w["lm_head"].double().cpu().numpy().T
    err = np.abs(logits - ref).max()
    # split-bf16 operand: ~2^-16 relative per element, fp32 accumulation
    assert err <= 2e-5 * np.abs(ref).max(), err
    assert list(np.argmax(logits, 1)[:a + 1]) == list(np.argmax(ref, 1)[:a + 1])
