import sys, numpy as np, torch
sys.path.insert(0, '.')
from dataclasses import replace
import synth
from paper_2505_01572_b200 import Stage
base = synth.preset("toy-verifier")
cases = {
 "toy": base,
 "vocab32k": replace(base, vocab=32000),
 "vocab1000": replace(base, vocab=1000),
 "d768": replace(base, d_model=768, n_heads=12, n_kv_heads=12),
 "d256": replace(base, d_model=256, n_heads=4, n_kv_heads=4),
 "ffn3072": replace(base, d_ffn=3072),
 "eps1e-6": replace(base, rms_eps=1e-6),
 "68m": synth.preset("llama-68m"),
 "68m_v256": replace(synth.preset("llama-68m"), vocab=256),
}
for name, s in cases.items():
    for plen in (64, 96):
        w = synth.make_weights(s, seed=7, device="cuda")
        st = Stage(s, w, max_seq=plen + 40)
        prompt = list(synth.make_prompt(s.vocab, plen, seed=8))
        st.prefill(prompt)
        a, n, lg = st.verify([], want_logits=True)
        print(name, plen, "nan" if np.isnan(lg).any() else "ok", a, n, float(np.abs(lg).max()), flush=True)
        st.close()
