"""Attention parity probe: verify logits vs the oracle for several window sizes
(R = w + 1) and shapes; prints the relative logit error per case."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from dataclasses import replace
import numpy as np
import synth
from oracle import llama as L
from paper_2505_01572_b200 import Stage

for name, kw in [("llama3.1-8b", dict(n_layers=2, vocab=4096)), ("llama3.2-1b", dict(n_layers=2, vocab=4096))]:
    base = synth.preset("llama3.1-8b" if name != "llama3.2-1b" else "llama3.2-1b")
    s = replace(base, name=name, **kw)
    wt = synth.make_weights(s, seed=3, device="cuda")
    w64 = synth.weights_to_numpy(wt)
    for plen in (40, 100):
        prompt = list(synth.make_prompt(s.vocab, plen, seed=4))
        st = Stage(s, wt, max_seq=plen + 40, max_window=31)
        for w in (0, 4, 15, 16, 20, 31):
            st.prefill(prompt)
            window = list(synth.make_prompt(s.vocab, w, seed=5)) if w else []
            a, nxt, lg = st.verify(window, want_logits=True)
            z = L.forward_full(w64, s, prompt + window)[plen - 1:]
            err = np.abs(lg - z).max(axis=1) / np.abs(z).max()
            print(f"{name:12s} plen {plen:4d} w {w:2d}: max rel err {err.max():.2e}  per-row {np.array2string(err, precision=1)}",
                  flush=True)
        st.close()
