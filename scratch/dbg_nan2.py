import sys, ctypes, numpy as np, torch
sys.path.insert(0, '.')
from dataclasses import replace
import synth
from paper_2505_01572_b200 import Stage, abi
base = synth.preset("toy-verifier")
def rd(st, which, shape, dt):
    a = np.zeros(shape, dtype=dt)
    abi.check(abi.lib().ps_test_read(st.handle, which, a.ctypes.data, a.nbytes))
    return a
for plen in (64, 65, 66, 80, 95, 96, 97, 128):
  for ms in (104, 136, 300):
    if plen + 8 > ms: continue
    for g in (True, False):
        w = synth.make_weights(base, seed=7, device="cuda")
        st = Stage(base, w, max_seq=ms, use_graphs=g)
        prompt = list(synth.make_prompt(base.vocab, plen, seed=8))
        st.prefill(prompt)
        x = rd(st, 0, (32, 128), np.float32)
        q = rd(st, 2, (32, 128), np.float32)
        att = rd(st, 3, (32, 128), np.uint16)
        ss = rd(st, 5, (32, 1), np.float32)
        pt = rd(st, 8, (2,), np.int32)
        a, n, lg = st.verify([], want_logits=True)
        R = (plen - 1) % 32 or 32
        print(plen, ms, g, "nan" if np.isnan(lg).any() else "ok", "x", np.isnan(x[:R]).any(), "q", np.isnan(q[:R]).any(), "ss", ss[:R, 0].min(), "pt", pt, flush=True)
        st.close()
