"""One verify pass of a paper-shaped model, bracketed by cudaProfilerStart/Stop
so `ncu --profile-from-start off` sees exactly that pass (launch list / full
capture).  Usage: python scripts/prof_verify.py [--shape llama3.1-8b] [--ctx 512] [--w 8] [--reps 1]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synth
from paper_2505_01572_b200 import Stage

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="llama3.1-8b")
ap.add_argument("--layers", type=int, default=None)
ap.add_argument("--ctx", type=int, default=512)
ap.add_argument("--w", type=int, default=4)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--graphs", type=int, default=1)
a = ap.parse_args()
s = synth.preset(a.shape)
if a.layers:
    s = synth.reduced_depth(s, a.layers)
w = synth.make_weights(s, seed=1, device="cuda")
st = Stage(s, w, max_seq=a.ctx + 64, max_window=max(a.w, 1), use_graphs=bool(a.graphs))
prompt = [int(x) for x in synth.make_prompt(s.vocab, a.ctx, seed=2)]
st.prefill(prompt)
win = [int(x) for x in synth.make_prompt(s.vocab, a.w, seed=3)]
st.verify(win)                       # warm (graph capture)
st.kv_rollback(a.ctx)
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(a.reps):
    st.verify(win)
    st.kv_rollback(a.ctx)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("kernels per verify:", st.info()["launches_per_verify"])
