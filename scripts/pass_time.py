"""Average verify-pass / draft-step time of one stage (in-library CUDA events
around each forward, ps_stage_info.sum_fwd_ms), for quick A/B sweeps of
kernel variants selected through the environment.

Usage: python scripts/pass_time.py [--shape llama3.1-8b] [--ctx 600] [--w 4] [--reps 30]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synth
from paper_2505_01572_b200 import Stage

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="llama3.1-8b")
ap.add_argument("--ctx", type=int, default=600)
ap.add_argument("--w", type=int, default=4)
ap.add_argument("--reps", type=int, default=30)
ap.add_argument("--gbs", type=float, default=6542.0)
a = ap.parse_args()
s = synth.preset(a.shape)
w = synth.make_weights(s, seed=1, device="cuda")
st = Stage(s, w, max_seq=a.ctx + 64, max_window=max(a.w, 1))
prompt = [int(x) for x in synth.make_prompt(s.vocab, a.ctx, seed=2)]
st.prefill(prompt)
win = [int(x) for x in synth.make_prompt(s.vocab, a.w, seed=3)]


def one():
    if a.w:
        st.verify(win)
    else:
        st.draft(1)
    st.kv_rollback(a.ctx)


for _ in range(5):
    one()
torch.cuda.synchronize()
st.reset_timers()
for _ in range(a.reps):
    one()
torch.cuda.synchronize()
inf = st.info()
ms = inf["sum_fwd_ms"] / max(1, inf["n_fwd"])
R = a.w + 1
byts = s.streamed_bytes_per_pass(R) + (a.ctx + R) * s.kv_bytes_per_token()
print(f"{a.shape} R={R} ctx={a.ctx} env PS_RA={os.environ.get('PS_RA')} : {ms:.4f} ms  "
      f"{byts / ms / 1e6:.0f} GB/s  frac {byts / ms / 1e6 / a.gbs:.3f}")
st.close()
