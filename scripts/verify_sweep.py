"""Verify-kernel sweep (BASELINE.json configs[4]): one LLaMA-3.1-8B-shaped
stage, verify-pass time for gamma in {0, 1, 2, 4, 8, 16} (R = gamma + 1 rows)
and context 512 .. 32K, each the average of in-library CUDA-event timings of
the pass (ps_stage_info.sum_fwd_ms).  Algorithmic bytes per pass = streamed
weights (R embedding rows) + KV read (ctx x KV bytes/token) + KV write
(R x KV bytes/token) -- SURVEY.md 8(d); GB/s against MEASURED_PEAKS.json.

Usage: python scripts/verify_sweep.py [--shape llama3.1-8b] [--reps 10] [--out profiles/r01_verify_sweep.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import synth
from paper_2505_01572_b200 import Stage

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="llama3.1-8b")
ap.add_argument("--ctxs", default="512,1024,2048,4096,8192,16384,32768")
ap.add_argument("--gammas", default="0,1,2,4,8,16")
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--out", default=None)
a = ap.parse_args()

peaks = {}
try:
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
except OSError:
    pass
peak = float(peaks.get("hbm_gbs", 7700.0))
ctxs = [int(x) for x in a.ctxs.split(",")]
gammas = [int(x) for x in a.gammas.split(",")]
s = synth.preset(a.shape)
w = synth.make_weights(s, seed=1, device="cuda")
toks = [int(x) for x in synth.make_prompt(s.vocab, max(ctxs) + 1, seed=2)]
win = [int(x) for x in synth.make_prompt(s.vocab, max(gammas), seed=3)]
rows = []
for c in ctxs:
    # one stage per context, sized for it (max_seq sets the attention work-item
    # size, DESIGN §5 "long context"); prompt through the 64-row prefill bucket
    st = Stage(s, w, max_seq=c + max(gammas) + 64, max_window=max(1, max(gammas)))
    st.prefill(toks[:c])
    for g in gammas:
        for _ in range(2):
            st.verify(win[:g])
            st.kv_rollback(c)
        torch.cuda.synchronize()
        st.reset_timers()
        for _ in range(a.reps):
            st.verify(win[:g])
            st.kv_rollback(c)
        inf = st.info()
        ms = inf["sum_fwd_ms"] / max(1, inf["n_fwd"])
        R = g + 1
        byts = s.streamed_bytes_per_pass(R) + (c + R) * s.kv_bytes_per_token()
        gbs = byts / (ms * 1e-3) / 1e9
        rows.append({"ctx": c, "gamma": g, "rows": R, "ms": ms, "bytes": byts, "GB/s": gbs, "frac": gbs / peak})
        print(f"ctx {c:6d} gamma {g:2d} R {R:2d}: {ms:7.3f} ms  {gbs:7.0f} GB/s  {gbs / peak:.3f}", flush=True)
    st.close()
res = {"shape": a.shape, "peak_gbs": peak, "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 7700",
       "reps": a.reps, "rows": rows}
if a.out:
    json.dump(res, open(a.out, "w"), indent=1)
