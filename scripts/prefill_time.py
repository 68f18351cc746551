"""Prefill timing (NEXT-3): a whole prompt through ps_prefill on one
stage, CUDA events on the stage stream, for the prefill kernels (tcgen05
GEMMs with the tokens as M, causal prefill attention; PS_PREFILL_AUTO) and the
decode megakernel's 64-row bucket (PS_PREFILL_ROWS).  FLOPs = 2 x params x
tokens (linear layers, lm_head excluded: prefill stops at the KV) + causal
attention 4 x L x q_dim x n^2 / 2; the split-bf16 operand doubles the MMA work
but not these algorithmic FLOPs.

Usage: python scripts/prefill_time.py [--shape llama3.1-8b] [--n 511] [--reps 3]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import synth
from paper_2505_01572_b200 import Stage, abi

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="llama3.1-8b")
ap.add_argument("--n", type=int, default=512, help="prompt tokens (n - 1 positions are forwarded)")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--paths", default="auto,rows")
a = ap.parse_args()
s = synth.preset(a.shape)
w = synth.make_weights(s, seed=1, device="cuda")
peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
tf_peak = peaks.get("bf16_tflops_sustained")
n = a.n - 1
lin = s.streamed_bytes_per_pass(1) / 2 - s.vocab * s.d_model   # linear-layer params (+ norms, 1 embed row)
flops = 2.0 * lin * n + 4.0 * s.n_layers * s.q_dim * n * n / 2
out = {"shape": a.shape, "tokens": n, "flops": flops}
for path in a.paths.split(","):
    st = Stage(s, w, max_seq=a.n + 64)
    st.set_prefill_path(abi.PS_PREFILL_AUTO if path == "auto" else abi.PS_PREFILL_ROWS)
    prompt = [int(x) for x in synth.make_prompt(s.vocab, a.n, seed=2)]
    other = [(t + 1) % s.vocab for t in prompt]
    ms = []
    for rep in range(a.reps + 1):
        st.prefill(other[:1])                     # drop the KV (no common prefix with `prompt`)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st.stream)
        st.prefill(prompt)
        e1.record(st.stream)
        e1.synchronize()
        if rep:
            ms.append(e0.elapsed_time(e1))
    m = min(ms)
    out[path] = {"ms": m, "ms_all": ms, "TFLOP/s": flops / (m * 1e-3) / 1e12,
                 "frac_bf16_sustained": flops / (m * 1e-3) / 1e12 / tf_peak if tf_peak else None}
    print(f"{a.shape} n={n} {path:5s}: {m:8.2f} ms  {flops / (m * 1e-3) / 1e12:7.1f} TFLOP/s", flush=True)
    st.close()
print(json.dumps(out))
