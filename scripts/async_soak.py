"""Soak test of the async runtime (PS_MODE_PIPESPEC, one host thread per stage)
on the toy pair: N runs per alpha, each output compared with M_K AR; prints
every mismatch with its first differing index.  Usage:
python scripts/async_soak.py [--runs 100]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_2505_01572_b200 import Stage, pipeline_run
from paper_2505_01572_b200.abi import PS_MODE_AR, PS_MODE_PIPESPEC

ap = argparse.ArgumentParser()
ap.add_argument("--runs", type=int, default=100)
ap.add_argument("--gen", type=int, default=40)
a = ap.parse_args()
sd_, sv = synth.preset("toy-drafter"), synth.preset("toy-verifier")
wd = synth.make_weights(sd_, seed=31, device="cuda")
wv = synth.make_weights(sv, seed=32, device="cuda")
d, v = Stage(sd_, wd, max_seq=256, max_window=8), Stage(sv, wv, max_seq=256, max_window=8)
prompt = [int(x) for x in synth.make_prompt(256, 64, seed=33)]
ar, _ = pipeline_run([d, v], prompt, a.gen, mode=PS_MODE_AR)
bad = 0
for alpha in (0.0, 0.6, 0.9, 1.0):
    d.set_synthetic(ar + [0] * 16, len(prompt), level=0, top=1, alphas=[alpha], seed=5)
    for r in range(a.runs):
        ps, stats = pipeline_run([d, v], prompt, a.gen, mode=PS_MODE_PIPESPEC, gammas=[0, 6])
        if ps != ar:
            bad += 1
            i = next((j for j in range(min(len(ps), len(ar))) if ps[j] != ar[j]), min(len(ps), len(ar)))
            print(f"MISMATCH alpha={alpha} run={r} first_diff={i} ps[{i}:{i+4}]={ps[i:i+4]} ar[{i}:{i+4}]={ar[i:i+4]} "
                  f"len ps={len(ps)} steps={list(stats.steps[:2])} verify={list(stats.verify_steps[:2])} "
                  f"rollbacks={list(stats.rollbacks[:2])}", flush=True)
    d.clear_synthetic()
print(f"async soak: {bad} mismatches in {4 * a.runs} runs")
