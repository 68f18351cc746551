"""The bench's step (bench.py, BASELINE configs[1]) alone, for ncu launch lists:
prefill of both stages, M_1's AR reference stream, then --warmup + --steps
sync-SD rounds (gamma drafter forwards + one verify forward each).  Prints the
number of megakernel launches before the timed steps so the launch list can
be cut there (ncu -s), and the steps' launches (gamma + 1 per step).

Usage: python scripts/step_launches.py [--steps 10] [--warmup 3] [--gamma 4]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synth
from paper_2505_01572_b200 import Stage, abi

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--gamma", type=int, default=4)
ap.add_argument("--prompt", type=int, default=512)
ap.add_argument("--gen", type=int, default=256)
a = ap.parse_args()
ds, ts = synth.preset("llama3.2-1b"), synth.preset("llama3.1-8b")
wd = synth.make_weights(ds, seed=0, device="cuda")
wt = synth.make_weights(ts, seed=1, device="cuda")
max_seq = a.prompt + a.gen + 4 * a.gamma + 128
drafter = Stage(ds, wd, max_seq=max_seq, max_window=8)
target = Stage(ts, wt, max_seq=max_seq, max_window=8)
prompt = [int(x) for x in synth.make_prompt(ts.vocab, a.prompt, seed=17)]
L = abi.lib()
target.prefill(prompt)
S = target.draft(a.gen + 2 * a.gamma + 2)
target.kv_rollback(a.prompt)
drafter.prefill(prompt)
drafter.set_synthetic(S, a.prompt, level=0, top=1, alphas=[0.8], seed=1234)
gen = []


def step():
    global gen
    if len(gen) >= a.gen:
        target.kv_rollback(a.prompt)
        drafter.resync(prompt)
        gen = []
    d = drafter.draft(a.gamma)
    acc, nxt = target.verify(d)
    gen += d[:acc] + [nxt]
    drafter.resync(prompt + gen)


for _ in range(a.warmup):
    step()
torch.cuda.synchronize()
n0 = L.ps_kernel_launch_count()
for _ in range(a.steps):
    step()
torch.cuda.synchronize()
print(f"launches before the timed steps: {n0}; in the steps: {L.ps_kernel_launch_count() - n0}", flush=True)
drafter.close()
target.close()
