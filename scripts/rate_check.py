"""BASELINE configs[4] closed-form check on the GPU runtime (SURVEY §8(d)
config 5): measured verify probability rho and tokens per
verifier step E(N) of async PipeSpec (ps_pipeline_run, PS_MODE_PIPESPEC, two
stages on one GPU) against Eq.3 rho = alpha / (1 - alpha^(gamma+1) + alpha)
and Eq.1 E(N) = (1 - rho) + rho * sum_{j=0}^{gamma} alpha^j, under reading R4:
the drafter produces >= gamma + 1 tokens per verifier step (a light drafter;
the verifier's steps are padded to a virtual latency with ps_run_opts.virtual_ns
so the drafter's kernels run between them on the one GPU), windows capped at
gamma, lookahead 0, AR steps when no valid draft.

Acceptance is synthetic (reading R24): the verifier's emitted token follows a
fixed random stream S (chained override with alpha = 1 above it) and the
drafter agrees with it with probability alpha (a new counter seed per
generation: with one seed every generation would replay the same acceptance
pattern); both still run their real forwards.  Generations of --gen tokens restart from a 64-token prompt until
--steps verifier steps per (alpha, gamma) cell.

Usage: python scripts/rate_check.py [--steps 10000] [--out profiles/r02_rate_check.json]
"""
import argparse
import json
import os
import sys
from dataclasses import replace

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import synth
from paper_2505_01572_b200 import Stage, pipeline_run
from paper_2505_01572_b200.abi import PS_MODE_PIPESPEC

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=10000)
ap.add_argument("--gen", type=int, default=512)
ap.add_argument("--verifier", default="llama3.1-8b")
ap.add_argument("--out", default=None)
ap.add_argument("--pad", type=float, default=1.5, help="drafter steps of slack per verifier step (x (gamma + 3))")
ap.add_argument("--alphas", default="0.5,0.8,0.95")
ap.add_argument("--gammas", default="2,4,8")
a = ap.parse_args()


def eq3(al, g):
    return al / (1 - al ** (g + 1) + al)


def eq1(al, g, rho):
    return (1 - rho) + rho * sum(al ** j for j in range(g + 1))


vs = synth.preset(a.verifier)
ds = replace(synth.preset("llama-68m"), name="light-drafter", vocab=vs.vocab)   # ~0.1 ms per draft step
wv = synth.make_weights(vs, seed=1, device="cuda")
wd = synth.make_weights(ds, seed=2, device="cuda")
max_seq = 64 + a.gen + 128
ver = Stage(vs, wv, max_seq=max_seq, max_window=8)
dra = Stage(ds, wd, max_seq=max_seq, max_window=8)
prompt = [int(x) for x in synth.make_prompt(vs.vocab, 64, seed=3)]
rng = np.random.default_rng(5)
S = [int(x) for x in rng.integers(0, vs.vocab, a.gen + 64)]
# verifier step time (one verify pass) for the virtual-latency padding
ver.prefill(prompt)
ver.draft(8)
pass_ms = ver.info()["last_fwd_ms"]
dra.prefill(prompt)
dra.draft(8)
draft_ms = dra.info()["last_fwd_ms"]
cells = []
for alpha in [float(x) for x in a.alphas.split(",")]:
    for gamma in [int(x) for x in a.gammas.split(",")]:
        pad_ns = int((pass_ms + (gamma + 3) * draft_ms * a.pad + 0.5) * 1e6)
        steps = verify = tokens = 0
        runs = 0
        wins = []
        while steps < a.steps:
            # the verifier emits S (alpha 1 above it); the drafter agrees with it
            # w.p. alpha -- a fresh counter seed per generation, so the acceptance
            # pattern over positions is a new draw every time
            seed = 1000 * runs + 77
            ver.set_synthetic(S, len(prompt), level=1, top=2, alphas=[1.0], seed=seed)
            dra.set_synthetic(S, len(prompt), level=0, top=2, alphas=[alpha, 1.0], seed=seed)
            out, st, ev = pipeline_run([dra, ver], prompt, a.gen, mode=PS_MODE_PIPESPEC, gammas=[0, gamma],
                                       lookaheads=[0, 0], virtual_ns=[0, pad_ns], event_cap=20000, return_events=True)
            assert out == S[:a.gen], "output differs from the verifier's stream"
            steps += int(st.steps[1])
            verify += int(st.verify_steps[1])
            tokens += len(out)
            runs += 1
            wins += [e["w"] for e in ev if e["stage"] == 1 and e["kind"] == 1]
        rho, en = verify / steps, tokens / steps
        cell = {"alpha": alpha, "gamma": gamma, "verifier_steps": steps, "generations": runs,
                "rho_measured": rho, "rho_eq3": eq3(alpha, gamma), "EN_measured": en,
                "EN_eq1": eq1(alpha, gamma, eq3(alpha, gamma)), "virtual_step_ms": pad_ns / 1e6,
                "mean_window": float(np.mean(wins)) if wins else 0.0,
                "full_windows": float(np.mean([w == gamma for w in wins])) if wins else 0.0}
        cell["rho_abs_err"] = abs(rho - cell["rho_eq3"])
        cell["EN_rel_err"] = abs(en - cell["EN_eq1"]) / cell["EN_eq1"]
        cells.append(cell)
        print(json.dumps(cell), flush=True)
res = {"verifier": a.verifier, "drafter": "llama-68m shape, vocab 128256", "verify_pass_ms": pass_ms,
       "draft_step_ms": draft_ms, "cells": cells,
       "max_rho_abs_err": max(c["rho_abs_err"] for c in cells), "max_EN_rel_err": max(c["EN_rel_err"] for c in cells)}
print(json.dumps({k: v for k, v in res.items() if k != "cells"}), flush=True)
if a.out:
    json.dump(res, open(a.out, "w"), indent=1)
