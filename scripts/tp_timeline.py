"""Share of a tensor-parallel verify pass spent in the in-kernel all-reduce
(a14): the TPRED phases (sum of the T ranks' O / down partials from peer
memory + residual + next RMSNorm operand) and the wait that precedes them.
Phase spans from the %globaltimer stamps of the trace build
(libpipespec_trace.so, selected here through PS_LIB), rank 0 of a TP group
whose ranks run concurrently on disjoint SM partitions of ONE GPU (peer memory
is local HBM here, not NVLink: an upper-bound-free stand-in for the protocol's
latency, not NVLink bandwidth).

Usage: python scripts/tp_timeline.py [--shape llama3.1-8b] [--layers 8] [--tp 2] [--ctx 512] [--w 4]
"""
import argparse
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("PS_LIB", os.path.join(ROOT, "paper_2505_01572_b200", "libpipespec_trace.so"))
import numpy as np
import torch

import synth
from paper_2505_01572_b200 import Stage, abi, shard_weights, tp_connect_local

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="llama3.1-8b")
ap.add_argument("--layers", type=int, default=8)
ap.add_argument("--tp", type=int, default=2)
ap.add_argument("--ctx", type=int, default=512)
ap.add_argument("--w", type=int, default=4)
ap.add_argument("--reps", type=int, default=4)
a = ap.parse_args()
s = synth.reduced_depth(synth.preset(a.shape), a.layers)
T = a.tp
w = synth.make_weights(s, seed=1, device="cuda")
n_sm = torch.cuda.get_device_properties(0).multi_processor_count
stages = [Stage(s, shard_weights(s, w, r, T), max_seq=a.ctx + 64, max_window=max(a.w, 1), tp_rank=r, tp_size=T,
                max_ctas=n_sm // T) for r in range(T)]
tp_connect_local(stages)


def run_all(fn):
    out = [None] * T
    def body(i):
        out[i] = fn(stages[i])
    th = [threading.Thread(target=body, args=(i,)) for i in range(T)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    return out


prompt = [int(x) for x in synth.make_prompt(s.vocab, a.ctx, seed=2)]
win = [int(x) for x in synth.make_prompt(s.vocab, a.w, seed=3)]
run_all(lambda st: st.prefill(prompt))
L = s.n_layers
G = n_sm // T
n_ph = 1 + 8 * L + 2
names = ["EMBED"] + ["QKV", "ATTN", "ACOMB", "O", "TPRED", "GU", "DOWN", "TPRED"] * L + ["LMHEAD", "ARGMAX"]
acc = {}
total = []
for rep in range(a.reps + 1):
    run_all(lambda st: (st.verify(win), st.kv_rollback(a.ctx)))
    torch.cuda.synchronize()
    buf = np.zeros(n_sm * (8 * L + 8) * 8, dtype=np.uint64)
    abi.check(abi.lib().ps_trace_read(stages[0].handle, 9, buf.ctypes.data, buf.nbytes))
    if rep == 0:
        continue
    t = buf[:G * n_ph * 8].reshape(G, n_ph, 8).astype(np.int64)
    pub = t[:, :, 1]
    t0 = t[:, 0, 0].min()
    done = pub.max(axis=0)
    for p in range(n_ph):
        prev = done[p - 1] if p else t0
        acc.setdefault(names[p], []).append(done[p] - prev)
    total.append(done[n_ph - 1] - t0)
tot = np.mean(total) / 1e3
print(f"{a.shape} L={L} TP{T} on {G} SMs each, R={a.w + 1} ctx={a.ctx}: pass {tot:.1f} us")
for k, v in acc.items():
    v = np.array(v, dtype=np.float64) / 1e3
    n = len(v) // a.reps
    print(f"  {k:7s} x{n:3d}: {v.mean():7.2f} us each, {v.sum() / a.reps:8.1f} us per pass, "
          f"{100 * v.sum() / a.reps / tot:5.1f}% of the pass")
for st in stages:
    st.close()
