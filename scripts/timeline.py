"""Per-phase timeline of the verify megakernel from its %globaltimer stamps
(the PS_TRACE build libpipespec_trace.so -- `python -m paper_2505_01572_b200._build
--trace`, selected here through PS_LIB -- ps_trace_read 9: [G][n_ph][8] u64 per CTA and phase:
0 epilogue start (after the phase wait), 1 publish, 2 X loader ready,
3 first full ring slot (MMA), 4 MMA done, 5 first accumulator, 6 last
accumulator, 7 last epilogue end).

Prints, per phase kind, the mean over layers of
  span  = T_done(p) - T_done(p-1)     (T_done = max over CTAs of the publish stamp)
  seen  = min over CTAs of the next start - T_done(p)     (publication latency)
  tail  = T_done(p) - median over CTAs of their publish stamp  (straggler tail)
and the ideal streaming time of the phase's weights at --gbs.

Usage: python scripts/timeline.py [--shape llama3.1-8b] [--ctx 512] [--w 4] [--layers N]
"""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("PS_LIB", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                             "paper_2505_01572_b200", "libpipespec_trace.so"))
import numpy as np
import torch

import synth
from paper_2505_01572_b200 import Stage, abi

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="llama3.1-8b")
ap.add_argument("--layers", type=int, default=None)
ap.add_argument("--ctx", type=int, default=512)
ap.add_argument("--w", type=int, default=4)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--gbs", type=float, default=6542.0)
a = ap.parse_args()
s = synth.preset(a.shape)
if a.layers:
    s = synth.reduced_depth(s, a.layers)
w = synth.make_weights(s, seed=1, device="cuda")
st = Stage(s, w, max_seq=a.ctx + 64, max_window=max(a.w, 1))
prompt = [int(x) for x in synth.make_prompt(s.vocab, a.ctx, seed=2)]
st.prefill(prompt)
win = [int(x) for x in synth.make_prompt(s.vocab, a.w, seed=3)]
L = s.n_layers
G = torch.cuda.get_device_properties(0).multi_processor_count
nph_max = 8 * L + 8
acc = {}
attn_st = []
sk = {}
mil = {}
for rep in range(a.reps + 1):
    if a.w:
        st.verify(win)
        st.kv_rollback(a.ctx)
    else:
        st.draft(1)
        st.kv_rollback(a.ctx)
    torch.cuda.synchronize()
    buf = np.zeros(G * nph_max * 8, dtype=np.uint64)
    abi.check(abi.lib().ps_trace_read(st.handle, 9, buf.ctypes.data, buf.nbytes))
    ebuf = np.zeros(nph_max * G * 4, dtype=np.uint64)
    abi.check(abi.lib().ps_trace_read(st.handle, 11, ebuf.ctypes.data, ebuf.nbytes))
    et = ebuf.reshape(nph_max, G, 4).astype(np.int64)
    if rep == 0:
        continue
    n_ph = 1 + 6 * L + 2
    t = buf[:G * n_ph * 8].reshape(G, n_ph, 8).astype(np.int64)
    pub = t[:, :n_ph, 1]
    start = t[:, :n_ph, 0]
    t0 = start[:, 0].min()
    done = pub.max(axis=0)
    names = ["EMBED"] + ["QKV", "ATTN", "ACOMB", "O", "GU", "DOWN"] * L + ["LMHEAD", "ARGMAX"]
    for p in range(n_ph):
        prev = done[p - 1] if p else t0
        span = done[p] - prev
        seen = (start[:, p + 1].min() - done[p]) if p + 1 < n_ph else 0
        tail = done[p] - np.median(pub[:, p])
        k = names[p]
        acc.setdefault(k, []).append((span, seen, tail))
        # within-phase milestones relative to T_done(p-1): median / max over CTAs
        row = []
        for j in (2, 3, 4, 6, 7, 1):
            col = t[:, p, j]
            col = col[col > 0]
            row += [np.median(col) - prev, col.max() - prev] if len(col) else [np.nan, np.nan]
        mil.setdefault(k, []).append(row)
        # stream-K fixup stamps of this phase: reducers have s1 (after the wait) in range
        e0, e1, e2 = et[p, :, 0] - prev, et[p, :, 1] - prev, et[p, :, 2] - prev
        red_ = (e1 > 0) & (e1 < 1e6) & (e2 >= e1)
        if red_.any():
            sk.setdefault(k, []).append([e0[red_].max(), e1[red_].max(), e2[red_].max(),
                                         np.median(e1[red_] - e0[red_]), (e1[red_] - e0[red_]).max(),
                                         np.median(e2[red_] - e1[red_]), (e2[red_] - e1[red_]).max(),
                                         (t[red_, p, 7] - prev - e2[red_]).max(),
                                         np.median(e0[~red_ & (e0 > 0) & (e0 < 1e6)]) if (~red_ & (e0 > 0) & (e0 < 1e6)).any() else np.nan,
                                         e0[~red_ & (e0 > 0) & (e0 < 1e6)].max() if (~red_ & (e0 > 0) & (e0 < 1e6)).any() else np.nan,
                                         np.median(t[red_, p, 6] - prev), (t[red_, p, 6] - prev).max()])
    acc.setdefault("TOTAL", []).append((done[n_ph - 1] - t0, 0, 0))
    # attention item stamps of the LAST layer's ATTN phase (first item per CTA)
    abuf = np.zeros(1024 * 8, dtype=np.uint64)
    abi.check(abi.lib().ps_trace_read(st.handle, 10, abuf.ctypes.data, abuf.nbytes))
    at = abuf.reshape(1024, 8)[:G].astype(np.int64)
    pa = 1 + 6 * (L - 1) + 1                       # last ATTN phase index
    ok = (at[:, 0] > done[pa - 1]) & (at[:, 0] < done[pa])
    if ok.any():
        rel = at[ok, :5] - done[pa - 1]
        attn_st.append([np.median(rel[:, j]) for j in range(5)] + [rel[:, 4].max(), ok.sum()]
                       + [np.median(at[ok, j]) for j in (5, 6, 7)])

R = a.w + 1
d, f, hq, hkv = s.d_model, s.d_ffn, s.n_heads * s.head_dim, s.n_kv_heads * s.head_dim
wbytes = {"QKV": (hq + 2 * hkv) * d * 2, "O": d * hq * 2, "GU": 2 * f * d * 2, "DOWN": d * f * 2,
          "LMHEAD": s.vocab * d * 2, "ATTN": (a.ctx + R) * 2 * hkv * 2}
print(f"{a.shape} L={L} R={R} ctx={a.ctx} G={G}")
print(f"{'phase':8s} {'n':>4s} {'span us':>9s} {'ideal us':>9s} {'seen us':>8s} {'tail us':>8s} {'sum us':>9s}")
for k, v in acc.items():
    v = np.array(v, dtype=np.float64) / 1e3
    n = len(v) // a.reps
    ideal = wbytes.get(k, 0) / (a.gbs * 1e9) * 1e6
    print(f"{k:8s} {n:4d} {v[:, 0].mean():9.2f} {ideal:9.2f} {v[:, 1].mean():8.2f} {v[:, 2].mean():8.2f} "
          f"{v[:, 0].mean() * n:9.1f}")
print("milestones (us after the previous phase completed; med/max over CTAs):")
print(f"{'phase':8s} {'Xready':>13s} {'MMA1st':>13s} {'MMAdone':>13s} {'lastacc':>13s} {'epiend':>13s} {'publish':>13s}")
for k, v in mil.items():
    v = np.nanmean(np.array(v, dtype=np.float64), axis=0) / 1e3
    print(f"{k:8s} " + " ".join(f"{v[2*i]:6.2f}/{v[2*i+1]:6.2f}" for i in range(6)))
if attn_st:
    v = np.array(attn_st, dtype=np.float64).mean(axis=0)
    print(f"ATTN (last layer, us after QKV done, median over CTAs): start {v[0]/1e3:.2f} "
          f"first softmax {v[2]/1e3:.2f} end {v[4]/1e3:.2f} (max {v[5]/1e3:.2f}, {v[6]:.0f} CTAs); "
          f"warp 0 time in: wait+bar {v[7]/1e3:.2f} QK {v[8]/1e3:.2f} softmax+PV {v[9]/1e3:.2f}")
print("stream-K reducers (us after the previous phase; max over reducer CTAs; wait/reduce med/max; epi after reduce max):")
for k, v in sk.items():
    v = np.nanmean(np.array(v, dtype=np.float64), axis=0) / 1e3
    print(f"{k:8s} s0 {v[0]:6.2f} s1 {v[1]:6.2f} s2 {v[2]:6.2f} wait {v[3]:5.2f}/{v[4]:5.2f} reduce {v[5]:5.2f}/{v[6]:5.2f} epi {v[7]:5.2f} nonred pub {v[8]:5.2f}/{v[9]:5.2f} red lastacc {v[10]:5.2f}/{v[11]:5.2f}")
st.close()
