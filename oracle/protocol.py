"""Virtual-clock discrete-event simulation of the k-model protocol.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Modes:
  'ar'        autoregressive M_K (§3.1, Fig.2(1)); the lossless target.
  'sd'        synchronous (tiered) speculative decoding: the drafter produces
              exactly gamma tokens, then the verifier verifies them, in lockstep
              ("Synchronous Execution"; Eq.5; Tab.1 "Synchronous"/
              "Multi-Draft" = tiered when k > 2).
  'pipespec'  asynchronous PipeSpec, Algorithm 1: every stage runs
              concurrently; M_0 drafts continuously; stage i>0 takes
              its window from O_{i-1}, verifies, appends the matching prefix and
              its own correction / bonus token (reading R1), and on a mismatch
              signals rejection: every stage j<i is resynced to O_i (P:97,
              P:106-107, reading R2) and its in-flight step is discarded
              ("discarded and regenerated").

Rules where the paper is silent (readings R3, R7, R9):
  * a verify step costs t_i regardless of window size (R3);
  * window = the next min(valid drafts, gamma_i) tokens; with lookahead L_i = 0
    a stage verifies whenever >= 1 valid draft exists and otherwise takes an AR
    step (the 1-token branch of Eq.1); L_i >= 1 waits for L_i drafts (R7);
  * before taking a window, stage i checks the drafter's token at its pending
    position n-1; a mismatch resyncs the stages below (R2);
  * messages are instantaneous; simultaneous events are ordered by
    (time, stage index, sequence); a stage whose buffer is resynced
    bumps its epoch and restarts immediately, so stale results are dropped and
    the highest-origin rollback wins (R9);
  * a drafter idles while it is `max_lead` tokens ahead of its verifier
    (bounded draft ring; must exceed gamma so Eq.1/Eq.3 can hold, R4).

`model.predict(i, toks, H)` returns stage i's greedy next token for context
`toks` (numpy int64 view); `H` is the context's rolling hash when the model
asks for one (`model.uses_hash`), else None.  `verify` below is Alg.1's
compare-and-append evaluated lazily (predictions after the first mismatch
cannot change the result).
"""
from __future__ import annotations

import heapq
from dataclasses import dataclass, field

import numpy as np

from .synthetic import sm


@dataclass
class StageCfg:
    t: float              # t_i, per-step latency
    gamma: int = 8        # gamma_i, verify window cap
    lookahead: int = 0    # L_i


@dataclass
class StageStats:
    steps: int = 0
    verify_steps: int = 0
    ar_steps: int = 0
    discarded: int = 0
    rollbacks: int = 0
    busy: float = 0.0
    appended: int = 0


@dataclass
class RunResult:
    tokens: list
    time: float
    stats: list
    accept_hist: dict = field(default_factory=dict)   # tokens appended per stage-K verify step
    events: list = field(default_factory=list)        # (time, stage, kind, payload)


class Buf:
    """Token buffer O_i as a growable int64 array, with optional prefix hashes."""

    def __init__(self, toks, cap, hashed, seed):
        self.t = np.zeros(cap, dtype=np.int64)
        self.n = 0
        self.hashed = hashed
        self.h = [sm(seed ^ 0xC0FFEE)] if hashed else None
        self.extend(toks)

    def view(self):
        return self.t[:self.n]

    def extend(self, toks):
        for x in toks:
            self.t[self.n] = int(x)
            self.n += 1
            if self.hashed:
                self.h.append(sm(self.h[-1] ^ int(x)))

    def truncate(self, m):
        self.n = m
        if self.hashed:
            del self.h[m + 1:]

    def first_mismatch(self, src) -> int:
        L = min(self.n, src.n)
        diff = np.nonzero(self.t[:L] != src.t[:L])[0]
        return int(diff[0]) if diff.size else L

    def resync(self, src) -> bool:
        """Make this buffer consistent with src (no-op if it already extends src,
        S:332).  Returns True if the content changed."""
        m = self.first_mismatch(src)
        if m == src.n:
            return False
        self.truncate(m)
        self.extend(src.t[m:src.n])
        return True


def _hash_ext(H, tok):
    return sm(H ^ int(tok))


def verify(model, i, buf, window):
    """Alg.1 P:101-105 with correction/bonus: returns (a, next)."""
    n = buf.n
    ctx = buf.t.copy()[: n + len(window) + 1]
    H = buf.h[n] if buf.hashed else None
    a = 0
    while True:
        p = model.predict(i, ctx[: n + a], H)
        if a < len(window) and p == window[a]:
            ctx[n + a] = window[a]
            if H is not None:
                H = _hash_ext(H, window[a])
            a += 1
            continue
        return a, p


def _predict_next(model, i, buf):
    return model.predict(i, buf.view(), buf.h[buf.n] if buf.hashed else None)


def _done(O, n_prompt, max_new, eos):
    gen = O.t[n_prompt:O.n]
    return gen.size >= max_new or (eos is not None and (gen == eos).any())


def _finish(O, n_prompt, max_new, eos):
    gen = [int(x) for x in O.t[n_prompt:O.n]]
    if eos is not None and eos in gen:
        gen = gen[: gen.index(eos) + 1]
    return gen[:max_new]


# ----------------------------------------------------------------------------- AR
def run_ar(cfgs, model, prompt, max_new, eos=None, seed=0):
    K = len(cfgs) - 1
    O = Buf(prompt, len(prompt) + max_new + 1, model.uses_hash, seed)
    st = [StageStats() for _ in cfgs]
    T = 0.0
    while not _done(O, len(prompt), max_new, eos):
        O.extend([_predict_next(model, K, O)])
        T += cfgs[K].t
        st[K].steps += 1
        st[K].ar_steps += 1
        st[K].busy += cfgs[K].t
        st[K].appended += 1
    return RunResult(_finish(O, len(prompt), max_new, eos), T, st)


# ----------------------------------------------------------------------------- sync SD
def run_sd(cfgs, model, prompt, max_new, eos=None, seed=0):
    """Tiered synchronous SD: stage i (i>0) obtains gamma_i drafts from stage i-1
    (itself running synchronous SD when i-1 > 0), then verifies them."""
    K = len(cfgs) - 1
    cap = len(prompt) + max_new + sum(c.gamma for c in cfgs) * (K + 1) + 8
    st = [StageStats() for _ in cfgs]
    hist, events = {}, []
    clock = [0.0]

    def produce(i, ctx, m):
        """m greedy tokens of stage i after buffer ctx (ctx is not modified)."""
        buf = Buf([], cap, model.uses_hash, seed)
        buf.extend(ctx.view())
        out = []
        while len(out) < m:
            if i == 0 or cfgs[i].gamma == 0:
                tok = _predict_next(model, i, buf)
                clock[0] += cfgs[i].t
                st[i].steps += 1
                st[i].ar_steps += 1
                st[i].busy += cfgs[i].t
                buf.extend([tok])
                out.append(tok)
                continue
            d = produce(i - 1, buf, cfgs[i].gamma)
            a, nxt = verify(model, i, buf, d)
            clock[0] += cfgs[i].t
            st[i].steps += 1
            st[i].verify_steps += 1
            st[i].busy += cfgs[i].t
            app = list(d[:a]) + [nxt]
            if a < len(d):
                st[i - 1].rollbacks += 1
            if i == K:
                hist[len(app)] = hist.get(len(app), 0) + 1
                events.append((clock[0], i, "verify", (buf.n, list(d), a, nxt)))
            buf.extend(app)
            out.extend(app)
        return out[:m] if i < K else out

    O = Buf(prompt, cap, model.uses_hash, seed)
    while not _done(O, len(prompt), max_new, eos):
        need = max_new - (O.n - len(prompt))
        if K == 0:
            O.extend(produce(0, O, need))
        else:
            # one verify round of the top stage
            d = produce(K - 1, O, cfgs[K].gamma) if cfgs[K].gamma > 0 else []
            if d:
                a, nxt = verify(model, K, O, d)
                st[K].verify_steps += 1
                if a < len(d):
                    st[K - 1].rollbacks += 1
                app = list(d[:a]) + [nxt]
                hist[len(app)] = hist.get(len(app), 0) + 1
                events.append((clock[0] + cfgs[K].t, K, "verify", (O.n, list(d), a, nxt)))
            else:
                app = [_predict_next(model, K, O)]
                st[K].ar_steps += 1
            clock[0] += cfgs[K].t
            st[K].steps += 1
            st[K].busy += cfgs[K].t
            st[K].appended += len(app)
            O.extend(app)
        del need
    return RunResult(_finish(O, len(prompt), max_new, eos), clock[0], st, hist, events)


# ----------------------------------------------------------------------------- PipeSpec
def run_pipespec(cfgs, model, prompt, max_new, eos=None, seed=0, max_lead=None,
                 record=False, max_steps=None):
    K = len(cfgs) - 1
    if K == 0:
        return run_ar(cfgs, model, prompt, max_new, eos, seed)
    if max_lead is None:
        max_lead = 2 * max(c.gamma for c in cfgs) + max(c.lookahead for c in cfgs) + 2
    assert max_lead > max(max(c.gamma, c.lookahead) for c in cfgs[1:])
    n_prompt = len(prompt)
    cap = n_prompt + max_new + (max_lead + max(c.gamma for c in cfgs) + 2) * (K + 1) + 8
    bufs = [Buf(prompt, cap, model.uses_hash, seed) for _ in range(K + 1)]
    st = [StageStats() for _ in cfgs]
    epoch = [0] * (K + 1)
    started = [0.0] * (K + 1)
    step = [None] * (K + 1)
    waiting = [False] * (K + 1)
    heap, seqc = [], [0]
    hist, events = {}, []
    finished = [False]

    def push(i, T):
        seqc[0] += 1
        heapq.heappush(heap, (T + cfgs[i].t, i, seqc[0], epoch[i]))
        started[i] = T

    def rollback_below(i, T):
        for j in range(i - 1, -1, -1):
            if bufs[j].resync(bufs[i]):
                st[j].rollbacks += 1
                epoch[j] += 1
                if record:
                    events.append((T, j, "rollback", (i, bufs[i].n)))
                if step[j] is not None:          # discard in-flight work, restart now
                    st[j].discarded += 1
                    st[j].busy += T - started[j]
                    step[j] = None
                    start(j, T)
                else:
                    wake(j, T)

    def wake(j, T):
        if 0 <= j <= K and waiting[j]:
            waiting[j] = False
            start(j, T)

    def start(i, T):
        if finished[0] or step[i] is not None:
            return
        O = bufs[i]
        if i < K and (O.n >= bufs[i + 1].n + max_lead or O.n >= cap - cfgs[i].gamma - 2):
            waiting[i] = True                # bounded draft ring: idle while far ahead
            return
        if i == 0:
            step[0] = ("draft", None)
            push(0, T)
            return
        P = bufs[i - 1]
        n = O.n
        if P.n >= n and P.first_mismatch(O) < n:
            # the drafter's buffer disagrees with mine somewhere in O_i[0:n] (its
            # token at my pending position, or -- after a higher stage's rollback
            # left it on a short prefix of O_i -- earlier): resync it to O_i
            # (Alg.1 P:97 "Rollback O_i", reading R2)
            rollback_below(i, T)
        m = P.first_mismatch(O)
        avail = P.n - n if m >= n else 0
        w = min(max(avail, 0), cfgs[i].gamma)
        if avail >= max(1, cfgs[i].lookahead):
            step[i] = ("verify", P.t[n:n + w].copy())
        elif cfgs[i].lookahead == 0:
            step[i] = ("ar", np.zeros(0, dtype=np.int64))
        else:
            waiting[i] = True
            return
        push(i, T)

    def end(i, T):
        kind, window = step[i]
        step[i] = None
        O = bufs[i]
        st[i].steps += 1
        st[i].busy += cfgs[i].t
        if i == 0:
            O.extend([_predict_next(model, 0, O)])
            st[0].appended += 1
            wake(1, T)
        else:
            a, nxt = verify(model, i, O, window)
            w = len(window)
            if kind == "verify":
                st[i].verify_steps += 1
            else:
                st[i].ar_steps += 1
            app = [int(x) for x in window[:a]] + [nxt]
            if record:
                events.append((T, i, kind, (O.n, [int(x) for x in window], a, nxt)))
            if i == K and kind == "verify":
                hist[len(app)] = hist.get(len(app), 0) + 1
            O.extend(app)
            st[i].appended += len(app)
            if a < w:
                rollback_below(i, T)
            if i == K and _done(O, n_prompt, max_new, eos):
                finished[0] = True
                return
            wake(i + 1, T)
            wake(i - 1, T)
        start(i, T)

    for i in range(K + 1):
        start(i, 0.0)
    T = 0.0
    while heap and not finished[0]:
        T, i, _, ep = heapq.heappop(heap)
        if ep != epoch[i] or step[i] is None:
            continue
        end(i, T)
        if max_steps is not None and st[K].steps >= max_steps:
            break
    if not finished[0] and (max_steps is None or st[K].steps < max_steps):
        raise RuntimeError("pipespec DES stalled (no runnable stage)")
    return RunResult(_finish(bufs[K], n_prompt, max_new, eos), T, st, hist, events)


def run(mode, cfgs, model, prompt, max_new, eos=None, seed=0, **kw):
    if mode == "ar":
        return run_ar(cfgs, model, prompt, max_new, eos, seed)
    if mode == "sd":
        return run_sd(cfgs, model, prompt, max_new, eos, seed)
    if mode == "pipespec":
        return run_pipespec(cfgs, model, prompt, max_new, eos, seed, **kw)
    raise ValueError(mode)


# ----------------------------------------------------------------------------- models
class LlamaModels:
    """Stage models backed by oracle.llama (greedy argmax), with a context cache."""
    uses_hash = False

    def __init__(self, stages):
        """stages: list of (weights64, shape) for M_0..M_K."""
        from . import llama
        self._llama = llama
        self.stages = stages
        self.cache = {}

    def predict(self, i, toks, H=None):
        key = (i, tuple(int(x) for x in toks))
        r = self.cache.get(key)
        if r is None:
            w, s = self.stages[i]
            r = self._llama.greedy(self._llama.forward_full(w, s, list(key[1]))[-1])
            self.cache[key] = r
        return r


class HashModels:
    """All stages synthetic (oracle.synthetic.HashChain)."""
    uses_hash = True

    def __init__(self, chain):
        self.chain = chain

    def predict(self, i, toks, H):
        return self.chain.predict_h(i, H)


class StreamModels:
    """Stages < K synthetic against stream S (oracle.synthetic.StreamChain),
    stage K and off-path predictions from `base` (e.g. LlamaModels)."""
    uses_hash = False

    def __init__(self, chain, base):
        self.chain = chain
        self.base = base

    def predict(self, i, toks, H=None):
        if i < self.chain.K and self.chain.on_path(toks):
            p = len(toks) - self.chain.n_prompt
            from .synthetic import chained_token
            return chained_token(self.chain.S[p], i, self.chain.K, p, self.chain.seed,
                                 self.chain.thrs, self.chain.vocab)
        return self.base.predict(i, toks, H)
