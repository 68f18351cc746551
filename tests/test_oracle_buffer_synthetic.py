"""Pins for oracle/buffer.py and oracle/synthetic.py
(alpha definition §3.3)."""
import math

import numpy as np
import pytest

from oracle import buffer as B
from oracle import synthetic as S


def test_buffer_examples_spec():
    b = B.TokenBuffer([])
    b.append([5, 7]); assert b.tokens == [5, 7]
    b = B.TokenBuffer([1]); b.append([]); assert b.tokens == [1]
    b = B.TokenBuffer([1, 2]); b.append([3]); assert b.tokens == [1, 2, 3]
    b = B.TokenBuffer([1, 2, 3, 4]); b.rollback(2); assert b.tokens == [1, 2]
    b = B.TokenBuffer([1, 2, 3]); b.rollback(3); assert b.tokens == [1, 2, 3]
    b = B.TokenBuffer([1, 2, 3]); b.rollback(0); assert b.tokens == []
    with pytest.raises(B.ContractError):
        B.TokenBuffer([1, 2]).rollback(3)


def test_kv_len_and_pages():
    b = B.TokenBuffer(list(range(100)))
    assert b.kv_len == 99 and b.pages(16) == 7
    b.rollback(33)
    assert b.kv_len == 32 and b.pages(16) == 2 and b.tokens[-1] == 32
    b.append([1, 2, 3])
    assert b.kv_len == 35 and b.pages(16) == 3
    b.rollback(36)   # no-op
    assert b.kv_len == 35


def test_resync_rules():
    # stage 0 at length 12 resynced to stage 1's 7 tokens
    lo = B.TokenBuffer(list(range(12)))
    hi = list(range(6)) + [99]
    m = lo.resync(hi)
    assert lo.tokens == hi and m == 6 and lo.kv_len == 5
    # no-op when already an extension
    lo = B.TokenBuffer(list(range(12)))
    assert lo.resync(list(range(7))) == 12 and lo.tokens == list(range(12))


def test_counter_generator_reference_values():
    # splitmix64 reference outputs for seed 0 (Vigna's splitmix64.c: first outputs
    # of the sequence x += golden; z = mix(x)) -- an external pin of `sm`.
    x, outs = 0, []
    for _ in range(3):
        outs.append(S.sm(x))
        x = (x + 0x9E3779B97F4A7C15) & S.M64
    assert outs == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


def test_agreement_frequency_binomial():
    """Empirical agreement within a binomial 3-sigma band."""
    seed, V = 12345, 32768
    for a in (0.0, 0.3, 0.8, 1.0):
        thr = S.alpha_threshold(a)
        n = 100_000
        k = sum(S.agree(seed, 0, p, thr) for p in range(n))
        sig = math.sqrt(n * a * (1 - a))
        assert abs(k - n * a) <= 3 * sig + 1e-9


def test_other_token_differs_and_in_range():
    V = 7
    for p in range(2000):
        for t in range(V):
            o = S.other(t, 3, 1, p, V)
            assert o != t and 0 <= o < V


def test_chain_transitive_agreement():
    """Stage 0 agrees with stage K iff every link agrees; rate ~ product."""
    seed, V, alphas = 77, 1000, [0.9, 0.7]
    thrs = [S.alpha_threshold(a) for a in alphas]
    n, k0K, k01 = 50_000, 0, 0
    for p in range(n):
        tK = p % V
        t1 = S.chained_token(tK, 1, 2, p, seed, thrs, V)
        t0 = S.chained_token(tK, 0, 2, p, seed, thrs, V)
        assert t1 == (tK if S.agree(seed, 1, p, thrs[1]) else S.other(tK, seed, 1, p, V))
        k0K += t0 == tK
        k01 += t0 == t1
    pr = 0.9 * 0.7
    assert abs(k0K - n * pr) <= 3 * math.sqrt(n * pr * (1 - pr)) + 0.001 * n  # + rare re-collisions
    assert abs(k01 - n * 0.9) <= 3 * math.sqrt(n * 0.09)


def test_hash_chain_replay_stable():
    ch = S.HashChain(5, [0.8], 100)
    c = [1, 2, 3, 4]
    assert ch.predict(0, c) == ch.predict(0, list(c))
    assert ch.predict(1, c) == ch.predict_h(1, ch.ctx_hash(c))
