"""Pins for oracle/protocol.py: losslessness (output == AR of M_K, the central
property implied by exact-match greedy verification, Alg.1),
Eq.5 for sync SD, Eqs.1/3 for async PipeSpec (conditions of reading R4), and
qualitative shapes (§4.3 long tail)."""
import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

import synth
from oracle import analytic as A
from oracle import llama as L
from oracle import protocol as P
from oracle import synthetic as S


def hash_models(seed, alphas, V=500):
    return P.HashModels(S.HashChain(seed, alphas, V))


@settings(max_examples=120, deadline=None)
@given(k=st.integers(2, 4), seed=st.integers(0, 2**31), data=st.data())
def test_lossless_random_configs(k, seed, data):
    """SPEC criterion 5: >= 100 random configs, PS and sync SD == AR."""
    alphas = [data.draw(st.floats(0.1, 0.99)) for _ in range(k - 1)]
    cfgs = [P.StageCfg(t=data.draw(st.floats(0.2, 20.0)), gamma=data.draw(st.integers(1, 12)),
                       lookahead=data.draw(st.integers(0, 3))) for _ in range(k)]
    m = hash_models(seed, alphas)
    prompt = [int(x) for x in np.random.default_rng(seed).integers(0, 500, 5)]
    n = data.draw(st.integers(1, 60))
    ar = P.run("ar", cfgs, m, prompt, n)
    assert len(ar.tokens) == n
    assert P.run("sd", cfgs, m, prompt, n).tokens == ar.tokens
    assert P.run("pipespec", cfgs, m, prompt, n).tokens == ar.tokens


def test_lossless_real_models_and_synthetic_alpha():
    """Toy config (BASELINE configs[0]): toy-drafter -> toy-verifier, gamma=4,
    natural alpha and synthetic alpha in {0, 0.5, 0.9, 1} (StreamChain)."""
    sd_, sv = synth.preset("toy-drafter"), synth.preset("toy-verifier")
    wd = synth.weights_to_numpy(synth.make_weights(sd_, seed=10))
    wv = synth.weights_to_numpy(synth.make_weights(sv, seed=11))
    prompt = list(synth.make_prompt(sv.vocab, 64, seed=12))
    base = P.LlamaModels([(wd, sd_), (wv, sv)])
    stream, _ = L.ar_decode(wv, sv, prompt, 40)   # S longer than the run: no end effects
    cfgs = [P.StageCfg(1.0), P.StageCfg(4.0, gamma=4)]
    for mode in ("ar", "sd", "pipespec"):
        assert P.run(mode, cfgs, base, prompt, 32).tokens == stream[:32]
    for alpha in (0.0, 0.5, 0.9, 1.0):
        m = P.StreamModels(S.StreamChain(stream, len(prompt), 5, [alpha], sv.vocab, base.predict), base)
        for mode in ("sd", "pipespec"):
            r = P.run(mode, cfgs, m, prompt, 32)
            assert r.tokens == stream[:32]
        if alpha == 1.0:   # every sync-SD window fully accepted: gamma + 1 tokens per round
            r = P.run("sd", cfgs, m, prompt, 32)
            assert set(r.accept_hist) <= {5}
        if alpha == 0.0:
            r = P.run("sd", cfgs, m, prompt, 32)
            assert set(r.accept_hist) == {1}


def test_three_stage_real_models_lossless():
    s0, s1 = synth.preset("toy-drafter"), synth.preset("toy-verifier")
    w0 = synth.weights_to_numpy(synth.make_weights(s0, seed=1))
    w1 = synth.weights_to_numpy(synth.make_weights(s1, seed=2))
    w2 = synth.weights_to_numpy(synth.make_weights(s1, seed=3))
    prompt = list(synth.make_prompt(256, 24, seed=4))
    base = P.LlamaModels([(w0, s0), (w1, s1), (w2, s1)])
    stream, _ = L.ar_decode(w2, s1, prompt, 20)
    m = P.StreamModels(S.StreamChain(stream, len(prompt), 9, [0.9, 0.8], 256, base.predict), base)
    cfgs = [P.StageCfg(1.0, 0), P.StageCfg(3.0, 4), P.StageCfg(9.0, 4)]
    for mode in ("sd", "pipespec"):
        assert P.run(mode, cfgs, m, prompt, 20).tokens == stream


@pytest.mark.parametrize("alpha,gamma,c", [(0.8, 4, 4.0), (0.95, 8, 10.0), (1.0, 4, 10.0),
                                           (0.8, 8, 4.0)])
def test_sync_sd_matches_eq5(alpha, gamma, c):
    """SPEC criterion 4: simulated sync-SD speedup vs Eq.5 within 3%."""
    m = hash_models(21, [alpha], V=1000)
    cfgs = [P.StageCfg(1.0), P.StageCfg(c, gamma)]
    n = 6000
    ar = P.run("ar", cfgs, m, [1, 2, 3], n)
    sd = P.run("sd", cfgs, m, [1, 2, 3], n)
    assert sd.tokens == ar.tokens
    assert ar.time / sd.time == pytest.approx(A.sd_speedup(alpha, gamma, c), rel=0.03)


def test_sync_sd_alpha0_slower_than_ar():
    m = hash_models(2, [0.0], V=1000)
    cfgs = [P.StageCfg(1.0), P.StageCfg(10.0, 8)]
    ar = P.run("ar", cfgs, m, [1], 300)
    sd = P.run("sd", cfgs, m, [1], 300)
    assert ar.time / sd.time < 1.0


@pytest.mark.parametrize("alpha,gamma", [(0.5, 2), (0.8, 4), (0.95, 8)])
def test_async_rates_match_eq1_eq3(alpha, gamma):
    """SPEC criterion 2 under reading R4 (c = gamma+1, gamma-capped windows,
    lookahead 0): verify probability within 0.01 of Eq.3, tokens/step within 2%
    of Eq.1 over 2e4 stage-K steps."""
    m = hash_models(7, [alpha], V=1000)
    cfgs = [P.StageCfg(1.0), P.StageCfg(float(gamma + 1), gamma=gamma)]
    r = P.run_pipespec(cfgs, m, list(range(10)), 20000 * (gamma + 2), max_steps=20000)
    sK = r.stats[1]
    assert sK.verify_steps / sK.steps == pytest.approx(A.rho_steady_state(alpha, gamma), abs=0.01)
    assert sK.appended / sK.steps == pytest.approx(A.pipespec_rate(alpha, gamma), rel=0.02)


def test_async_beats_sync_and_long_tail():
    """Tab.1 'async > sync' for the same models; §4.3 long tail with an unbounded
    window at alpha=0.9 while sync SD stays <= gamma+1 = 9 (SPEC criterion 9)."""
    m = hash_models(3, [0.9], V=1000)
    ar = P.run("ar", [P.StageCfg(1.0), P.StageCfg(40.0, 8)], m, [0], 2000)
    sd = P.run("sd", [P.StageCfg(1.0), P.StageCfg(40.0, 8)], m, [0], 2000)
    ps = P.run("pipespec", [P.StageCfg(1.0), P.StageCfg(40.0, 64)], m, [0], 2000)
    assert ar.tokens == sd.tokens == ps.tokens
    assert ps.time < sd.time < ar.time
    assert max(sd.accept_hist) <= 9
    assert max(ps.accept_hist) > 20


def test_deterministic():
    m = hash_models(4, [0.7, 0.8])
    cfgs = [P.StageCfg(1.0, 0), P.StageCfg(3.0, 4), P.StageCfg(12.0, 6)]
    a = P.run("pipespec", cfgs, m, [1, 2], 200, record=True)
    b = P.run("pipespec", cfgs, m, [1, 2], 200, record=True)
    assert a.tokens == b.tokens and a.events == b.events and a.time == b.time
