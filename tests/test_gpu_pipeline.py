"""GPU: ps_pipeline_run (Alg.1) over the toy config (BASELINE configs[0]):
output identical to M_K autoregressive decoding, and the sync-SD accept trace
identical to the oracle DES under the same synthetic-alpha construction."""
import numpy as np
import pytest

import synth
from oracle import llama as L
from oracle import protocol as P
from oracle import synthetic as SY
from tests._parity import check_tokens_teacher_forced

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pair():
    from paper_2505_01572_b200 import Stage
    sd_, sv = synth.preset("toy-drafter"), synth.preset("toy-verifier")
    wd = synth.make_weights(sd_, seed=31, device="cuda")
    wv = synth.make_weights(sv, seed=32, device="cuda")
    d, v = Stage(sd_, wd, max_seq=256, max_window=8), Stage(sv, wv, max_seq=256, max_window=8)
    prompt = [int(x) for x in synth.make_prompt(256, 64, seed=33)]
    yield sd_, sv, wd, wv, d, v, prompt
    d.close()
    v.close()


def test_ar_and_sd_lossless(pair):
    from paper_2505_01572_b200 import pipeline_run
    from paper_2505_01572_b200.abi import PS_MODE_AR, PS_MODE_SYNC_SD
    sd_, sv, wd, wv, d, v, prompt = pair
    ar, _ = pipeline_run([d, v], prompt, 32, mode=PS_MODE_AR)
    check_tokens_teacher_forced(synth.weights_to_numpy(wv), sv, prompt, ar)
    # natural alpha (random-init drafter ~1/V agreement)
    sd, stats = pipeline_run([d, v], prompt, 32, mode=PS_MODE_SYNC_SD, gammas=[0, 4])
    assert sd == ar
    S = ar + [0] * 8
    for alpha in (0.0, 0.5, 0.9, 1.0):
        d.set_synthetic(S, len(prompt), level=0, top=1, alphas=[alpha], seed=77)
        sd, stats = pipeline_run([d, v], prompt, 32, mode=PS_MODE_SYNC_SD, gammas=[0, 4])
        assert sd == ar, alpha
        gpu_hist = {k: int(c) for k, c in enumerate(stats.accept_hist) if c}
        # oracle DES with the same chained construction against the same stream
        wd64, wv64 = synth.weights_to_numpy(wd), synth.weights_to_numpy(wv)
        base = P.LlamaModels([(wd64, sd_), (wv64, sv)])
        chain = SY.StreamChain(S, len(prompt), 77, [alpha], 256, base.predict)
        r = P.run("sd", [P.StageCfg(1.0), P.StageCfg(4.0, 4)], P.StreamModels(chain, base), prompt, 32)
        assert r.tokens == ar
        assert gpu_hist == r.accept_hist, (alpha, gpu_hist, r.accept_hist)
    d.clear_synthetic()


@pytest.mark.parametrize("alpha", [0.0, 0.6, 0.9, 1.0])
def test_async_pipespec_lossless_two_stage(pair, alpha):
    """PS_MODE_PIPESPEC (Alg.1, one host thread per stage) == M_K AR output."""
    from paper_2505_01572_b200 import pipeline_run
    from paper_2505_01572_b200.abi import PS_MODE_AR, PS_MODE_PIPESPEC
    sd_, sv, wd, wv, d, v, prompt = pair
    d.clear_synthetic()
    ar, _ = pipeline_run([d, v], prompt, 40, mode=PS_MODE_AR)
    d.set_synthetic(ar + [0] * 16, len(prompt), level=0, top=1, alphas=[alpha], seed=5)
    ps, stats = pipeline_run([d, v], prompt, 40, mode=PS_MODE_PIPESPEC, gammas=[0, 6])
    assert ps == ar
    assert stats.tokens == 40
    assert stats.steps[1] >= 1
    if alpha == 1.0:
        assert stats.verify_steps[1] >= 1
    d.clear_synthetic()


def test_async_pipespec_three_stage_and_lookahead():
    from paper_2505_01572_b200 import Stage, pipeline_run
    from paper_2505_01572_b200.abi import PS_MODE_AR, PS_MODE_PIPESPEC, PS_MODE_SYNC_SD
    s0, s1 = synth.preset("toy-drafter"), synth.preset("toy-verifier")
    st = [Stage(s0, synth.make_weights(s0, seed=41, device="cuda"), max_seq=256, max_window=8),
          Stage(s1, synth.make_weights(s1, seed=42, device="cuda"), max_seq=256, max_window=8),
          Stage(s1, synth.make_weights(s1, seed=43, device="cuda"), max_seq=256, max_window=8)]
    prompt = [int(x) for x in synth.make_prompt(256, 48, seed=44)]
    ar, _ = pipeline_run(st, prompt, 36, mode=PS_MODE_AR)
    S = ar + [0] * 16
    st[0].set_synthetic(S, len(prompt), level=0, top=2, alphas=[0.9, 0.8], seed=9)
    st[1].set_synthetic(S, len(prompt), level=1, top=2, alphas=[0.8], seed=9)
    for la in (0, 2):
        ps, stats = pipeline_run(st, prompt, 36, mode=PS_MODE_PIPESPEC, gammas=[0, 4, 6], lookaheads=[0, la, la])
        assert ps == ar
    sd, _ = pipeline_run(st, prompt, 36, mode=PS_MODE_SYNC_SD, gammas=[0, 4, 6])
    assert sd == ar
    for x in st:
        x.close()
