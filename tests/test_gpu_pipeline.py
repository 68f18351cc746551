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
    i = next((j for j in range(min(len(ps), len(ar))) if ps[j] != ar[j]), None)
    assert ps == ar, (f"first diff at {i}: ps {ps[i:i + 4] if i is not None else ps[len(ar):]} "
                      f"ar {ar[i:i + 4] if i is not None else []}; steps {list(stats.steps[:2])} "
                      f"verify {list(stats.verify_steps[:2])} rollbacks {list(stats.rollbacks[:2])} "
                      f"hist {[int(x) for x in stats.accept_hist[:8]]}")
    assert stats.tokens == 40
    assert stats.steps[1] >= 1
    if alpha == 1.0:
        # With lookahead 0 the verifier takes an AR step whenever no draft is
        # waiting (reading R7), so on one GPU the schedule may never verify a
        # window (the two stages' kernels serialise).  Lookahead 1 makes it
        # wait for a draft: every verifier step is then a verification.
        ps1, st1 = pipeline_run([d, v], prompt, 40, mode=PS_MODE_PIPESPEC, gammas=[0, 6], lookaheads=[0, 1])
        assert ps1 == ar
        assert st1.verify_steps[1] >= 1 and st1.verify_steps[1] == st1.steps[1]
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


def _stage_process(rank, board, S, n, q):
    """One stage per process: M_0 (toy drafter, synthetic alpha 0.8 against S)
    or M_1 (toy verifier), both on cuda:0, through ps_pipeline_run_rank."""
    import os
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import synth as sy
    from paper_2505_01572_b200 import Stage, pipeline_run_rank
    name, seed = ("toy-drafter", 31) if rank == 0 else ("toy-verifier", 32)
    s = sy.preset(name)
    w = sy.make_weights(s, seed=seed, device="cuda")
    st = Stage(s, w, max_seq=256, max_window=8)
    prompt = [int(x) for x in sy.make_prompt(256, 64, seed=33)]
    if rank == 0:
        st.set_synthetic(S, len(prompt), level=0, top=1, alphas=[0.8], seed=78)
    try:
        out, stats = pipeline_run_rank(st, rank, 2, board, prompt, n, gammas=[0, 4], lookaheads=[0, 2])
        q.put((rank, "ok", out, int(stats.verify_steps[1]), int(stats.rollbacks[0])))
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e), [], 0, 0))
    st.close()


def test_stage_per_process_pipespec_lossless(pair):
    """The paper's layout -- each model in its own process (its own GPU in a
    deployment; here both on cuda:0, so the verifier waits for 2 drafts
    (lookahead 2) instead of racing the time-sliced drafter) -- through the
    shared-memory board:
    output == M_K autoregressive decoding, verify steps taken."""
    import os
    import torch.multiprocessing as mp
    from paper_2505_01572_b200 import board_create, board_unlink, pipeline_run
    from paper_2505_01572_b200.abi import PS_MODE_AR
    sd_, sv, wd, wv, d, v, prompt = pair
    n = 40
    ar, _ = pipeline_run([d, v], prompt, n + 8, mode=PS_MODE_AR)
    board = f"/pipespec-gpu-{os.getpid()}"
    board_create(board, 2, 64 + n + 400)
    try:
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        procs = [ctx.Process(target=_stage_process, args=(r, board, ar, n, q)) for r in range(2)]
        for p in procs:
            p.start()
        res = sorted(q.get(timeout=240) for _ in range(2))
        for p in procs:
            p.join(timeout=60)
    finally:
        board_unlink(board)
    for rank, status, out, vsteps, rb in res:
        assert status == "ok", (rank, status)
        assert out == ar[:n], rank
        assert vsteps > 0
