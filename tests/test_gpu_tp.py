"""GPU parity of the tensor-parallel verify pass.

T ranks of one stage, each a megakernel on its own partition of the GPU's SMs
(`max_ctas`), connected with ps_tp_connect_local: the multi-GPU layout with the
peer buffers in local instead of NVLink memory -- the same kernel code, the same
exchange protocol.  Every rank holds only its Megatron shard; the results are
checked against the fp64 oracle of the FULL model, and the ranks must agree
bit for bit (same a, next, tokens)."""
import threading

import numpy as np
import pytest
import torch

import synth
from oracle import llama as L
from tests._parity import check_logits, check_tokens_teacher_forced, check_verify

pytestmark = pytest.mark.gpu


def run_all(stages, fn, timeout=300):
    """fn(stage) on every rank concurrently (one host thread per rank, as the
    ABI requires); returns the per-rank results, re-raising the first error."""
    res, err = [None] * len(stages), [None] * len(stages)

    def go(i):
        try:
            res[i] = fn(stages[i])
        except BaseException as e:  # noqa: BLE001
            err[i] = e

    th = [threading.Thread(target=go, args=(i,)) for i in range(len(stages))]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout)
    assert not any(t.is_alive() for t in th), "tensor-parallel call hung"
    for e in err:
        if e is not None:
            raise e
    return res


def make_group(shape, w, T, max_seq=512, max_window=31):
    from paper_2505_01572_b200 import Stage, shard_weights, tp_connect_local
    n_sm = torch.cuda.get_device_properties(0).multi_processor_count
    stages = [Stage(shape, shard_weights(shape, w, r, T), max_seq=max_seq, max_window=max_window,
                    tp_rank=r, tp_size=T, max_ctas=n_sm // T) for r in range(T)]
    tp_connect_local(stages)
    return stages


def agree(res):
    for r in res[1:]:
        assert r == res[0], (r, res[0])
    return res[0]


@pytest.fixture(scope="module", params=[2, 4])
def toy_group(request):
    T = request.param
    s = synth.preset("toy-tp")
    w = synth.make_weights(s, seed=31, device="cuda")
    w64 = synth.weights_to_numpy(w)
    prompt = list(synth.make_prompt(s.vocab, 48, seed=32))
    stages = make_group(s, w, T, max_seq=256)
    yield s, w64, stages, prompt, T
    for st in stages:
        st.close()


@pytest.mark.parametrize("case", ["w0", "full", "reject0", "reject_mid", "w16", "w31"])
def test_tp_verify_matches_oracle(toy_group, case):
    s, w64, stages, prompt, T = toy_group
    x = list(prompt)
    stream, _ = L.ar_decode(w64, s, x, 32)
    W = {"w0": [], "full": stream[:8], "reject0": [(stream[0] + 5) % s.vocab] + stream[1:4],
         "reject_mid": stream[:5] + [(stream[5] + 1) % s.vocab] + stream[6:9],
         "w16": stream[:16], "w31": stream[:31]}[case]
    run_all(stages, lambda st: st.prefill(x))
    res = run_all(stages, lambda st: st.verify(W, want_logits=True))
    a, nxt = agree([(r[0], r[1]) for r in res])
    logits = np.concatenate([r[2] for r in res], axis=1)   # rank r holds vocab slice r
    ref = L.verify(w64, s, x, W)
    check_logits(logits, ref["logits"])
    check_verify((a, nxt), ref, len(W))
    toks = agree(run_all(stages, lambda st: st.tokens()))
    assert toks == x + W[:a] + [nxt]
    infos = run_all(stages, lambda st: st.info())
    assert all(i["kv_len"] == len(x) + a for i in infos)


def test_tp_ar_stream_and_rollback(toy_group):
    """Draft (rows = 1), reject, roll back and resync: every rank identical,
    the stream the oracle's greedy choice on the GPU's own tokens."""
    s, w64, stages, prompt, T = toy_group
    run_all(stages, lambda st: st.prefill(prompt))
    toks = agree(run_all(stages, lambda st: st.draft(16)))
    check_tokens_teacher_forced(w64, s, prompt, toks)
    keep = len(prompt) + 6
    run_all(stages, lambda st: st.kv_rollback(keep))
    ctx = agree(run_all(stages, lambda st: st.tokens()))
    assert ctx == list(prompt) + toks[:6]
    more = agree(run_all(stages, lambda st: st.draft(10)))
    assert more == toks[6:16]          # same KV-consistent continuation after rollback
    # lazy resync to a foreign prefix, then verify a window over it
    foreign = list(prompt) + toks[:3] + [(toks[3] + 7) % s.vocab]
    run_all(stages, lambda st: st.resync(foreign))
    r = agree(run_all(stages, lambda st: st.verify([5, 6, 7])))
    ref = L.verify(w64, s, foreign, [5, 6, 7])
    check_verify(r, ref, 3)


def test_tp_matches_single_rank_decisions(toy_group):
    """TP=T and TP=1 on the same weights reach the same greedy stream (the
    fp32 partial sums differ only in summation order)."""
    from paper_2505_01572_b200 import Stage
    s, w64, stages, prompt, T = toy_group
    w = synth.make_weights(s, seed=31, device="cuda")
    one = Stage(s, w, max_seq=256)
    one.prefill(prompt)
    ref = one.draft(24)
    one.close()
    run_all(stages, lambda st: st.prefill(prompt))
    got = agree(run_all(stages, lambda st: st.draft(24)))
    if got != ref:   # only a near-tie may split them
        j = next(i for i in range(24) if got[i] != ref[i])
        z = L.forward_full(w64, s, list(prompt) + got[:j + 1])[-1]
        top = np.sort(z)[-2:]
        assert top[1] - top[0] < 1e-2, (j, got[j], ref[j])


@pytest.mark.parametrize("name,layers,T", [("llama3.1-8b", 2, 2), ("llama3.1-8b", 1, 4),
                                           ("llama3.1-70b", 1, 2), ("llama3.1-70b", 2, 4)])
def test_tp_paper_widths(name, layers, T):
    """8B (TP2 / TP4) and 70B (TP2, the paper's "split across 2 GPUs", P:181;
    TP4, the 8-GPU layout of config 4) widths with the FULL 128256 vocabulary
    at reduced depth: logits and decisions vs the fp64 oracle."""
    s = synth.reduced_depth(synth.preset(name), layers)
    w = synth.make_weights(s, seed=41, device="cuda")
    w64 = synth.weights_to_numpy(w)
    prompt = list(synth.make_prompt(s.vocab, 40, seed=42))
    stages = make_group(s, w, T, max_seq=128, max_window=16)
    try:
        stream, _ = L.ar_decode(w64, s, prompt, 5)
        W = stream[:3] + [(stream[3] + 11) % s.vocab]
        run_all(stages, lambda st: st.prefill(prompt))
        res = run_all(stages, lambda st: st.verify(W, want_logits=True))
        a, nxt = agree([(r[0], r[1]) for r in res])
        ref = L.verify(w64, s, prompt, W)
        check_logits(np.concatenate([r[2] for r in res], axis=1), ref["logits"])
        check_verify((a, nxt), ref, len(W))
    finally:
        for st in stages:
            st.close()
