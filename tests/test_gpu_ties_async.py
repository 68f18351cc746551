"""GPU: the greedy tie rule (SURVEY §8(c) c.3 "all-equal logits (tie -> lowest
index)", reading R12) and the asynchronous verification pass (§8(b)
ps_verify_async / ps_verify_wait).

Exact fp32 ties are built into the lm_head: rows that are the same ONE-HOT
vector c * e_j give logits c * xhat_j computed by a single product, so they are
bit-identical whatever the split of the K reduction -- within one 128-row
tile, across tiles, and across the ranks of a vocabulary-parallel lm_head.
The GPU must then pick the lower vocabulary id, like np.argmax."""
import numpy as np
import pytest
import torch

import synth
from oracle import llama as L
from tests._parity import check_logits, check_verify

pytestmark = pytest.mark.gpu


def _final_hidden(w64, s, tokens):
    """Oracle: the final-norm output of the last row (the lm_head's operand)."""
    sess = L.Session(w64, s)
    x = sess.hidden(tokens)
    return L.rms_norm(x, w64["final_norm"], s.rms_eps)[-1]


@pytest.fixture(scope="module")
def toy():
    s = synth.preset("toy-verifier")
    w = synth.make_weights(s, seed=41, device="cuda")
    prompt = [int(x) for x in synth.make_prompt(s.vocab, 40, seed=42)]
    return s, w, prompt


@pytest.mark.parametrize("lo,hi", [(5, 100), (5, 200), (130, 250), (0, 255)])
def test_exact_tie_picks_lowest_index(toy, lo, hi):
    """Rows lo < hi of the lm_head set to the same one-hot vector: within a tile
    (5, 100), across tiles (5, 200), (130, 250), and at the vocabulary ends."""
    from paper_2505_01572_b200 import Stage
    s, w0, prompt = toy
    w = {**w0, "lm_head": w0["lm_head"].clone()}
    w64 = synth.weights_to_numpy(w)
    h = _final_hidden(w64, s, prompt)
    j = int(np.argmax(h))                       # the largest positive normalised feature
    onehot = torch.zeros(s.d_model, dtype=torch.bfloat16, device="cuda")
    onehot[j] = 16.0
    for t in (hi, lo):
        w["lm_head"][t] = onehot
    w64 = synth.weights_to_numpy(w)
    st = Stage(s, w, max_seq=128, max_window=4)
    st.prefill(prompt)
    a, nxt, logits = st.verify([], want_logits=True)
    assert logits[0, lo] == logits[0, hi] and logits[0].max() == logits[0, lo]   # an exact tie, and the max
    ref = L.verify(w64, s, prompt, [])
    assert ref["next"] == lo and nxt == lo
    st.close()


def test_all_equal_logits_pick_index_zero(toy):
    """An all-zero lm_head: every logit is +-0.0 (signed zeros compare equal,
    np.argmax takes index 0); with drafts of token 0 every row accepts."""
    from paper_2505_01572_b200 import Stage
    s, w0, prompt = toy
    w = {**w0, "lm_head": torch.zeros_like(w0["lm_head"])}
    w64 = synth.weights_to_numpy(w)
    st = Stage(s, w, max_seq=128, max_window=4)
    st.prefill(prompt)
    a, nxt = st.verify([0, 0, 0])
    ref = L.verify(w64, s, prompt, [0, 0, 0])
    assert (a, nxt) == (ref["a"], ref["next"]) == (3, 0)
    st.prefill(prompt)
    a, nxt = st.verify([7, 0])
    assert (a, nxt) == (0, 0)
    st.close()


def test_tensor_parallel_tie_across_ranks():
    """Vocabulary-parallel lm_head (TP2): the tied rows live on different ranks;
    the max over the ranks' greedy keys must still pick the lower id."""
    from tests.test_gpu_tp import agree, make_group, run_all
    s = synth.preset("toy-tp")
    w = synth.make_weights(s, seed=43, device="cuda")
    prompt = [int(x) for x in synth.make_prompt(s.vocab, 40, seed=44)]
    w64 = synth.weights_to_numpy(w)
    h = _final_hidden(w64, s, prompt)
    j = int(np.argmax(h))
    lo, hi = 3, s.vocab // 2 + 9                # rank 0's slice and rank 1's slice
    w["lm_head"] = w["lm_head"].clone()
    for t in (lo, hi):
        w["lm_head"][t].zero_()
        w["lm_head"][t, j] = 16.0
    stages = make_group(s, w, 2, max_seq=128, max_window=4)
    run_all(stages, lambda st: st.prefill(prompt))
    res = agree(run_all(stages, lambda st: st.verify([])))
    assert res == (0, lo)
    for st in stages:
        st.close()


# ----------------------------------------------------------------------------- async verify
def test_verify_async_host_and_device_windows(toy):
    """ps_verify_async + ps_verify_wait equal ps_verify, for a host window and a
    device-resident window; the ticket's pinned record carries a, next, kv_len
    and the predictions."""
    from paper_2505_01572_b200 import Stage
    s, w, prompt = toy
    w64 = synth.weights_to_numpy(w)
    st = Stage(s, w, max_seq=160, max_window=8)
    st.prefill(prompt)
    stream = st.draft(8)
    window = stream[:3] + [(stream[3] + 1) % s.vocab] + stream[4:6]
    ref = L.verify(w64, s, prompt, window)
    results = []
    for dev in (False, True):
        st.prefill(prompt)
        win = torch.tensor(window, dtype=torch.int32, device="cuda") if dev else window
        tk = st.verify_async(win)
        a, nxt = st.verify_wait()
        r = tk.h_result.contents
        assert (r.a, r.next, r.kv_len, r.rows) == (a, nxt, len(prompt) + a, len(window) + 1)
        assert list(r.pred[:a]) == window[:a]
        assert st.tokens() == prompt + window[:a] + [nxt]
        results.append((a, nxt))
    st.prefill(prompt)
    assert st.verify(window) == results[0] == results[1]
    check_verify(results[0], ref, len(window), where="async")
    st.close()


def test_verify_async_guards(toy):
    """While a pass is in flight every call that uses the stage is refused; a
    device window with an out-of-range token is reported without a commit."""
    from paper_2505_01572_b200 import PipeSpecError, Stage
    s, w, prompt = toy
    st = Stage(s, w, max_seq=160, max_window=8)
    st.prefill(prompt)
    st.verify_async([1, 2])
    for call in (lambda: st.verify([]), lambda: st.draft(1), lambda: st.prefill(prompt),
                 lambda: st.kv_rollback(5), lambda: st.resync(prompt), lambda: st.verify_async([])):
        with pytest.raises(PipeSpecError):
            call()
    assert st.tokens() == prompt            # read-only calls are allowed; O_i unchanged
    st.verify_wait()
    assert st.verify_query()                # nothing in flight
    with pytest.raises(PipeSpecError):
        st.verify_wait()
    st.prefill(prompt)
    bad = torch.tensor([3, s.vocab + 7], dtype=torch.int32, device="cuda")
    st.verify_async(bad)
    with pytest.raises(PipeSpecError):
        st.verify_wait()
    assert st.tokens() == prompt and st.info()["kv_len"] == len(prompt) - 1
    a, nxt = st.verify([])                  # the stage is usable afterwards
    assert st.tokens() == prompt + [nxt]
    st.close()
