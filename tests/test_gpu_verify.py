"""GPU parity of the verify hot path (ps_verify / ps_draft / ps_prefill /
ps_kv_rollback) against the fp64 oracle, on the toy shapes (BASELINE configs[0])
and on paper-shaped widths (LLaMA-3.2-1B full depth, LLaMA-3.1-8B and
LLaMA-2-7B widths at reduced depth, LLaMA-68M full)."""
from dataclasses import replace

import numpy as np
import pytest
import torch

import synth
from oracle import buffer as B
from oracle import llama as L
from oracle import synthetic as SY
from tests._parity import check_logits, check_tokens_teacher_forced, check_verify

pytestmark = pytest.mark.gpu


def make(shape_name, seed, layers=None, max_seq=512, **kw):
    from paper_2505_01572_b200 import Stage
    s = synth.preset(shape_name)
    if layers is not None:
        s = synth.reduced_depth(s, layers)
    w = synth.make_weights(s, seed=seed, device="cuda")
    return s, w, Stage(s, w, max_seq=max_seq, **kw)


@pytest.fixture(scope="module")
def toy():
    s, w, st = make("toy-verifier", 21, max_seq=256)
    w64 = synth.weights_to_numpy(w)
    prompt = synth.make_prompt(s.vocab, 64, seed=22)
    yield s, w, w64, st, prompt
    st.close()


def test_ar_stream_matches_oracle(toy):
    s, w, w64, st, prompt = toy
    st.prefill(prompt)
    toks = st.draft(32)
    assert st.tokens() == list(prompt) + toks
    check_tokens_teacher_forced(w64, s, prompt, toks)


@pytest.mark.parametrize("case", ["w0", "full", "reject0", "reject_mid", "w15", "w16", "w31"])
def test_verify_windows(toy, case):
    s, w, w64, st, prompt = toy
    x = list(prompt)
    stream, _ = L.ar_decode(w64, s, x, 32)
    W = {"w0": [], "full": stream[:8], "reject0": [(stream[0] + 5) % s.vocab] + stream[1:4],
         "reject_mid": stream[:5] + [(stream[5] + 1) % s.vocab] + stream[6:9],
         "w15": stream[:15], "w16": stream[:16], "w31": stream[:31]}[case]
    st.prefill(x)
    a, nxt, logits = st.verify(W, want_logits=True)
    ref = L.verify(w64, s, x, W)
    check_logits(logits, ref["logits"])
    check_verify((a, nxt), ref, len(W))
    assert st.tokens() == x + W[:a] + [nxt]
    info = st.info()
    buf = B.TokenBuffer(x)
    buf.append(W[:a] + [nxt])
    assert info["kv_len"] == buf.kv_len == len(x) + a
    assert info["pages_in_use"] == buf.pages(64)


def test_row_bucket_invariance_verify_equals_ar(toy):
    """GPU self-consistency: a verify over w accepted drafts
    yields bit-identical logits rows to w+1 single-token steps."""
    s, w, w64, st, prompt = toy
    st.prefill(prompt)
    rows = []
    for _ in range(20):
        a, nxt, lg = st.verify([], want_logits=True)
        rows.append(lg[0])
    gpu_stream = st.tokens()[len(prompt):]
    st.prefill(prompt)
    a, nxt, lg = st.verify(gpu_stream[:19], want_logits=True)
    assert a == 19 and nxt == gpu_stream[19]
    assert np.array_equal(lg, np.stack(rows)), np.abs(lg - np.stack(rows)).max()


def test_rollback_semantics_and_recompute(toy):
    s, w, w64, st, prompt = toy
    st.prefill(prompt)
    toks = st.draft(12)
    n = len(prompt) + 12
    from paper_2505_01572_b200 import PipeSpecError
    with pytest.raises(PipeSpecError):
        st.kv_rollback(n + 1)               # keep > len: contract violation
    with pytest.raises(PipeSpecError):
        st.kv_rollback(0)
    st.kv_rollback(n)                       # no-op
    assert st.info()["kv_len"] == n - 1
    st.kv_rollback(len(prompt) + 3)
    info = st.info()
    assert st.tokens() == list(prompt) + toks[:3]
    assert info["kv_len"] == len(prompt) + 2
    assert info["pages_in_use"] == B.pages_for(len(prompt) + 2, 64)
    # after truncation the KV is consistent: re-drafting reproduces the stream
    assert st.draft(9) == toks[3:]


def test_prefill_resync_keeps_common_prefix(toy):
    s, w, w64, st, prompt = toy
    st.prefill(prompt)
    st.draft(10)
    other = list(prompt[:40]) + list(synth.make_prompt(s.vocab, 30, seed=99))
    st.prefill(other)                        # truncate to the common prefix, extend
    a, nxt, lg = st.verify([], want_logits=True)
    ref = L.verify(w64, s, other, [])
    check_logits(lg, ref["logits"])
    check_verify((a, nxt), ref, 0)


def test_synthetic_override_matches_counter_generator(toy):
    """The drafter's emitted tokens follow the chained construction exactly
    (bit-exact integers) while on the target stream."""
    s, w, w64, st, prompt = toy
    S = [int(x) for x in synth.make_prompt(s.vocab, 40, seed=5)]
    for alpha in (1.0, 0.0, 0.6):
        st.prefill(prompt)
        st.set_synthetic(S, len(prompt), level=0, top=1, alphas=[alpha], seed=1234)
        thrs = [SY.alpha_threshold(alpha)]
        got = st.draft(1)[0]
        want = SY.chained_token(S[0], 0, 1, 0, 1234, thrs, s.vocab)
        assert got == want
        if alpha == 1.0:
            assert st.draft(20) == S[1:21]
        if alpha == 0.0:
            assert got != S[0]
    st.clear_synthetic()


def test_chained_draft_equals_single_steps(toy):
    """ps_draft of n tokens launches the n forwards back to back, each taking
    its row token (and the synthetic on-path bit) from the previous forward on
    the device; the result equals n single-step drafts bit for bit -- greedy,
    with the synthetic override (on and off the target stream), and after a
    lazy resync (the chain's first forward carries the catch-up rows)."""
    s, w, w64, st, prompt = toy
    for mode in ("greedy", "synthetic"):
        st.prefill(prompt)
        if mode == "synthetic":
            base = st.draft(1)
            st.kv_rollback(len(prompt))
            # the target stream: the greedy token first (on path), then random
            S = base + [int(x) for x in synth.make_prompt(s.vocab, 60, seed=6)]
            st.set_synthetic(S, len(prompt), level=0, top=1, alphas=[0.6], seed=99)
        chained = st.draft(12)
        st.kv_rollback(len(prompt))
        single = [st.draft(1)[0] for _ in range(12)]
        assert chained == single, mode
        other = list(prompt) + single[:3] + [(single[3] + 1) % s.vocab] + single[4:7]
        st.resync(other)
        c2 = st.draft(5)
        assert st.tokens() == other + c2
        st.resync(other)
        s2 = [st.draft(1)[0] for _ in range(5)]
        assert c2 == s2, mode
    st.clear_synthetic()


@pytest.mark.parametrize("name,layers,plen,w", [
    ("llama-68m", None, 96, 8),
    ("llama3.2-1b", None, 96, 16),
    ("llama3.1-8b", 2, 160, 16),
    ("llama2-7b", 2, 96, 7),
    ("llama2-13b", 2, 96, 8),        # config 3's target: MHA (40 / 40 heads), d = 5120
])
def test_paper_shapes_parity(name, layers, plen, w):
    """Full-width shapes: logits within 2e-2*max|logit| of the fp64 oracle,
    (a, next) exact unless the deciding rows are near-ties."""
    s, wt, st = make(name, 7, layers=layers, max_seq=plen + 40)
    w64 = synth.weights_to_numpy(wt)
    prompt = list(synth.make_prompt(s.vocab, plen, seed=8))
    st.prefill(prompt)
    stream = st.draft(w + 2)
    st.prefill(prompt)
    window = stream[:w // 2] + [(stream[w // 2] + 3) % s.vocab] + stream[w // 2 + 1:w]
    a, nxt, logits = st.verify(window, want_logits=True)
    ref = L.verify(w64, s, prompt, window)
    check_logits(logits, ref["logits"])
    check_verify((a, nxt), ref, w)
    st.close()
    del wt
    torch.cuda.empty_cache()


def test_lazy_resync_catch_up_equals_eager(toy):
    """ps_resync defers the KV of a resynced suffix into the next forward's
    leading rows; the result equals an eager ps_prefill bit-exactly."""
    s, w, w64, st, prompt = toy
    st.prefill(prompt)
    base = st.draft(6)
    other = list(prompt) + base[:2] + [(base[2] + 9) % s.vocab] + list(synth.make_prompt(s.vocab, 5, 3))
    st.resync(other)
    assert st.tokens() == other
    a1, n1, l1 = st.verify(base[:3], want_logits=True)
    st.prefill(prompt)
    st.prefill(other)
    a2, n2, l2 = st.verify(base[:3], want_logits=True)
    assert (a1, n1) == (a2, n2) and np.array_equal(l1, l2)
    # a long pending suffix (> 31 rows) is caught up in chunks
    longer = list(prompt[:10]) + list(synth.make_prompt(s.vocab, 70, 4))
    st.resync(longer)
    a3, n3, l3 = st.verify([], want_logits=True)
    ref = L.verify(w64, s, longer, [])
    check_logits(l3, ref["logits"])
    check_verify((a3, n3), ref, 0)


@pytest.mark.slow
def test_bench_config_self_consistency():
    """BASELINE configs[1] at full size (LLaMA-3.2-1B -> LLaMA-3.1-8B shapes,
    512-token prompt, bench.py's launch configuration): properties that hold at
    any size -- sync-SD and async PipeSpec output == M_K autoregressive output,
    and a verify over w accepted drafts reproduces the AR logits bit-exactly."""
    from paper_2505_01572_b200 import Stage, pipeline_run
    from paper_2505_01572_b200.abi import PS_MODE_AR, PS_MODE_PIPESPEC, PS_MODE_SYNC_SD
    ds, ts = synth.preset("llama3.2-1b"), synth.preset("llama3.1-8b")
    wd = synth.make_weights(ds, seed=0, device="cuda")
    wt = synth.make_weights(ts, seed=1, device="cuda")
    d = Stage(ds, wd, max_seq=700, max_window=8)
    t = Stage(ts, wt, max_seq=700, max_window=8)
    prompt = [int(x) for x in synth.make_prompt(ts.vocab, 512, seed=17)]
    ar, _ = pipeline_run([d, t], prompt, 48, mode=PS_MODE_AR)
    d.set_synthetic(ar + [0] * 16, 512, level=0, top=1, alphas=[0.8], seed=1234)
    sd, st = pipeline_run([d, t], prompt, 48, mode=PS_MODE_SYNC_SD, gammas=[0, 8])
    assert sd == ar and st.verify_steps[1] >= 1
    ps, _ = pipeline_run([d, t], prompt, 48, mode=PS_MODE_PIPESPEC, gammas=[0, 8])
    assert ps == ar
    # row-bucket invariance at full size: AR rows vs one verify of 8 accepted drafts
    t.prefill(prompt)
    rows = []
    for _ in range(9):
        a, nxt, lg = t.verify([], want_logits=True)
        rows.append(lg[0])
    t.prefill(prompt)
    a, nxt, lg = t.verify(ar[:8], want_logits=True)
    assert a == 8 and nxt == ar[8]
    assert np.array_equal(lg, np.stack(rows))
    d.close()
    t.close()


def test_long_context_many_attention_items():
    """LLaMA-68M shape (12 KV heads) at ~2K context: more attention work items
    than CTAs (strided item loop), 33 chunks per row combined; parity vs oracle."""
    s, wt, st = make("llama-68m", 3, max_seq=2200)
    w64 = synth.weights_to_numpy(wt)
    prompt = list(synth.make_prompt(s.vocab, 2040, seed=4))
    st.prefill(prompt)
    stream = st.draft(6)
    st.prefill(prompt)
    window = stream[:3] + [(stream[3] + 7) % s.vocab] + stream[4:5]
    a, nxt, logits = st.verify(window, want_logits=True)
    ref = L.verify(w64, s, prompt, window)
    check_logits(logits, ref["logits"])
    check_verify((a, nxt), ref, len(window))
    st.close()


def test_70b_width_one_layer():
    """LLaMA-3.1-70B widths (d=8192, 64/8 heads, ffn 28672; vocab cut to 32000
    to bound the oracle's RAM): GQA g=8 -> 4 attention row blocks at R=32."""
    from dataclasses import replace
    s = replace(synth.preset("llama3.1-70b"), n_layers=1, vocab=32000)
    from paper_2505_01572_b200 import Stage
    wt = synth.make_weights(s, seed=5, device="cuda")
    st = Stage(s, wt, max_seq=200)
    w64 = synth.weights_to_numpy(wt)
    prompt = list(synth.make_prompt(s.vocab, 80, seed=6))
    st.prefill(prompt)
    stream = st.draft(31)
    st.prefill(prompt)
    window = stream[:31]
    a, nxt, logits = st.verify(window, want_logits=True)
    ref = L.verify(w64, s, prompt, window)
    check_logits(logits, ref["logits"])
    check_verify((a, nxt), ref, len(window))
    st.close()


def test_long_context_head_dim_128():
    """head_dim 128 (the LLaMA-3.1-8B attention geometry: llama3 RoPE, GQA
    g=4) at a 4.2K context: 66 chunks per row (the combine's > 32-chunk path),
    264 attention items > 148 CTAs; parity vs the oracle, and a verify over
    accepted drafts reproduces the AR steps' logits bit-exactly (row-bucket
    invariance with rows crossing a chunk boundary)."""
    from paper_2505_01572_b200 import Stage
    s = replace(synth.preset("llama3.1-8b"), name="hd128-long", n_layers=2, d_model=2048, n_heads=16,
                n_kv_heads=4, d_ffn=2048, vocab=4096)
    wt = synth.make_weights(s, seed=9, device="cuda")
    w64 = synth.weights_to_numpy(wt)
    n = 4222                                   # rows of the window straddle position 4224 = 66 * 64
    st = Stage(s, wt, max_seq=n + 64)
    prompt = list(synth.make_prompt(s.vocab, n, seed=10))
    st.prefill(prompt)
    rows = []
    for _ in range(5):
        a, nxt, lg = st.verify([], want_logits=True)
        rows.append(lg[0])
    stream = st.tokens()[n:]
    st.prefill(prompt)
    window = stream[:4]
    a, nxt, logits = st.verify(window, want_logits=True)
    assert a == 4 and nxt == stream[4]
    assert np.array_equal(logits, np.stack(rows))
    st.prefill(prompt)
    window = stream[:2] + [(stream[2] + 5) % s.vocab]
    a, nxt, logits = st.verify(window, want_logits=True)
    ref = L.verify(w64, s, prompt, window)
    check_logits(logits, ref["logits"])
    check_verify((a, nxt), ref, len(window))
    st.close()


@pytest.mark.parametrize("name,layers,n", [("toy-verifier", None, 150), ("llama3.1-8b", 2, 200)])
def test_prefill_64_row_chunks(name, layers, n):
    """NEXT-3 prefill: the prompt runs through the 64-row bucket (64-token
    chunks + a ragged tail, split-bf16 N = 128 MMAs, 16-row epilogue chunks).
    Its KV is bit-identical to a one-token-at-a-time prefill (row-bucket
    invariance), and the next verify matches the oracle."""
    from paper_2505_01572_b200 import abi
    s, w, st = make(name, 31, layers=layers, max_seq=n + 40)
    st.set_prefill_path(abi.PS_PREFILL_ROWS)   # the decode megakernel's bucket (not the prefill kernels)
    w64 = synth.weights_to_numpy(w)
    prompt = list(synth.make_prompt(s.vocab, n, seed=32))
    st.prefill(prompt)                       # 64 + 64 + 21 (+ ragged) rows
    a1, n1, l1 = st.verify([], want_logits=True)
    st.prefill(prompt[:1])
    for i in range(2, n + 1):                # one row per forward (the 16-row bucket)
        st.prefill(prompt[:i])
    a2, n2, l2 = st.verify([], want_logits=True)
    assert (a1, n1) == (a2, n2) and np.array_equal(l1, l2)
    ref = L.verify(w64, s, prompt, [])
    check_logits(l1, ref["logits"])
    check_verify((a1, n1), ref, 0)
    st.close()


@pytest.mark.parametrize("name,layers,n", [("toy-verifier", None, 150), ("llama-68m", None, 1030),
                                            ("llama3.2-1b", 2, 700), ("llama3.1-8b", 2, 512)])
def test_prefill_gemm_path(name, layers, n):
    """NEXT-3: runs of >= 64 prompt positions go through the prefill
    kernels -- tcgen05 GEMMs with the tokens as the M = 128 side (split-bf16
    operand, fused RoPE/KV-append, residual and SwiGLU epilogues) and the
    causal prefill attention -- in chunks of <= 512 tokens (1030: 512 + 512 +
    5 through the megakernel; 150, 700: ragged M tiles).  The next verify
    matches the oracle, and its logits agree with those after a prefill
    through the megakernel's 64-row bucket (PS_PREFILL_ROWS) within the
    parity tolerance (the two paths sum in different orders)."""
    from paper_2505_01572_b200 import Stage, abi
    s, w, st = make(name, 41, layers=layers, max_seq=n + 40)
    w64 = synth.weights_to_numpy(w)
    prompt = list(synth.make_prompt(s.vocab, n, seed=42))
    ar, _ = L.ar_decode(w64, s, prompt, 2)
    window = ar[:2] + [(ar[1] + 7) % s.vocab]
    st.prefill(prompt)
    a1, n1, l1 = st.verify(window, want_logits=True)
    ref = L.verify(w64, s, prompt, window)
    check_logits(l1, ref["logits"])
    check_verify((a1, n1), ref, len(window))
    assert st.info()["kv_len"] == n + a1
    st.close()
    st2 = Stage(s, w, max_seq=n + 40)
    st2.set_prefill_path(abi.PS_PREFILL_ROWS)
    st2.prefill(prompt)
    a2, n2, l2 = st2.verify(window, want_logits=True)
    check_logits(l1, np.asarray(l2, dtype=np.float64))
    st2.close()


@pytest.mark.parametrize("page_size", [128, 256])
def test_prefill_gemm_path_page_sizes(page_size):
    """The prefill kernels' KV append (per-token page lookup) and attention
    tiles (32 keys inside one page) with 128- and 256-token pages; a prompt of
    700 tokens = 512 + 187 positions spans several pages and two chunks."""
    s, w, st = make("toy-verifier", 43, max_seq=760, page_size=page_size)
    w64 = synth.weights_to_numpy(w)
    prompt = list(synth.make_prompt(s.vocab, 700, seed=44))
    st.prefill(prompt)
    window = [int(t) for t in synth.make_prompt(s.vocab, 3, seed=45)]
    a, nxt, lg = st.verify(window, want_logits=True)
    ref = L.verify(w64, s, prompt, window)
    check_logits(lg, ref["logits"])
    check_verify((a, nxt), ref, len(window))
    st.close()


def test_prefill_gemm_path_gqa8_wide():
    """The prefill kernels at the LLaMA-3.1-70B attention geometry (d = 8192,
    64 query heads over 8 KV heads: GQA group 8, so a 64-row attention CTA
    covers 8 positions) and its 28672-wide FFN (gate/up tiles of 112 + 112
    rows), one layer, vocabulary cut to 4096; 300-token prompt."""
    from paper_2505_01572_b200 import Stage
    s = replace(synth.preset("llama3.1-70b"), name="70b-1l", n_layers=1, vocab=4096)
    w = synth.make_weights(s, seed=47, device="cuda")
    w64 = synth.weights_to_numpy(w)
    prompt = list(synth.make_prompt(s.vocab, 300, seed=48))
    st = Stage(s, w, max_seq=340)
    st.prefill(prompt)
    window = [int(t) for t in synth.make_prompt(s.vocab, 2, seed=49)]
    a, nxt, lg = st.verify(window, want_logits=True)
    ref = L.verify(w64, s, prompt, window)
    check_logits(lg, ref["logits"])
    check_verify((a, nxt), ref, len(window))
    st.close()
    del w
    torch.cuda.empty_cache()


def test_prefill_path_rejects_unknown():
    from paper_2505_01572_b200 import abi
    s, w, st = make("toy-verifier", 5, max_seq=128)
    with pytest.raises(abi.PipeSpecError):
        st.set_prefill_path(7)
    st.close()


def _oracle_verify_incremental(w64, shape, x, d, chunk=512):
    """oracle.llama.verify computed through the oracle's incremental Session
    (prompt fed in `chunk`-token pieces, pinned equal to the full forward in
    the CPU suite), so a 16K context never builds a 16K x 16K score matrix."""
    sess = L.Session(w64, shape)
    for i in range(0, len(x) - 1, chunk):
        sess.hidden(x[i:min(i + chunk, len(x) - 1)])
    z = sess.forward([x[-1]] + list(d))
    pred = [L.greedy(r) for r in z]
    a = L.first_mismatch(pred, d)
    return dict(a=a, next=pred[a], pred=pred, logits=z, gaps=[L.top2_gap(r) for r in z])


def test_long_context_16k_multichunk_items():
    """a ~16.6K context with the long-context attention items
    (sc > 1 64-key chunks per work item, streamed through the 16-key TMA ring
    with an online softmax; sc is the stage's choice for max_seq 32K).  The
    window's rows straddle an item boundary: a verify over accepted drafts
    equals the AR steps bit-exactly, and a verify with a rejection matches the
    oracle."""
    from paper_2505_01572_b200 import Stage
    s = replace(synth.preset("llama3.1-8b"), name="hd128-16k", n_layers=2, d_model=1024, n_heads=8,
                n_kv_heads=4, d_ffn=1024, vocab=4096)
    wt = synth.make_weights(s, seed=41, device="cuda")
    w64 = synth.weights_to_numpy(wt)
    st = Stage(s, wt, max_seq=32768)
    item = 64 * st.info()["attn_sc"]         # keys per work item
    assert item >= 128
    n = -(-16600 // item) * item - 2          # rows n-1 .. n+3 straddle the item boundary at n + 2
    prompt = list(synth.make_prompt(s.vocab, n, seed=42))
    st.prefill(prompt)
    rows = []
    for _ in range(5):
        a, nxt, lg = st.verify([], want_logits=True)
        rows.append(lg[0])
    stream = st.tokens()[n:]
    st.prefill(prompt)
    a, nxt, logits = st.verify(stream[:4], want_logits=True)
    assert a == 4 and nxt == stream[4]
    assert np.array_equal(logits, np.stack(rows))
    st.prefill(prompt)
    window = stream[:2] + [(stream[2] + 5) % s.vocab]
    a, nxt, logits = st.verify(window, want_logits=True)
    ref = _oracle_verify_incremental(w64, s, prompt, window)
    check_logits(logits, ref["logits"])
    check_verify((a, nxt), ref, len(window))
    st.close()


@pytest.mark.parametrize("hd", [64, 128])
def test_attention_ragged_last_item(hd):
    """Key-split attention (warp w takes the stages w mod 4 of an item and
    writes its own partial) at a context whose last item is ragged (3 of its 4
    stages hold keys; the padded stage is fully masked): a verify over accepted
    drafts equals the AR steps bit-exactly, and a verify with a rejection
    matches the oracle."""
    from paper_2505_01572_b200 import Stage
    s = replace(synth.preset("llama3.1-8b"), name=f"ragged-hd{hd}", n_layers=2, d_model=8 * hd, n_heads=8,
                n_kv_heads=2, head_dim=hd, d_ffn=1024, vocab=4096)
    wt = synth.make_weights(s, seed=51, device="cuda")
    w64 = synth.weights_to_numpy(wt)
    n = 713                                   # 11 full 64-key chunks + a ragged one
    st = Stage(s, wt, max_seq=n + 64)
    prompt = list(synth.make_prompt(s.vocab, n, seed=52))
    st.prefill(prompt)
    rows = []
    for _ in range(9):
        a, nxt, lg = st.verify([], want_logits=True)
        rows.append(lg[0])
    stream = st.tokens()[n:]
    st.prefill(prompt)
    a, nxt, logits = st.verify(stream[:8], want_logits=True)
    assert a == 8 and nxt == stream[8]
    assert np.array_equal(logits, np.stack(rows))
    st.prefill(prompt)
    window = stream[:3] + [(stream[3] + 5) % s.vocab] + stream[4:6]
    a, nxt, logits = st.verify(window, want_logits=True)
    ref = L.verify(w64, s, prompt, window)
    check_logits(logits, ref["logits"])
    check_verify((a, nxt), ref, len(window))
    st.close()
