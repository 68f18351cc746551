"""CPU tests of the async PipeSpec runtime's protocol (Alg.1) through
the library's board code -- the same code the GPU stages run -- with the
closed-form host test double of include/pipespec_test.h: stages as threads of
one process (ps_pipeline_run's layout) and as one process per stage over the
shared-memory board (ps_pipeline_run_rank's layout).  The output must equal
the target's autoregressive stream, whatever the acceptance rate, timing or
interleaving (the method is lossless, Eq.1 P:128 / S:49)."""
import ctypes as C
import os
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def target_ar(prompt, n, V):
    """The test double's stage-K model written out: next(c) = (c[-1]*7919 + |c|*104729 + 13) mod V."""
    c = list(prompt)
    for _ in range(n):
        c.append((c[-1] * 7919 + len(c) * 104729 + 13) % V)
    return c[len(prompt):]


def _opts(k, n, gamma, look=0, lead=0):
    from paper_2505_01572_b200 import abi
    g = (C.c_int32 * k)(*([0] + [gamma] * (k - 1)))
    la = (C.c_int32 * k)(*([0] + [look] * (k - 1)))
    return abi.RunOpts(abi.PS_MODE_PIPESPEC, n, -1, g, la, lead), (g, la)


@pytest.mark.parametrize("k,alpha,gamma,look,sleep", [(2, 0.8, 4, 0, 0), (2, 0.5, 8, 0, 50), (2, 1.0, 4, 0, 0),
                                                      (2, 0.0, 4, 0, 0), (3, 0.9, 4, 0, 20), (3, 0.6, 6, 2, 0),
                                                      (4, 0.8, 3, 0, 10)])
def test_threads_lossless(k, alpha, gamma, look, sleep):
    from paper_2505_01572_b200 import abi
    V, n = 997, 120
    prompt = np.arange(5, 21, dtype=np.int32)
    opts, keep = _opts(k, n, gamma, look)
    out = np.zeros(n, dtype=np.int32)
    ln = C.c_int32()
    st = abi.RunStats()
    abi.check(abi.lib().ps_test_fake_pipeline(k, prompt.ctypes.data, len(prompt), C.byref(opts), V, alpha, 7,
                                              sleep, out.ctypes.data, C.byref(ln), C.byref(st)))
    assert out[:ln.value].tolist() == target_ar(prompt.tolist(), n, V)
    assert st.steps[k - 1] > 0 and st.steps[0] > 0
    if alpha == 1.0:
        assert sum(st.rollbacks[:k]) == 0


def _rank_worker(rank, k, board, n, alpha, gamma, sleep, q):
    sys.path.insert(0, ROOT)
    from paper_2505_01572_b200 import abi
    V = 997
    prompt = np.arange(5, 21, dtype=np.int32)
    opts, keep = _opts(k, n, gamma)
    out = np.zeros(n, dtype=np.int32)
    ln = C.c_int32()
    st = abi.RunStats()
    s = abi.lib().ps_test_fake_run_rank(rank, k, board.encode(), prompt.ctypes.data, len(prompt), C.byref(opts),
                                        V, alpha, 11, sleep, out.ctypes.data, C.byref(ln), C.byref(st))
    q.put((rank, s, out[:ln.value].tolist(), [int(x) for x in st.steps[:k]], int(st.verify_steps[k - 1])))


@pytest.mark.parametrize("k,alpha,gamma,sleep", [(2, 0.8, 4, 30), (3, 0.7, 4, 10)])
def test_processes_lossless(k, alpha, gamma, sleep):
    from paper_2505_01572_b200 import abi
    n = 80
    board = f"/pipespec-test-{os.getpid()}-{k}"
    abi.check(abi.lib().ps_board_create(board.encode(), k, 16 + n + 400))
    try:
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        procs = [ctx.Process(target=_rank_worker, args=(r, k, board, n, alpha, gamma, sleep, q)) for r in range(k)]
        for p in procs:
            p.start()
        res = sorted(q.get(timeout=180) for _ in range(k))
        for p in procs:
            p.join(timeout=60)
    finally:
        abi.lib().ps_board_unlink(board.encode())
    want = target_ar(list(range(5, 21)), n, 997)
    for rank, status, out, steps, vsteps in res:
        assert status == 0, (rank, status)
        assert out == want, rank
        assert all(s > 0 for s in steps) and vsteps > 0


def test_board_rank_mismatch_fails_cleanly():
    from paper_2505_01572_b200 import abi
    board = f"/pipespec-test-{os.getpid()}-bad"
    abi.check(abi.lib().ps_board_create(board.encode(), 2, 400))
    try:
        opts, keep = _opts(3, 10, 4)
        out = np.zeros(10, dtype=np.int32)
        ln = C.c_int32()
        prompt = np.arange(3, dtype=np.int32)
        s = abi.lib().ps_test_fake_run_rank(0, 3, board.encode(), prompt.ctypes.data, 3, C.byref(opts), 97, 0.5,
                                            1, 0, out.ctypes.data, C.byref(ln), None)
        assert s == abi.PS_E_INVALID
        assert abi.lib().ps_test_fake_run_rank(0, 2, b"/pipespec-missing-board", prompt.ctypes.data, 3,
                                               C.byref(opts), 97, 0.5, 1, 0, out.ctypes.data, C.byref(ln),
                                               None) == abi.PS_E_INVALID
    finally:
        abi.lib().ps_board_unlink(board.encode())
