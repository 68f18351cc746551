"""GPU: the ONE-PROCESS-PER-RANK tensor-parallel path (ps_tp_handle /
ps_tp_connect over CUDA IPC handles, all-gathered with torch.distributed --
the wiring a multi-GPU stage uses).  Two processes, each one
rank of a TP2 stage on its own half of cuda:0's SMs (max_ctas), exchange their
partials through IPC-mapped peer memory inside the megakernel.  (Two processes
share one GPU by time-slicing, so every exchange waits for a context switch:
correct but slow -- this checks the wiring, not the speed.)  Results are
compared with the fp64 oracle of the FULL model; both ranks must agree."""
import os
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _rank(rank, port, q):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    import synth
    from paper_2505_01572_b200 import Stage, shard_weights
    from paper_2505_01572_b200.stage import tp_connect_group
    try:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=2)
        s = synth.preset("toy-tp")
        w = synth.make_weights(s, seed=61, device="cuda")
        n_sm = torch.cuda.get_device_properties(0).multi_processor_count
        st = Stage(s, shard_weights(s, w, rank, 2), max_seq=128, max_window=8, tp_rank=rank, tp_size=2,
                   max_ctas=n_sm // 2)
        tp_connect_group(st)
        prompt = [int(x) for x in synth.make_prompt(s.vocab, 40, seed=62)]
        st.prefill(prompt)
        stream = st.draft(4)
        st.prefill(prompt)
        window = stream[:2] + [(stream[2] + 1) % s.vocab]
        a, nxt, logits = st.verify(window, want_logits=True)
        q.put((rank, "ok", stream, (a, nxt), logits))
        dist.barrier()
        st.close()
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e), None, None, None))


def test_tp2_over_ipc_handles_matches_oracle():
    import socket

    import numpy as np
    import torch.multiprocessing as mp

    import synth
    from oracle import llama as L
    from tests._parity import check_logits, check_verify
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=300) for _ in range(2)), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert r[1] == "ok", r[:2]
    assert res[0][2] == res[1][2] and res[0][3] == res[1][3]      # the ranks agree bit for bit
    s = synth.preset("toy-tp")
    w = synth.make_weights(s, seed=61, device="cuda")
    w64 = synth.weights_to_numpy(w)
    prompt = [int(x) for x in synth.make_prompt(s.vocab, 40, seed=62)]
    stream = res[0][2]
    window = stream[:2] + [(stream[2] + 1) % s.vocab]
    ref = L.verify(w64, s, prompt, window)
    logits = np.concatenate([res[0][4], res[1][4]], axis=1)       # vocab slices in rank order
    check_logits(logits, ref["logits"])
    check_verify(res[0][3], ref, len(window), where="tp2-ipc")
