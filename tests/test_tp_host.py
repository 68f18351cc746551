"""CPU tests of the tensor-parallel host logic: the Megatron
shard layout of shard_weights and the handle exchange of tp_connect_group
(gloo, world_size 2).  The device half is tests/test_gpu_tp.py."""
import os
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _shard(*a, **k):
    from paper_2505_01572_b200.stage import shard_weights
    return shard_weights(*a, **k)


@pytest.mark.parametrize("T", [2, 4])
def test_shards_reassemble(T):
    s = synth.preset("toy-tp")
    w = synth.make_weights(s, seed=5)
    sh = [_shard(s, w, r, T) for r in range(T)]
    assert torch.equal(torch.cat([x["lm_head"] for x in sh]), w["lm_head"])
    for l, lw in enumerate(w["layers"]):
        for k, dim in (("wq", 0), ("wk", 0), ("wv", 0), ("wg", 0), ("wu", 0), ("wo", 1), ("wd", 1)):
            parts = [x["layers"][l][k] for x in sh]
            assert all(p.is_contiguous() for p in parts)
            assert torch.equal(torch.cat(parts, dim=dim), lw[k]), k
        for x in sh:
            assert x["layers"][l]["n_attn"] is lw["n_attn"] and x["embed"] is w["embed"]


@pytest.mark.parametrize("T", [2, 4])
def test_shard_layout_is_megatron(T):
    """Row-parallel O and down pair with the column split of Q and gate/up:
    sum_r (h_r W_r^T) equals the full product, and rank-local GQA (local query
    head j reads local KV head j // g) addresses the global KV head."""
    s = synth.preset("toy-tp")
    w = synth.make_weights(s, seed=6)
    rng = np.random.default_rng(0)
    R = 5
    att = rng.standard_normal((R, s.q_dim))
    hid = rng.standard_normal((R, s.d_ffn))
    f64 = lambda t: t.to(torch.float64).numpy()   # noqa: E731
    lw = w["layers"][0]
    full_o, full_d = att @ f64(lw["wo"]).T, hid @ f64(lw["wd"]).T
    qh, fr = s.n_heads // T, s.d_ffn // T
    po = sum(att[:, r * qh * s.head_dim:(r + 1) * qh * s.head_dim] @ f64(_shard(s, w, r, T)["layers"][0]["wo"]).T
             for r in range(T))
    pd = sum(hid[:, r * fr:(r + 1) * fr] @ f64(_shard(s, w, r, T)["layers"][0]["wd"]).T for r in range(T))
    assert np.allclose(po, full_o, rtol=1e-12, atol=1e-12) and np.allclose(pd, full_d, rtol=1e-12, atol=1e-12)
    g = s.n_heads // s.n_kv_heads
    kh = s.n_kv_heads // T
    for r in range(T):
        for j in range(qh):
            assert (r * qh + j) // g == r * kh + j // g


class _FakeStage:
    def __init__(self, rank, T):
        self.tp_size, self.rank, self.got = T, rank, None

    def tp_handle(self):
        return bytes([self.rank + 1]) * 64

    def tp_connect(self, handles):
        self.got = handles


def _worker(rank, world, port, out):
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    from paper_2505_01572_b200.stage import tp_connect_group
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    st = _FakeStage(rank, world)
    tp_connect_group(st)
    out.put((rank, st.got))
    dist.destroy_process_group()


def test_tp_connect_group_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 30500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    for _, got in res:
        assert got == [bytes([1]) * 64, bytes([2]) * 64]


def test_sharded_generation_equals_slicing_the_full_model():
    """synth.make_weights_sharded (used for the 70B stages) is bit-identical to
    slicing the full model with stage.shard_weights."""
    import torch

    import synth
    from paper_2505_01572_b200.stage import shard_weights
    s = synth.preset("toy-tp")
    full = synth.make_weights(s, seed=5)
    for T in (2, 4):
        for r in range(T):
            a = synth.make_weights_sharded(s, seed=5, rank=r, tp=T)
            b = shard_weights(s, full, r, T)
            for k in ("embed", "lm_head", "final_norm"):
                assert torch.equal(a[k], b[k]), k
            for la, lb in zip(a["layers"], b["layers"]):
                for k in la:
                    assert torch.equal(la[k], lb[k]), k
