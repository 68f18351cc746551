"""CPU tests of bench.py's host logic: the N>1 cross-rank aggregation (gloo,
world_size 2) and the --impl reference arm (the oracle) on toy shapes."""
import json
import os
import subprocess
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, out):
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dev, wall, tok = bench.aggregate(1.0 + rank, 2.0 + 3 * rank, 10 + rank, world, device="cpu")
    out.put((rank, dev, wall, tok))
    dist.destroy_process_group()


def test_aggregate_two_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    for _, dev, wall, tok in res:
        assert (dev, wall, tok) == (2.0, 5.0, 21.0)   # max, max, sum


def test_reference_arm_toy():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--draft",
                        "toy-drafter", "--target", "toy-verifier", "--steps", "3", "--warmup", "1"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "tokens/s" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0


def test_reference_arm_nonzero_rank_exits_silently():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--draft",
                        "toy-drafter", "--target", "toy-verifier", "--steps", "1", "--warmup", "0"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert r.returncode == 0 and r.stdout.strip() == ""


@pytest.mark.parametrize("n,cfg,want", [
    (2, "c2", [[0], [1]]),
    (3, "c3", [[0], [1], [2]]),
    (4, "c4", [[0], [1], [2, 3]]),
    (8, "c4", [[0], [1], [4, 5, 6, 7]]),
])
def test_layouts_follow_the_paper(n, cfg, want):
    """N > 1: each model on its own GPU(s), the target tensor parallel over the
    rest (8 GPUs 1B@0, 8B@1, 70B TP4@4-7; 4 GPUs 70B TP2@2-3)."""
    sys.path.insert(0, ROOT)
    import bench
    import synth
    shapes = [synth.preset(m) for m in bench.LAYOUT_CONFIGS[cfg]["models"]]
    assert bench.layout_for(n, cfg, shapes) == want
