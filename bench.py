#!/usr/bin/env python
"""bench.py — PipeSpec verify hot path on B200 (BASELINE.json configs[1]).

Workload (N=1): k=2 LLaMA-3.2-1B-shape -> LLaMA-3.1-8B-shape, random-init bf16
weights, 512-token synthetic prompt, 256 greedy tokens, both stages co-resident
on one B200.  A *step* is one pass of the whole hot path (SURVEY.md §8(a)
a1-a13): M_0 drafts gamma tokens (gamma rows=1 forwards, synthetic alpha
override on the emitted token), M_1 verifies the window (one rows=gamma+1
forward + argmax/compare/scan), appends the accepted prefix + correction/bonus
token, truncates its KV, and the drafter is resynced to M_1's buffer (the
rollback signal).  Output is lossless: identical to M_1's autoregressive
greedy stream, which the bench checks on every run.

value    tokens/s of the whole job (device time, CUDA events, max over ranks)
e2e      the same through the C ABI with host buffers, wall clock
roofline the dominant kernel (gate/up GEMM of M_1) timed live with CUDA events
cpu_baseline / --impl reference: the fp64 oracle on the host cores (bounded
         sample, extrapolated in depth)

N>1 (torchrun): every rank runs an independent replica of the batch-1 job
(weak scaling, no data-path collective); the stage-per-GPU pipeline is the
NEXT-1 runtime.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "tokens/s batch-1 greedy & speedup vs M_k autoregressive; verify HBM GB/s"
STEP_IN_BYTES = 176     # sizeof(StepIn): uploaded per forward (host -> device)
STEP_OUT_BYTES = 144    # sizeof(StepOut): read back per forward (device -> host, mapped pinned)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--draft", default="llama3.2-1b")
    ap.add_argument("--target", default="llama3.1-8b")
    ap.add_argument("--prompt", type=int, default=512)
    ap.add_argument("--gen", type=int, default=256)
    ap.add_argument("--gamma", type=int, default=4)   # SD window tuned on B200 over {3,4,5,8} (paper SD: 8)
    ap.add_argument("--alpha", type=float, default=0.8)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--multi-gpu-extras", action="store_true",
                    help="N>1: also time M_1 tensor-parallel over the N GPUs and the stage-per-GPU async pipeline")
    return ap.parse_args()


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clocks, throttle reasons and power sampled during the timed region
    (NVML every 10 ms; nvidia-smi every 200 ms if NVML is unavailable), plus
    the board's energy counter across the region (J per token, P:296 4.5)."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index):
        self.index = index
        self.samples = []            # (sm_mhz, max_mhz, [reason names], power_w)
        self.energy_j = None
        self._stop = threading.Event()
        self._nv = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
        except Exception:
            self._nv = None
        self._t = threading.Thread(target=self._run, daemon=True)

    def _sample_nvml(self):
        nv, h = self._nv, self._h
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
        reasons = [n for n, b in zip(self.NAMES, bits) if r & b]
        pw = nv.nvmlDeviceGetPowerUsage(h) / 1e3
        self.samples.append((float(sm), float(mx), reasons, pw))

    def _sample_smi(self):
        out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True,
                             timeout=5).stdout.strip()
        if out:
            f = [x.strip() for x in out.split(",")]
            reasons = [self.NAMES[i] for i in range(4) if "Active" in f[2 + i] and not f[2 + i].startswith("Not")]
            num = lambda x: float(x) if x.replace(".", "").isdigit() else float("nan")
            self.samples.append((num(f[0]), num(f[1]), reasons, float("nan")))

    def _run(self):
        while not self._stop.is_set():
            try:
                self._sample_nvml() if self._nv else self._sample_smi()
            except Exception:
                pass
            self._stop.wait(0.01 if self._nv else 0.2)

    def _energy_mj(self):
        try:
            return self._nv.nvmlDeviceGetTotalEnergyConsumption(self._h) if self._nv else None
        except Exception:
            return None

    def __enter__(self):
        self._e0 = self._energy_mj()
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)
        e1 = self._energy_mj()
        if self._e0 is not None and e1 is not None:
            self.energy_j = (e1 - self._e0) / 1e3

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [s[0] for s in self.samples if s[0] == s[0]]
        mx = [s[1] for s in self.samples if s[1] == s[1]]
        pw = [s[3] for s in self.samples if s[3] == s[3]]
        reasons = sorted({n for s in self.samples for n in s[2]})
        out = {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
               "reasons": reasons, "samples": len(self.samples), "source": "nvml" if self._nv else "nvidia-smi"}
        if pw:
            out["power_w_median"] = statistics.median(pw)
        return out


# ----------------------------------------------------------------------------- dist
def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


def aggregate(dev_s, wall_s, tokens, world, device="cpu"):
    """Whole-job numbers over ranks: times are the MAX over ranks (the job ends
    when its slowest replica does), tokens the SUM (weak scaling)."""
    if world <= 1:
        return dev_s, wall_s, float(tokens)
    import torch
    import torch.distributed as dist
    times = torch.tensor([dev_s, wall_s], device=device, dtype=torch.float64)
    tok = torch.tensor([float(tokens)], device=device, dtype=torch.float64)
    dist.all_reduce(times, op=dist.ReduceOp.MAX)
    dist.all_reduce(tok, op=dist.ReduceOp.SUM)
    return float(times[0]), float(times[1]), float(tok[0])


def multi_gpu_extras(args, rank, world, ts, wt, drafter, target, prompt, S, g):
    """N > 1 only (beside the replica line): (1) M_1's verify pass tensor-
    parallel over all N GPUs -- Megatron shards, the all-reduces and the
    vocab-parallel argmax inside the megakernel over NVLink peer memory
    (SURVEY §8(e), a14); (2) the paper's stage-per-GPU layout, M_0 on rank 0's
    GPU and M_1 on rank 1's, async PipeSpec through the shared-memory board.
    Each part reports an error string instead of failing the bench."""
    import torch
    import torch.distributed as dist
    from paper_2505_01572_b200 import (Stage, board_create, board_unlink, pipeline_run_rank, shard_weights,
                                       tp_connect_group)
    out = {}
    obj = [prompt, S, f"/pipespec-bench-{os.getpid()}"]
    dist.broadcast_object_list(obj, src=0)        # every rank works on rank 0's prompt and stream
    p0, S0, board = obj
    try:
        tps = Stage(ts, shard_weights(ts, wt, rank, world), max_seq=args.prompt + 64, max_window=g,
                    tp_rank=rank, tp_size=world)
        tp_connect_group(tps)
        tps.prefill(p0)
        win = S0[:g]
        res = None
        for it in range(13):
            if it == 3:
                torch.cuda.synchronize()
                dist.barrier()
                tps.reset_timers()
            res = tps.verify(win)
            tps.kv_rollback(len(p0))
        inf = tps.info()
        ms = torch.tensor([inf["sum_fwd_ms"] / max(1, inf["n_fwd"])], device="cuda", dtype=torch.float64)
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        R = g + 1
        byts = ts.streamed_bytes_per_pass(R) + (len(p0) + R) * ts.kv_bytes_per_token()
        out["tp_verify_pass"] = {"tp": world, "ms": float(ms[0]), "rows": R, "ctx": len(p0),
                                 "accepted": res[0], "agg_GB/s": byts / (float(ms[0]) * 1e-3) / 1e9}
        tps.close()
    except Exception as e:  # noqa: BLE001
        out["tp_verify_pass"] = {"error": repr(e)[:300]}
    try:
        if rank == 0:
            board_create(board, 2, len(p0) + args.gen + 512)
            drafter.set_synthetic(S0, len(p0), level=0, top=1, alphas=[args.alpha], seed=args.seed + 1234)
        dist.barrier()
        if rank < 2:
            stage = drafter if rank == 0 else target
            torch.cuda.synchronize()
            w0 = time.perf_counter()
            got, st = pipeline_run_rank(stage, rank, 2, board, p0, args.gen, gammas=[0, g])
            dt = time.perf_counter() - w0
            ok = got == S0[:args.gen]
        dist.barrier()
        if rank == 0:
            board_unlink(board)
            out["stage_per_gpu_pipespec"] = {"layout": "M_0 on GPU 0, M_1 on GPU 1, one process each",
                                             "tokens_per_s": len(got) / dt,
                                             "tokens_per_s_decode": len(got) / (st.wall_ns / 1e9),
                                             "lossless": ok, "verify_steps": int(st.verify_steps[1]),
                                             "rollbacks": int(st.rollbacks[0])}
    except Exception as e:  # noqa: BLE001
        out["stage_per_gpu_pipespec"] = {"error": repr(e)[:300]}
    return out


def oracle_sample(draft_shape, target_shape, wd, wt, gamma, alpha, seed, n_rounds, ctx=64, layers=2):
    """The fp64 oracle (as it stands) on the host cores: sync-SD rounds of the
    same two shapes at `layers` of their L layers (full width and vocab), ctx
    tokens of context; per-round time extrapolated linearly in depth:
      t(L) = t(0) + (L / layers) * (t(layers) - t(0))   for each model.
    Accepted lengths follow the same counter-based construction as the GPU run."""
    import numpy as np

    import synth
    from oracle import llama as OL
    from oracle import synthetic as SY

    def np64(w, nl):
        sub = {"embed": w["embed"], "lm_head": w["lm_head"], "final_norm": w["final_norm"],
               "layers": w["layers"][:nl]}
        return synth.weights_to_numpy(sub)

    d2, t2 = synth.reduced_depth(draft_shape, layers), synth.reduced_depth(target_shape, layers)
    d0, t0 = synth.reduced_depth(draft_shape, 0), synth.reduced_depth(target_shape, 0)
    wd2, wt2 = np64(wd, layers), np64(wt, layers)
    wd0, wt0 = dict(wd2, layers=[]), dict(wt2, layers=[])
    prompt = [int(x) for x in synth.make_prompt(target_shape.vocab, ctx, seed + 99)]
    thr = SY.alpha_threshold(alpha)
    times, toks = [], 0
    p = 0
    for _ in range(n_rounds):
        t_start = time.perf_counter()
        per = {}
        for name, (w, s) in {"d2": (wd2, d2), "d0": (wd0, d0), "t2": (wt2, t2), "t0": (wt0, t0)}.items():
            sess = OL.Session(w, s)
            sess.forward(prompt)                       # context (not timed)
            t1 = time.perf_counter()
            if name.startswith("d"):
                z = sess.forward(prompt[-1:])
                for _ in range(gamma - 1):
                    z = sess.forward([OL.greedy(z[-1])])
            else:
                sess.forward(prompt[-1:] + prompt[:gamma])   # one verify forward, R = gamma + 1
            per[name] = time.perf_counter() - t1
        tD = per["d0"] + draft_shape.n_layers / layers * (per["d2"] - per["d0"])
        tT = per["t0"] + target_shape.n_layers / layers * (per["t2"] - per["t0"])
        a = 0
        while a < gamma and SY.agree(seed, 0, p + a, thr):
            a += 1
        p += a + 1
        toks += a + 1
        times.append(tD + tT)
        del t_start
    cores = len(os.sched_getaffinity(0))
    try:
        from threadpoolctl import threadpool_info
        blas = max((i.get("num_threads", 0) for i in threadpool_info()), default=cores)
    except Exception:
        blas = cores
    return toks / sum(times), min(cores, blas), times, toks


def run_reference(args):
    """--impl reference: the oracle on the host cores, same metric/config."""
    rank, _, world = dist_env()
    if rank != 0:
        return
    import torch

    import synth
    ds, ts = synth.preset(args.draft), synth.preset(args.target)
    # the oracle only needs the first 2 layers + embeddings (CPU generation)
    wd = synth.make_weights(synth.reduced_depth(ds, 2), seed=args.seed, device="cpu")
    wt = synth.make_weights(synth.reduced_depth(ts, 2), seed=args.seed + 1, device="cpu")
    del torch
    tot_t, tot_tok = 0.0, 0
    _, _, _, _ = oracle_sample(ds, ts, wd, wt, args.gamma, args.alpha, args.seed, 1) if args.warmup else (0, 0, 0, 0)
    val, cores, times, toks = oracle_sample(ds, ts, wd, wt, args.gamma, args.alpha, args.seed, args.steps)
    tot_t, tot_tok = sum(times), toks
    line = {"metric": METRIC, "value": val, "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / max(1, args.steps), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": f"k=2 {args.draft}->{args.target} sync-SD round, gamma={args.gamma}, "
                                   f"alpha={args.alpha} synthetic", "prompt": args.prompt, "gen": args.gen},
            "cpu_baseline": {"value": val, "unit": "tokens/s", "cores": cores, "kind": "oracle",
                             "sample": f"{args.steps} oracle sync-SD rounds at 2 of L layers (full width/vocab), "
                                       "64-token context, extrapolated linearly in depth"},
            "e2e": {"value": val, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- ours
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import numpy as np
    import torch
    import torch.distributed as dist

    import synth
    from paper_2505_01572_b200 import Stage, abi

    rank, local, world = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ds, ts = synth.preset(args.draft), synth.preset(args.target)
    g = args.gamma
    max_seq = args.prompt + args.gen + 4 * g + 64
    wd = synth.make_weights(ds, seed=args.seed, device="cuda")
    wt = synth.make_weights(ts, seed=args.seed + 1, device="cuda")
    drafter = Stage(ds, wd, max_seq=max_seq, max_window=g)
    target = Stage(ts, wt, max_seq=max_seq, max_window=g)
    prompt = [int(x) for x in synth.make_prompt(ts.vocab, args.prompt, seed=args.seed + 17 + rank)]
    L = abi.lib()

    # --- M_K autoregressive: the lossless reference stream S and the AR baseline
    target.prefill(prompt)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(target.stream)
    S = target.draft(args.gen + 2 * g + 2)
    e1.record(target.stream)
    e1.synchronize()
    ar_tok_s = len(S) / (e0.elapsed_time(e1) / 1e3)
    target.kv_rollback(args.prompt)
    drafter.prefill(prompt)
    drafter.set_synthetic(S, args.prompt, level=0, top=1, alphas=[args.alpha], seed=args.seed + 1234)

    state = {"gen": [], "pass_ctx": []}

    def step(record):
        if len(state["gen"]) >= args.gen:          # job restarts from the prompt
            assert state["gen"][:args.gen] == S[:args.gen], "lossless check failed"
            target.kv_rollback(args.prompt)
            drafter.resync(prompt)
            state["gen"] = []
        d = drafter.draft(g)
        a, nxt = target.verify(d)
        if record:
            state["pass_ctx"].append(args.prompt + len(state["gen"]))
        new = d[:a] + [nxt]
        state["gen"] += new
        drafter.resync(prompt + state["gen"])     # rollback signal: O_0 := O_1 (lazy KV catch-up)
        return len(new)

    for _ in range(args.warmup):
        step(False)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    target.reset_timers()
    drafter.reset_timers()
    launches0 = L.ps_kernel_launch_count()
    t0e, t1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tokens = 0
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        t0e.record(drafter.stream)
        for _ in range(args.steps):
            tokens += step(True)
        t1e.record(target.stream)
        torch.cuda.synchronize()
        w1 = time.perf_counter()
    launches = L.ps_kernel_launch_count() - launches0
    dev_s = t0e.elapsed_time(t1e) / 1e3
    wall_s = w1 - w0
    dev_s, wall_s, tot_tokens = aggregate(dev_s, wall_s, tokens, world, device="cuda")

    # --- dominant kernel: M_1's verify forward = ONE persistent megakernel launch
    # (embed, 32 x {QKV, attention, combine, O, gate/up, down}, lm_head, argmax);
    # its device time is measured live by CUDA events around the launch on the
    # stage stream (ps_stage_info.sum_fwd_ms over the timed verify passes).
    R = g + 1
    ti, di = target.info(), drafter.info()
    pass_ms = ti["sum_fwd_ms"] / max(1, ti["n_fwd"])
    draft_ms = di["sum_fwd_ms"] / max(1, di["n_fwd"])
    ctx = statistics.mean(state["pass_ctx"]) if state["pass_ctx"] else args.prompt
    pass_bytes = ts.streamed_bytes_per_pass(R) + (ctx + R) * ts.kv_bytes_per_token()
    pass_gbs = pass_bytes / (pass_ms * 1e-3) / 1e9
    draft_bytes = ds.streamed_bytes_per_pass(1) + (ctx + 1) * ds.kv_bytes_per_token()
    draft_gbs = draft_bytes / (draft_ms * 1e-3) / 1e9
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = peaks.get("hbm_gbs", 6650.0)
    traffic, draft_traffic = None, None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        traffic = tr.get("verify_megakernel_8b_r5", {}).get("dram_bytes_per_launch")
        draft_traffic = tr.get("draft_megakernel_1b_r1", {}).get("dram_bytes_per_launch")
    except Exception:
        pass
    step_ms = 1e3 * dev_s / args.steps
    share = (pass_ms + g * draft_ms) / step_ms if step_ms > 0 else None

    # --- whole-generation runs through ps_pipeline_run (Alg.1) in each mode, wall clock
    from paper_2505_01572_b200 import pipeline_run
    from paper_2505_01572_b200.abi import PS_MODE_AR, PS_MODE_PIPESPEC, PS_MODE_SYNC_SD
    modes = {}
    # async PipeSpec with lookahead 0 (the paper's setting) and, as Fig.5's
    # lookahead sweep, with the verifier waiting for L >= 1 drafts (reading R7)
    runs = [("ar", PS_MODE_AR, 0), ("sync_sd", PS_MODE_SYNC_SD, 0), ("pipespec_async", PS_MODE_PIPESPEC, 0)]
    runs += [(f"pipespec_async_lookahead{la}", PS_MODE_PIPESPEC, la) for la in (1, 2, 4)]
    for mname, mode, la in runs:
        torch.cuda.synchronize()
        w0m = time.perf_counter()
        out, st_ = pipeline_run([drafter, target], prompt, args.gen, mode=mode, gammas=[0, g], lookaheads=[0, la])
        torch.cuda.synchronize()
        dtm = time.perf_counter() - w0m
        assert out == S[:args.gen], f"{mname}: output differs from M_K autoregressive decoding"
        modes[mname] = {"tokens_per_s": len(out) / dtm, "decode_s": st_.wall_ns / 1e9,
                        "tokens_per_s_decode": len(out) / (st_.wall_ns / 1e9) if st_.wall_ns else None,
                        "verify_steps": int(st_.verify_steps[1]), "rollbacks": int(st_.rollbacks[0]),
                        # tokens appended per verify step of M_K (Fig.4's histogram)
                        "accept_hist": {int(k): int(c) for k, c in enumerate(st_.accept_hist) if c}}
    value = tot_tokens / dev_s
    e2e = tot_tokens / wall_s
    fwd_per_step = g + 1
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * dev_s / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": f"k=2 {args.draft}->{args.target} (BASELINE configs[1]), sync-SD round "
                               f"gamma={args.gamma}, synthetic alpha={args.alpha}, co-resident on 1 GPU",
                   "prompt": args.prompt, "gen": args.gen, "global_batch": world,
                   "parallelism": f"replicas{world}" if world > 1 else "single",
                   "l2": "inputs > L2 (16 GB of 8B weights streamed per verify pass)"},
        "speedup_vs_ar": value / ar_tok_s, "ar_tokens_per_s": ar_tok_s,
        "pipeline_run": modes,
        "tokens_per_step": tot_tokens / world / args.steps,
        "verify_pass": {"ms": pass_ms, "rows": R, "ctx": ctx, "bytes": pass_bytes, "GB/s": pass_gbs,
                        "frac": pass_gbs / peak},
        "draft_step": {"ms": draft_ms, "rows": 1, "bytes": draft_bytes, "GB/s": draft_gbs, "frac": draft_gbs / peak,
                       "traffic": draft_traffic},
        "kernel_share_of_step": share,
        "roofline": {"kernel": "M_1 verify forward: persistent tcgen05/TMA megakernel (1 launch per pass)",
                     "bound": "hbm", "achieved": pass_gbs, "peak": peak, "unit": "GB/s", "frac": pass_gbs / peak,
                     "traffic": traffic, "algorithmic_bytes_per_launch": pass_bytes, "rows": R,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback"},
        "e2e": {"value": e2e, "unit": "tokens/s",
                "h2d_bytes_per_step": fwd_per_step * STEP_IN_BYTES + g * 4,
                "d2h_bytes_per_step": fwd_per_step * STEP_OUT_BYTES},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    if clk.energy_j is not None and tokens > 0:
        # board energy counter across the timed region (this GPU's tokens; paper 4.5)
        line["energy"] = {"joules": clk.energy_j, "j_per_token": clk.energy_j / tokens,
                          "avg_w": clk.energy_j / max(wall_s, 1e-9), "source": "nvmlDeviceGetTotalEnergyConsumption"}
    if world > 1 and args.multi_gpu_extras:
        line["multi_gpu"] = multi_gpu_extras(args, rank, world, ts, wt, drafter, target, prompt, S, g)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, cores, times, toks = oracle_sample(ds, ts, wd, wt, g, args.alpha, args.seed + 1234, 2)
        line["cpu_baseline"] = {"value": v, "unit": "tokens/s", "cores": cores, "kind": "oracle",
                                "sample": f"2 oracle sync-SD rounds (gamma={g}) at 2 of L layers, full width/vocab, "
                                          "64-token context, extrapolated linearly in depth"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    drafter.close()
    target.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
