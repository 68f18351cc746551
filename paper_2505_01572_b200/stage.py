"""Thin Python binding over the C ABI (same names as include/pipespec.h).

PyTorch only provides device memory (weights, the KV pool) and streams; every
step of the verify pass runs in libpipespec.so's sm_100a kernels.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import abi

LAYER_KEYS = ("wq", "wk", "wv", "wo", "wg", "wu", "wd", "n_attn", "n_mlp")


def model_shape(s) -> abi.ModelShape:
    """ps_model_shape from any object with the ModelShape attributes."""
    return abi.ModelShape(s.vocab, s.d_model, s.n_layers, s.n_heads, s.n_kv_heads, s.head_dim, s.d_ffn,
                          s.rms_eps, s.rope_theta, s.rope_kind, s.rope_factor, s.lo_ff, s.hi_ff,
                          s.rope_orig_max, int(bool(s.tied)))


def kv_pool_bytes(shape, max_seq: int, page_size: int, tp_size: int = 1) -> int:
    sh = model_shape(shape)
    return int(abi.lib().ps_kv_pool_bytes_tp(C.byref(sh), max_seq, page_size, tp_size))


def shard_weights(shape, weights: dict, rank: int, tp_size: int) -> dict:
    """Rank `rank`'s Megatron shard of a full weight dict (include/pipespec.h,
    ps_placement): column-parallel Q/K/V (by heads) and gate/up (by FFN rows),
    row-parallel O and down (matching input columns), vocab-parallel lm_head;
    embed and norm gains replicated.  Pure slicing (copies where a slice is not
    contiguous); no arithmetic."""
    T, r = tp_size, rank
    hd = shape.head_dim
    qh, kh, fr, vr = shape.n_heads // T, shape.n_kv_heads // T, shape.d_ffn // T, shape.vocab // T
    out = {"embed": weights["embed"], "final_norm": weights["final_norm"],
           "lm_head": weights["lm_head"][r * vr:(r + 1) * vr].contiguous(), "layers": []}
    for lw in weights["layers"]:
        out["layers"].append({
            "wq": lw["wq"][r * qh * hd:(r + 1) * qh * hd].contiguous(),
            "wk": lw["wk"][r * kh * hd:(r + 1) * kh * hd].contiguous(),
            "wv": lw["wv"][r * kh * hd:(r + 1) * kh * hd].contiguous(),
            "wo": lw["wo"][:, r * qh * hd:(r + 1) * qh * hd].contiguous(),
            "wg": lw["wg"][r * fr:(r + 1) * fr].contiguous(),
            "wu": lw["wu"][r * fr:(r + 1) * fr].contiguous(),
            "wd": lw["wd"][:, r * fr:(r + 1) * fr].contiguous(),
            "n_attn": lw["n_attn"], "n_mlp": lw["n_mlp"]})
    return out


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


class Stage:
    """One model M_i: ps_stage_create over borrowed bf16 CUDA weights."""

    def __init__(self, shape, weights: dict, max_seq: int = 1024, max_window: int = 31,
                 page_size: int = 64, device: int = 0, stream: torch.cuda.Stream | None = None,
                 use_graphs: bool = True, megakernel: bool = True, tp_rank: int = 0, tp_size: int = 1,
                 max_ctas: int = 0):
        """`weights`: the full model, or with tp_size > 1 this rank's shard
        (shard_weights); `shape` is always the full model's."""
        self.shape = shape
        self.weights = weights            # keep the borrowed tensors alive
        self._sh = model_shape(shape)
        dev = torch.device("cuda", device)
        for k in ("embed", "lm_head", "final_norm"):
            t = weights[k]
            assert t.is_cuda and t.dtype == torch.bfloat16 and t.is_contiguous(), k
        ptrs = []
        for lw in weights["layers"]:
            for k in LAYER_KEYS:
                t = lw[k]
                assert t.is_cuda and t.dtype == torch.bfloat16 and t.is_contiguous(), k
                ptrs.append(t.data_ptr())
        self._layer_ptrs = (C.c_void_p * max(1, len(ptrs)))(*ptrs)
        self._w = abi.Weights(weights["embed"].data_ptr(), weights["lm_head"].data_ptr(),
                              weights["final_norm"].data_ptr(),
                              C.cast(self._layer_ptrs, C.POINTER(C.c_void_p)))
        nbytes = kv_pool_bytes(shape, max_seq, page_size, tp_size)
        self.kv_pool = torch.empty(max(nbytes, 16), dtype=torch.uint8, device=dev)
        self.stream = stream if stream is not None else torch.cuda.Stream(device=dev)
        self._pl = abi.Placement(device, None, tp_rank, tp_size)
        self._opts = abi.StageOpts(max_seq, max_window, page_size, self.kv_pool.data_ptr(), nbytes,
                                   self.stream.cuda_stream, int(use_graphs), int(megakernel), max_ctas)
        self.tp_rank, self.tp_size = tp_rank, tp_size
        h = C.c_void_p()
        abi.check(abi.lib().ps_stage_create(C.byref(self._sh), C.byref(self._w), C.byref(self._pl),
                                            C.byref(self._opts), C.byref(h)))
        self._h = h
        self.max_window = max_window
        self.max_seq = max_seq

    # ---------------------------------------------------------------- calls
    def close(self):
        if getattr(self, "_h", None):
            abi.lib().ps_stage_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def prefill(self, tokens):
        t = _i32(tokens)
        abi.check(abi.lib().ps_prefill(self._h, t.ctypes.data, len(t)))

    def set_prefill_path(self, path: int):
        """abi.PS_PREFILL_AUTO (prefill kernels for runs of >= 64 tokens) or
        abi.PS_PREFILL_ROWS (the megakernel's 64-row bucket only)."""
        abi.check(abi.lib().ps_set_prefill_path(self._h, int(path)))

    def resync(self, tokens):
        """Lazy rollback-and-extend to `tokens` (KV catch-up folded into the next forward)."""
        t = _i32(tokens)
        abi.check(abi.lib().ps_resync(self._h, t.ctypes.data, len(t)))

    def draft(self, n_steps: int) -> list[int]:
        out = np.zeros(max(1, n_steps), dtype=np.int32)
        abi.check(abi.lib().ps_draft(self._h, n_steps, out.ctypes.data))
        return out[:n_steps].tolist()

    def verify(self, window, want_logits: bool = False):
        """Returns (accepted_len, next_token[, logits float32 [w+1, V] numpy])."""
        if isinstance(window, torch.Tensor) and window.is_cuda:
            win = window.to(torch.int32).contiguous()
            ptr, w = win.data_ptr(), win.numel()
        else:
            win = _i32(window)
            ptr, w = win.ctypes.data, len(win)
        a, nxt = C.c_int32(), C.c_int32()
        logits = None
        lptr = None
        if want_logits:
            logits = np.zeros((w + 1, self.shape.vocab // self.tp_size), dtype=np.float32)
            lptr = logits.ctypes.data
        abi.check(abi.lib().ps_verify(self._h, ptr if w else None, w, C.byref(a), C.byref(nxt), lptr))
        if want_logits:
            return a.value, nxt.value, logits
        return a.value, nxt.value

    def tp_handle(self) -> bytes:
        """This rank's exchange-buffer handle (ps_tp_handle)."""
        buf = (C.c_uint8 * abi.PS_TP_HANDLE_BYTES)()
        abi.check(abi.lib().ps_tp_handle(self._h, buf))
        return bytes(buf)

    def tp_connect(self, handles):
        """Map the peers' exchange buffers: handles = every rank's tp_handle() in rank order."""
        assert len(handles) == self.tp_size and all(len(h) == abi.PS_TP_HANDLE_BYTES for h in handles)
        buf = (C.c_uint8 * (abi.PS_TP_HANDLE_BYTES * self.tp_size)).from_buffer_copy(b"".join(handles))
        abi.check(abi.lib().ps_tp_connect(self._h, buf))

    def verify_async(self, window):
        """Enqueue a verification pass (ps_verify_async); `window` may be a CUDA
        int32 tensor (gathered on-stream, never read by the host).  Returns the
        ticket's pinned result record (valid after verify_wait)."""
        if isinstance(window, torch.Tensor) and window.is_cuda:
            self._async_win = window.to(torch.int32).contiguous()    # alive until the pass ran
            ptr, w = self._async_win.data_ptr(), self._async_win.numel()
        else:
            self._async_win = _i32(window)
            ptr, w = self._async_win.ctypes.data, len(self._async_win)
        tk = abi.VerifyTicket()
        abi.check(abi.lib().ps_verify_async(self._h, ptr if w else None, w, C.byref(tk)))
        return tk

    def verify_query(self) -> bool:
        d = C.c_int32()
        abi.check(abi.lib().ps_verify_query(self._h, C.byref(d)))
        return bool(d.value)

    def verify_wait(self):
        """Commit the in-flight pass: returns (accepted_len, next_token)."""
        a, nxt = C.c_int32(), C.c_int32()
        abi.check(abi.lib().ps_verify_wait(self._h, C.byref(a), C.byref(nxt)))
        self._async_win = None
        return a.value, nxt.value

    def kv_rollback(self, keep_len: int):
        abi.check(abi.lib().ps_kv_rollback(self._h, keep_len))

    def tokens(self) -> list[int]:
        n = C.c_int64()
        abi.check(abi.lib().ps_stage_tokens(self._h, None, 0, C.byref(n)))
        out = np.zeros(max(1, n.value), dtype=np.int32)
        abi.check(abi.lib().ps_stage_tokens(self._h, out.ctypes.data, n.value, C.byref(n)))
        return out[:n.value].tolist()

    def info(self) -> dict:
        i = abi.StageInfo()
        abi.check(abi.lib().ps_stage_get_info(self._h, C.byref(i)))
        return dict(n_tokens=i.n_tokens, kv_len=i.kv_len, pages_in_use=i.pages_in_use,
                    pages_total=i.pages_total, launches_per_verify=i.launches_per_verify,
                    last_fwd_ms=i.last_fwd_ms, sum_fwd_ms=i.sum_fwd_ms, n_fwd=i.n_fwd,
                    max_window=i.max_window, max_seq=i.max_seq, attn_sc=i.attn_sc)

    def reset_timers(self):
        abi.check(abi.lib().ps_stage_reset_timers(self._h))

    def set_synthetic(self, S, n_prompt: int, level: int, top: int, alphas, seed: int):
        s = _i32(S)
        al = (C.c_double * max(1, len(alphas)))(*alphas)
        abi.check(abi.lib().ps_set_synthetic(self._h, s.ctypes.data if len(s) else None, len(s), n_prompt,
                                             level, top, al, seed))

    def clear_synthetic(self):
        abi.check(abi.lib().ps_set_synthetic(self._h, None, 0, 0, 0, 0, None, 0))


def tp_connect_local(stages):
    """Link the ranks of one tensor-parallel group created in this process (rank order)."""
    hs = (C.c_void_p * len(stages))(*[s.handle for s in stages])
    abi.check(abi.lib().ps_tp_connect_local(hs, len(stages)))


def tp_connect_group(stage, group=None):
    """One process per rank: all-gather the exchange handles over a
    torch.distributed group (any backend) and connect."""
    import torch.distributed as dist
    handles = [None] * stage.tp_size
    dist.all_gather_object(handles, stage.tp_handle(), group=group)
    stage.tp_connect(handles)


class RunOptions:
    """ps_run_opts with its ctypes arrays kept alive.  gammas None -> NULL
    (window cap 8 per verifier); alphas (k-1 floats) turn on the synthetic
    override; virtual_ns pads every step of stage i to that many ns;
    event_cap > 0 records the run's event log (see events())."""

    def __init__(self, k, max_new_tokens, mode, gammas=None, lookaheads=None, eos_id=-1, max_lead=0,
                 alphas=None, seed=0, virtual_ns=None, event_cap=0):
        self.g = (C.c_int32 * k)(*gammas) if gammas is not None else None
        self.la = (C.c_int32 * k)(*lookaheads) if lookaheads is not None else None
        self.al = (C.c_double * max(1, k - 1))(*alphas) if alphas is not None else None
        self.vn = (C.c_int64 * k)(*virtual_ns) if virtual_ns is not None else None
        self.ev = (abi.Event * event_cap)() if event_cap > 0 else None
        self.opts = abi.RunOpts(mode, max_new_tokens, eos_id,
                                C.cast(self.g, C.POINTER(C.c_int32)) if self.g else None,
                                C.cast(self.la, C.POINTER(C.c_int32)) if self.la else None, max_lead,
                                C.cast(self.al, C.POINTER(C.c_double)) if self.al else None, seed,
                                C.cast(self.vn, C.POINTER(C.c_int64)) if self.vn else None,
                                C.cast(self.ev, C.POINTER(abi.Event)) if self.ev else None, event_cap)

    def events(self, stats) -> list[dict]:
        out = []
        for e in (self.ev[:stats.n_events] if self.ev else []):
            out.append(dict(t_ns=e.t_ns, stage=e.stage, kind=e.kind, n=e.n, w=e.w, a=e.a, next=e.next,
                            origin=e.origin, window=list(e.window[:e.w])))
        return out


def board_create(name: str, k: int, capacity: int):
    """Shared-memory board for one process per stage (ps_board_create)."""
    abi.check(abi.lib().ps_board_create(name.encode(), k, capacity))


def board_unlink(name: str):
    abi.check(abi.lib().ps_board_unlink(name.encode()))


def pipeline_run_rank(stage, rank: int, k: int, board: str, prompt, max_new_tokens: int, gammas=None,
                      lookaheads=None, eos_id: int = -1, max_lead: int = 0, virtual_ns=None, event_cap: int = 0,
                      return_events: bool = False):
    """This process's stage M_rank of a k-stage async PipeSpec run
    (ps_pipeline_run_rank); `stage` may be a list of the members of a
    tensor-parallel group driven by this process (ps_pipeline_run_rank_group)."""
    group = list(stage) if isinstance(stage, (list, tuple)) else [stage]
    ro = RunOptions(k, max_new_tokens, abi.PS_MODE_PIPESPEC, gammas, lookaheads, eos_id, max_lead,
                    virtual_ns=virtual_ns, event_cap=event_cap)
    p = _i32(prompt)
    out = np.zeros(max_new_tokens, dtype=np.int32)
    n = C.c_int32()
    stats = abi.RunStats()
    hs = (C.c_void_p * len(group))(*[s.handle for s in group])
    abi.check(abi.lib().ps_pipeline_run_rank_group(hs, len(group), rank, k, board.encode(), p.ctypes.data, len(p),
                                                   C.byref(ro.opts), out.ctypes.data, C.byref(n), C.byref(stats)))
    if return_events:
        return out[:n.value].tolist(), stats, ro.events(stats)
    return out[:n.value].tolist(), stats


def pipeline_run(stages, prompt, max_new_tokens: int, mode: int = abi.PS_MODE_PIPESPEC, gammas=None,
                 lookaheads=None, eos_id: int = -1, max_lead: int = 0, alphas=None, seed: int = 0,
                 virtual_ns=None, event_cap: int = 0, return_events: bool = False):
    """ps_pipeline_run over `stages` (M_0 .. M_K).  Returns (tokens, stats[, events])."""
    k = len(stages)
    hs = (C.c_void_p * k)(*[s.handle for s in stages])
    ro = RunOptions(k, max_new_tokens, mode, gammas, lookaheads, eos_id, max_lead, alphas, seed, virtual_ns,
                    event_cap)
    opts = ro.opts
    p = _i32(prompt)
    out = np.zeros(max_new_tokens, dtype=np.int32)
    n = C.c_int32()
    stats = abi.RunStats()
    abi.check(abi.lib().ps_pipeline_run(hs, k, p.ctypes.data, len(p), C.byref(opts), out.ctypes.data,
                                        C.byref(n), C.byref(stats)))
    if return_events:
        return out[:n.value].tolist(), stats, ro.events(stats)
    return out[:n.value].tolist(), stats


def group_call(group, fn):
    """fn(member) on every member of a tensor-parallel group concurrently (one
    thread each, as the ABI requires); returns the leader's result after
    checking the members agree."""
    import threading
    res, err = [None] * len(group), [None] * len(group)

    def go(i):
        try:
            res[i] = fn(group[i])
        except BaseException as e:  # noqa: BLE001
            err[i] = e

    th = [threading.Thread(target=go, args=(i,)) for i in range(1, len(group))]
    for t in th:
        t.start()
    go(0)
    for t in th:
        t.join()
    for e in err:
        if e is not None:
            raise e
    for r in res[1:]:
        if r != res[0]:
            raise RuntimeError(f"tensor-parallel members disagree: {r} vs {res[0]}")
    return res[0]
