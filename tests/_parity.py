"""Shared parity helpers for the -m gpu tests (compare CUDA path vs oracle)."""
import numpy as np

from oracle import llama as L

REL_LOGIT_TOL = 2e-2      # north star: max|dlogit| <= 2e-2 * max|logit|
TIE_GAP = 1e-2            # north star: decisions exempt where oracle top-2 gap < 1e-2,
                          # read relative to the row's max|logit| (reading R25)


def check_logits(gpu, ref, tol=REL_LOGIT_TOL):
    gpu = np.asarray(gpu, dtype=np.float64)
    err = np.abs(gpu - ref).max()
    scale = np.abs(ref).max()
    assert err <= tol * scale, f"max|dlogit| {err:.3e} > {tol} * {scale:.3e}"
    return err / scale


def check_tokens_teacher_forced(w64, shape, prompt, gpu_tokens):
    """Every GPU-chosen token equals the oracle argmax on the GPU's own stream,
    or the oracle prefers another token by less than TIE_GAP (reading R21)."""
    z = L.forward_full(w64, shape, list(prompt) + list(gpu_tokens))[len(prompt) - 1:-1]
    exempt = 0
    for j, t in enumerate(gpu_tokens):
        best = int(np.argmax(z[j]))
        if best != t:
            assert z[j][best] - z[j][t] < TIE_GAP * np.abs(z[j]).max(), (j, t, best, z[j][best] - z[j][t])
            exempt += 1
    return exempt


def check_verify(res, ref, w):
    """(a, next) bit-exact unless the deciding rows are near-ties."""
    a, nxt = res[0], res[1]
    if (a, nxt) == (ref["a"], ref["next"]):
        return True
    k = min(a, ref["a"])
    rel = [g / np.abs(z).max() for g, z in zip(ref["gaps"][: k + 1], ref["logits"][: k + 1])]
    assert min(rel) < TIE_GAP, (a, nxt, ref["a"], ref["next"], rel)
    return False
