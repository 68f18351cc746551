"""Seeded synthetic prompts and draft windows.

Prompts are uniform random token ids (SURVEY.md §8(d) "Prompts are uniform
random token ids from seed_prompt"); the paper's datasets are out of scope.
"""
from __future__ import annotations

import numpy as np


def make_prompt(vocab: int, length: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(np.random.SeedSequence([seed, 0x9209]))
    return rng.integers(0, vocab, size=length, dtype=np.int64).astype(np.int32)


def make_window(vocab: int, w: int, seed: int) -> np.ndarray:
    """A random draft window of w tokens (arbitrary drafts, mostly rejected)."""
    rng = np.random.default_rng(np.random.SeedSequence([seed, 0x3141]))
    return rng.integers(0, vocab, size=w, dtype=np.int64).astype(np.int32)
