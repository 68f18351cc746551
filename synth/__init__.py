"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds NO arithmetic of the method (no forward pass, no argmax,
no verification, no hashing used by the synthetic-alpha drafters).  It only
produces data: model shape presets (public HF configs),
seeded bf16 random-init weights and seeded prompts / draft windows.

Both `oracle/` and `paper_2505_01572_b200/` may import it; neither imports
the other.
"""
from .shapes import ModelShape, PRESETS, preset, reduced_depth  # noqa: F401
from .weights import make_weights, make_weights_sharded, weights_to_numpy  # noqa: F401
from .prompts import make_prompt, make_window  # noqa: F401
