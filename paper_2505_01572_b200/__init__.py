"""paper_2505_01572_b200 — B200-native (sm_100a) PipeSpec verify hot path.

The product is libpipespec.so (C ABI in include/pipespec.h); this package is
its thin Python binding.  There is no CPU fallback: without the built library
the import of `stage` fails, and without an sm_100a GPU every call raises
PipeSpecError(PS_E_CUDA).
"""
from .abi import PipeSpecError  # noqa: F401
from .stage import (Stage, pipeline_run, kv_pool_bytes, model_shape, shard_weights,  # noqa: F401
                    tp_connect_local, tp_connect_group, board_create, board_unlink, pipeline_run_rank,
                    group_call, RunOptions)
