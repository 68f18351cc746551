"""CPU pins of the shape presets and of the roofline byte accounting that
bench.py and scripts/verify_sweep.py divide by.

The presets follow the public HF configs of the models the paper names (P:181,
names only): their parameter counts must match the published model sizes, and
the per-pass algorithmic bytes (streamed weights + KV read + KV write) must
match the values derived in SURVEY.md 8(d) from the same configs."""
import pytest

import synth

# published parameter counts (HF model cards / config arithmetic)
PARAMS = {
    "llama-68m": 68.0e6,        # JackFram/llama-68m
    "llama2-7b": 6.74e9,
    "llama2-13b": 13.0e9,
    "llama3.2-1b": 1.24e9,
    "llama3.1-8b": 8.03e9,
    "llama3.1-70b": 70.6e9,
}


@pytest.mark.parametrize("name,n", sorted(PARAMS.items()))
def test_preset_parameter_counts(name, n):
    s = synth.preset(name)
    assert abs(s.n_params() - n) / n < 5e-3, (name, s.n_params())


# KV bytes per token and streamed weight bytes per pass
@pytest.mark.parametrize("name,kv,stream_gb", [
    ("llama-68m", 6144, 0.087),
    ("llama2-7b", 512 * 1024, 13.2),
    ("llama2-13b", 800 * 1024, 25.7),
    ("llama3.2-1b", 32 * 1024, 2.47),
    ("llama3.1-8b", 128 * 1024, 15.0),
    ("llama3.1-70b", 320 * 1024, 139.0),
])
def test_kv_and_streamed_bytes(name, kv, stream_gb):
    s = synth.preset(name)
    assert s.kv_bytes_per_token_bf16() == kv
    assert s.kv_bytes_per_token() == 2 * kv          # split-bf16 (hi + lo) planes as stored (R28)
    assert abs(s.streamed_bytes_per_pass(1) / 1e9 - stream_gb) / stream_gb < 5e-3


@pytest.mark.parametrize("ctx,gb", [(512, 15.08), (4096, 15.55), (32768, 19.31)])
def test_verify_pass_bytes_8b_r17(ctx, gb):
    """SURVEY.md 8(d) 'Algorithmic bytes per verify pass', LLaMA-3.1-8B, R = 17."""
    s = synth.preset("llama3.1-8b")
    R = 17
    b = s.streamed_bytes_per_pass(R) + (ctx + R) * s.kv_bytes_per_token_bf16()
    assert abs(b / 1e9 - gb) < 0.01
