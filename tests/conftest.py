import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running oracle checks")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    """Report every near-tie exemption the parity checks took (R25)."""
    try:
        from tests._parity import EXEMPTIONS
    except Exception:  # pragma: no cover
        return
    tr = terminalreporter
    tr.write_sep("-", f"R25 near-tie exemptions taken: {len(EXEMPTIONS)}")
    for e in EXEMPTIONS:
        tr.write_line(f"  {e['where']}: gap {e['abs_gap']:.3e} abs / {e['rel_gap']:.3e} rel "
                      f"(max|logit| {e['scale']:.2f}, {e['criterion']} bound)")
    out = os.environ.get("PS_EXEMPTIONS_JSON")
    if out:
        import json
        with open(out, "w") as f:
            json.dump(EXEMPTIONS, f, indent=1)
