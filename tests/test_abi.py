"""CPU-side checks of the C ABI boundary: the library builds/loads and exports
every function that include/*.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions(header="pipespec.h"):
    names = set()
    for h in [header]:
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\**\s+\**(ps_[a-z0-9_]+)\s*\(", src, re.M):
            names.add(m.group(1))
    return sorted(names)


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ("ps_stage_create", "ps_stage_destroy", "ps_prefill", "ps_draft", "ps_verify",
                     "ps_kv_rollback", "ps_pipeline_run", "ps_last_error"):
        assert required in names


def test_library_exports_every_declared_symbol():
    from paper_2505_01572_b200 import abi
    lib = abi.lib()
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    # ctypes prototypes cover every declared function
    assert set(declared_functions()) <= set(abi._PROTOS)


def test_product_library_carries_no_test_hooks():
    """The protocol test double and kernel probes live in libpipespec_test.so
    only; the trace accessor only in the PS_TRACE build."""
    from paper_2505_01572_b200 import abi
    lib = abi.lib()
    for n in declared_functions("pipespec_test.h"):
        assert not hasattr(lib, n), n


def test_test_library_exports_its_header():
    from paper_2505_01572_b200 import abi
    tl = abi.test_lib()
    names = [n for n in declared_functions("pipespec_test.h") if n != "ps_trace_read"]
    missing = [n for n in names if not hasattr(tl, n)]
    assert not missing, missing
    assert set(names) <= set(abi._TEST_PROTOS)


def test_pure_host_calls_without_gpu():
    import synth
    from paper_2505_01572_b200 import abi, stage
    lib = abi.lib()
    assert lib.ps_version() >= 100
    s = synth.preset("llama3.1-8b")
    sh = stage.model_shape(s)
    # 32 layers x 4 planes (K hi/lo, V hi/lo) x 8 heads x 64 tokens x 128 x 2 bytes per page, 8 pages
    assert lib.ps_kv_pool_bytes(ctypes.byref(sh), 512, 64) == 8 * 32 * 4 * 8 * 64 * 128 * 2
    # invalid arguments are rejected before any device work
    h = ctypes.c_void_p()
    st = lib.ps_stage_create(ctypes.byref(sh), None, None, None, ctypes.byref(h))
    assert st == abi.PS_E_INVALID and lib.ps_last_error()
    assert lib.ps_kv_rollback(None, 1) == abi.PS_E_INVALID
