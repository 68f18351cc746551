"""Build the sm_100a shared libraries in-tree with nvcc.

  libpipespec.so        the product: the C ABI of include/pipespec.h
                        (csrc/ps_stage.cu + csrc/ps_pipeline.cu)
  libpipespec_test.so   test infrastructure only (include/pipespec_test.h:
                        the runtime's protocol test double, GEMM probes)
  libpipespec_trace.so  the product with %globaltimer phase stamps (PS_TRACE=1,
                        scripts/timeline.py); built on request only

nvcc cross-compiles for sm_100a without a GPU.  The libraries link the CUDA
runtime statically, so loading one needs no GPU; every compute entry point
fails with PS_E_CUDA when no sm_100a device is present (no CPU fallback).
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libpipespec.so")
TEST_LIB = os.path.join(PKG, "libpipespec_test.so")
TRACE_LIB = os.path.join(PKG, "libpipespec_trace.so")
TARGETS = {
    LIB: (["ps_stage.cu", "ps_pipeline.cu"], []),
    TEST_LIB: (["ps_testlib.cu"], []),
    TRACE_LIB: (["ps_stage.cu", "ps_pipeline.cu"], ["-DPS_TRACE=1"]),
}
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-Xcompiler", "-fPIC", "-shared", "-cudart", "static", "-Xptxas", "-v"]


def _stale(lib: str) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cuh", ".h"))]
    deps += [os.path.join(ROOT, "include", f) for f in os.listdir(os.path.join(ROOT, "include"))]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False, trace: bool = False) -> str:
    """Build the product and test libraries (and the trace library if asked),
    in parallel nvcc processes; returns the product library's path."""
    libs = [LIB, TEST_LIB] + ([TRACE_LIB] if trace else [])
    procs = []
    for lib in libs:
        if not force and not _stale(lib):
            continue
        srcs, extra = TARGETS[lib]
        cmd = [NVCC, *FLAGS, *extra, "-o", lib + ".tmp", *[os.path.join(CSRC, s) for s in srcs]]
        procs.append((lib, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
    for lib, p in procs:
        out, err = p.communicate()
        if p.returncode != 0:
            sys.stderr.write(out + err)
            raise RuntimeError(f"nvcc failed building {os.path.basename(lib)}")
        if verbose:
            sys.stderr.write(err)
        os.replace(lib + ".tmp", lib)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, trace="--trace" in sys.argv))
