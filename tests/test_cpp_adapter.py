"""The header-only C++ drop-in (include/opfuse_fk.hpp): reference-spelled opfuse
code (tests/cpp/adapter_example.cpp, `opfuse::` via the namespace alias) —
builders, validation errors, the api:: facade with its cast handle and cache,
execute_batch, the sc:: static chain — compiled and run over the fk.h C-ABI.

CPU: against the oracle (and the unmodified reference behind its shim), with
the known answers checked. GPU (-m gpu): the same program against
libfk_cuda.so with device planes must print exactly the oracle's lines.
"""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBS = {"oracle": (os.path.join(ROOT, "oracle", "build"), "fk_oracle"),
        "reference": (os.path.join(ROOT, "oracle", "_ref"), "fk_ref"),
        "cuda": (os.path.join(ROOT, "paper_2508_07071_b200", "lib"), "fk_cuda")}


def build_and_run(tmp_path, backend):
    lib_dir, name = LIBS[backend]
    exe = tmp_path / f"adapter_{backend}"
    subprocess.run(["g++", "-std=c++17", "-O1", "-Wall", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "adapter_example.cpp"), "-L", lib_dir, f"-l{name}",
                    f"-Wl,-rpath,{lib_dir}", "-o", str(exe)], check=True)
    return subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.splitlines()


def test_cpp_adapter_against_the_oracle(tmp_path):
    out = build_and_run(tmp_path, "oracle")
    src = (np.arange(60 * 40) % 97).astype(np.float32) / np.float32(97.0)
    v = ((src * np.float32(400) + np.float32(2)) - np.float32(1.5)) / np.float32(1.25)
    want = int(np.clip(np.rint(v.astype(np.float64)), 0, 255).sum())
    assert out[0] == f"passes=1 sum={want} savings={60 * 40 * (4 * 4 + 1)}"
    assert out[1] == "errc=3 pos=1"                                  # KindMismatch at chain position 1
    assert out[2] == "api errc=3 provenance=multiply (handle #2)"    # the facade names the handle
    assert out[3].startswith("facade passes=1/1 ")
    assert out[4].startswith("batch passes=1 ")
    assert out[5].startswith("static digest=")


def test_cpp_adapter_oracle_equals_reference(tmp_path):
    """The same program over the unmodified reference (minus the extensions the
    reference lacks: it has no cast handle, so only lines 0-2 compare)."""
    assert build_and_run(tmp_path, "reference")[:3] == build_and_run(tmp_path, "oracle")[:3]


@pytest.mark.gpu
def test_cpp_adapter_on_the_gpu(tmp_path):
    assert build_and_run(tmp_path, "cuda") == build_and_run(tmp_path, "oracle")
