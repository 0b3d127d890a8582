"""The header-only C++ adapter (include/opfuse_fk.hpp) compiles and runs against the
oracle library: the reference's C++ spelling of a pipeline, unchanged, over fk.h."""
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_adapter_runs_against_the_c_abi(tmp_path):
    exe = tmp_path / "adapter"
    lib_dir = os.path.join(ROOT, "oracle", "build")
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "adapter_example.cpp"), "-L", lib_dir, "-lfk_oracle",
                    f"-Wl,-rpath,{lib_dir}", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout
    src = (np.arange(60 * 40) % 97).astype(np.float32) / np.float32(97.0)
    v = ((src * np.float32(400) + np.float32(2)) - np.float32(1.5)) / np.float32(1.25)
    want = int(np.clip(np.rint(v.astype(np.float64)), 0, 255).sum())
    assert f"passes=1 sum={want} savings={60 * 40 * (4 * 4 + 1)}" in out
    assert "errc=3 pos=1" in out  # KindMismatch at chain position 1
