"""The roofline-grade unfused comparator (csrc/fk_stream.cu) against the oracle.

execute_unfused (executor.cpp:134-217) runs one compiled streaming pass per
compute op over planar intermediates, then the write pass, when every pass is
streamable — the configs the bench reports `unfused` for. Its output must equal
the oracle's unfused (and fused) output bit for bit, its counters the
reference's, and it must really take the compiled passes (last_kernel).
"""
import numpy as np
import pytest
import torch

from paper_2508_07071_b200 import workloads as wl

pytestmark = pytest.mark.gpu


def unfused_both(build, cuda, oracle):
    wc, wo = build(cuda), build(oracle)
    rep = cuda.execute_unfused(wc.pipeline)
    assert cuda.last_kernel() == "fk_stream", cuda.last_kernel()
    orep = oracle.execute_unfused(wo.pipeline)
    torch.cuda.synchronize()
    for a, b in zip(wc.outputs, wo.outputs):
        assert torch.equal(a.cpu(), b), f"{wc.name}: unfused output differs from the oracle"
    assert rep.passes == orep.passes == wc.pipeline.n_compute + 1
    assert rep.kernels_launched == rep.passes
    assert (rep.bytes_read, rep.bytes_written, rep.intermediate_bytes_allocated) == \
        (orep.bytes_read, orep.bytes_written, orep.intermediate_bytes_allocated)
    return rep


def test_unfused_c1_small(cuda, oracle):
    unfused_both(lambda lib: wl.c1(lib, W=256, H=96), cuda, oracle)


@pytest.mark.parametrize("n", [1, 5, 64, 300])
def test_unfused_c3_chains(cuda, oracle, n):
    unfused_both(lambda lib: wl.c3(lib, n, W=128, H=64), cuda, oracle)


@pytest.mark.parametrize("per_crop", [False, True])
def test_unfused_crops(cuda, oracle, per_crop):
    unfused_both(lambda lib: wl.crops_224(lib, 12, per_crop_norm=per_crop, name="C4" if per_crop else "C5"),
                 cuda, oracle)


def test_unfused_c2(cuda, oracle):
    unfused_both(wl.c2, cuda, oracle)
