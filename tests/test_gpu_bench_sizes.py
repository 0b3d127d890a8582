"""Parity at the sizes bench.py times (VERDICT r01 "parity at the benchmarked sizes").

Each benchmarked workload is built by the same builder bench.py uses
(paper_2508_07071_b200.workloads) on the CUDA product and on the C oracle, run
once, and compared bit for bit over every output byte:

  C5  configs[4]: all 8192 crops of 224x224x3 (the timed launch itself)
  C4  configs[3]: B = 1024 crops with per-crop normalize constants
  C2  configs[1]: the cvGS 50-crop batch
  C1  configs[0]: 3840x2160 f32 5-op chain -> u8
  C3  configs[2]: 4096x4096 f32, N in {1, 64, 1000} chained ops

The oracle is the plain-C restatement pinned to the reference in
test_oracle.py; outputs are compared on the GPU as raw bytes (no tolerance).
"""
import numpy as np
import pytest
import torch

from paper_2508_07071_b200 import workloads as wl
from paper_2508_07071_b200.opfuse import Library

pytestmark = pytest.mark.gpu


def same_bytes(cuda_outs, oracle_outs):
    for a, b in zip(cuda_outs, oracle_outs):
        bb = b.to(a.device) if b.device != a.device else b
        if not torch.equal(a, bb):
            diff = (a != bb).nonzero()
            return False, f"{diff.numel()} differing bytes, first at {diff[:8].flatten().tolist()}"
    return True, ""


def run_both(build, cuda, oracle):
    wc = build(cuda)
    wo = build(oracle)
    rep = cuda.execute_fused(wc.pipeline)
    oracle.execute_fused(wo.pipeline)
    torch.cuda.synchronize()
    ok, why = same_bytes(wc.outputs, wo.outputs)
    assert ok, f"{wc.name}: {why}"
    return rep, wc


def test_c5_all_8192_crops(cuda, oracle):
    rep, w = run_both(lambda lib: wl.crops_224(lib, 8192, per_crop_norm=False, name="C5"), cuda, oracle)
    assert rep.kernels_launched == 1
    assert cuda.last_kernel() == "fk_walk", cuda.last_kernel()


def test_c5_shards_match_whole(cuda, oracle):
    """The bench's strong-scaling shards (first = rank * 8192 / G) are the same
    crops as the whole batch: shard 3 of 4 equals the oracle too."""
    rep, w = run_both(lambda lib: wl.crops_224(lib, 2048, per_crop_norm=False, name="C5", first=6144), cuda, oracle)
    assert cuda.last_kernel() == "fk_walk"


def test_c4_1024_crops_per_crop_normalize(cuda, oracle):
    rep, w = run_both(lambda lib: wl.crops_224(lib, 1024, per_crop_norm=True, name="C4"), cuda, oracle)
    assert cuda.last_kernel() == "fk_walk"


@pytest.mark.parametrize("b", [1, 2, 16, 128])
def test_c4_small_batches_row_bands(cuda, oracle, b):
    """Small batches split each plane into row bands (more CTAs than planes)."""
    run_both(lambda lib: wl.crops_224(lib, b, per_crop_norm=True, name="C4"), cuda, oracle)
    assert cuda.last_kernel() == "fk_walk"


def test_c2_cvgs_50_crops(cuda, oracle):
    run_both(wl.c2, cuda, oracle)
    assert cuda.last_kernel() == "fk_walk"


def test_c1_4k(cuda, oracle):
    rep, _ = run_both(lambda lib: wl.c1(lib), cuda, oracle)
    assert cuda.last_kernel() == "fk_direct"


@pytest.mark.parametrize("n", [1, 64, 1000])
def test_c3_4096(cuda, oracle, n):
    run_both(lambda lib: wl.c3(lib, n), cuda, oracle)
    assert cuda.last_kernel() == "fk_direct"
