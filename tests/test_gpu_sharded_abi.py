"""The multi-device and plane-ownership entry points of the C-ABI on the GPU.

* fk_execute_sharded (SURVEY.md §8(b),(e)): the configs[4] batch cut into
  contiguous z-shards (shard_range), one pipeline per shard, all enqueued by one
  call; the shard outputs equal the unsharded run and the oracle bit for bit.
  This box has one GPU, so every shard targets device 0 — the code path per
  shard (set device, enqueue on its stream, no wait) is the multi-GPU one.
* fk_gather: the shards' planes copied into one buffer (peer copies; the same
  device here) equal the unsharded output.
* fk_plane_alloc / fk_plane_free: a library-owned frame stays alive while a
  pipeline built from a view of it exists (plane.hpp:97 shared ownership), even
  after the caller's handle is freed.
"""
import numpy as np
import pytest
import torch

from paper_2508_07071_b200 import workloads as wl
from paper_2508_07071_b200._ffi import BILINEAR, F32, F32X3, U8X3
from paper_2508_07071_b200.opfuse import ExecConfig
from paper_2508_07071_b200.shard import shard_range

pytestmark = pytest.mark.gpu


def test_execute_sharded_equals_unsharded(cuda, oracle):
    n, shards = 96, 4
    whole = wl.crops_224(cuda, n, per_crop_norm=False)
    cuda.execute_fused(whole.pipeline)
    parts = [wl.crops_224(cuda, hi - lo, per_crop_norm=False, first=lo)
             for lo, hi in (shard_range(n, r, shards) for r in range(shards))]
    stream = torch.cuda.Stream()
    reps = cuda.execute_sharded([p.pipeline for p in parts], [0] * shards,
                                [ExecConfig(stream=stream.cuda_stream, timed=True)] * shards)
    torch.cuda.synchronize()
    assert len(reps) == shards and all(r.kernels_launched == 1 for r in reps)
    assert all(r.device_ms > 0 for r in reps)
    got = torch.cat([p.outputs[0] for p in parts])
    assert torch.equal(got, whole.outputs[0])
    wo = wl.crops_224(oracle, n, per_crop_norm=False)
    oracle.execute_fused(wo.pipeline)
    assert torch.equal(got.cpu(), wo.outputs[0])


def test_gather_collects_shards(cuda):
    n, shards = 24, 3
    whole = wl.crops_224(cuda, n, per_crop_norm=False)
    cuda.execute_fused(whole.pipeline)
    parts = [wl.crops_224(cuda, hi - lo, per_crop_norm=False, first=lo)
             for lo, hi in (shard_range(n, r, shards) for r in range(shards))]
    cuda.execute_sharded([p.pipeline for p in parts], [0] * shards)
    dst = torch.empty_like(whole.outputs[0])
    off, plan = 0, []
    for p in parts:
        out = p.outputs[0]
        plan.append((off, out.data_ptr(), 0, out.numel()))
        off += out.numel()
    cuda.gather(dst.data_ptr(), 0, plan, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert torch.equal(dst, whole.outputs[0])


def test_shared_plane_outlives_its_handle(cuda, oracle):
    rng = np.random.default_rng(5)
    frame = rng.integers(0, 256, (90, 160, 3), dtype=np.uint8)
    owned = cuda.plane_alloc_shared(160, 90, U8X3)
    # fill the library-owned plane through the API: a plain read -> write pipeline
    src = cuda.plane_from_numpy(frame)
    cuda.execute_fused(cuda.validate_chain([cuda.op_read_per_thread(src), cuda.op_write_per_thread(owned)]))
    # a crop + resize of a VIEW of it; then the caller's handle goes away
    view = owned.view(10, 5, 120, 80)
    dst = cuda.plane_alloc(48, 32, F32X3)
    rd = cuda.fold_unary_into_read(cuda.op_resize(cuda.op_read_per_thread(view), 48, 32, BILINEAR),
                                   cuda.op_cast(U8X3, F32X3))
    p = cuda.validate_chain([rd, cuda.op_write_per_thread(dst)])
    owned.free()
    assert owned.data_ptr == 0
    torch.cuda.empty_cache()
    cuda.execute_fused(p)
    got = dst.to_numpy()
    osrc = oracle.plane_from_numpy(frame)
    odst = oracle.plane_alloc(48, 32, F32X3)
    orr = oracle.fold_unary_into_read(oracle.op_resize(oracle.op_crop(osrc, 10, 5, 120, 80), 48, 32, BILINEAR),
                                      oracle.op_cast(U8X3, F32X3))
    oracle.execute_fused(oracle.validate_chain([orr, oracle.op_write_per_thread(odst)]))
    assert np.array_equal(got.view(np.uint32), odst.to_numpy().view(np.uint32))


def test_shared_plane_errors(cuda):
    from paper_2508_07071_b200.opfuse import OpfuseError
    with pytest.raises(OpfuseError):
        cuda.plane_alloc_shared(0, 4, F32)
    p = cuda.plane_alloc_shared(8, 4, F32)
    p.free()
    p.free()  # a second free is a no-op
