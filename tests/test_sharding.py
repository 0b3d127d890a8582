"""Multi-process sharding path on CPU: world_size 2 over gloo (127.0.0.1).

Each rank builds the batched crop pipeline over its own contiguous shard of the
crops (paper_2508_07071_b200.shard.shard_range) on the C oracle, runs it, and
the shards gathered on rank 0 must equal one unsharded run bit for bit; the
timing reduction is the max over ranks. This is the host logic bench.py uses
on N GPUs (there with NCCL and the CUDA library).
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2508_07071_b200.shard import shard_range


def test_shard_range_partitions_exactly():
    for n in (0, 1, 7, 8, 50, 8192, 8193):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def _crops(n):
    rng = np.random.default_rng(11)
    rects = []
    for _ in range(n):
        w, h = int(rng.integers(20, 90)), int(rng.integers(20, 70))
        rects.append((int(rng.integers(0, 120 - w)), int(rng.integers(0, 80 - h)), w, h))
    return rects


def _run_shard(lib, frames, rects, lo, hi):
    from fkchains import ChainSpec, ReadSpec, run
    from paper_2508_07071_b200._ffi import BILINEAR, F32X3, OP_DIV, OP_SUB, U8X3
    reads = [ReadSpec(z % len(frames), *rects[z], 24, 16, BILINEAR, [("cast", U8X3, F32X3)]) for z in range(lo, hi)]
    spec = ChainSpec(frames, reads, [("arith", OP_SUB, F32X3, (123.675, 116.28, 103.53)),
                                     ("arith", OP_DIV, F32X3, (58.395, 57.12, 57.375))],
                     F32X3, split=True, batch=True, active_read=hi - lo, active_write=hi - lo)
    outs, rep = run(lib, spec)
    return outs, rep


def _worker(rank, world, port, n, result_q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import torch.distributed as dist
    from paper_2508_07071_b200.opfuse import Library
    from paper_2508_07071_b200.shard import max_over_ranks, sum_over_ranks
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(3)
    frames = [rng.integers(0, 256, (80, 120, 3), dtype=np.uint8) for _ in range(2)]
    rects = _crops(n)
    lo, hi = shard_range(n, rank, world)
    outs, rep = _run_shard(Library("oracle"), frames, rects, lo, hi)
    slowest = max_over_ranks(rep.wall_time_ns)
    total_points = sum_over_ranks(rep.points_visited)
    gathered = [None] * world if rank == 0 else None
    dist.gather_object([[a.tobytes() for a in d] for d in outs], gathered, dst=0)
    if rank == 0:
        full, _ = _run_shard(Library("oracle"), frames, rects, 0, n)
        flat = [plane for shard in gathered for plane in shard]
        same = all(x == y.tobytes() for got, want in zip(flat, full) for x, y in zip(got, want))
        result_q.put((same, len(flat), slowest >= rep.wall_time_ns, int(total_points)))
    dist.destroy_process_group()


def test_two_rank_gloo_sharding_matches_unsharded_run():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    n = 13
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    same, planes, max_ok, points = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert same and planes == n and max_ok and points == n * 24 * 16


def test_execute_sharded_cpu_backends(oracle, reference):
    """fk_execute_sharded on the CPU backends runs the shards one after another:
    the shard outputs concatenate to the unsharded output."""
    import torch
    from paper_2508_07071_b200 import workloads as wl
    for lib in (oracle,):
        n, shards = 10, 3
        whole = wl.crops_224(lib, n, per_crop_norm=False)
        lib.execute_fused(whole.pipeline)
        parts = [wl.crops_224(lib, hi - lo, per_crop_norm=False, first=lo)
                 for lo, hi in (shard_range(n, r, shards) for r in range(shards))]
        reps = lib.execute_sharded([p.pipeline for p in parts], [0] * shards)
        assert len(reps) == shards
        assert torch.equal(torch.cat([p.outputs[0] for p in parts]), whole.outputs[0])
        dst = torch.empty_like(whole.outputs[0])
        off, plan = 0, []
        for p in parts:
            plan.append((off, p.outputs[0].data_ptr(), 0, p.outputs[0].numel()))
            off += p.outputs[0].numel()
        lib.gather(dst.data_ptr(), 0, plan)
        assert torch.equal(dst, whole.outputs[0])


def test_plane_alloc_cpu_backends(oracle, reference):
    from paper_2508_07071_b200._ffi import F32X3
    from paper_2508_07071_b200.opfuse import OpfuseError
    for lib in (oracle, reference):
        p = lib.plane_alloc_shared(5, 3, F32X3)
        assert p.data_ptr != 0 and p.row_stride == 5
        v = p.view(1, 1, 2, 2)
        assert v.width == 2 and v.c().data == p.data_ptr + (5 + 1) * 12
        p.free()
        assert p.data_ptr == 0
        with pytest.raises(OpfuseError):
            lib.plane_alloc_shared(0, 3, F32X3)
