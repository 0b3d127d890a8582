"""CUDA product vs the C oracle (itself pinned to the reference in test_oracle.py).

Bit-exact everywhere: integer/u8 paths and the f32/f64 paths alike (the kernels
use explicitly rounded intrinsics in the reference's operation order, so no
tolerance is needed; NaN payloads compare as equal, see fkchains.same).
"""
import numpy as np
import pytest

from fkchains import (ChainSpec, ReadSpec, mismatch_report, outputs_equal, random_chain, run)
from paper_2508_07071_b200._ffi import (BILINEAR, F32, F32X3, F64, NEAREST, OP_ADD, OP_DIV, OP_MUL, OP_SUB,
                                        SWAP_RB, U8, U8X3, PATH_GENERIC, PATH_COMPILED)
from paper_2508_07071_b200.opfuse import ExecConfig

pytestmark = pytest.mark.gpu


def check(cuda, oracle, spec, unfused=False, cfg=None):
    got, rep = run(cuda, spec, unfused=unfused, cfg=cfg)
    want, wrep = run(oracle, spec, unfused=unfused)
    assert outputs_equal(got, want), mismatch_report(got, want)
    assert (rep.bytes_read, rep.bytes_written, rep.passes, rep.points_visited, rep.intermediate_bytes_allocated) == \
        (wrep.bytes_read, wrep.bytes_written, wrep.passes, wrep.points_visited, wrep.intermediate_bytes_allocated)
    return rep


@pytest.mark.parametrize("seed", range(8))
def test_random_chains_fused(cuda, oracle, seed):
    rng = np.random.default_rng(1000 + seed)
    for _ in range(60):
        spec = random_chain(rng, allow_batch_arith=True)
        rep = check(cuda, oracle, spec)
        assert rep.kernels_launched == 1


@pytest.mark.parametrize("seed", range(3))
def test_random_chains_interpreter_only(cuda, oracle, seed):
    """Same chains with the compiled kernels and the u8 LUT disabled: the interpreted path alone."""
    rng = np.random.default_rng(1000 + seed)
    for _ in range(60):
        spec = random_chain(rng, allow_batch_arith=True)
        rep = check(cuda, oracle, spec, cfg=ExecConfig(force_generic=True, no_lut=True))
        assert rep.path == PATH_GENERIC


def test_u8_chains_take_compiled_kernels(cuda, oracle):
    """u8 crop/resize reads with lane-wise chains run the compiled resample kernel (LUT or AFFINE)."""
    rng = np.random.default_rng(77)
    frame = rng.integers(0, 256, (97, 131, 3), dtype=np.uint8)
    gray = rng.integers(0, 256, (60, 70), dtype=np.uint8)
    norm = [("arith", OP_SUB, F32X3, (123.675, 116.28, 103.53)), ("arith", OP_DIV, F32X3, (58.395, 57.12, 57.375))]
    cases = [
        # AFFINE: swap + cast folded, f32 normalise, split
        ChainSpec([frame], [ReadSpec(0, 3, 4, 50, 60, 37, 29, BILINEAR, [("swap", U8X3), ("cast", U8X3, F32X3)])],
                  norm, F32X3, split=True),
        # AFFINE: cast in the compute chain (not folded), packed write, nearest
        ChainSpec([frame], [ReadSpec(0, 0, 0, 131, 97, 64, 48, NEAREST)], [("cast", U8X3, F32X3)] + norm, F32X3),
        # LUT: u8 arithmetic with a swap between per-lane constants
        ChainSpec([frame], [ReadSpec(0, 10, 10, 40, 40, 40, 40, BILINEAR)],
                  [("arith", OP_MUL, U8X3, (3, 5, 7)), ("swap", U8X3), ("arith", OP_ADD, U8X3, (1, 2, 3))], U8X3),
        # LUT: gray u8 plane, cast to f64, StaticLoop
        ChainSpec([gray], [ReadSpec(0, 2, 3, 33, 44, 100, 90, BILINEAR)],
                  [("cast", U8, F64), ("loop", ("arith", OP_MUL, F64, (1.01,)), 7)], F64),
        # LUT: direct (non-resizing) crop
        ChainSpec([frame], [ReadSpec(0, 5, 6, 77, 55)], [("cast", U8X3, F32X3), ("arith", OP_DIV, F32X3, (3.0, 7.0, 9.0))],
                  F32X3, split=True),
    ]
    for spec in cases:
        rep = check(cuda, oracle, spec)
        assert rep.path == PATH_COMPILED, spec


@pytest.mark.parametrize("seed", range(3))
def test_random_chains_unfused(cuda, oracle, seed):
    rng = np.random.default_rng(2000 + seed)
    for _ in range(40):
        spec = random_chain(rng)
        rep = check(cuda, oracle, spec, unfused=True)
        assert rep.kernels_launched == rep.passes


def test_random_chains_large_planes(cuda, oracle):
    rng = np.random.default_rng(7)
    for _ in range(12):
        spec = random_chain(rng, max_dim=300, max_batch=3, max_ops=5)
        check(cuda, oracle, spec)


def test_c1_vertical_chain_small(cuda, oracle):
    """configs[0] at a parity size: Read f32 -> Mul,Add,Sub,Div -> Cast u8 -> Write."""
    rng = np.random.default_rng(42)
    src = rng.random((217, 389), dtype=np.float32)
    spec = ChainSpec([src], [ReadSpec(0)],
                     [("arith", OP_MUL, F32, (400.0,)), ("arith", OP_ADD, F32, (2.0,)),
                      ("arith", OP_SUB, F32, (1.5,)), ("arith", OP_DIV, F32, (1.25,)), ("cast", F32, U8)], U8)
    assert check(cuda, oracle, spec).path == PATH_COMPILED          # fk_direct<MUL,ADD,SUB,DIV; ->u8>
    assert check(cuda, oracle, spec, cfg=ExecConfig(force_generic=True)).path == PATH_GENERIC
    check(cuda, oracle, spec, unfused=True)
    # odd widths, a crop view and f32 output exercise the tails of the 16-wide tiles
    src2 = rng.random((33, 101), dtype=np.float32) * 300 - 20
    for rd in (ReadSpec(0), ReadSpec(0, 3, 2, 77, 29)):
        for comp, wk in (([("arith", OP_MUL, F32, (3.0,)), ("arith", OP_ADD, F32, (0.5,))], F32),
                         ([("arith", OP_SUB, F32, (7.0,)), ("arith", OP_DIV, F32, (3.0,)), ("cast", F32, U8)], U8)):
            assert check(cuda, oracle, ChainSpec([src2], [rd], comp, wk, dst_stride_pad=3)).path == PATH_COMPILED


def test_cvgs_batch_50(cuda, oracle):
    """configs[1] exactly: 50 crops of a 1920x1080 u8x3 frame -> bilinear 64x128 ->
    SwapRB -> f32x3 -> sub mean / div std -> split into 3 planar f32 planes."""
    rng = np.random.default_rng(42)
    frame = rng.integers(0, 256, (1080, 1920, 3), dtype=np.uint8)
    r7 = np.random.default_rng(7)
    reads = []
    for _ in range(50):
        w, h = 64 + int(r7.integers(0, 448)), 128 + int(r7.integers(0, 448))
        x0, y0 = int(r7.integers(0, 1921 - w)), int(r7.integers(0, 1081 - h))
        reads.append(ReadSpec(0, x0, y0, w, h, 64, 128, BILINEAR, [("swap", U8X3), ("cast", U8X3, F32X3)]))
    spec = ChainSpec([frame], reads, [("arith", OP_SUB, F32X3, (123.675, 116.28, 103.53)),
                                      ("arith", OP_DIV, F32X3, (58.395, 57.12, 57.375))],
                     F32X3, split=True, batch=True, active_read=50, active_write=50)
    rep = check(cuda, oracle, spec)
    assert rep.kernels_launched == 1
    check(cuda, oracle, spec, unfused=True)


def test_per_crop_normalize_matches_single_plane_pipelines(cuda, oracle):
    """configs[3] extension: per-crop Sub/Div constants (BatchArith) in ONE launch equal
    B independent single-plane oracle pipelines (the reference cannot express per-z
    compute params; bench.cpp:199-202 builds one pipeline per plane)."""
    rng = np.random.default_rng(3)
    frame = rng.integers(0, 256, (300, 400, 3), dtype=np.uint8)
    B = 6
    rects = [(int(rng.integers(0, 200)), int(rng.integers(0, 100)), int(rng.integers(20, 200)),
              int(rng.integers(20, 200))) for _ in range(B)]
    rects = [(x, y, min(w, 400 - x), min(h, 300 - y)) for x, y, w, h in rects]
    means = [tuple(float(np.float32(v)) for v in 255 * np.array([0.485, 0.456, 0.406]) + rng.normal(0, 2, 3))
             for _ in range(B)]
    stds = [tuple(float(np.float32(v)) for v in 255 * np.array([0.229, 0.224, 0.225]) + rng.normal(0, 1, 3))
            for _ in range(B)]
    post = [("cast", U8X3, F32X3)]
    batched = ChainSpec([frame], [ReadSpec(0, *r, 56, 56, BILINEAR, post) for r in rects],
                        [("batch_arith", OP_SUB, F32X3, means), ("batch_arith", OP_DIV, F32X3, stds)],
                        F32X3, split=True, batch=True, active_read=B, active_write=B)
    got, rep = run(cuda, batched)
    assert rep.kernels_launched == 1
    for z in range(B):
        single = ChainSpec([frame], [ReadSpec(0, *rects[z], 56, 56, BILINEAR, post)],
                           [("arith", OP_SUB, F32X3, means[z]), ("arith", OP_DIV, F32X3, stds[z])], F32X3, split=True)
        want, _ = run(oracle, single)
        assert outputs_equal([got[z]], want), f"crop {z}: " + mismatch_report([got[z]], want)


def test_static_loop_long_chain(cuda, oracle):
    """configs[2] structure: ceil(N/2) Mul then floor(N/2) Add, StaticLoop above 64 (bench.cpp:100-108)."""
    rng = np.random.default_rng(42)
    src = rng.random((64, 96), dtype=np.float32)
    for n in (1, 2, 63, 64, 65, 1000):
        comp = []
        for op, c, k in ((OP_MUL, 1.0000001, (n + 1) // 2), (OP_ADD, 1e-7, n // 2)):
            inner = ("arith", op, F32, (float(np.float32(c)),))
            comp += [inner] * k if k <= 64 else [("loop", inner, k)]
        comp = [c for c in comp]
        check(cuda, oracle, ChainSpec([src], [ReadSpec(0)], comp, F32))


def test_default_value_and_inactive_writes(cuda, oracle):
    rng = np.random.default_rng(5)
    srcs = [rng.integers(0, 256, (9, 13), dtype=np.uint8) for _ in range(5)]
    spec = ChainSpec(srcs, [ReadSpec(i) for i in range(5)], [("cast", U8, F32), ("arith", OP_MUL, F32, (2.0,))],
                     F32, batch=True, active_read=3, active_write=4, default=(7,))
    got, _ = run(cuda, spec)
    want, _ = run(oracle, spec)
    assert outputs_equal(got, want)
    assert np.all(got[3][0] == 14.0)          # default value 7 -> cast -> x2
    assert np.all(got[4][0] == 0.0)           # inactive write: untouched (zero-initialised)


def test_kernel_selection_reports_path(cuda):
    import torch
    lib = cuda
    src = lib.plane_from_numpy(np.ones((8, 8), np.float32))
    dst = lib.plane_alloc(8, 8, F32)
    p = lib.validate_chain([lib.op_read_per_thread(src), lib.op_mul(lib_f32(3.0)), lib.op_write_per_thread(dst)])
    rep = lib.execute_fused(p, ExecConfig(timed=True, force_generic=True))
    torch.cuda.synchronize()
    assert rep.path == PATH_GENERIC and rep.device_ms > 0
    assert np.all(dst.to_numpy() == 3.0)


def lib_f32(v):
    from paper_2508_07071_b200.opfuse import f32
    return f32(v)


def test_golden_vectors_on_gpu(cuda):
    """The reference's own outputs (tests/golden, generated from oracle/_ref) reproduced on sm_100a."""
    import json
    import os
    from fkchains import spec_from_dict
    here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    manifest = json.load(open(os.path.join(here, "golden.json")))
    arrays = np.load(os.path.join(here, "golden.npz"))
    for case in manifest["cases"]:
        name = case["name"]
        srcs = [arrays[f"{name}/src{j}"] for j in range(case["spec"]["n_sources"])]
        spec = spec_from_dict(case["spec"], srcs)
        want = [[arrays[f"{name}/out{z}_{l}"] for l in range(n)] for z, n in enumerate(case["n_out"])]
        for cfg in (None, ExecConfig(force_generic=True, no_lut=True)):
            got, rep = run(cuda, spec, cfg=cfg)
            assert outputs_equal(got, want), name + ": " + mismatch_report(got, want)
            assert [rep.bytes_read, rep.bytes_written, rep.passes, rep.points_visited] == case["fused"], name
        got, _ = run(cuda, spec, unfused=True)
        assert outputs_equal(got, want), name + " (unfused): " + mismatch_report(got, want)
