"""The column-streaming resample kernel's exact-result filter (fk_resample_sep.cuh).

The kernel lerps in FP32 and recomputes in the reference's double arithmetic
only the pixels whose FP32 value lies within 2^-13 of a rounding boundary. These
cases aim at exactly the places where that could go wrong — ties that are exact
in binary (dyadic fx/fy: 448 -> 224, 2x upscales), ties that are exact only as
rationals (8 -> 7 scale with tap differences of 7, where the double's own
rounding decides nearbyint), a band in which every pixel is flagged (the fix
list overflows), and the configs[4] workload itself on a 256-crop sample — and
compare with the C oracle bit for bit.
"""
import numpy as np
import pytest

from fkchains import ChainSpec, ReadSpec, mismatch_report, outputs_equal, run
from paper_2508_07071_b200._ffi import BILINEAR, F32X3, OP_DIV, OP_SUB, PATH_COMPILED, U8, U8X3

pytestmark = pytest.mark.gpu

NORM = [("arith", OP_SUB, F32X3, (123.675, 116.28, 103.53)), ("arith", OP_DIV, F32X3, (58.395, 57.12, 57.375))]
POST = [("swap", U8X3), ("cast", U8X3, F32X3)]


def check(cuda, oracle, spec):
    got, rep = run(cuda, spec)
    want, _ = run(oracle, spec)
    assert outputs_equal(got, want), mismatch_report(got, want)
    return rep


def batch_spec(frames, rects, out_w, out_h, post=POST, compute=NORM, write=F32X3, split=True):
    reads = [ReadSpec(i % len(frames), x, y, w, h, out_w, out_h, BILINEAR, list(post))
             for i, (x, y, w, h) in enumerate(rects)]
    return ChainSpec(frames, reads, compute, write, split=split, batch=True,
                     active_read=len(reads), active_write=len(reads))


def test_c5_sample_256_crops(cuda, oracle):
    """configs[4]'s pipeline on 256 of its crops (16 frames, w/h in [112, 448] -> 224x224)."""
    rng = np.random.default_rng(42)
    frames = [rng.integers(0, 256, (1080, 1920, 3), dtype=np.uint8) for _ in range(16)]
    r = np.random.default_rng(7)
    rects = []
    for _ in range(256):
        w, h = int(r.integers(112, 449)), int(r.integers(112, 449))
        rects.append((int(r.integers(0, 1921 - w)), int(r.integers(0, 1081 - h)), w, h))
    rep = check(cuda, oracle, batch_spec(frames, rects, 224, 224, post=[("cast", U8X3, F32X3)]))
    assert rep.path == PATH_COMPILED and rep.kernels_launched == 1


@pytest.mark.parametrize("levels", [2, 8, 256])
def test_dyadic_scales_exact_ties(cuda, oracle, levels):
    """Integer and half-integer scale factors: fx, fy in {0, 1/4, 1/2, 3/4}, where
    (a + b + c + d) / 4 lands exactly on k + 0.5 and nearbyint must tie to even."""
    rng = np.random.default_rng(levels)
    frames = [rng.integers(0, levels, (300, 500, 3), dtype=np.uint8)]
    rects = [(0, 0, 448, 224), (1, 3, 448, 112), (2, 2, 112, 56), (5, 7, 336, 168), (9, 1, 56, 28), (0, 0, 224, 224),
             (3, 0, 450, 226), (4, 4, 224, 112)]
    check(cuda, oracle, batch_spec(frames, rects, 224, 56))
    # the u8 value itself (no chain after the resize): LUT mode, u8x3 packed output
    check(cuda, oracle, batch_spec(frames, rects, 224, 56, post=[], compute=[], write=U8X3, split=False))


def test_rational_ties_decided_by_double_rounding(cuda, oracle):
    """Scale 8 -> 7: fx = odd/14 is not a binary fraction, and columns alternating
    0 / 7 make 7 * fx an exact half-integer as a rational, so the reference's
    result hangs on the rounding of fx in double. Every pixel of these crops is
    flagged, so the per-band fix list also overflows into the whole-pair path."""
    row = np.where(np.arange(512) % 2 == 0, 0, 7).astype(np.uint8)
    frame = np.repeat(np.repeat(row[None, :, None], 3, axis=2), 200, axis=0)
    frame[:, :, 1] = 7 - frame[:, :, 1]
    frames = [np.ascontiguousarray(frame)]
    rects = [(0, 0, 448, 128), (1, 0, 64, 64), (3, 5, 256, 112)]
    for rect in rects:
        w, h = rect[2], rect[3]
        check(cuda, oracle, batch_spec(frames, [rect], w * 7 // 8, h * 7 // 8, post=[], compute=[], write=U8X3,
                                       split=False))
    check(cuda, oracle, batch_spec(frames, rects, 392, 112))


def test_gray_and_odd_widths(cuda, oracle):
    """Single-lane u8 sources, odd output widths (the last thread's second column
    is outside the plane) and unaligned source rows."""
    rng = np.random.default_rng(5)
    gray = rng.integers(0, 256, (130, 257), dtype=np.uint8)
    reads = [ReadSpec(0, 1, 2, 255, 101, 97, 61, BILINEAR), ReadSpec(0, 0, 0, 257, 130, 97, 61, BILINEAR)]
    spec = ChainSpec([gray], reads, [], U8, batch=True, active_read=2, active_write=2)
    check(cuda, oracle, spec)
    odd = rng.integers(0, 256, (99, 131, 3), dtype=np.uint8)   # row pitch 393: rows not 4-byte aligned
    check(cuda, oracle, batch_spec([odd], [(0, 0, 131, 99), (3, 1, 100, 90)], 101, 47))
