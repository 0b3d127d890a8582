"""The column-walk crop kernel (csrc/fk_walk.cu) against the C oracle, bit for bit.

fk_walk runs every bilinear u8x3 crop batch with an AFFINE chain and a split f32
write whose frames have 16-byte aligned rows (the cvGS / configs[1], [3], [4]
family). These cases aim at its own structure: 64-column strips and the paired
half strips (two planes of equal crop height in one warp), the row bands, the
TMA-staged spans at the frame's right and bottom edges (the last row's copy is
cut to the readable bytes), clamped taps, upscales where one source row
completes several output rows, the exact-result filter (dyadic rows/columns
with exact ties, and rational ties that only the reference's double rounding
decides, which go through the fix queue), per-crop constants and lane swaps.
Every case asserts that fk_walk really ran.
"""
import numpy as np
import pytest

from fkchains import ChainSpec, ReadSpec, mismatch_report, outputs_equal, run
from paper_2508_07071_b200._ffi import BILINEAR, F32X3, OP_DIV, OP_MUL, OP_SUB, U8X3

pytestmark = pytest.mark.gpu

NORM = [("arith", OP_SUB, F32X3, (123.675, 116.28, 103.53)), ("arith", OP_DIV, F32X3, (58.395, 57.12, 57.375))]


def spec_of(frames, rects, out_w, out_h, swap=True, compute=NORM, frame_of=None):
    post = ([("swap", U8X3)] if swap else []) + [("cast", U8X3, F32X3)]
    frame_of = frame_of or (lambda i: i % len(frames))
    reads = [ReadSpec(frame_of(i), x, y, w, h, out_w, out_h, BILINEAR, list(post))
             for i, (x, y, w, h) in enumerate(rects)]
    return ChainSpec(frames, reads, compute, F32X3, split=True, batch=True,
                     active_read=len(reads), active_write=len(reads))


def check_walk(cuda, oracle, spec):
    got, rep = run(cuda, spec)
    assert cuda.last_kernel() == "fk_walk", cuda.last_kernel()
    want, _ = run(oracle, spec)
    assert outputs_equal(got, want), mismatch_report(got, want)
    return rep


def random_rects(rng, n, lo, hi, fw, fh):
    out = []
    for _ in range(n):
        w, h = int(rng.integers(lo, hi + 1)), int(rng.integers(lo, hi + 1))
        out.append((int(rng.integers(0, fw - w + 1)), int(rng.integers(0, fh - h + 1)), w, h))
    return out


@pytest.mark.parametrize("out_w,out_h", [(224, 224), (64, 128), (96, 40), (160, 33), (130, 17), (2, 5)])
def test_strip_shapes(cuda, oracle, out_w, out_h):
    """Full 64-column strips, half strips paired across planes (96, 160, 224:
    16 lanes), a 1-lane remainder (130) and a 2-column plane; odd crop counts
    leave one half strip unpaired."""
    rng = np.random.default_rng(out_w * 1000 + out_h)
    frames = [rng.integers(0, 256, (300, 512, 3), dtype=np.uint8) for _ in range(3)]
    rects = random_rects(rng, 13, 8, 300, 512, 300)
    rects += [(0, 0, 512, 300), (511, 299, 1, 1)]   # the whole frame; a 1x1 crop at the corner
    check_walk(cuda, oracle, spec_of(frames, rects, out_w, out_h))


def test_equal_heights_pair(cuda, oracle):
    """Many crops of one height (every half strip paired) at different x0/y0/widths."""
    rng = np.random.default_rng(3)
    frames = [rng.integers(0, 256, (400, 1024, 3), dtype=np.uint8)]
    rects = [(int(rng.integers(0, 500)), int(rng.integers(0, 100)), int(rng.integers(50, 500)), 300)
             for _ in range(10)]
    check_walk(cuda, oracle, spec_of(frames, rects, 224, 96))


def test_frame_edges_last_row(cuda, oracle):
    """Crops whose last source row is the frame's last row and whose span ends
    at the frame's last byte: the staged copy of that row is cut to the bytes
    that exist (the frame is its own allocation)."""
    rng = np.random.default_rng(9)
    frames = [rng.integers(0, 256, (120, 320, 3), dtype=np.uint8)]
    rects = [(320 - 77, 120 - 51, 77, 51), (0, 120 - 120, 320, 120), (319, 0, 1, 120), (200, 119, 120, 1),
             (250, 60, 70, 60)]
    check_walk(cuda, oracle, spec_of(frames, rects, 224, 64))


@pytest.mark.parametrize("levels", [2, 16, 256])
def test_exact_scales_ties(cuda, oracle, levels):
    """Dyadic fractions (448 -> 224, 336, 280, 2x / 4x upscales, rect % 7 == 0):
    FP32 is exact there, ties are real and must round to even like nearbyint."""
    rng = np.random.default_rng(levels)
    frames = [rng.integers(0, levels, (480, 512, 3), dtype=np.uint8)]
    rects = [(0, 0, 448, 448), (16, 8, 336, 280), (5, 3, 280, 112), (7, 9, 112, 56), (1, 1, 56, 224),
             (2, 0, 224, 224), (3, 3, 448, 112), (64, 64, 49, 70), (0, 31, 217, 203)]
    check_walk(cuda, oracle, spec_of(frames, rects, 224, 224))


def test_rational_ties_fix_queue(cuda, oracle):
    """Scale 8 -> 7 with taps alternating 0 / 7: the exact lerp is a half-integer
    as a rational, the reference's double rounding decides, and every such value
    goes through the fix queue (a whole 32-row band of flagged lanes)."""
    row = np.where(np.arange(512) % 2 == 0, 0, 7).astype(np.uint8)
    frame = np.repeat(np.repeat(row[None, :, None], 3, axis=2), 256, axis=0)
    frame[:, :, 1] = 7 - frame[:, :, 1]
    frame[::2, :, 2] = 7 - frame[::2, :, 2]
    frames = [np.ascontiguousarray(frame)]
    check_walk(cuda, oracle, spec_of(frames, [(0, 0, 448, 128), (1, 0, 64, 64), (3, 5, 256, 112)], 392, 112,
                                     swap=False, compute=[]))
    check_walk(cuda, oracle, spec_of(frames, [(0, 0, 256, 256), (8, 8, 128, 240)], 224, 210))


def test_per_crop_constants_and_mixed_swaps(cuda, oracle):
    """BatchArith (per-crop mean/std) and a batch mixing swapped and plain crops
    (per-plane constants, swap folded into the output pointers)."""
    rng = np.random.default_rng(21)
    frames = [rng.integers(0, 256, (200, 384, 3), dtype=np.uint8) for _ in range(2)]
    rects = random_rects(rng, 9, 20, 200, 384, 200)
    means = [tuple(float(np.float32(m + rng.normal(0, 3))) for m in (123.675, 116.28, 103.53)) for _ in rects]
    stds = [tuple(float(np.float32(s + rng.normal(0, 2))) for s in (58.395, 57.12, 57.375)) for _ in rects]
    compute = [("batch_arith", OP_SUB, F32X3, means), ("batch_arith", OP_DIV, F32X3, stds)]
    check_walk(cuda, oracle, spec_of(frames, rects, 224, 100, compute=compute))
    spec = spec_of(frames, rects, 224, 100)
    for i in range(0, len(spec.reads), 2):
        spec.reads[i].post = [("cast", U8X3, F32X3)]   # no swap on every other crop
    check_walk(cuda, oracle, spec)


def test_other_chains(cuda, oracle):
    """Other registered AFFINE chains: none, one multiply, mul-sub-div."""
    rng = np.random.default_rng(8)
    frames = [rng.integers(0, 256, (160, 256, 3), dtype=np.uint8)]
    rects = random_rects(rng, 5, 30, 160, 256, 160)
    for compute in ([], [("arith", OP_MUL, F32X3, (0.5, 2.0, 1.0 / 255))],
                    [("arith", OP_MUL, F32X3, (1.0 / 255,) * 3), ("arith", OP_SUB, F32X3, (0.485, 0.456, 0.406)),
                     ("arith", OP_DIV, F32X3, (0.229, 0.224, 0.225))]):
        check_walk(cuda, oracle, spec_of(frames, rects, 128, 64, compute=compute))
