"""The BASELINE.json configurations as pipelines on any backend.

C1  vertical fusion: 3840x2160 f32 -> Mul, Add, Sub, Div, Cast(u8) -> u8          (configs[0])
C2  cvGS preprocessing: 50 crops of a 1920x1080 u8x3 frame -> bilinear 64x128 ->
    SwapRB -> f32x3 -> sub mean / div std -> split to 3 planar f32              (configs[1])
C3  long vertical chain: N chained ops on 4096x4096 f32 (StaticLoop above 64)     (configs[2])
C4  horizontal fusion: B crops 224x224x3, per-crop resize + per-crop normalize     (configs[3])
C5  batch-sharded preprocessing: 8192 crops 224x224x3 resize+normalize+split      (configs[4])

Inputs are synthetic and seeded (numpy default_rng). Parameters follow
SURVEY.md §8(d). Every builder returns a Workload with the validated pipeline,
its planes, and the algorithmic byte count the roofline uses.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from ._ffi import BILINEAR, F32, F32X3, SWAP_RB, U8, U8X3
from .opfuse import Library, Plane, f32, f32x3

MEAN = (123.675, 116.28, 103.53)   # ImageNet mean x 255
STD = (58.395, 57.12, 57.375)      # ImageNet std x 255


@dataclass
class Workload:
    name: str
    pipeline: object
    points: int                  # output pixels per execute
    alg_bytes: int               # minimal input + output footprint per execute
    out_bytes: int
    in_bytes: int
    sources: list = field(default_factory=list)   # Planes read (for e2e H2D)
    outputs: list = field(default_factory=list)   # torch storages written (for e2e D2H)
    keep: list = field(default_factory=list)
    info: dict = field(default_factory=dict)
    rotate: list = field(default_factory=list)    # extra identical pipelines on their own planes
                                                  # (timed steps cycle through them: sets > L2)


def _touched_bilinear(lo: int, n: int, out: int) -> np.ndarray:
    """Source indices (relative) the bilinear taps touch along one axis (ops.cpp:259-270)."""
    i = np.arange(out, dtype=np.float64)
    c = (i + 0.5) * n / out - 0.5
    f = np.floor(c).astype(np.int64)
    return np.unique(np.concatenate([np.clip(f, 0, n - 1), np.clip(f + 1, 0, n - 1)])) + lo


def crop_rects(n: int, rng: np.random.Generator, lo: int, hi: int, fw: int = 1920, fh: int = 1080):
    rects = []
    for _ in range(n):
        w, h = int(rng.integers(lo, hi + 1)), int(rng.integers(lo, hi + 1))
        x0, y0 = int(rng.integers(0, fw - w + 1)), int(rng.integers(0, fh - h + 1))
        rects.append((x0, y0, w, h))
    return rects


def unique_input_bytes(rects, frame_of, out_w, out_h, n_frames, fw=1920, fh=1080, bpe=3):
    masks = np.zeros((n_frames, fh, fw), dtype=bool)
    for z, (x0, y0, w, h) in enumerate(rects):
        ys = _touched_bilinear(y0, h, out_h) if h != out_h or w != out_w else np.arange(y0, y0 + h)
        xs = _touched_bilinear(x0, w, out_w) if h != out_h or w != out_w else np.arange(x0, x0 + w)
        masks[frame_of(z)][np.ix_(ys, xs)] = True
    return int(masks.sum()) * bpe


def c1(lib: Library, seed: int = 42, W: int = 3840, H: int = 2160, sets: int = 1) -> Workload:
    """configs[0]; `sets` > 1 adds copies on their own planes (4 sets = 166 MB > L2)."""
    rng = np.random.default_rng(seed)
    pipes, keep = [], []
    for _ in range(sets):
        src = lib.plane_from_numpy(rng.random((H, W), dtype=np.float32))
        dst = lib.plane_alloc(W, H, U8)
        pipes.append((lib.validate_chain([lib.op_read_per_thread(src), lib.op_mul(f32(400.0)), lib.op_add(f32(2.0)),
                                          lib.op_sub(f32(1.5)), lib.op_div(f32(1.25)), lib.op_cast(F32, U8),
                                          lib.op_write_per_thread(dst)]), src, dst))
        keep += [src, dst]
    p, src, dst = pipes[0]
    return Workload("C1", p, W * H, W * H * 5, W * H, W * H * 4, [src], [dst.storage], keep,
                    {"shape": f"{W}x{H}", "chain": "read f32 -> mul,add,sub,div -> cast u8 -> write"},
                    [q for q, _, _ in pipes[1:]])


def c3(lib: Library, n_ops: int, seed: int = 42, W: int = 4096, H: int = 4096, sets: int = 1) -> Workload:
    """configs[2]; `sets` > 1 adds copies on their own planes (2 sets = 268 MB > L2)."""
    rng = np.random.default_rng(seed)
    pipes, keep = [], []
    for _ in range(sets):
        src = lib.plane_from_numpy(rng.random((H, W), dtype=np.float32))
        dst = lib.plane_alloc(W, H, F32)
        chain = [lib.op_read_per_thread(src)]
        for op, c, k in ((lib.op_mul, 1.0000001, (n_ops + 1) // 2), (lib.op_add, 1e-7, n_ops // 2)):
            if k:  # bench.cpp:100-108: literal ops up to 64, a StaticLoop beyond
                o = op(f32(c))
                chain += [o] * k if k <= 64 else [lib.op_static_loop(o, k)]
        chain.append(lib.op_write_per_thread(dst))
        pipes.append((lib.validate_chain(chain), src, dst))
        keep += [src, dst]
    p, src, dst = pipes[0]
    return Workload(f"C3[N={n_ops}]", p, W * H, W * H * 8, W * H * 4, W * H * 4, [src], [dst.storage], keep,
                    {"shape": f"{W}x{H}", "n_ops": n_ops}, [q for q, _, _ in pipes[1:]])


def crops_pipeline(lib: Library, frames: list, rects: list, frame_of, out_w: int, out_h: int,
                   swap_rb: bool, means=None, stds=None, out_storage=None) -> tuple:
    """Batch of crop -> bilinear resize -> [SwapRB] -> cast f32x3 -> sub -> div -> split.

    means/stds: one (r,g,b) triple shared by all crops, or a list per crop (BatchArith)."""
    import torch
    B = len(rects)
    plane_bytes = out_w * out_h * 4
    if out_storage is None:
        out_storage = torch.empty(B * 3 * plane_bytes, dtype=torch.uint8, device=lib.device)
    reads, writes = [], []
    for z, (x0, y0, w, h) in enumerate(rects):
        r = lib.op_resize(lib.op_crop(frames[frame_of(z)], x0, y0, w, h), out_w, out_h, BILINEAR)
        if swap_rb:
            r = lib.fold_unary_into_read(r, lib.op_color_convert(SWAP_RB, U8X3))
        reads.append(lib.fold_unary_into_read(r, lib.op_cast(U8X3, F32X3)))
        planes = [Plane(out_storage, (3 * z + l) * plane_bytes, out_w, out_h, out_w, F32) for l in range(3)]
        writes.append(lib.op_split_write(planes))
    means = means or MEAN
    stds = stds or STD
    if isinstance(means[0], (tuple, list)):
        sub = lib.op_batch_arith(9, [f32x3(*m) for m in means])     # OP_SUB
        div = lib.op_batch_arith(10, [f32x3(*s) for s in stds])     # OP_DIV
    else:
        sub, div = lib.op_sub(f32x3(*means)), lib.op_div(f32x3(*stds))
    p = lib.validate_chain([lib.op_batch_read(reads), sub, div, lib.op_batch_write(writes)])
    return p, out_storage


def c2(lib: Library, seed: int = 42) -> Workload:
    rng = np.random.default_rng(seed)
    frame = lib.plane_from_numpy(rng.integers(0, 256, (1080, 1920, 3), dtype=np.uint8))
    r7 = np.random.default_rng(7)
    rects = []
    for _ in range(50):  # w = 64 + r%448, h = 128 + r%448
        w, h = 64 + int(r7.integers(0, 448)), 128 + int(r7.integers(0, 448))
        rects.append((int(r7.integers(0, 1921 - w)), int(r7.integers(0, 1081 - h)), w, h))
    p, out = crops_pipeline(lib, [frame], rects, lambda z: 0, 64, 128, swap_rb=True)
    out_b = 50 * 64 * 128 * 12
    in_b = unique_input_bytes(rects, lambda z: 0, 64, 128, 1)
    return Workload("C2", p, 50 * 64 * 128, out_b + in_b, out_b, in_b, [frame], [out], [frame, out],
                    {"crops": 50, "out": "64x128", "chain": "crop->resize->SwapRB->f32->sub->div->split"})


def c4_reference_planes(lib: Library, n: int, seed: int = 42, n_frames: int = 16) -> list:
    """C4's crops as n single-plane pipelines, each with its own normalize
    constants: the reference cannot express per-plane constants in one batch,
    so its C4 is one pipeline per crop (the bench.cpp:199-202 pattern). Same
    frames, rects and constants as crops_224(..., per_crop_norm=True)."""
    rng = np.random.default_rng(seed)
    frames = [lib.plane_from_numpy(rng.integers(0, 256, (1080, 1920, 3), dtype=np.uint8))
              for _ in range(n_frames)]
    rects = crop_rects(n, np.random.default_rng(7), 112, 448)
    jr = np.random.default_rng(11)
    means = [tuple(float(np.float32(m + jr.normal(0, 2.0))) for m in MEAN) for _ in range(n)]
    stds = [tuple(float(np.float32(s + jr.normal(0, 1.0))) for s in STD) for _ in range(n)]
    out = []
    for z in range(n):
        p, o = crops_pipeline(lib, frames, [rects[z]], lambda _z, z=z: z % n_frames, 224, 224, swap_rb=False,
                              means=means[z], stds=stds[z])
        out.append((p, o))
    return out, frames


def crops_224(lib: Library, n: int, per_crop_norm: bool, seed: int = 42, n_frames: int = 16,
              name: str = "C5", first: int = 0) -> Workload:
    """C4/C5: crops of 16 frames (crop z from frame z % 16), w,h in [112, 448] -> 224x224."""
    rng = np.random.default_rng(seed)
    frames = [lib.plane_from_numpy(rng.integers(0, 256, (1080, 1920, 3), dtype=np.uint8))
              for _ in range(n_frames)]
    all_rects = crop_rects(first + n, np.random.default_rng(7), 112, 448)
    rects = all_rects[first:first + n]
    frame_of = lambda z: (first + z) % n_frames  # noqa: E731
    means = stds = None
    if per_crop_norm:
        jr = np.random.default_rng(11)
        means = [tuple(float(np.float32(m + jr.normal(0, 2.0))) for m in MEAN) for _ in range(first + n)][first:]
        stds = [tuple(float(np.float32(s + jr.normal(0, 1.0))) for s in STD) for _ in range(first + n)][first:]
    p, out = crops_pipeline(lib, frames, rects, frame_of, 224, 224, swap_rb=False, means=means, stds=stds)
    out_b = n * 224 * 224 * 12
    in_b = unique_input_bytes(rects, frame_of, 224, 224, n_frames)
    return Workload(name, p, n * 224 * 224, out_b + in_b, out_b, in_b, frames, [out], frames + [out],
                    {"crops": n, "out": "224x224x3 f32 planar", "frames": f"{n_frames}x1920x1080 u8x3",
                     "per_crop_normalize": per_crop_norm, "rects": rects})
