"""Generate tests/golden/golden.npz + golden.json from the UNMODIFIED reference.

Run in the build container (needs oracle/_ref/libfk_ref.so, compiled from
/root/reference by oracle/Makefile):   python tests/golden/make_golden.py

Each case is a chain description (JSON), its seeded inputs and the reference's
outputs and ExecReport counters (npz). tests/test_oracle.py checks the C oracle
against them on CPU; tests/test_gpu_parity.py checks the CUDA library against
them on the GPU. Nothing reads /root/reference at test time.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from fkchains import ChainSpec, ReadSpec, random_chain, run, spec_to_dict  # noqa: E402
from paper_2508_07071_b200._ffi import (BILINEAR, F32, F32X3, NEAREST, OP_ADD, OP_DIV, OP_MUL, OP_SUB,  # noqa: E402
                                        U8, U8X3)
from paper_2508_07071_b200.opfuse import Library  # noqa: E402


def named_cases():
    rng = np.random.default_rng(42)
    cases = []
    # configs[0] shape at a small size: Read f32 -> Mul, Add, Sub, Div -> Cast u8 (SURVEY §8(d) constants)
    src = rng.random((48, 80), dtype=np.float32)
    src.reshape(-1)[:8] = np.array([0.0, 0.00125, 0.63375, 0.635, 0.6362, np.nan, -1.0, 1.0], np.float32)
    cases.append(("c1_vertical", ChainSpec([src], [ReadSpec(0)],
                  [("arith", OP_MUL, F32, (400.0,)), ("arith", OP_ADD, F32, (2.0,)), ("arith", OP_SUB, F32, (1.5,)),
                   ("arith", OP_DIV, F32, (1.25,)), ("cast", F32, U8)], U8)))
    # configs[1] shape: crops of a u8x3 frame -> bilinear 64x128 -> SwapRB -> f32 -> normalise -> split
    frame = rng.integers(0, 256, (270, 480, 3), dtype=np.uint8)
    r7 = np.random.default_rng(7)
    reads = []
    for _ in range(6):
        w, h = 16 + int(r7.integers(0, 200)), 32 + int(r7.integers(0, 200))
        reads.append(ReadSpec(0, int(r7.integers(0, 481 - w)), int(r7.integers(0, 271 - h)), w, h, 64, 128, BILINEAR,
                              [("swap", U8X3), ("cast", U8X3, F32X3)]))
    cases.append(("c2_cvgs", ChainSpec([frame], reads, [("arith", OP_SUB, F32X3, (123.675, 116.28, 103.53)),
                                                        ("arith", OP_DIV, F32X3, (58.395, 57.12, 57.375))],
                                       F32X3, split=True, batch=True, active_read=6, active_write=6)))
    # configs[2] shape: StaticLoop chains (bench.cpp:319-330 constants)
    src3 = rng.random((32, 64), dtype=np.float32)
    cases.append(("c3_static_loop", ChainSpec([src3], [ReadSpec(0)],
                  [("loop", ("arith", OP_MUL, F32, (float(np.float32(1.0000001)),)), 500),
                   ("loop", ("arith", OP_ADD, F32, (float(np.float32(1e-7)),)), 500)], F32)))
    # nearest resize, u8 wrap arithmetic, batch default values and inactive writes
    g = rng.integers(0, 256, (40, 50), dtype=np.uint8)
    cases.append(("nearest_u8_wrap", ChainSpec([g, g], [ReadSpec(0, 3, 4, 30, 20, 47, 33, NEAREST),
                                                        ReadSpec(1, 0, 0, 50, 40, 47, 33, NEAREST)],
                                               [("arith", OP_MUL, U8, (37,)), ("arith", OP_ADD, U8, (200,)),
                                                ("arith", OP_DIV, U8, (3,))], U8, batch=True, active_read=1,
                                               active_write=2, default=(9,))))
    # gray conversion and f64 paths
    f = rng.random((20, 30, 3)) * 255
    cases.append(("togray_f64", ChainSpec([f], [ReadSpec(0, 1, 1, 25, 15, 40, 10, BILINEAR, [("gray", 5)])],
                                          [("cast", F32, 2), ("arith", OP_MUL, 2, (1.5,))], 2)))
    return cases


def main():
    ref = Library("reference")
    cases = named_cases()
    rng = np.random.default_rng(20250811)
    for i in range(40):
        cases.append((f"random_{i:02d}", random_chain(rng)))
    manifest, arrays = [], {}
    for name, spec in cases:
        outs, rep = run(ref, spec)
        _, urep = run(ref, spec, unfused=True)
        for j, s in enumerate(spec.sources):
            arrays[f"{name}/src{j}"] = s
        for z, ds in enumerate(outs):
            for l, a in enumerate(ds):
                arrays[f"{name}/out{z}_{l}"] = a
        manifest.append({"name": name, "spec": spec_to_dict(spec), "n_out": [len(d) for d in outs],
                         "fused": [rep.bytes_read, rep.bytes_written, rep.passes, rep.points_visited],
                         "unfused": [urep.bytes_read, urep.bytes_written, urep.passes, urep.points_visited,
                                     urep.intermediate_bytes_allocated]})
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py", "backend": ref.name, "cases": manifest}, f, indent=1)
    print(f"{len(cases)} cases, {sum(a.nbytes for a in arrays.values())} bytes of arrays")


if __name__ == "__main__":
    main()
