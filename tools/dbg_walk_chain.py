"""Which chain op makes fk_walk differ from the oracle (debug helper)."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests")); sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
from fkchains import run, outputs_equal
from test_gpu_walk import spec_of, random_rects
from paper_2508_07071_b200._ffi import F32X3, OP_DIV, OP_MUL, OP_SUB
from paper_2508_07071_b200.opfuse import Library
cuda, oracle = Library("cuda"), Library("oracle")
rng = np.random.default_rng(8)
frames = [rng.integers(0, 256, (160, 256, 3), dtype=np.uint8)]
rects = random_rects(rng, 5, 30, 160, 256, 160)
M = ("arith", OP_MUL, F32X3, (1.0 / 255,) * 3); S = ("arith", OP_SUB, F32X3, (0.485, 0.456, 0.406)); D = ("arith", OP_DIV, F32X3, (0.229, 0.224, 0.225))
for name, comp in [("M", [M]), ("S", [S]), ("D", [D]), ("MS", [M, S]), ("SD", [S, D]), ("MD", [M, D]), ("MSD", [M, S, D])]:
    for swap in (False, True):
        spec = spec_of(frames, rects, 128, 64, swap=swap, compute=comp)
        got, _ = run(cuda, spec); k = cuda.last_kernel()
        want, _ = run(oracle, spec)
        n = sum(int((np.asarray(a).view(np.uint32) != np.asarray(b).view(np.uint32)).sum()) for ga, wa in zip(got, want) for a, b in zip(ga, wa))
        print(name, "swap" if swap else "    ", k, "mismatches", n)
