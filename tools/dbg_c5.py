"""Debug: a few C5-style crops through the CUDA library vs the oracle; per-plane mismatch maps."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from fkchains import run
from test_gpu_filter import batch_spec
from paper_2508_07071_b200._ffi import U8X3, F32X3
from paper_2508_07071_b200.opfuse import Library
cuda, oracle = Library("cuda"), Library("oracle")
rng = np.random.default_rng(42)
frames = [rng.integers(0, 256, (1080, 1920, 3), dtype=np.uint8) for _ in range(2)]
r = np.random.default_rng(7)
rects = []
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 4):
    w, h = int(r.integers(112, 449)), int(r.integers(112, 449))
    rects.append((int(r.integers(0, 1921 - w)), int(r.integers(0, 1081 - h)), w, h))
if os.environ.get("DBG_AFFINE"):
    spec = batch_spec(frames, rects, 224, 224, post=[("cast", U8X3, F32X3)])
else:
    spec = batch_spec(frames, rects, 224, 224, post=[], compute=[], write=U8X3, split=False)
a, _ = run(cuda, spec); b, _ = run(oracle, spec)
for z, (da, db) in enumerate(zip(a, b)):
    x, y = np.stack(da, -1) if len(da) > 1 else da[0], np.stack(db, -1) if len(db) > 1 else db[0]
    x, y = x.view(np.int32) if x.dtype == np.float32 else x.astype(int), y.view(np.int32) if y.dtype == np.float32 else y.astype(int)
    bad = np.argwhere(np.any(x != y, axis=-1) if x.ndim == 3 else x != y)
    print("z", z, rects[z], "shape", x.shape, "bad px", len(bad))
    if len(bad):
        cols = np.unique(bad[:, 1]); rows = np.unique(bad[:, 0])
        print("  bad cols", cols[:40], "... n", len(cols), " bad rows", rows[:20], "n", len(rows))
        i = tuple(bad[0]); print("  first", i, x[i], y[i])
