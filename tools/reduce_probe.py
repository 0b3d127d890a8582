"""ReduceDPP probe: Sum/Max/Min in one traversal over large planes (run under ncu for kernel times)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2508_07071_b200.opfuse import Library
from paper_2508_07071_b200._ffi import REDUCE_SUM, REDUCE_MAX, REDUCE_MIN
lib = Library("cuda")
rng = np.random.default_rng(0)
for shape, dt in (((2160, 3840), np.float32), ((8192, 8192), np.float32), ((1080, 1920, 3), np.uint8), ((8192, 8192), np.uint8), ((4320, 7680, 3), np.uint8)):
    a = (rng.random(shape, dtype=np.float32) if dt == np.float32 else rng.integers(0, 256, shape, dtype=np.uint8))
    r = lib.op_read_per_thread(lib.plane_from_numpy(a))
    which = os.environ.get("SPECS", "sum,max,min").split(",")
    specs = [({"sum": REDUCE_SUM, "max": REDUCE_MAX, "min": REDUCE_MIN}[w], None, None) for w in which]
    for _ in range(3):
        res, n = lib.multi_reduce_plane(r, specs)
    t = time.time()
    for _ in range(10):
        res, n = lib.multi_reduce_plane(r, specs)
    dt_ms = (time.time() - t) / 10 * 1e3
    print(shape, a.dtype, f"{a.nbytes/1e6:.0f} MB", f"host-timed {dt_ms:.2f} ms per call (incl. program build + sync)", res[1:])
