"""Debug: first random reduce case where CUDA and the oracle disagree; isolate the spec."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from fkchains import random_chain, make_read
from test_reduce import random_specs, close, reduce_on
from paper_2508_07071_b200.opfuse import Library
cuda, oracle = Library("cuda"), Library("oracle")
seed = 0
rng = np.random.default_rng(700 + seed)
for i in range(40):
    spec = random_chain(rng, max_dim=40, max_batch=5)
    a, ra, kinds = reduce_on(cuda, spec, 7000 + 100 * seed + i, 0)
    b, rb, _ = reduce_on(oracle, spec, 7000 + 100 * seed + i, 1)
    for j, (x, y, (c, k)) in enumerate(zip(a, b, kinds)):
        try:
            close(x, y, c, k)
        except AssertionError:
            print("case", i, "spec", j, "combine", c, "kind", k, x, y)
            print(" reads", spec.reads[:2], len(spec.reads), "batch", spec.batch, spec.active_read, "src", spec.sources[0].shape, spec.sources[0].dtype)
            r2 = np.random.default_rng(7000 + 100 * seed + i)
            for lib in (cuda, oracle):
                rd, _ = make_read(lib, spec)
                specs = random_specs(np.random.default_rng(7000 + 100 * seed + i), lib, rd, spec)
                print(" ", lib.name, "specs", [(s[0], s[1].name if s[1] else None, s[2]) for s in specs])
                print(" ", lib.name, "single", lib.multi_reduce_plane(rd, [specs[j]], 1)[0])
            sys.exit(0)
print("no mismatch")
