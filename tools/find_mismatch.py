"""Print the first random chain on which the CUDA library and the oracle disagree."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from fkchains import random_chain, run, outputs_equal, mismatch_report
from paper_2508_07071_b200.opfuse import Library
cuda, oracle = Library("cuda"), Library("oracle")
seeds = [int(a) for a in sys.argv[1:]] or [1000]
for seed in seeds:
    rng = np.random.default_rng(seed)
    for i in range(60):
        spec = random_chain(rng, allow_batch_arith=True)
        a, _ = run(cuda, spec); b, _ = run(oracle, spec)
        if not outputs_equal(a, b):
            print("seed", seed, "chain", i)
            print(" reads", spec.reads[:2], "n", len(spec.reads), "src", [s.shape + (s.dtype,) for s in spec.sources[:2]])
            print(" compute", spec.compute, "write", spec.write_kind, "split", spec.split, "batch", spec.batch,
                  spec.active_read, spec.active_write, spec.default, "pad", spec.dst_stride_pad)
            print(" ", mismatch_report(a, b)[:2000])
            break
