"""Scratch timing of the first kernels (not the bench contract; see bench.py)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2508_07071_b200.opfuse import Library, Plane, ExecConfig, f32, f32x3
from paper_2508_07071_b200._ffi import *

lib = Library("cuda")
torch.cuda.set_device(0)
st = torch.cuda.current_stream()
cfg = ExecConfig(stream=st.cuda_stream)

def timeit(fn, n=20):
    for _ in range(3): fn()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n

# C1
rng = np.random.default_rng(42)
W, H = 3840, 2160
srcs = [lib.plane_from_numpy(rng.random((H, W), dtype=np.float32)) for _ in range(4)]
dsts = [lib.plane_alloc(W, H, U8) for _ in range(4)]
pipes = [lib.validate_chain([lib.op_read_per_thread(s), lib.op_mul(f32(400)), lib.op_add(f32(2)), lib.op_sub(f32(1.5)),
                             lib.op_div(f32(1.25)), lib.op_cast(F32, U8), lib.op_write_per_thread(d)]) for s, d in zip(srcs, dsts)]
i = [0]
def c1():
    lib.execute_fused(pipes[i[0] % 4], cfg); i[0] += 1
ms = timeit(c1, 40)
print(f"C1 fused: {ms*1e3:.1f} us  {W*H/ms/1e6:.0f} Mpx/s  {W*H*5/ms/1e6:.0f} GB/s")
def c1u():
    lib.execute_unfused(pipes[i[0] % 4], cfg); i[0] += 1
ms = timeit(c1u, 10)
print(f"C1 unfused: {ms*1e3:.1f} us  {W*H*39/ms/1e6:.0f} GB/s(traffic)")

# C3 N=1000
src = lib.plane_from_numpy(rng.random((4096, 4096), dtype=np.float32)); dst = lib.plane_alloc(4096, 4096, F32)
for N in (1, 16, 64, 1000):
    comp = []
    for op, c, k in ((lib.op_mul, 1.0000001, (N + 1)//2), (lib.op_add, 1e-7, N//2)):
        if k == 0: continue
        o = op(f32(c)); comp += [o]*k if k <= 64 else [lib.op_static_loop(o, k)]
    p = lib.validate_chain([lib.op_read_per_thread(src)] + comp + [lib.op_write_per_thread(dst)])
    ms = timeit(lambda: lib.execute_fused(p, cfg), 10)
    print(f"C3 N={N}: {ms*1e3:.1f} us  {4096*4096*8/ms/1e6:.0f} GB/s  {N*4096*4096/ms/1e9:.1f} Gop/s")

# C5-like: 8192 crops 224x224 from 16 frames
B = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
frames = [lib.plane_from_numpy(rng.integers(0, 256, (1080, 1920, 3), dtype=np.uint8)) for _ in range(16)]
out = torch.empty(B * 3 * 224 * 224 * 4, dtype=torch.uint8, device="cuda")
r = np.random.default_rng(7)
t0 = time.time()
reads, writes = [], []
for z in range(B):
    w, h = int(r.integers(112, 449)), int(r.integers(112, 449))
    x0, y0 = int(r.integers(0, 1921 - w)), int(r.integers(0, 1081 - h))
    rd = lib.op_resize(lib.op_crop(frames[z % 16], x0, y0, w, h), 224, 224, BILINEAR)
    rd = lib.fold_unary_into_read(rd, lib.op_cast(U8X3, F32X3))
    reads.append(rd)
    planes = [Plane(out, (z * 3 + l) * 224 * 224 * 4, 224, 224, 224, F32) for l in range(3)]
    writes.append(lib.op_split_write(planes))
p = lib.validate_chain([lib.op_batch_read(reads), lib.op_sub(f32x3(123.675, 116.28, 103.53)),
                        lib.op_div(f32x3(58.395, 57.12, 57.375)), lib.op_batch_write(writes)])
print(f"C5 build {time.time()-t0:.2f}s")
ms = timeit(lambda: lib.execute_fused(p, cfg), 10)
px = B * 224 * 224
print(f"C5 fused B={B}: {ms*1e3:.1f} us  {px/ms/1e6:.0f} Mpx/s  out {px*12/ms/1e6:.0f} GB/s")
