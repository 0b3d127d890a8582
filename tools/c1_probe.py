"""Probe: C1 kernel time vs size and vs a torch copy of the same bytes (events, no flush, rotated)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2508_07071_b200 import workloads as wl
from paper_2508_07071_b200.opfuse import Library, ExecConfig
lib = Library("cuda")
st = torch.cuda.current_stream()
cfg = ExecConfig(stream=st.cuda_stream)

def t(fn, n=40):
    for i in range(5): fn(i)
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); a.record()
    for i in range(n): fn(i)
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1000

for H in (2160, 4320, 8640):
    w = wl.c1(lib, H=H, sets=4)
    ps = [w.pipeline] + w.rotate
    us = t(lambda i: lib.execute_fused(ps[i % 4], cfg))
    print(f"C1 3840x{H}: {us:.1f} us  {w.alg_bytes/us/1e3:.0f} GB/s")
for mb in (33, 66, 132):
    xs = [torch.empty(mb * 2**20 // 4, device="cuda") for _ in range(4)]
    ys = [torch.empty(mb * 2**20 // 16, device="cuda") for _ in range(4)]
    us = t(lambda i: ys[i % 4].copy_(xs[i % 4][::4]))
    print(f"torch strided read {mb} MB -> {mb//4} MB: {us:.1f} us {(mb*1.25)*2**20/us/1e3:.0f} GB/s")
    us = t(lambda i: torch.sum(xs[i % 4]))
    print(f"torch sum {mb} MB: {us:.1f} us {mb*2**20/us/1e3:.0f} GB/s")
