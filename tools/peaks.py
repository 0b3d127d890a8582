"""HBM peaks on this box (CUDA events, best of 10): copy (read+write bytes),
write-only (fill) and read-only (sum) over buffers far larger than L2."""
import json
import torch

def best(fn, reps=10):
    ts = []
    for _ in range(reps + 2):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts[2:])

n = 4 << 30
x = torch.empty(n, dtype=torch.uint8, device="cuda")
y = torch.empty(n, dtype=torch.uint8, device="cuda")
out = {}
out["write_gbs"] = n / best(lambda: x.fill_(3)) / 1e6
out["copy_gbs"] = 2 * n / best(lambda: y.copy_(x)) / 1e6
xf = x.view(torch.float32)
out["read_gbs"] = n / best(lambda: xf.sum()) / 1e6
w = torch.empty(4932501504 // 4, dtype=torch.float32, device="cuda")
out["write_c5_4.93GB_gbs"] = w.numel() * 4 / best(lambda: w.fill_(1.0)) / 1e6
print(json.dumps(out))
