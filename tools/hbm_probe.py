"""HBM bandwidth for pure writes, pure reads and copies (CUDA events, 4 GiB buffers)."""
import torch

n = 1 << 31  # 2^31 bf16 = 4 GiB
a = torch.empty(n, dtype=torch.bfloat16, device="cuda")
b = torch.empty(n, dtype=torch.bfloat16, device="cuda")
a.fill_(1.0)
b.fill_(2.0)
out = torch.empty(1, dtype=torch.float32, device="cuda")


def t(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e))
    return best


B = n * 2
w = t(lambda: a.fill_(3.0))
r = t(lambda: torch.sum(a.view(-1, 4096), dim=(0,), dtype=torch.float32))
c = t(lambda: b.copy_(a))
print(f"write {B / w / 1e6:.0f} GB/s  read {B / r / 1e6:.0f} GB/s  copy {2 * B / c / 1e6:.0f} GB/s (read+write)")
