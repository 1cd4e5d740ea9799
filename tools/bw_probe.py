"""HBM bandwidth probe: write-only (fill_), read-only (sum), copy, on 4 GiB buffers (CUDA events)."""
import torch

n = 1 << 30  # floats = 4 GiB
a = torch.empty(n, device="cuda")
b = torch.empty(n, device="cuda")
a.fill_(1.0)
torch.cuda.synchronize()


def t(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    return best / 1e3


tw = t(lambda: b.fill_(2.0))
tr = t(lambda: a.sum())
tc = t(lambda: b.copy_(a))
print(f"write-only {4 * n / tw / 1e12:.2f} TB/s, read-only {4 * n / tr / 1e12:.2f} TB/s, copy (r+w) {8 * n / tc / 1e12:.2f} TB/s")
