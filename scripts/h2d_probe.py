"""Does a pinned H2D copy overlap with kernels on this box?  Times (a) the host
cost of issuing copy_(non_blocking), (b) a compute loop alone, (c) the same
loop with the copy issued on a side stream."""
import time
import torch

x = torch.empty((3072, 32768), dtype=torch.float64).pin_memory()
print("pinned:", x.is_pinned())
d = torch.empty_like(x, device="cuda")
a = torch.randn(8192, 8192, device="cuda")
side = torch.cuda.Stream()


def work(n=60):
    for _ in range(n):
        torch.mm(a, a)


work(5)
torch.cuda.synchronize()
t = time.perf_counter()
d.copy_(x, non_blocking=True)
t_issue = time.perf_counter() - t
torch.cuda.synchronize()
t_copy = time.perf_counter() - t
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); work(); e1.record(); torch.cuda.synchronize()
alone = e0.elapsed_time(e1)
e0.record()
with torch.cuda.stream(side):
    t = time.perf_counter()
    d.copy_(x, non_blocking=True)
    t_issue2 = time.perf_counter() - t
work()
e1.record(); torch.cuda.synchronize()
both = e0.elapsed_time(e1)
print(f"copy issue {t_issue*1e3:.2f} ms, copy total {t_copy*1e3:.2f} ms; work alone {alone:.1f} ms, "
      f"work + concurrent copy {both:.1f} ms (issue {t_issue2*1e3:.2f} ms)")
