"""PCIe copy ceilings on the box: contiguous vs interior-strided, one and both directions."""
import time

import torch

n = 128
dev = torch.device("cuda", 0)
pad = torch.zeros((n + 6,) * 4, dtype=torch.float64, device=dev)
inner = (slice(3, 3 + n),) * 4
hin = torch.empty((n,) * 4, dtype=torch.float64).pin_memory()
hout = torch.empty((n,) * 4, dtype=torch.float64).pin_memory()
dcont = torch.empty((n,) * 4, dtype=torch.float64, device=dev)
s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
GB = hin.numel() * 8 / 1e9


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps


for name, fn in [
    ("H2D contiguous", lambda: dcont.copy_(hin, non_blocking=True)),
    ("D2H contiguous", lambda: hout.copy_(dcont, non_blocking=True)),
    ("H2D into padded interior", lambda: pad[inner].copy_(hin, non_blocking=True)),
    ("D2H from padded interior", lambda: hout.copy_(pad[inner], non_blocking=True)),
]:
    t = timeit(fn)
    print(f"{name:28s} {GB / t:6.1f} GB/s")


def both():
    with torch.cuda.stream(s1):
        dcont.copy_(hin, non_blocking=True)
    with torch.cuda.stream(s2):
        hout.copy_(pad[inner], non_blocking=True)
    s1.synchronize()
    s2.synchronize()


t = timeit(both)
print(f"{'both directions concurrently':28s} {GB / t:6.1f} GB/s per direction")
