"""Host-link probe for the e2e pipeline (runner.HostPipeline) at 128^4.

Times, with CUDA events, 2 GiB of pinned host <-> device traffic:
  h2d / d2h alone and both at once on two streams, contiguous;
  the same into / out of the padded (134^4-style) device layout through
  torch's strided copy_ (what HostPipeline does) and through
  cudaMemcpy3DAsync-equivalent chunked copies of contiguous planes.
  python scripts/probes/pcie_bw.py
"""
import time

import torch

N, G = 128, 3
P = N + 2 * G
dev = torch.device("cuda:0")
nbytes = N ** 4 * 8


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        t = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    return best


h_in = torch.empty(N, N, N, N, dtype=torch.float64).pin_memory()
h_out = torch.empty_like(h_in).pin_memory()
h_in.fill_(1.0)
d_c = torch.empty(N, N, N, N, dtype=torch.float64, device=dev)
d_c2 = torch.empty_like(d_c)
d_p = torch.zeros(P, P, P, P, dtype=torch.float64, device=dev)
d_p2 = torch.zeros_like(d_p)
sl = (slice(G, G + N),) * 4
s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)


def gbs(t):
    return nbytes / t / 1e9


def both(fa, fb):
    def run():
        with torch.cuda.stream(s1):
            fa()
        with torch.cuda.stream(s2):
            fb()
        s1.synchronize()
        s2.synchronize()
    return run


t = timed(lambda: d_c.copy_(h_in, non_blocking=True))
print(f"h2d contiguous            {gbs(t):6.1f} GB/s")
t = timed(lambda: h_out.copy_(d_c, non_blocking=True))
print(f"d2h contiguous            {gbs(t):6.1f} GB/s")
t = timed(both(lambda: d_c.copy_(h_in, non_blocking=True), lambda: h_out.copy_(d_c2, non_blocking=True)))
print(f"h2d+d2h contiguous        {gbs(t):6.1f} GB/s each way")
t = timed(lambda: d_p[sl].copy_(h_in, non_blocking=True))
print(f"h2d strided copy_         {gbs(t):6.1f} GB/s")
t = timed(lambda: h_out.copy_(d_p[sl], non_blocking=True))
print(f"d2h strided copy_         {gbs(t):6.1f} GB/s")
t = timed(both(lambda: d_p[sl].copy_(h_in, non_blocking=True), lambda: h_out.copy_(d_p2[sl], non_blocking=True)))
print(f"h2d+d2h strided copy_     {gbs(t):6.1f} GB/s each way")


# staged: contiguous DMA into a device staging buffer, then a device-side
# scatter into the padded layout (one strided copy kernel), chunked by x planes
def staged_h2d(chunks=8):
    step = N // chunks
    for c in range(chunks):
        a, b = c * step, (c + 1) * step
        d_c[a:b].copy_(h_in[a:b], non_blocking=True)
        d_p[G + a:G + b, G:G + N, G:G + N, G:G + N].copy_(d_c[a:b], non_blocking=True)


def staged_d2h(chunks=8):
    step = N // chunks
    for c in range(chunks):
        a, b = c * step, (c + 1) * step
        d_c2[a:b].copy_(d_p2[G + a:G + b, G:G + N, G:G + N, G:G + N], non_blocking=True)
        h_out[a:b].copy_(d_c2[a:b], non_blocking=True)


for ch in (1, 8, 32):
    t = timed(lambda: staged_h2d(ch))
    print(f"h2d staged x{ch:<3d}           {gbs(t):6.1f} GB/s")
    t = timed(lambda: staged_d2h(ch))
    print(f"d2h staged x{ch:<3d}           {gbs(t):6.1f} GB/s")
    t = timed(both(lambda: staged_h2d(ch), lambda: staged_d2h(ch)))
    print(f"h2d+d2h staged x{ch:<3d}       {gbs(t):6.1f} GB/s each way")
