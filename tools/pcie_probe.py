"""Host<->device copy bandwidth from pinned memory: H2D alone, D2H alone,
both directions concurrently (for the e2e figure)."""
import torch

n = 2 * 4198401  # one 2048^2 state (fp64)
h = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(2)]
d = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(2)]
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def h2d():
    with torch.cuda.stream(s1):
        d[0].copy_(h[0], non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h[1].copy_(d[1], non_blocking=True)


def both():
    h2d()
    d2h()


B = n * 8
for name, fn in [("h2d", h2d), ("d2h", d2h), ("both", both)]:
    ms = timeit(fn)
    print(f"{name}: {ms:.3f} ms for {B / 1e6:.0f} MB per direction -> {B / ms / 1e6:.1f} GB/s per direction")
