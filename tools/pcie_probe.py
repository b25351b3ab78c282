"""PCIe probe: pinned H2D / D2H bandwidth alone and concurrently (the floor
of the host-buffer path: x + y in, y' out)."""
import time
import torch

n_in, n_out = 107_412_496, 53_706_248  # Laplacian: x + y (f64) in, y' out
hi = torch.empty(n_in, dtype=torch.uint8).pin_memory()
ho = torch.empty(n_out, dtype=torch.uint8).pin_memory()
di = torch.empty(n_in, dtype=torch.uint8, device="cuda")
do = torch.empty(n_out, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(f, reps=10):
    for _ in range(2):
        f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


h2d = t(lambda: di.copy_(hi, non_blocking=True))
d2h = t(lambda: ho.copy_(do, non_blocking=True))


def both():
    with torch.cuda.stream(s1):
        di.copy_(hi, non_blocking=True)
    with torch.cuda.stream(s2):
        ho.copy_(do, non_blocking=True)


bo = t(both)
print(f"H2D {n_in/1e6:.1f} MB {h2d:.3f} ms ({n_in/h2d/1e6:.1f} GB/s); D2H {n_out/1e6:.1f} MB {d2h:.3f} ms "
      f"({n_out/d2h/1e6:.1f} GB/s); both concurrently {bo:.3f} ms")
