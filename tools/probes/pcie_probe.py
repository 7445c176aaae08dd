"""Host<->device copy rates: contiguous vs the store's pitched (9396 B rows in 9408 B) copies,
each direction alone and both directions at once."""
import sys, time
sys.path.insert(0, '/root/repo')
import torch
from paper_1611_08769_b200 import DEFAULT_PARAMS, GswScheme

GB = 1e9
n = 1 << 18                                   # ciphertexts per copy (2.46 GB)
s = GswScheme(DEFAULT_PARAMS)
ctx = s.ctx
words = DEFAULT_PARAMS.n_ct * DEFAULT_PARAMS.k
h_in = torch.zeros((n, words), dtype=torch.int32).pin_memory()
h_out = torch.empty((n, words), dtype=torch.int32).pin_memory()
d_a = torch.empty((n, words), dtype=torch.int32, device="cuda")
d_b = torch.empty((n, words), dtype=torch.int32, device="cuda")
nbytes = n * words * 4
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=3):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps


def h2d():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)


def both():
    h2d(); d2h()


for name, fn, b in (("h2d contiguous", h2d, nbytes), ("d2h contiguous", d2h, nbytes),
                    ("h2d+d2h concurrent", both, 2 * nbytes)):
    t = timed(fn)
    print(f"{name:28s} {b / t / GB:7.1f} GB/s")
ctx.reserve(n)
t = timed(lambda: ctx.write_range(0, n, h_in.data_ptr(), sync=False))
print(f"{'h2d pitched (store)':28s} {nbytes / t / GB:7.1f} GB/s")
t = timed(lambda: ctx.read_range(0, n, h_out.data_ptr(), sync=False))
print(f"{'d2h pitched (store)':28s} {nbytes / t / GB:7.1f} GB/s")
