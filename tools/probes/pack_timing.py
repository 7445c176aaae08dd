"""Time the device (de)serialisation kernels: store range <-> reference-packed rows."""
import sys, time
sys.path.insert(0, '/root/repo')
import torch
from paper_1611_08769_b200 import DEFAULT_PARAMS, GswScheme
s = GswScheme(DEFAULT_PARAMS); ctx = s.ctx
n = 1 << 16
ctx.reserve(n)
pb = (261 * 261 + 7) // 8
host = torch.empty((n, pb), dtype=torch.uint8).pin_memory()
for name, fn in (("read_packed", lambda: ctx.read_packed(0, n, host.data_ptr())),
                 ("write_packed", lambda: ctx.write_packed(0, n, host.data_ptr()))):
    fn(); torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(3): fn()
    dt = (time.perf_counter() - t) / 3
    print(f"{name}: {n} cts in {dt*1e3:.1f} ms incl. PCIe ({n*pb/dt/1e9:.1f} GB/s of packed bytes)")
