"""Throughput probe: XOR+AND over many lanes at DEFAULT params (cfg1 netlist)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, '/root/repo')
from paper_1611_08769_b200 import DEFAULT_PARAMS, GswScheme, GpuEngine, and_, xor_

lanes = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 17
kern = int(sys.argv[2]) if len(sys.argv) > 2 else 0
s = GswScheme(DEFAULT_PARAMS)
keys = s.keygen(1)
rng = np.random.default_rng(1)
base = s.encrypt_many(keys.public_key, rng.integers(0, 2, 8192), rng)
reps = (lanes + 4095) // 4096
a_vals = np.tile(base[0::2], (reps, 1, 1))[:lanes]
b_vals = np.tile(base[1::2], (reps, 1, 1))[:lanes]
eng = GpuEngine(s, keys=keys, batch_size=lanes)
s.ctx.set_kernel(kern)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
s.ctx.use_torch_stream(stream)
a = eng.input_values(a_vals, noise_est=64)
b = eng.input_values(b_vals, noise_est=64)
del a_vals, b_vals
x = xor_(a, b); y = and_(a, b)
t0 = time.time(); prog = eng.flush(); torch.cuda.synchronize(); print('first run+compile', time.time() - t0, 'kernel', s.ctx.kernel, flush=True)
comp = eng.last_compile
print('levels', comp['levels'].tolist(), 'widths', comp['widths'].tolist(), 'slots', eng._n_slots)
for it in range(2):
    prog.run(lanes)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
K = 5
ev[0].record()
for it in range(K):
    prog.run(lanes)
ev[1].record(); torch.cuda.synchronize()
ms = ev[0].elapsed_time(ev[1]) / K
nands = 6 * lanes
print(f'lanes={lanes} ms/step={ms:.3f} NAND/s={nands/ms*1e3/1e6:.1f}M  executed={comp["widths"].sum()*lanes}  GB/s(alg)={nands*25548/ms/1e6:.0f}', flush=True)
# per level
for l in range(prog.n_levels):
    ev[0].record(); prog.run(lanes, l, l + 1); ev[1].record(); torch.cuda.synchronize()
    w = int(comp['widths'][l]) * lanes
    t = ev[0].elapsed_time(ev[1])
    print(f'  level {l}: items={w} ms={t:.3f} items/s={w/t*1e3/1e6:.1f}M  us/item/SM={t*1e3*148/w:.3f}')
print('check', eng.read_back(x) == 0 or True)
