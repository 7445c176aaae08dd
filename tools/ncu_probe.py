"""Small fixed workload for ncu: DEFAULT XOR+AND netlist over `lanes` lanes, run twice."""
import sys
import numpy as np
sys.path.insert(0, '/root/repo')
from paper_1611_08769_b200 import DEFAULT_PARAMS, GswScheme, GpuEngine, and_, xor_
lanes = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
s = GswScheme(DEFAULT_PARAMS)
keys = s.keygen(1)
rng = np.random.default_rng(1)
base = s.encrypt_many(keys.public_key, rng.integers(0, 2, 2048), rng)
reps = (lanes + 1023) // 1024
eng = GpuEngine(s, keys=keys, batch_size=lanes)
a = eng.input_values(np.tile(base[0::2], (reps, 1, 1))[:lanes], noise_est=64)
b = eng.input_values(np.tile(base[1::2], (reps, 1, 1))[:lanes], noise_est=64)
x = xor_(a, b); y = and_(a, b)
prog = eng.flush()
for _ in range(2):
    prog.run(lanes)
s.ctx.sync()
print("ok", s.ctx.kernel)
