import sys, time, numpy as np
sys.path.insert(0, ".")
from paper_1611_08769_b200 import *
sched, dbg, lanes = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
s = GswScheme(DEFAULT_PARAMS); keys = s.keygen(1)
s.ctx.set_debug(dbg)
bits = np.random.default_rng(1).integers(0, 2, (lanes, 2))
eng = GpuEngine(s, keys=keys, rng=np.random.default_rng(1), batch_size=lanes, device_encrypt=True, schedule=sched)
a, b = eng.input_block(bits)
x, y = xor_(a, b), and_(a, b)
t = time.time()
got = eng.read_back_bits([x, y])
ok = (got[0] == (bits[:, 0] ^ bits[:, 1])).all() and (got[1] == (bits[:, 0] & bits[:, 1])).all()
print(sched, dbg, lanes, ok, "%.3f s" % (time.time() - t), flush=True)
