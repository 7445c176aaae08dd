"""In-pipeline MMA issue time per gate (commit - d_free) under ablations (timeline probe)."""
import sys, ctypes
import numpy as np
sys.path.insert(0, '/root/repo')
from paper_1611_08769_b200 import DEFAULT_PARAMS, GswScheme, GpuEngine, and_, xor_, _native
lanes = 65536
s = GswScheme(DEFAULT_PARAMS); keys = s.keygen(1)
rng = np.random.default_rng(1)
eng = GpuEngine(s, keys=keys, rng=rng, batch_size=lanes, device_encrypt=True)
a, b = eng.input_block(rng.integers(0, 2, (lanes, 2)))
x = xor_(a, b); y = and_(a, b)
prog = eng.flush(); s.ctx.sync()
for dbg, name in [(0, "full"), (16, "no A build (no STTM)"), (32, "no B build"), (64, "no epi math"),
                  (4096, "no tile LDTM"), (16 | 32 | 64 | 4096, "no A,B,epi,LDTM"), (256 | 512, "no loads/stores")]:
    s.ctx.set_debug(16384 | dbg)
    prog.run(lanes, 1, 2); s.ctx.sync()
    buf = np.zeros(64 * 16, dtype=np.uint64)
    _native._lib.fhegpu_debug_ws_trace(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)))
    tr = buf.reshape(64, 16).astype(np.int64)
    issue = np.median(tr[8:48, 4] - tr[8:48, 3])
    period = np.median(np.diff(tr[8:48, 4]))
    print(f"{name:26s} MMA issue/gate={issue:7.0f} cycles ({issue/27:5.1f}/MMA)  commit period={period:7.0f}")
s.ctx.set_debug(0)
