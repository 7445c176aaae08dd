"""Timeline probe of the pipelined kernel on CTA 0 (clock64 per gate and event).

Needs a library built with the probes compiled in:
  nvcc ... -DFHEGPU_TRACE=1 -o paper_1611_08769_b200/libfhegpu.so paper_1611_08769_b200/csrc/fhegpu.cu"""
import sys, ctypes
import numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_1611_08769_b200 import DEFAULT_PARAMS, GswScheme, GpuEngine, and_, xor_, _native
lanes = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
extra = int(sys.argv[2]) if len(sys.argv) > 2 else 0
schedule = sys.argv[3] if len(sys.argv) > 3 else "levels"     # "tiled": whole program, window
window = int(sys.argv[4]) if len(sys.argv) > 4 else 0          # trace gates [64w, 64w + 64)
s = GswScheme(DEFAULT_PARAMS); keys = s.keygen(1)
rng = np.random.default_rng(1)
eng = GpuEngine(s, keys=keys, rng=rng, batch_size=lanes, device_encrypt=True, schedule=schedule)
a, b = eng.input_block(rng.integers(0, 2, (lanes, 2)))
x = xor_(a, b); y = and_(a, b)
prog = eng.flush(); s.ctx.sync()
s.ctx.set_debug(16384 | extra | (window << 20))
if schedule == "levels":
    prog.run(lanes, 1, 2)
else:
    prog.run(lanes)
s.ctx.sync()
buf = np.zeros(64 * 16, dtype=np.uint64)
_native._lib.fhegpu_debug_ws_trace(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)))
tr = buf.reshape(64, 16).astype(np.int64)
t0 = tr[0, 0]
names = {0: "P:got_empty", 2: "M:op_full", 3: "M:d_free", 4: "M:commit", 5: "B:in_full", 6: "B:a_free",
         7: "B:done", 8: "E:bar1", 9: "E:main_done", 11: "E:bar2",
         12: "T:top", 13: "T:maindone", 10: "T:a_free", 14: "T:out_free", 1: "T:math_done", 15: "T:tail_ready"}
print("cycles relative to gate 0 producer start; per-gate rows")
print("gate " + " ".join(f"{names[e]:>12s}" for e in sorted(names)))
for g in range(16, 24):
    print(f"{g:4d} " + " ".join(f"{tr[g, e] - t0:12d}" for e in sorted(names)))
d = np.diff(tr[8:40, 7]); print("builder done period (median cycles):", np.median(d))
d = np.diff(tr[8:40, 4]); print("MMA commit period:", np.median(d))
d = np.diff(tr[8:40, 11]); print("epilogue period:", np.median(d))
