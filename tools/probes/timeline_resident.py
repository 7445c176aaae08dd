"""Per-slot timeline of the lane-resident kernel on CTA 0 (needs a -DFHEGPU_TRACE=1 build).

usage: timeline_resident.py [LANES] [WINDOW]  -- slots [64 WINDOW, 64 WINDOW + 64) of CTA 0"""
import sys, ctypes
import numpy as np
sys.path.insert(0, '/root/repo')
from paper_1611_08769_b200 import DEFAULT_PARAMS, GswScheme, GpuEngine, and_, xor_, _native
lanes = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
window = int(sys.argv[2]) if len(sys.argv) > 2 else 4
s = GswScheme(DEFAULT_PARAMS); keys = s.keygen(1)
rng = np.random.default_rng(1)
eng = GpuEngine(s, keys=keys, rng=rng, batch_size=lanes, device_encrypt=True, schedule="resident")
a, b = eng.input_block(rng.integers(0, 2, (lanes, 2)))
x = xor_(a, b); y = and_(a, b)
prog = eng.flush(); s.ctx.sync()
s.ctx.set_debug(16384 | (window << 20))
prog.run(lanes)
s.ctx.sync()
buf = np.zeros(64 * 16, dtype=np.uint64)
_native._lib.fhegpu_debug_ws_trace(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)))
tr = buf.reshape(64, 16).astype(np.int64)
t0 = tr[0, 5]
names = {5: "B:start", 6: "B:raw", 7: "B:afree", 8: "B:done", 2: "M:opfull", 3: "M:dfree", 4: "M:commit",
         12: "T:main", 13: "T:outfree", 14: "T:ready", 9: "E:main", 10: "E:bar", 11: "E:pub"}
order = [5, 6, 7, 8, 2, 3, 4, 12, 13, 14, 9, 10, 11]
print("slot(gate,lane) " + " ".join(f"{names[e]:>9s}" for e in order))
gates = ["t1", "t2", "u", "v", "y", "x"]
for i in range(16, 40):
    print(f"{i:3d} {gates[(i % 18) // 3]:>2s}{i % 3}     " + " ".join(f"{tr[i, e] - t0:9d}" for e in order))
for e, nm in ((8, "builder done"), (4, "MMA commit"), (10, "epilogue barrier"), (11, "epi_done publish")):
    print(f"{nm} period (median cycles): {np.median(np.diff(tr[8:56, e]))}")
raw = tr[8:56, 6] - tr[8:56, 5]
print("RAW wait per slot (cycles): median", np.median(raw), "mean", raw.mean(), "max", raw.max())
af = tr[8:56, 7] - tr[8:56, 6]
print("a_free wait per slot: median", np.median(af), "mean", af.mean())
