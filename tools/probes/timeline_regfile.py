"""Per-slot timeline of the register-file kernel on CTA 0 (FHEGPU_LIB=<-DFHEGPU_TRACE=1 build>).

usage: timeline_regfile.py [WINDOW] -- slots [64 WINDOW, 64 WINDOW + 64) of CTA 0, cfg4 netlist"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1611_08769_b200 import DEFAULT0_PARAMS, FixedFormat, GpuEngine, GswScheme, _native, fft_1d, input_signal  # noqa
from tests.helpers import config_signal  # noqa

window = int(sys.argv[1]) if len(sys.argv) > 1 else 40
lanes = 148
s = GswScheme(DEFAULT0_PARAMS)
keys = s.keygen(4)
rngs, vals = zip(*[config_signal("cfg4", l) for l in range(lanes)])
eng = GpuEngine(s, keys=keys, batch_size=lanes, lane_rngs=list(rngs), device_encrypt=True, schedule="regfile")
out = fft_1d(input_signal(eng, np.array(vals), FixedFormat(16, 12)))
prog = eng.flush()
s.ctx.sync()
s.ctx.set_debug(16384 | (window << 20) | (int(os.environ.get("RF_TRACE_BUILDER", "0")) & 7) << 8)
prog.run(lanes)
s.ctx.sync()
buf = np.zeros(64 * 16, dtype=np.uint64)
_native._lib.fhegpu_debug_ws_trace(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)))
tr = buf.reshape(64, 16).astype(np.int64)
t0 = tr[0, 5]
names = {0: "C:start", 1: "C:done", 5: "B:start", 7: "B:afree", 6: "B:ops", 8: "B:done", 2: "M:opfull",
         3: "M:dfree", 4: "M:commit", 12: "T:main", 13: "T:outfree", 14: "T:ready", 9: "E:main", 10: "E:bar",
         11: "E:end", 15: "E:top"}
order = [0, 1, 5, 7, 6, 8, 2, 3, 4, 12, 13, 14, 15, 9, 10, 11]
print("slot " + " ".join(f"{names[e]:>9s}" for e in order))
for i in range(16, 40):
    print(f"{i:3d}  " + " ".join(f"{tr[i, e] - t0:9d}" for e in order))
for e in order:
    print(f"{names[e]:>10s} period (median cycles): {np.median(np.diff(tr[8:56, e]))}")
for a, b, nm in ((5, 7, "builder a_free wait"), (7, 6, "builder operand wait"), (6, 8, "builder build"),
                 (0, 1, "B copier slot"), (2, 3, "MMA d_free wait"), (12, 13, "tail out_free wait"),
                 (9, 10, "epilogue main->barrier"), (10, 11, "epilogue thread-0 tail"),
                 (15, 9, "epilogue top->main")):
    d = tr[8:56, b] - tr[8:56, a]
    print(f"{nm:>26s}: median {np.median(d):7.0f}  mean {d.mean():7.0f}")
