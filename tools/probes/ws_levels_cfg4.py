"""configs[4] on level launches (warp-specialised kernel): completes? (graphs / PDL knobs)"""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1611_08769_b200 import DEFAULT0_PARAMS, FixedFormat, GpuEngine, GswScheme, fft_1d, input_signal
from paper_1611_08769_b200.fft import read_signal_ints
from tests.helpers import config_signal, golden_npz
lanes, graphs, dbg = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
s = GswScheme(DEFAULT0_PARAMS)
s.ctx.set_graphs(bool(graphs))
s.ctx.set_debug(dbg)
rngs, vals = zip(*[config_signal("cfg4", l) for l in range(lanes)])
eng = GpuEngine(s, keys=s.keygen(4), batch_size=lanes, lane_rngs=list(rngs), device_encrypt=True, schedule="levels")
out = fft_1d(input_signal(eng, np.array(vals), FixedFormat(16, 12)))
t = time.time()
got = read_signal_ints(eng, out)
print(lanes, graphs, dbg, np.array_equal(got, golden_npz("clear_cfg4.npz")["words"][:lanes]), "%.2f s" % (time.time() - t), flush=True)
