"""Time one encrypted FFT program (cfg2 / cfg3 / cfg0) on the GPU: per-level launch profile."""
import sys, time
import numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_1611_08769_b200 import FixedFormat, GpuEngine, GswScheme, fft_1d, fft_2d, input_signal
from tests.helpers import FFT_CONFIGS, config_signal
from paper_1611_08769_b200 import DEFAULT0_PARAMS, EXACT_PARAMS
cfg = sys.argv[1]
dbg = int(sys.argv[2]) if len(sys.argv) > 2 else 0
schedule = sys.argv[3] if len(sys.argv) > 3 else 'levels'
pname, seed, (F, f), dims, _ = FFT_CONFIGS[cfg]
params = {"EXACT": EXACT_PARAMS, "DEFAULT0": DEFAULT0_PARAMS}[pname]
s = GswScheme(params); keys = s.keygen(seed)
rng, x = config_signal(cfg)
t0 = time.time()
eng = GpuEngine(s, keys=keys, rng=rng, device_encrypt=True, schedule=schedule)
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream); s.ctx.use_torch_stream(stream)
sig = input_signal(eng, x, FixedFormat(F, f), dims=dims if isinstance(dims, tuple) else None)
out = fft_2d(sig) if isinstance(dims, tuple) else fft_1d(sig)
build = time.time() - t0
prog = eng.flush(); torch.cuda.synchronize()
s.ctx.set_debug(dbg)
comp = eng.last_compile
w = comp["widths"]
print(f"{cfg} [{schedule}, launches={prog.launches}]: nands={eng.nand_count} levels={len(w)} build_s={build:.2f} slots={eng._n_slots} widths min/med/max={w.min()}/{int(np.median(w))}/{w.max()}")
for _ in range(2): prog.run(1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
for _ in range(5): prog.run(1)
e1.record(stream); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"  ms/FFT={ms:.3f}  FFT/s={1e3/ms:.1f}  NAND/s={eng.nand_count/ms/1e3:.1f}M  (HBM-roofline time {eng.nand_count*25548/6516.7e9*1e3:.2f} ms)")
# time by width bucket
lv_ms = []
for l in range(prog.n_levels):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream); prog.run(1, l, l + 1); b.record(stream); torch.cuda.synchronize()
    lv_ms.append(a.elapsed_time(b))
lv_ms = np.array(lv_ms)
for lo, hi in ((0, 148), (148, 1000), (1000, 10**9)):
    m = (w >= lo) & (w < hi)
    print(f"  widths [{lo},{hi}): levels={m.sum():4d} gates={w[m].sum():8d} ms={lv_ms[m].sum():7.3f}")
