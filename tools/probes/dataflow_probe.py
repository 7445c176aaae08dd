"""Dataflow vs level scheduling on one single-signal FFT program (timing only).

(a) dataflow, real dependencies   (b) dataflow, no waits (deps = -1; results invalid)
(c) the same SSA program launched level by level (debug bit 15)."""
import sys
import numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_1611_08769_b200 import FixedFormat, GpuEngine, GswScheme, fft_1d, fft_2d, input_signal
from paper_1611_08769_b200 import DEFAULT0_PARAMS
from tests.helpers import FFT_CONFIGS, config_signal
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
pname, seed, (F, f), dims, _ = FFT_CONFIGS[cfg]
s = GswScheme(DEFAULT0_PARAMS); keys = s.keygen(seed)
rng, x = config_signal(cfg)
eng = GpuEngine(s, keys=keys, rng=rng, device_encrypt=True, schedule="dataflow")
st = torch.cuda.Stream(); torch.cuda.set_stream(st); s.ctx.use_torch_stream(st)
sig = input_signal(eng, x, FixedFormat(F, f), dims=dims if isinstance(dims, tuple) else None)
out = fft_2d(sig) if isinstance(dims, tuple) else fft_1d(sig)
prog = eng.flush(); torch.cuda.synchronize()
deps = eng.last_compile["deps"]

def t(n=5):
    prog.run(1); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(n): prog.run(1)
    b.record(st); torch.cuda.synchronize()
    return a.elapsed_time(b) / n

print(f"{cfg}: (a) dataflow {t():.3f} ms")
s.ctx.set_debug(65536); print(f"{cfg}: (a') dataflow, publish only when blocked {t():.3f} ms"); s.ctx.set_debug(0)
prog.set_deps(np.full_like(deps, -1)); print(f"{cfg}: (b) dataflow, no waits {t():.3f} ms")
s.ctx.set_debug(65536); print(f"{cfg}: (b') no waits, publish only when blocked {t():.3f} ms"); s.ctx.set_debug(0)
prog.set_deps(deps); s.ctx.set_debug(32768); print(f"{cfg}: (c) SSA program, level launches {t():.3f} ms")
s.ctx.set_debug(0)
# lag structure: how far back (in items) is the nearest dependency of each item?
n = len(deps); idx = np.arange(n)
d = np.maximum(deps[:, 0], deps[:, 1])
gap = idx - d
print(f"  items={n}  dep distance (items): min {gap[d>=0].min()}  p10 {np.percentile(gap[d>=0],10):.0f}  median {np.median(gap[d>=0]):.0f}")
