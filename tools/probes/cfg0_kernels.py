"""configs[0] (8-pt, EXACT params, 148 levels) per-FFT device time with each level kernel:
tcgen05 two-CTA (default for N = 51) vs the CUDA-core SIMT kernel, graphs on."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_1611_08769_b200 import EXACT_PARAMS, FixedFormat, GpuEngine, GswScheme, fft_1d, input_signal  # noqa: E402
from paper_1611_08769_b200._native import KERNEL_SIMT, KERNEL_TCGEN05  # noqa: E402
from paper_1611_08769_b200.fft import read_signal_ints  # noqa: E402
from tests.helpers import config_signal, golden_npz  # noqa: E402

for name, kern in (("tcgen05", KERNEL_TCGEN05), ("simt", KERNEL_SIMT)):
    scheme = GswScheme(EXACT_PARAMS)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    scheme.ctx.use_torch_stream(stream)
    scheme.ctx.set_kernel(kern)
    rng, vals = config_signal("cfg0")
    eng = GpuEngine(scheme, keys=scheme.keygen(0), rng=rng, device_encrypt=True)
    out = fft_1d(input_signal(eng, vals, FixedFormat(16, 12)))
    prog = eng.flush()
    ok = read_signal_ints(eng, out)[0].tolist() == golden_npz("clear_cfg0.npz")["words"][0].tolist()
    for _ in range(3):
        prog.run(1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(20):
        prog.run(1)
    e1.record(stream)
    torch.cuda.synchronize()
    print(f"{name}: {e0.elapsed_time(e1) / 20:.4f} ms per FFT, launches {prog.launches}, ok {ok}", flush=True)
