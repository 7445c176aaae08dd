"""Wall time of whole API calls (encrypt -> fft -> flush -> decrypt) per FFT config: the first
call records + compiles, later calls replay the circuit template's cached program."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_1611_08769_b200 import (DEFAULT0_PARAMS, EXACT_PARAMS, FixedFormat, GpuEngine, GswScheme,  # noqa: E402
                                   fft_1d, fft_2d, input_signal)
from paper_1611_08769_b200.fft import read_signal_ints  # noqa: E402
from tests.helpers import FFT_CONFIGS, config_signal  # noqa: E402

PARAMS = {"EXACT": EXACT_PARAMS, "DEFAULT0": DEFAULT0_PARAMS}


def main(cfgs, reps=5):
    for cfg in cfgs:
        pname, seed, (F, f), dims, _ = FFT_CONFIGS[cfg]
        lanes = 1024 if cfg == "cfg4" else 1
        scheme = GswScheme(PARAMS[pname])
        keys = scheme.keygen(seed)
        if lanes == 1:
            rng, values = config_signal(cfg)
            eng = GpuEngine(scheme, keys=keys, rng=rng, device_encrypt=True)
        else:
            rngs, vals = zip(*[config_signal(cfg, l) for l in range(lanes)])
            values = np.array(vals)
            eng = GpuEngine(scheme, keys=keys, batch_size=lanes, lane_rngs=list(rngs), device_encrypt=True)
        times = []
        for r in range(reps + 1):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            sig = input_signal(eng, values, FixedFormat(F, f), dims=dims if isinstance(dims, tuple) else None)
            t1 = time.perf_counter()
            out = fft_2d(sig) if isinstance(dims, tuple) else fft_1d(sig)
            t2 = time.perf_counter()
            eng.flush()
            t3 = time.perf_counter()
            words = read_signal_ints(eng, out)
            t4 = time.perf_counter()
            times.append((t1 - t0, t2 - t1, t3 - t2, t4 - t3, t4 - t0))
            del sig, out
        print(cfg, "first: input %.4f record %.4f flush %.4f read %.4f total %.4f s" % times[0])
        rest = np.array(times[1:])
        print(cfg, "replay median: input %.4f record %.4f flush %.4f read %.4f total %.4f s" %
              tuple(np.median(rest, axis=0)), "hits", eng.template_hits, flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["cfg0", "cfg3", "cfg2", "cfg4"])
