"""configs[4] (1024 x 16-pt FFT) as one register-file launch vs level launches: device time per
step (CUDA events), FFT/s, NAND/s, and the plan's traffic (fills + stores per gate)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_1611_08769_b200 import DEFAULT0_PARAMS, FixedFormat, GpuEngine, GswScheme, fft_1d, input_signal  # noqa: E402
from paper_1611_08769_b200.fft import read_signal_ints  # noqa: E402
from tests.helpers import config_signal, golden_npz  # noqa: E402


def main(schedules, lanes=1024, reps=5):
    scheme = GswScheme(DEFAULT0_PARAMS)
    keys = scheme.keygen(4)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    scheme.ctx.use_torch_stream(stream)
    want = golden_npz("clear_cfg4.npz")["words"][:lanes]
    rngs0 = None
    for sched in schedules:
        GpuEngine._TEMPLATES.clear()
        rngs, vals = zip(*[config_signal("cfg4", l) for l in range(lanes)])
        eng = GpuEngine(scheme, keys=keys, batch_size=lanes, lane_rngs=list(rngs), device_encrypt=True,
                        schedule=sched)
        out = fft_1d(input_signal(eng, np.array(vals), FixedFormat(16, 12)))
        t0 = time.perf_counter()
        prog = eng.flush()
        torch.cuda.synchronize()
        first = time.perf_counter() - t0
        ok = np.array_equal(read_signal_ints(eng, out), want)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        prog.run(lanes)
        torch.cuda.synchronize()
        import threading
        import pynvml
        pynvml.nvmlInit()
        hdl = pynvml.nvmlDeviceGetHandleByIndex(0)
        samples, stop = [], threading.Event()

        def sample():
            while not stop.is_set():
                samples.append((pynvml.nvmlDeviceGetClockInfo(hdl, pynvml.NVML_CLOCK_SM),
                                pynvml.nvmlDeviceGetPowerUsage(hdl) / 1000.0))
                time.sleep(0.02)
        th = threading.Thread(target=sample, daemon=True)
        th.start()
        e0.record(stream)
        for _ in range(reps):
            prog.run(lanes)
        e1.record(stream)
        torch.cuda.synchronize()
        stop.set()
        th.join()
        sm = np.median([a for a, _ in samples[len(samples) // 4:]]) if samples else 0
        pw = np.median([b for _, b in samples[len(samples) // 4:]]) if samples else 0
        print(f"  clocks: median {sm:.0f} MHz, power {pw:.0f} W over {len(samples)} samples", flush=True)
        ms = e0.elapsed_time(e1) / reps
        rf = eng.last_compile.get("regfile")
        print(f"{sched}: {ms:.1f} ms/step  {lanes / ms * 1e3:.0f} FFT/s  "
              f"{eng.nand_count * lanes / ms / 1e3:.1f}M NAND/s  launches {prog.launches}  "
              f"first {first:.2f}s  ok {ok}  plan {rf}", flush=True)
        del eng, out, prog


if __name__ == "__main__":
    args = sys.argv[1:]
    lanes = int(os.environ.get("RF_LANES", "1024"))
    main(args or ["regfile", "levels"], lanes=lanes, reps=int(os.environ.get("RF_REPS", "5")))
