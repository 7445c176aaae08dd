"""Would cfg4 (1024 x 16-pt FFTs) gain from running small lane chunks one after another
(working set in L2)?  Sustained FFT/s of one B-lane cfg4 program, repeated, per schedule.

usage: cfg4_chunk_probe.py LANES SCHEDULE [SECONDS]"""
import statistics, sys, threading, time
import numpy as np
import torch
sys.path.insert(0, '/root/repo')
from paper_1611_08769_b200 import DEFAULT0_PARAMS, FixedFormat, GpuEngine, GswScheme, fft_1d, input_signal

lanes, schedule = int(sys.argv[1]), sys.argv[2]
secs = float(sys.argv[3]) if len(sys.argv) > 3 else 4.0
s = GswScheme(DEFAULT0_PARAMS); keys = s.keygen(4)
rngs = [np.random.default_rng(4 + l) for l in range(lanes)]
vals = np.array([r.uniform(-1, 1, 16) + 1j * r.uniform(-1, 1, 16) for r in rngs])
eng = GpuEngine(s, keys=keys, batch_size=lanes, lane_rngs=rngs, device_encrypt=True, schedule=schedule)
st = torch.cuda.Stream(); torch.cuda.set_stream(st); s.ctx.use_torch_stream(st)
out = fft_1d(input_signal(eng, vals, FixedFormat(16, 12)))
prog = eng.flush(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st); prog.run(lanes); e1.record(st); torch.cuda.synchronize()
steps = max(3, int(secs / (e0.elapsed_time(e1) / 1e3)))
import pynvml
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
clk, pw, stop = [], [], threading.Event()
def samp():
    while not stop.is_set():
        clk.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
        pw.append(pynvml.nvmlDeviceGetPowerUsage(h) / 1000); time.sleep(0.02)
th = threading.Thread(target=samp); th.start()
e0.record(st)
for _ in range(steps): prog.run(lanes)
e1.record(st); torch.cuda.synchronize(); stop.set(); th.join()
ms = e0.elapsed_time(e1) / steps; hh = len(clk) // 2
print(f"cfg4 lanes={lanes:5d} {schedule:9s} launches={prog.launches:4d} {ms:7.2f} ms/run  "
      f"{lanes / ms * 1e3:7.1f} FFT/s  clk {statistics.median(clk[hh:]):.0f}  {statistics.median(pw[hh:]):.0f} W")
