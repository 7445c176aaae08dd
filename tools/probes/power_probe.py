"""Sustained cfg1 (XOR + AND) throughput vs lane count: NAND/s, SM clock, board power.

usage: power_probe.py LANES [SECONDS] -- runs the program back to back for ~SECONDS.
Small lane counts keep the whole working set in the 126 MB L2 (DRAM traffic ~inputs
+ outputs only); large ones stream every operand from HBM."""
import statistics, sys, threading, time
import numpy as np
import torch
sys.path.insert(0, '/root/repo')
from paper_1611_08769_b200 import DEFAULT_PARAMS, GswScheme, GpuEngine, and_, xor_

lanes = int(sys.argv[1]); seconds = float(sys.argv[2]) if len(sys.argv) > 2 else 3.0
dbg = int(sys.argv[3]) if len(sys.argv) > 3 else 0
schedule = sys.argv[4] if len(sys.argv) > 4 else "auto"
s = GswScheme(DEFAULT_PARAMS)
keys = s.keygen(1)
rng = np.random.default_rng(1)
base = s.encrypt_many(keys.public_key, rng.integers(0, 2, 2048), rng)
reps = (lanes + 1023) // 1024
eng = GpuEngine(s, keys=keys, batch_size=lanes, schedule=schedule)
a = eng.input_values(np.tile(base[0::2], (reps, 1, 1))[:lanes], noise_est=64)
b = eng.input_values(np.tile(base[1::2], (reps, 1, 1))[:lanes], noise_est=64)
x = xor_(a, b); y = and_(a, b)
st = torch.cuda.Stream()
s.ctx.use_torch_stream(st)
prog = eng.flush()
s.ctx.set_graphs(True)
s.ctx.set_debug(dbg)   # ablation bits (results invalid when nonzero)
for _ in range(3):
    prog.run(lanes)
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(st); prog.run(lanes); e1.record(st); torch.cuda.synchronize()
per = e0.elapsed_time(e1) / 1e3
steps = max(5, int(seconds / per))
import pynvml
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
clk, pw = [], []
stop = threading.Event()
def samp():
    while not stop.is_set():
        clk.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
        pw.append(pynvml.nvmlDeviceGetPowerUsage(h) / 1000)
        time.sleep(0.02)
t = threading.Thread(target=samp); t.start()
e0.record(st)
for _ in range(steps):
    prog.run(lanes)
e1.record(st); torch.cuda.synchronize()
stop.set(); t.join()
ms = e0.elapsed_time(e1) / steps
n = 6 * lanes
half = len(clk) // 2
print(f"{schedule} dbg={dbg:5d} lanes={lanes:8d} ws={eng._n_slots * lanes * 9408 / 1e6:8.1f}MB steps={steps:5d} "
      f"NAND/s={n / ms * 1e3 / 1e6:7.1f}M clk(med,2nd half)={statistics.median(clk[half:]):.0f} "
      f"power(med,2nd half)={statistics.median(pw[half:]):.0f}W limit={pynvml.nvmlDeviceGetEnforcedPowerLimit(h)/1000:.0f}W")
