"""Energy per gate (NVML total-energy counter) of sustained cfg1 (XOR + AND) runs per schedule,
plus idle board power: the gate kernels run at the board power limit, so throughput is set by
energy per gate.

usage: energy_probe.py [LANES] [SECONDS] [DBG] [SCHEDULES]   (DBG != 0: stage ablations, results invalid)"""
import sys, time
import numpy as np
import pynvml
import torch
sys.path.insert(0, '/root/repo')
from paper_1611_08769_b200 import DEFAULT_PARAMS, GswScheme, GpuEngine, and_, xor_

lanes = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
seconds = float(sys.argv[2]) if len(sys.argv) > 2 else 4.0
dbg = int(sys.argv[3]) if len(sys.argv) > 3 else 0
schedules = sys.argv[4].split(",") if len(sys.argv) > 4 else ["tiled", "levels"]
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
s = GswScheme(DEFAULT_PARAMS)
keys = s.keygen(1)
rng = np.random.default_rng(1)
base = s.encrypt_many(keys.public_key, rng.integers(0, 2, 2048), rng)
reps = (lanes + 1023) // 1024
time.sleep(2.0)
e0 = pynvml.nvmlDeviceGetTotalEnergyConsumption(h)
time.sleep(2.0)
idle_w = (pynvml.nvmlDeviceGetTotalEnergyConsumption(h) - e0) / 2.0 / 1000
print(f"idle board power {idle_w:.0f} W (limit {pynvml.nvmlDeviceGetEnforcedPowerLimit(h) / 1000:.0f} W)")
s.ctx.set_debug(dbg)
for schedule in schedules:
    eng = GpuEngine(s, keys=keys, batch_size=lanes, schedule=schedule)
    a = eng.input_values(np.tile(base[0::2], (reps, 1, 1))[:lanes], noise_est=64)
    b = eng.input_values(np.tile(base[1::2], (reps, 1, 1))[:lanes], noise_est=64)
    x = xor_(a, b); y = and_(a, b)
    st = torch.cuda.Stream()
    s.ctx.use_torch_stream(st)
    prog = eng.flush()
    for _ in range(5):
        prog.run(lanes)
    torch.cuda.synchronize()
    t0, en0 = time.perf_counter(), pynvml.nvmlDeviceGetTotalEnergyConsumption(h)
    steps = 0
    while time.perf_counter() - t0 < seconds:
        for _ in range(10):
            prog.run(lanes)
        torch.cuda.synchronize()
        steps += 10
    dt, de = time.perf_counter() - t0, (pynvml.nvmlDeviceGetTotalEnergyConsumption(h) - en0) / 1000
    gates = 6 * lanes * steps
    print(f"{schedule:7s} dbg={dbg:<7d} {gates / dt / 1e6:6.1f}M NAND/s  {de / dt:5.0f} W  {de / gates * 1e6:5.2f} uJ/gate "
          f"({(de / dt - idle_w) / (gates / dt) * 1e6:4.2f} uJ/gate above idle)  "
          f"SM clock {pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)} MHz")
    del eng, prog, a, b, x, y
