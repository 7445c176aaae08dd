"""Per-gate timeline of the warp-dataflow launch (configs[0]) from a -DFHEGPU_TRACE=1 build
(FHEGPU_LIB=...): where a gate's time goes (operand waits by path, compute) and how the real
critical path compares with the planner's model."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_1611_08769_b200 import EXACT_PARAMS, FixedFormat, GpuEngine, GswScheme, _native, fft_1d, input_signal  # noqa: E402
from tests.helpers import config_signal  # noqa: E402

scheme = GswScheme(EXACT_PARAMS)
keys = scheme.keygen(0)
rng, vals = config_signal("cfg0")
eng = GpuEngine(scheme, keys=keys, rng=rng, device_encrypt=True, schedule="flow")
out = fft_1d(input_signal(eng, vals, FixedFormat(16, 12)))
prog = eng.flush()
import time
t_end = time.perf_counter() + float(os.environ.get("FLOW_WARM_S", "1.5"))
while time.perf_counter() < t_end:                  # sustained load first: clocks ramp from idle
    for _ in range(50):
        prog.run(1)
    torch.cuda.synchronize()
n = len(eng.last_compile["ops"])
buf = np.zeros((n, 12), dtype=np.uint32)
_native._lib.fhegpu_debug_flow_trace(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), n)
if os.environ.get("FLOW_TRACE_OUT"):                # raw records for offline analysis
    np.savez_compressed(os.environ["FLOW_TRACE_OUT"], trace=buf, deps=eng.last_compile["deps"])
wr, wl, comp, tot, paths, gt1, gt2, gt3, c_ring, c_r, c_flag, smid = buf.T.astype(np.int64)
worker = paths >> 16
pr, pl = paths & 15, (paths >> 4) & 15
kr, kl = (paths >> 8) & 3, (paths >> 12) & 3
names = {0: "store", 1: "scratch", 2: "ring"}
print(f"gates {n}; mean per gate: wait_r {wr.mean():.0f} wait_l {wl.mean():.0f} compute {comp.mean():.0f} total {tot.mean():.0f} cycles")
print(f"compute: median {np.median(comp):.0f} p10 {np.percentile(comp, 10):.0f} p90 {np.percentile(comp, 90):.0f}")
print(f"service (total - waits): median {np.median(tot - wr - wl):.0f}")
deps = eng.last_compile["deps"]
WPC = int(os.environ.get("FLOW_WPC", "8"))
ghz = float(np.median((tot - wr)[gt3 > gt1] / (gt3 - gt1)[gt3 > gt1]))
print(f"SM clock from clock64 / globaltimer: {ghz:.3f} GHz")
for side, w, path, got, col in (("right", wr, pr, gt1, 1), ("left", wl, pl, gt2, 0)):      # deps: (left, right)
    d = deps[:, col]
    has = d >= 0
    hop = np.where(has, got - gt3[np.maximum(d, 0)], 0)            # ns, producer's end -> consumer has it
    waited = has & (w * (1 / ghz) > hop) & (hop > 0)                # the consumer was already waiting
    for pth in (1, 2):
        m = waited & (path == pth)
        if m.any():
            print(f"  {side} via {names[pth]:8s}: {m.sum():6d} waited-for operands, hop median {np.median(hop[m]):.0f} ns "
                  f"({np.median(hop[m]) * ghz:.0f} cyc) p10 {np.percentile(hop[m], 10):.0f} p90 {np.percentile(hop[m], 90):.0f}")
    for k in (0, 1, 2):
        for pth in (0, 1, 2):
            m = ((kr if side == "right" else kl) == k) & (path == pth)
            if m.any():
                print(f"  {side}: planned {names[k]:8s} took {names[pth]:8s}: {m.sum():6d} operands, wait median "
                      f"{np.median(w[m]):.0f} cyc")
# same-SM hops in SM clocks (clock64 is per SM): producer's ring store -> consumer holds the operand
for side, w, path, cgot, col in (("right", wr, pr, c_r, 1),):
    d = deps[:, col]
    m = (d >= 0) & (path == 2)
    dd = np.maximum(d, 0)
    m &= smid == smid[dd]
    hopc = (cgot - c_ring[dd]) & 0xFFFFFFFF
    hopc = np.where(hopc > 1 << 31, hopc - (1 << 32), hopc)
    waited = m & (w > hopc) & (hopc > 0)
    if waited.any():
        det = (c_flag - c_ring[dd]) & 0xFFFFFFFF
        det = np.where(det > 1 << 31, det - (1 << 32), det)
        post = (cgot - c_flag) & 0xFFFFFFFF
        print(f"  {side} ring hop split: store -> flag seen median {np.median(det[waited]):.0f} p10 {np.percentile(det[waited], 10):.0f} "
              f"p90 {np.percentile(det[waited], 90):.0f}; flag seen -> operand held median {np.median(post[waited]):.0f} "
              f"p90 {np.percentile(post[waited], 90):.0f}")
        same_w = waited & (worker == worker[dd])
        print(f"  (of these, producer on the same worker: {same_w.sum()})")
        print(f"  {side} ring hop in SM clocks (consumer already waiting): n {waited.sum()} median {np.median(hopc[waited]):.0f} "
              f"p10 {np.percentile(hopc[waited], 10):.0f} p90 {np.percentile(hopc[waited], 90):.0f}")
print(f"span: {(gt3.max() - gt1.min()) / 1e3:.1f} us; workers used {len(np.unique(worker))}")
# real critical path: walk back from the last gate through the operand that arrived last
g = int(np.argmax(gt3))
chain = []
while g >= 0:
    a, b = deps[g]
    cand = [(gt3[x], x) for x in (a, b) if x >= 0]
    chain.append(g)
    g = max(cand)[1] if cand else -1
chain = chain[::-1]
t = gt3[chain]
steps = np.diff(t)
same = worker[chain[1:]] == worker[chain[:-1]]
same_cta = (worker[chain[1:]] // WPC) == (worker[chain[:-1]] // WPC)
print(f"last-arrival chain: {len(chain)} gates, {(t[-1] - t[0]) / 1e3:.1f} us; step median {np.median(steps):.0f} ns; "
      f"same worker {same.sum()} (median {np.median(steps[same]) if same.any() else 0:.0f} ns), same CTA other warp "
      f"{(same_cta & ~same).sum()} (median {np.median(steps[same_cta & ~same]) if (same_cta & ~same).any() else 0:.0f} ns), "
      f"other CTA {(~same_cta).sum()} (median {np.median(steps[~same_cta]) if (~same_cta).any() else 0:.0f} ns)")
