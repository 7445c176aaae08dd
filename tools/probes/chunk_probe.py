"""Feasibility: cfg1 (XOR + AND over 2^20 pairs) as ONE dataflow launch tiled over lane chunks
(chunk-major, SSA temporaries) vs the level program -- sustained NAND/s, clock, power.

usage: chunk_probe.py [CHUNK_LANES] [SECONDS]"""
import statistics, sys, threading, time
import numpy as np
import torch
sys.path.insert(0, '/root/repo')
from paper_1611_08769_b200 import DEFAULT_PARAMS, GswScheme
from paper_1611_08769_b200._native import OP_DTYPE

C = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
SECS = float(sys.argv[2]) if len(sys.argv) > 2 else 4.0
R = int(sys.argv[3]) if len(sys.argv) > 3 else 0      # >0: temporaries in a ring of R chunk regions
                                                      # (timing only: no write-after-read deps)
TOTAL = 1 << 20
K = TOTAL // C
s = GswScheme(DEFAULT_PARAMS); ctx = s.ctx
keys = s.keygen(1); rng = np.random.default_rng(1)
st = torch.cuda.Stream(); torch.cuda.set_stream(st); ctx.use_torch_stream(st)
# store: a (K slots), b (K), x (K), y (K), then SSA temporaries 4 per chunk  (x C lanes each)
A, B, X, Y, T = 0, K, 2 * K, 3 * K, 4 * K
n_slots = 8 * K
ctx.reserve(n_slots * C)
base = s.encrypt_many(keys.public_key, rng.integers(0, 2, 65536), rng).astype(np.uint32)
pin = torch.from_numpy(base.view(np.int32).reshape(65536, -1)).pin_memory()
for first in range(0, 2 * K * C, 65536):            # a and b of every chunk: random fresh cts
    ctx.write_range(first, min(65536, 2 * K * C - first), pin.data_ptr())
# per chunk c: n1=NAND(a,b) n2=NAND(a,b) t1=NAND(n1,a) t2=NAND(n1,b) x=NAND(t1,t2) y=NAND(n2,n2)
ops = np.zeros(6 * K, dtype=OP_DTYPE); deps = np.full((6 * K, 2), -1, dtype=np.int32)
for c in range(K):
    a, b, x, y = A + c, B + c, X + c, Y + c
    t = T + 4 * (c % R if R else c)
    o = 6 * c
    rows = [(a, b, t + 0, -1, -1), (a, b, t + 1, -1, -1), (t + 0, a, t + 2, o, -1),
            (t + 0, b, t + 3, o, -1), (t + 2, t + 3, x, o + 2, o + 3), (t + 1, t + 1, y, o + 1, o + 1)]
    for j, (l, r, out, dl, dr) in enumerate(rows):
        ops[o + j] = (l, r, out, 0)
        deps[o + j] = (dl, dr)
WAVE = len(sys.argv) > 4 and sys.argv[4].startswith("wave")
SKEW = int(sys.argv[4][4:] or 1) if WAVE else 1
if WAVE:   # step s: level 0 of chunk s, level 1 of chunk s-SKEW, level 2 of chunk s-2*SKEW
    lvl = np.tile(np.array([0, 0, 1, 1, 2, 1]), K)
    chunk = np.repeat(np.arange(K), 6)
    perm = np.lexsort((np.tile(np.arange(6), K), lvl, chunk + SKEW * lvl))
    pos = np.empty_like(perm); pos[perm] = np.arange(len(perm))
    ops = ops[perm]
    d = deps[perm]
    deps = np.where(d >= 0, pos[np.maximum(d, 0)], -1).astype(np.int32)
    assert (deps < np.arange(len(deps))[:, None]).all()
prog = ctx.program(ops, np.array([0, 6 * K], dtype=np.uint64))
prog.set_deps(deps)
# the level program over all 2^20 lanes on the same inputs (slots: a=0 b=1 x=2 y=3 temps 4..7)
lv_ops = np.array([(0, 1, 4, 0), (0, 1, 5, 0), (4, 0, 6, 0), (4, 1, 7, 0), (6, 7, 2, 0), (5, 5, 3, 0)],
                  dtype=OP_DTYPE)
lv = ctx.program(lv_ops, np.array([0, 2, 4, 6], dtype=np.uint64))
import pynvml
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)


def measure(run, lanes_arg, label):
    run(lanes_arg); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st); run(lanes_arg); e1.record(st); torch.cuda.synchronize()
    steps = max(3, int(SECS / (e0.elapsed_time(e1) / 1e3)))
    clk, pw, stop = [], [], threading.Event()
    def samp():
        while not stop.is_set():
            clk.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
            pw.append(pynvml.nvmlDeviceGetPowerUsage(h) / 1000); time.sleep(0.02)
    th = threading.Thread(target=samp); th.start()
    e0.record(st)
    for _ in range(steps): run(lanes_arg)
    e1.record(st); torch.cuda.synchronize(); stop.set(); th.join()
    ms = e0.elapsed_time(e1) / steps; hh = len(clk) // 2
    print(f"{label:34s} {6 * TOTAL / ms / 1e3:7.1f}M NAND/s  {ms:6.2f} ms/step  clk {statistics.median(clk[hh:]):.0f}"
          f"  power {statistics.median(pw[hh:]):.0f} W")


measure(lambda n: lv.run(n), TOTAL, "levels (3 launches x 2^20 lanes)")
measure(lambda n: prog.run(n), C, f"dataflow, {K} chunks x {C} lanes" + (f", ring {R}" if R else "") + (", wavefront" if WAVE else ""))
