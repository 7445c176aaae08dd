"""Register-file debugging: every gate output kept (keep_all: all gates are program outputs),
regfile vs level launches, first differing gate in schedule order with its plan records."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1611_08769_b200 import DEFAULT0_PARAMS, GpuEngine, GswScheme  # noqa: E402
from paper_1611_08769_b200._native import rf_plan  # noqa: E402


def build(eng, n_in, n_gates, seed):
    rng = np.random.default_rng(seed)
    bits = np.random.default_rng(seed + 1).integers(0, 2, (eng.batch_size, n_in))
    wires = eng.input_block(bits)
    one = eng.constant(1)
    for g in range(n_gates):
        hi = len(wires)
        a = wires[int(rng.integers(max(0, hi - 30), hi))]
        b = a if rng.random() < 0.05 else wires[int(rng.integers(max(0, hi - 30), hi))]
        if rng.random() < 0.3:
            a = eng.nand(a, one)                    # folded NOT: a complemented operand
        if rng.random() < 0.3:
            b = eng.nand(b, one)
        w = eng.nand(a, b)
        wires.append(w)
    return wires


def build_fft(eng, *_):
    from paper_1611_08769_b200 import FixedFormat, fft_1d, input_signal
    from tests.helpers import config_signal
    vals = np.array([config_signal("cfg4", l)[1] for l in range(eng.batch_size)])
    rec = []
    orig = eng.nand

    def nand(a, b):
        n_before = len(eng._level)
        w = orig(a, b)
        if not w.const and w.node >= n_before:      # a new gate (not a folded NOT / constant)
            rec.append(w)
        return w
    eng.nand = nand
    eng._capturing = True                        # record gate by gate (no circuit template)
    sig = input_signal(eng, vals, FixedFormat(16, 12))
    ins = [h for p in sig.points for w in (p.re, p.im) for h in w.bits]
    fft_1d(sig)
    eng.nand = orig
    eng._capturing = False
    return ins[:12] + rec


def main(n_gates=400, lanes=1, keep=True):
    scheme = GswScheme(DEFAULT0_PARAMS)
    keys = scheme.keygen(5)
    vals = {}
    for sched in ("levels", "regfile"):
        eng = GpuEngine(scheme, keys=keys, rng=np.random.default_rng(3), batch_size=lanes, device_encrypt=True,
                        schedule=sched, keep_all=keep,
                        lane_rngs=[np.random.default_rng(9 + l) for l in range(lanes)] if n_gates == 0 else None)
        wires = (build_fft if n_gates == 0 else build)(eng, 12, n_gates, 7)
        if not keep:                                # hold a few outputs: the rest are temporaries
            rng = np.random.default_rng(11)
            pick = set(rng.choice(np.arange(12, len(wires)), 48, replace=False).tolist()) | {len(wires) - 1}
            wires = wires[:12] + [w if (12 + i) in pick else None for i, w in enumerate(wires[12:])]
            wires = wires[:12] + [w for w in wires[12:] if w is not None]
        eng.flush()
        vals[sched] = eng.node_values(wires[12:])
        if sched == "regfile":
            comp = eng.last_compile
            print("plan", comp.get("regfile"))
            gates, ins = GpuEngine._regfile_gates(comp)
            order, slots, fills, n_spill, st = rf_plan(gates, ins, eng.RF_BUFFERS, eng.RF_DIST, eng.RF_LOOK)
            # map: wires[12 + i] node -> gate index in comp
            node_gate = {int(o): i for i, o in enumerate(comp["nodes"][:, 2])}
            pos = np.empty(len(order), int)
            pos[order] = np.arange(len(order))
            bad = []
            for i, w in enumerate(wires[12:]):
                if not np.array_equal(vals["levels"][i], vals["regfile"][i]):
                    g = node_gate[w.node]
                    bad.append((pos[g], g, i))
            bad.sort()
            print(f"{len(bad)} of {len(wires) - 12} held gate outputs differ; spills {n_spill}")
            for t, g, i in bad[:5]:
                lanes_bad = [l for l in range(lanes) if not np.array_equal(vals['levels'][i][l], vals['regfile'][i][l])]
                print("slot", t, "gate", g, "lanes", lanes_bad[:8], "slot rec", slots[t], "gate rec", gates[g])
            if bad:
                t0 = bad[0][0]
                for t in range(max(0, t0 - 6), t0 + 1):
                    print("  t", t, slots[t], gates[order[t]])
                print("  fills near:", [f for f in fills if abs(int(f["consumer"]) - t0) < 8])


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 400, int(sys.argv[2]) if len(sys.argv) > 2 else 1,
         (sys.argv[3] != "0") if len(sys.argv) > 3 else True)
