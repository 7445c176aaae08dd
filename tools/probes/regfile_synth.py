"""Register-file pipeline rate on synthetic per-lane netlists: random NAND chains whose operands
come from the last `window` values (window 8: everything stays in buffers, no fills or spills;
larger windows: more fills/spills).  Device ms per step, cycles per gate slot, vs levels."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_1611_08769_b200 import DEFAULT0_PARAMS, GpuEngine, GswScheme  # noqa: E402


def main(n_gates=20000, lanes=148, windows=(6, 12, 40, 200), scheds=("regfile",)):
    scheme = GswScheme(DEFAULT0_PARAMS)
    keys = scheme.keygen(5)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    scheme.ctx.use_torch_stream(stream)
    for w in windows:
        for sched in scheds:
            GpuEngine._TEMPLATES.clear()
            eng = GpuEngine(scheme, keys=keys, rng=np.random.default_rng(3), batch_size=lanes, device_encrypt=True,
                            schedule=sched)
            rng = np.random.default_rng(7)
            wires = eng.input_block(np.random.default_rng(8).integers(0, 2, (lanes, 8)))
            vals = list(wires)
            for g in range(n_gates):
                hi = len(vals)
                a = vals[int(rng.integers(max(0, hi - w), hi))]
                b = vals[int(rng.integers(max(0, hi - w), hi))]
                vals.append(eng.nand(a, b))
            outs = vals[-4:]
            del vals
            prog = eng.flush()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            prog.run(lanes)
            e0.record(stream)
            for _ in range(3):
                prog.run(lanes)
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 3
            per_cta = -(-lanes // 148) * n_gates
            print(f"window {w:4d} {sched:8s} {ms:8.2f} ms  {ms * 1e-3 * 1.9e9 / per_cta:6.0f} cycles/slot@1.9GHz  "
                  f"{n_gates * lanes / ms / 1e3:.1f}M NAND/s  plan {eng.last_compile.get('regfile')}", flush=True)
            del eng, prog, outs


if __name__ == "__main__":
    main()
