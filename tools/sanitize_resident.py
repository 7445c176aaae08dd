"""Run the lane-resident XOR + AND launch (the gate benchmark's kernel) on LANES lanes and check it
against level launches -- the workload for compute-sanitizer racecheck / synccheck / memcheck:

    compute-sanitizer --tool racecheck python tools/sanitize_resident.py 4097

Covers the production instantiation (RAW waits compiled out) and, with dbg bit 21, the one that
waits on every in-group producer."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1611_08769_b200 import DEFAULT_PARAMS, GpuEngine, GswScheme, and_, xor_  # noqa: E402


def main(lanes: int):
    scheme = GswScheme(DEFAULT_PARAMS)
    keys = scheme.keygen(1)
    bits = np.random.default_rng(9).integers(0, 2, (lanes, 2))
    outs = {}
    for variant, dbg in (("levels", 0), ("resident", 0), ("resident-allwaits", 1 << 21)):
        eng = GpuEngine(scheme, keys=keys, rng=np.random.default_rng(1), batch_size=lanes,
                        device_encrypt=True, schedule=variant.split("-")[0])
        eng.ctx.set_debug(dbg)
        a, b = eng.input_block(bits)
        x, y = xor_(a, b), and_(a, b)
        eng.flush()
        outs[variant] = eng.node_values([x, y])
        eng.ctx.set_debug(0)
        print(variant, eng.last_compile["schedule"], flush=True)
    ok = all(np.array_equal(outs["levels"], outs[v]) for v in ("resident", "resident-allwaits"))
    print(f"lanes={lanes} resident == levels: {ok}")
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 4097)
