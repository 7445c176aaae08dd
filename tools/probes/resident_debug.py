"""Debug aid: the random small programs of tests/test_gpu_configs.py, resident vs levels, with
the kernel's debug bits (argv[1], e.g. 1048576 = no operand reuse); prints the failing trials'
plans and slot orders."""
import sys

import numpy as np

sys.path.insert(0, "/root/repo")
from paper_1611_08769_b200 import DEFAULT0_PARAMS, GswScheme  # noqa: E402
from paper_1611_08769_b200 import _native as nat  # noqa: E402
from paper_1611_08769_b200.engine import GpuEngine  # noqa: E402
from paper_1611_08769_b200.gates import and_, nor_, not_, or_, xnor_, xor_  # noqa: E402

dbg = int(sys.argv[1]) if len(sys.argv) > 1 else 0
scheme = GswScheme(DEFAULT0_PARAMS)
keys = scheme.keygen(2)
rng = np.random.default_rng(12)
gates = [not_, and_, or_, xor_, nor_, xnor_]
for trial in range(12):
    plan = [(int(rng.integers(0, len(gates))), int(rng.integers(0, 50)), int(rng.integers(0, 50)))
            for _ in range(int(rng.integers(1, 4)))]
    bits = rng.integers(0, 2, (512, int(rng.integers(1, 4))))
    res = {}
    for schedule in ("levels", "resident"):
        eng = GpuEngine(scheme, keys=keys, rng=np.random.default_rng(3), batch_size=512,
                        device_encrypt=True, schedule=schedule)
        eng.ctx.set_debug(dbg if schedule == "resident" else 0)
        pool = eng.input_block(bits)
        for g, i, j in plan:
            p1, p2 = pool[i % len(pool)], pool[j % len(pool)]
            pool.append(gates[g](p1) if gates[g] is not_ else gates[g](p1, p2))
        keep = [h for h in pool[len(bits[0]):] if not h.const][-3:]
        prog = eng.flush()
        if prog is None or not keep:
            break
        res[schedule] = (eng.node_values(keep), prog.launches)
        if schedule == "resident":
            rp = GpuEngine._resident_plan(eng.last_compile)
    if len(res) == 2:
        ok = np.array_equal(res["levels"][0], res["resident"][0])
        bad = [i for i in range(len(keep)) if not np.array_equal(res["levels"][0][i], res["resident"][0][i])]
        print(f"trial {trial}: launches {res['resident'][1]} ok={ok} bad outputs {bad}")
        if not ok and rp is not None:
            print(rp[0])
            print([(c & 7, (c >> 3) & 3, c >> 5) for c in nat.res_slot_order(rp[0], 3)])
