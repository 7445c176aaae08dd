"""Warp-dataflow schedules (CPU): the host planner of csrc/flow_nand.cuh places every gate of a
levelised program on one worker, names its operands by the path the kernel will try (store,
scratch, ring + scratch), and the worker lists run to completion -- under any interleaving of
the workers -- to the level program's results (a model of the kernel: in-order workers, a ring
of FLOW_RING outputs per worker, single-assignment scratch)."""

import numpy as np
import pytest

from paper_1611_08769_b200 import EXACT_PARAMS, FixedFormat, GpuEngine, GswScheme, fft_1d, input_signal
from paper_1611_08769_b200._native import FLOW_RING, FLOW_WARPS, OP_DTYPE, flow_plan
from tests.helpers import config_signal, replay_dry

K_STORE, K_SCRATCH, K_RING = 0, 1, 2
OP_TEMP, NO_STORE = 16, 0xFFFFFFFF


def _cfg0_program():
    eng = GpuEngine(GswScheme(EXACT_PARAMS), dry_run=True, schedule="flow")
    out = fft_1d(input_signal(eng, config_signal("cfg0")[1], FixedFormat(16, 12)))
    prog = eng.flush()
    assert prog["schedule"] == "flow" and "deps" in prog
    return eng, prog, out                            # (out: the handles that keep the outputs held)


def _run_model(ops, deps, ents, woff, store, mask, rng, late_ring):
    """Execute the worker lists: at every step a random worker whose next gate has its operands
    runs it.  late_ring: probability that a ring operand is treated as already overwritten (the
    kernel then takes the scratch copy).  Returns (store, ring hits)."""
    n_workers = len(woff) - 1
    ptr = woff[:-1].astype(np.int64).copy()
    end = woff[1:].astype(np.int64)
    scratch = {}                                     # gate -> bits
    rings = [dict() for _ in range(n_workers)]       # worker -> {ring slot: (pos1, bits)}
    placed = {}                                      # gate -> (worker, pos1)
    for w in range(n_workers):
        for i, e in enumerate(range(woff[w], woff[w + 1])):
            placed[int(ents[e, 3])] = (w, i + 1)
    live = [w for w in range(n_workers) if ptr[w] < end[w]]
    done, ring_hits = 0, 0
    while live:
        progressed = False
        for w in rng.permutation(live).tolist():
            e = ptr[w]
            left, right, out, g, lmeta, rmeta, pos1, _ = (int(x) for x in ents[e])
            vals = []
            for side, (idx, meta) in enumerate(((left, lmeta), (right, rmeta))):
                kind, comp = meta & 3, (meta >> 2) & 1
                if kind == K_STORE:
                    assert deps[g, side] < 0 and idx == int(ops[g]["right" if side else "left"])
                    v = store[idx]
                else:
                    assert idx == deps[g, side] >= 0
                    pw, ppos1 = placed[idx]
                    v = None
                    if kind == K_RING:
                        assert pw // FLOW_WARPS == w // FLOW_WARPS and pw % FLOW_WARPS == (meta >> 4) & 15
                        assert ppos1 == meta >> 8
                        ent = rings[pw].get((ppos1 - 1) % FLOW_RING)
                        if ent is not None and ent[0] == ppos1 and rng.random() >= late_ring:
                            v = ent[1]
                            ring_hits += 1
                    if v is None:
                        v = scratch.get(idx)
                    if v is None:
                        break                        # not produced yet: this worker waits
                vals.append(v ^ mask if comp else v)
            else:
                temp = int(ops[g]["flags"]) & OP_TEMP
                assert comp == ((int(ops[g]["flags"]) >> 1) & 1)
                assert out == (NO_STORE if temp else int(ops[g]["out"]))
                assert pos1 == e - woff[w] + 1
                res = mask ^ (vals[0] & vals[1])
                rings[w][(pos1 - 1) % FLOW_RING] = (pos1, res)
                scratch[g] = res
                if not temp:
                    store[out] = res
                ptr[w] += 1
                done += 1
                progressed = True
        live = [w for w in live if ptr[w] < end[w]]
        assert progressed or not live, f"deadlock after {done} gates"
    return store, scratch, ring_hits


@pytest.mark.parametrize("late_ring", [0.0, 0.5])
def test_cfg0_flow_schedule_runs_to_the_level_results(late_ring):
    eng, prog, out = _cfg0_program()
    ops, deps = prog["ops"], prog["deps"]
    n = len(ops)
    ents, woff, cycles = flow_plan(ops, deps, prog["offsets"], 148)
    assert sorted(ents[:, 3].tolist()) == list(range(n)), "every gate exactly once"
    assert woff[0] == 0 and woff[-1] == n and np.all(np.diff(woff.astype(np.int64)) >= 0)
    assert int(np.diff(woff.astype(np.int64)).max()) <= 32767
    # the model's makespan: a fraction of 148 levels x 2.45 us of level launches (~710k cycles)
    assert 0 < cycles < 400_000
    ref = replay_dry(eng)
    store = {s: b for s, b in eng.dry_inputs}
    got, scratch, ring_hits = _run_model(ops, deps, ents, woff, store, eng.mask, np.random.default_rng(5),
                                         late_ring)
    bad = [g for g in range(n) if scratch[g] != ref[int(ops["out"][g])]]
    assert not bad, f"{len(bad)} gate outputs differ"
    held = ops["out"][(ops["flags"] & OP_TEMP) == 0]
    assert 0 < len(held) < n and all(got[int(s)] == ref[int(s)] for s in held)   # only kept outputs are stored
    if late_ring == 0.0:
        assert ring_hits > n // 2                    # most operands travel through shared memory


def test_random_netlists_small_grids():
    rng = np.random.default_rng(11)
    for n_cta, n_in, n_gates in [(1, 3, 40), (2, 5, 300), (3, 8, 1500)]:
        level = np.zeros(n_in + n_gates, dtype=np.int64)
        rows = []
        for g in range(n_gates):
            a, b = rng.integers(0, n_in + g, 2)
            level[n_in + g] = 1 + max(level[a], level[b])
            rows.append((a, b, n_in + g, int(rng.integers(0, 4))))
        order = np.argsort(level[n_in:], kind="stable")
        ops = np.array([rows[i] for i in order], dtype=OP_DTYPE)
        lv = level[n_in:][order]
        offs = np.append(np.flatnonzero(np.diff(lv, prepend=lv[0] - 1)), n_gates).astype(np.uint64)
        producer = {int(o): i for i, o in enumerate(ops["out"])}
        deps = np.array([[producer.get(int(r["left"]), -1), producer.get(int(r["right"]), -1)] for r in ops],
                        dtype=np.int32)
        ents, woff, _ = flow_plan(ops, deps, offs, n_cta)
        mask = (1 << 16) - 1
        store0 = {s: int(rng.integers(0, 1 << 16)) for s in range(n_in)}
        ref = dict(store0)
        for r in ops:
            x = ref[int(r["left"])] ^ (mask if r["flags"] & 1 else 0)
            y = ref[int(r["right"])] ^ (mask if r["flags"] & 2 else 0)
            ref[int(r["out"])] = mask ^ (x & y)
        got, _, _ = _run_model(ops, deps, ents, woff, dict(store0), mask, rng, 0.3)
        assert got == ref
