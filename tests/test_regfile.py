"""Register-file plans (CPU): the planner's schedule, buffer allocation, fills, spills and
hazard conditions (csrc/rf_plan.h) evaluate every per-lane netlist to the level program's
results in a timed model of the kernel's pipeline (tests/helpers.replay_regfile), including
lags that expose any hazard the plan leaves uncovered."""

import numpy as np
import pytest

from paper_1611_08769_b200 import (DEFAULT0_PARAMS, EXACT_PARAMS, FixedFormat, GpuEngine, GswScheme, fft_1d,
                                   fft_2d, input_signal)
from paper_1611_08769_b200._csrc_consts import RF
from paper_1611_08769_b200._native import RF_GATE_DTYPE, rf_plan
from tests.helpers import FFT_CONFIGS, config_signal, regfile_gates, replay_dry, replay_regfile

PARAMS = {"EXACT": EXACT_PARAMS, "DEFAULT0": DEFAULT0_PARAMS}


def _program(cfg, lanes):
    pname, _, (F, f), dims, _ = FFT_CONFIGS[cfg]
    vals = np.array([config_signal(cfg, l)[1] for l in range(lanes)]) if cfg == "cfg4" else config_signal(cfg)[1]
    eng = GpuEngine(GswScheme(PARAMS[pname]), dry_run=True, batch_size=lanes, schedule="regfile")
    sig = input_signal(eng, vals, FixedFormat(F, f), dims=dims if isinstance(dims, tuple) else None)
    fft_2d(sig) if isinstance(dims, tuple) else fft_1d(sig)
    prog = eng.flush()
    assert prog["schedule"] == "regfile"
    return eng, prog


def _check(eng, prog, n_buf, lags, dist=5, look=4):
    gates, ins = regfile_gates(prog)
    order, slots, fills, n_spill, stats = rf_plan(gates, ins, n_buf, dist, look)
    assert sorted(order.tolist()) == list(range(len(gates)))
    ref = replay_dry(eng)
    store = {s: b for s, b in eng.dry_inputs}
    for E, R, W, L in lags:
        got = replay_regfile(gates, ins, order, slots, fills, n_buf, store, eng.mask, E=E, R=R, W=W, fill_lat=L)
        outs = gates["out_slot"][gates["held"] == 1].tolist()
        bad = [s for s in outs if got.get(int(s)) != ref[int(s)]]
        assert not bad, f"lags {(E, R, W, L)}: {len(bad)} outputs differ"
    return stats, n_spill


def test_cfg4_plan_moves_under_half_a_ciphertext_per_gate():
    eng, prog = _program("cfg4", 6)
    stats, n_spill = _check(eng, prog, 20, [(4, 1, 3, 2), (6, 3, 9, 7)])
    n = len(prog["ops"])
    assert (stats["fills"] + stats["stores"]) / n < 0.5      # level launches move 3 per gate
    assert stats["stalls"] < n // 1000


@pytest.mark.parametrize("cfg,n_buf", [("cfg0", 8), ("cfg3", 12)])
def test_other_netlists_and_tight_register_files(cfg, n_buf):
    eng, prog = _program(cfg, 1)
    _check(eng, prog, n_buf, [(4, 1, 3, 2), (5, 2, 6, 5)], look=2)


def _random_netlist(rng, n_in, n_gates, n_held):
    gates = np.zeros(n_gates, dtype=RF_GATE_DTYPE)
    for g in range(n_gates):
        hi = n_in + g
        lo = max(0, hi - 40)                              # mostly local, like ripple adders
        gates["left"][g] = rng.integers(lo, hi)
        gates["right"][g] = rng.integers(lo, hi) if rng.random() < 0.9 else rng.integers(0, hi)
        gates["flags"][g] = rng.integers(0, 4)
    held = rng.choice(n_gates, n_held, replace=False)
    gates["held"][held] = 1
    gates["out_slot"][held] = 1000 + np.arange(n_held)
    return gates


@pytest.mark.parametrize("seed", range(6))
def test_random_netlists_spill_and_refill(seed):
    rng = np.random.default_rng(seed)
    n_in, n_gates = 12, 1500
    gates = _random_netlist(rng, n_in, n_gates, 40)
    ins = np.arange(n_in, dtype=np.uint32)
    mask = (1 << 16) - 1
    store = {i: int(rng.integers(0, mask + 1)) for i in range(n_in)}
    # straight-line evaluation
    val = [store[i] for i in range(n_in)]
    for g in gates:
        a, b = val[g["left"]], val[g["right"]]
        a ^= mask if g["flags"] & 1 else 0
        b ^= mask if g["flags"] & 2 else 0
        val.append(~(a & b) & mask)
    n_buf = int(rng.integers(6, 11))
    order, slots, fills, n_spill, stats = rf_plan(gates, ins, n_buf, int(rng.integers(1, 6)), int(rng.integers(1, 4)))
    assert stats["stores"] > 40 and n_spill > 0                   # spills happen at this size
    for lags in ((4, 1, 3, 2), (7, 4, 11, 9), (0, 0, 0, 0)):
        got = replay_regfile(gates, ins, order, slots, fills, n_buf, store, mask, *lags)
        for g in np.flatnonzero(gates["held"]):
            assert got[int(gates["out_slot"][g])] == val[n_in + g]


def test_plan_records_are_consistent():
    rng = np.random.default_rng(7)
    gates = _random_netlist(rng, 8, 600, 20)
    order, slots, fills, n_spill, stats = rf_plan(gates, np.arange(8, dtype=np.uint32), 8, 5, 3)
    n = len(gates)
    assert (np.diff(fills["consumer"].astype(np.int64)) >= 0).all()            # fills in consumer order
    for f in fills:
        assert f["w_built"] <= f["consumer"] and f["w_epi"] <= f["consumer"] and f["w_st"] <= f["consumer"]
    for t, sl in enumerate(slots):
        for w in (int(sl["lwait"]), int(sl["rwait"])):
            if w != RF.NONE and not w & RF.WAIT_FILL:
                assert t - 5 < w < t                                          # only near producers wait
    with pytest.raises(Exception, match="n_buf"):
        rf_plan(gates, np.arange(8, dtype=np.uint32), 2, 5, 3)


def test_regfile_compile_keeps_input_slots_and_outputs_apart():
    """The register-file kernel fills inputs and stores outputs in its own order: the compile
    (pin_old) never hands an input's slot to an output, outputs get distinct slots, and the
    program's temporaries still reuse slots (the store stays level-launch sized)."""
    eng, prog = _program("cfg4", 4)
    gates, ins = regfile_gates(prog)
    outs = gates["out_slot"][gates["held"] == 1]
    assert len(set(outs.tolist())) == len(outs)
    assert not set(outs.tolist()) & set(ins.tolist())
    assert eng._n_slots < 6000                     # ~3.6k live values per signal, not 108k
