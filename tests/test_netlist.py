"""Netlist parity (CPU): the circuits built on the GPU engine emit the reference's
gate sequence, and the levelised + slot-allocated programs compute the right bits."""

import hashlib

import numpy as np
import pytest

from paper_1611_08769_b200 import (DEFAULT0_PARAMS, DEFAULT_PARAMS, EXACT_PARAMS, FixedFormat,
                                   GpuEngine, GswScheme, and_, fft_1d, fft_2d, input_signal, xor_)
from oracle import fixedfft
from paper_1611_08769_b200.fft import signal_words
from tests.helpers import (FFT_CONFIGS, config_signal, golden_json, golden_npz, model_outputs,
                           read_dry, replay_dry)

PARAMS = {"EXACT": EXACT_PARAMS, "DEFAULT0": DEFAULT0_PARAMS}


def _build(cfg, lanes=1, keep_all=False, values=None, schedule="levels"):
    pname, seed, (F, f), dims, _ = FFT_CONFIGS[cfg]
    scheme = GswScheme(PARAMS[pname])
    eng = GpuEngine(scheme, dry_run=True, record_trace=True, batch_size=lanes, keep_all=keep_all,
                    schedule=schedule)
    if values is None:
        values = config_signal(cfg)[1]
    sig = input_signal(eng, values, FixedFormat(F, f), dims=dims if isinstance(dims, tuple) else None)
    out = fft_2d(sig) if isinstance(dims, tuple) else fft_1d(sig)
    return eng, out


def _ops_digest(trace):
    ops = [t[:4] for t in trace if t[0] in (0, 1)]
    return hashlib.sha256(np.asarray(ops, dtype="<i8").tobytes()).hexdigest()[:16], ops


def test_cfg0_trace_matches_reference_gate_for_gate():
    eng, out = _build("cfg0")
    ref = golden_npz("trace_cfg0.npz")
    dig, ops = _ops_digest(eng.trace)
    assert np.array_equal(np.asarray(ops), ref["ops"])
    meta = golden_json("trace_cfg0.json")
    assert dig == meta["ops_digest"]
    assert (eng.nand_count, eng.max_depth) == (meta["nand_count"], meta["max_depth"])
    # output wires in reference order
    wires = [h.wire if not h.const else (-2 if h.plain else -1)
             for w in signal_words(out) for h in w.bits]
    assert wires == meta["outputs"]


@pytest.mark.parametrize("cfg", ["cfg2", "cfg3", "cfg4"])
def test_trace_digest_matches_reference(cfg):
    eng, out = _build(cfg)
    meta = golden_json(f"trace_{cfg}.json")
    dig, ops = _ops_digest(eng.trace)
    assert (eng.nand_count, eng.max_depth) == (meta["nand_count"], meta["max_depth"])
    assert len(ops) == meta["n_ops"] and sum(o[0] == 1 for o in ops) == meta["n_not"]
    assert dig == meta["ops_digest"]
    wires = [h.wire if not h.const else (-2 if h.plain else -1)
             for w in signal_words(out) for h in w.bits]
    assert wires == meta["outputs"]


def test_cfg1_pair_trace_matches_reference_with_swaps():
    """DEFAULT params: the noise rule swaps operands exactly like the reference."""
    meta = golden_json("trace_cfg1.json")
    scheme = GswScheme(DEFAULT_PARAMS)
    eng = GpuEngine(scheme, dry_run=True, record_trace=True)
    hs = [(eng.input_bit(0), eng.input_bit(1)) for _ in range(meta["pairs"])]
    outs = [(xor_(a, b), and_(a, b)) for a, b in hs]
    ops = [list(t[:4]) for t in eng.trace if t[0] in (0, 1)]
    assert ops == meta["ops"]
    assert [[x.wire, y.wire] for x, y in outs] == meta["outputs"]
    assert (eng.nand_count, eng.max_depth) == (meta["nand_count"], meta["max_depth"])


@pytest.mark.parametrize("cfg", ["cfg0", "cfg3"])
@pytest.mark.parametrize("keep_all", [False, True])
def test_compiled_program_replay_matches_oracle(cfg, keep_all):
    """Levelised ops + liveness slot reuse evaluate to the oracle's words (cleartext replay)."""
    eng, out = _build(cfg, keep_all=keep_all)
    eng.flush()
    store = replay_dry(eng)
    handles = [h for w in signal_words(out) for h in w.bits]
    bits = read_dry(eng, store, handles)
    F = FFT_CONFIGS[cfg][2][0]
    words = []
    for i in range(0, len(bits), F):
        u = sum((b & 1) << k for k, b in enumerate(bits[i:i + F]))
        words.append(u - (1 << F) if u >> (F - 1) else u)
    want = model_outputs(cfg, config_signal(cfg)[1][None])[0]
    assert words == want.tolist()
    comp = eng.dry_programs[0]
    assert comp["widths"].sum() == eng.executed_nands == eng.nand_count
    if not keep_all:
        assert eng._n_slots < len(eng._level) // 4      # slots are reused


def test_lanes_replay_and_slot_reuse_cfg4_subset():
    lanes = 8
    vals = np.array([config_signal("cfg4", l)[1] for l in range(lanes)])
    eng, out = _build("cfg4", lanes=lanes, values=vals)
    eng.flush()
    store = replay_dry(eng)
    handles = [h for w in signal_words(out) for h in w.bits]
    masks = read_dry(eng, store, handles)
    want = model_outputs("cfg4", vals)
    for lane in range(lanes):
        words = []
        for i in range(0, len(masks), 16):
            u = sum(((m >> lane) & 1) << k for k, m in enumerate(masks[i:i + 16]))
            words.append(u - (1 << 16) if u >> 15 else u)
        assert words == want[lane].tolist()


def test_incremental_flushes_and_dead_handles():
    """Several flushes with handles dropped in between keep results exact."""
    scheme = GswScheme(EXACT_PARAMS)
    eng = GpuEngine(scheme, dry_run=True, batch_size=4)
    a = eng.input_bit(0b0011)
    b = eng.input_bit(0b0101)
    x = xor_(a, b)
    eng.flush()
    y = and_(x, a)
    del a
    eng.flush()
    z = xor_(y, b)
    del x
    eng.flush()
    store = replay_dry(eng)
    got = read_dry(eng, store, [y, z])
    assert got == [0b0010, 0b0111]


def test_cse_keeps_reference_counts():
    scheme = GswScheme(DEFAULT_PARAMS)
    eng = GpuEngine(scheme, dry_run=True, cse=True, batch_size=4)
    a, b = eng.input_bit(0b0011), eng.input_bit(0b0101)
    x, y = xor_(a, b), and_(a, b)
    assert eng.nand_count == 6 and eng.executed_nands == 5 and eng.max_depth == 3
    eng.flush()
    store = replay_dry(eng)
    assert read_dry(eng, store, [x, y]) == [0b0110, 0b0001]


@pytest.mark.parametrize("cfg", ["cfg3", "cfg0"])
def test_dataflow_compile_is_single_assignment_with_exact_deps(cfg):
    """schedule='dataflow': no slot written twice, none overwritten after an earlier read in
    the program, deps name the producing op (< own index); replay still equals the oracle."""
    eng, out = _build(cfg, schedule="dataflow")
    eng.flush()
    comp = eng.dry_programs[0]
    ops, deps = comp["ops"], comp["deps"]
    outs = ops["out"].astype(np.int64)
    assert len(np.unique(outs)) == len(outs)                       # single assignment
    first_read = {}
    for i, (l, r) in enumerate(zip(ops["left"].tolist(), ops["right"].tolist())):
        first_read.setdefault(l, i)
        first_read.setdefault(r, i)
    for j, o in enumerate(outs.tolist()):                          # no write-after-read
        assert first_read.get(o, len(outs)) > j
    idx = np.arange(len(ops))
    for side, col in ((0, "left"), (1, "right")):
        d = deps[:, side]
        assert ((d >= -1) & (d < idx)).all()
        has = d >= 0
        assert np.array_equal(ops[col][has], ops["out"][d[has]])     # operand = producer's slot
    store = replay_dry(eng)
    handles = [h for w in signal_words(out) for h in w.bits]
    bits = read_dry(eng, store, handles)
    F = FFT_CONFIGS[cfg][2][0]
    words = []
    for i in range(0, len(bits), F):
        u = sum((b & 1) << k for k, b in enumerate(bits[i:i + F]))
        words.append(u - (1 << F) if u >> (F - 1) else u)
    assert words == model_outputs(cfg, config_signal(cfg)[1][None])[0].tolist()


@pytest.mark.parametrize("cfg,lanes,K", [("cfg0", 8, 4), ("cfg4", 6, 3)])
def test_tiled_program_equals_level_program(cfg, lanes, K):
    """Tiling (schedule 'tiled'): the SSA program replicated over K lane chunks in wavefront
    order computes the same store as the level program (a batch-wide slot s over B lanes IS
    chunk-slots s*K + c over B/K lanes), and its deps name earlier ops writing the operand."""
    vals = np.array([config_signal(cfg, lane)[1] for lane in range(lanes)]) if cfg == "cfg4" \
        else np.repeat(config_signal(cfg)[1][None], lanes, axis=0)
    eng, out = _build(cfg, lanes=lanes, values=vals, schedule="dataflow")
    eng.flush()
    comp = eng.dry_programs[0]
    C = lanes // K
    tops, tdeps = GpuEngine._tile(comp, K)
    n = len(tops)
    assert n == K * len(comp["ops"])
    idx = np.arange(n)
    for side, col in ((0, "left"), (1, "right")):
        d = tdeps[:, side]
        assert ((d >= -1) & (d < idx)).all()
        assert np.array_equal(tops[col][d >= 0], tops["out"][d[d >= 0]])
    # replay both on one flat lane-bit store (index = slot * lanes + lane)
    n_slots = max(int(comp["ops"][f].max()) for f in ("left", "right", "out")) + 1
    base = np.zeros(n_slots * lanes, dtype=np.uint8)
    for slot, bits in eng.dry_inputs:
        base[slot * lanes: (slot + 1) * lanes] = [(bits >> l) & 1 for l in range(lanes)]
    ref, til = base.copy(), base.copy()
    lane = np.arange(lanes)
    for l, r, o, f in comp["ops"].tolist():
        a, b = ref[l * lanes + lane] ^ (f & 1), ref[r * lanes + lane] ^ ((f >> 1) & 1)
        ref[o * lanes + lane] = 1 - (a & b)
    cl = np.arange(C)
    for l, r, o, f in tops.tolist():
        a, b = til[l * C + cl] ^ (f & 1), til[r * C + cl] ^ ((f >> 1) & 1)
        til[o * C + cl] = 1 - (a & b)
    assert np.array_equal(ref, til)


def test_tiled_ring_temporaries_replay_and_war_order():
    """Ring temporaries (tiled schedule): XOR+AND over 16 lanes in 8 chunks of 2 lanes, a ring
    of 5 chunk regions; sequential replay in tiled order equals the level program, every
    dependency (RAW and the roots' write-after-read deps on chunk c-5's sinks) points back."""
    from paper_1611_08769_b200 import and_, xor_
    lanes, K, ring = 16, 8, 5
    eng = GpuEngine(GswScheme(DEFAULT_PARAMS), dry_run=True, batch_size=lanes, schedule="dataflow")
    rng = np.random.default_rng(3)
    bits = rng.integers(0, 2, (lanes, 2))
    a = eng.input_bit(int(sum(int(v) << i for i, v in enumerate(bits[:, 0]))))
    b = eng.input_bit(int(sum(int(v) << i for i, v in enumerate(bits[:, 1]))))
    x, y = xor_(a, b), and_(a, b)
    assert eng._ring_ok()
    prog = eng._compile(ssa=True, ring_temps=True)
    assert prog["n_temp"] == 4 and eng._n_slots == 4          # a, b, x, y only
    C = lanes // K
    t_base = eng._n_slots * K
    tops, tdeps = GpuEngine._tile(prog, K, C, skew=2, ring=ring, t_base=t_base)
    idx = np.arange(len(tops))
    assert ((tdeps >= -1) & (tdeps < idx[:, None])).all()
    assert int(tops["out"].max()) < t_base + ring * prog["n_temp"]
    store = np.zeros((t_base + ring * prog["n_temp"]) * C, dtype=np.uint8)
    for slot, bmask in eng.dry_inputs:
        store[slot * lanes:(slot + 1) * lanes] = [(bmask >> l) & 1 for l in range(lanes)]
    cl = np.arange(C)
    for l, r, o, f in tops.tolist():
        u, v = store[l * C + cl] ^ (f & 1), store[r * C + cl] ^ ((f >> 1) & 1)
        store[o * C + cl] = 1 - (u & v)
    xs, ys = eng._slot[x.node], eng._slot[y.node]
    assert (store[xs * lanes:(xs + 1) * lanes] == (bits[:, 0] ^ bits[:, 1])).all()
    assert (store[ys * lanes:(ys + 1) * lanes] == (bits[:, 0] & bits[:, 1])).all()


def test_auto_schedule_policy():
    """'auto' on the tcgen05 geometry: resident for small per-lane programs (<= 8 gates) over
    >= 1024 lanes; regfile for deep (>= 16 levels) programs over >= 296 lanes; tiled for wide
    (batch % 128 == 0, >= 1024 lanes), shallow (<= 32 levels) programs whose store fits;
    levels otherwise."""
    from paper_1611_08769_b200 import and_, xor_

    def pick(lanes, params=DEFAULT_PARAMS, depth=1, kernel="tcgen05"):
        eng = GpuEngine(GswScheme(params), dry_run=True, batch_size=lanes)
        a, b = eng.input_bit(0), eng.input_bit(0)
        for _ in range(depth):
            a, b = xor_(a, b), and_(a, b)
        eng.dry_run = False                       # policy only; nothing is flushed
        eng.scheme._ctx = type("Ctx", (), {"kernel": kernel})()   # stand-in device context
        return eng._pick_schedule()

    assert pick(4096) == "resident"               # one XOR + AND per lane: 6 gates
    assert pick(1024) == "resident"
    assert pick(4000) == "resident"               # a partial last lane group is fine
    assert pick(4096, DEFAULT0_PARAMS, depth=2) == "tiled"   # 12 gates per lane
    assert pick(1024, DEFAULT0_PARAMS, depth=2) == "tiled"
    assert pick(512) == "levels"                  # too narrow to fill the SMs
    assert pick(4000, DEFAULT0_PARAMS, depth=2) == "levels"  # not a multiple of the tiled chunk
    assert pick(4096, EXACT_PARAMS) == "levels"   # no warp-specialised kernel for N = 51
    assert pick(4096, DEFAULT0_PARAMS, depth=12) == "regfile"  # 36 levels: one register-file launch
    assert pick(296, DEFAULT0_PARAMS, depth=12) == "regfile"
    assert pick(200, DEFAULT0_PARAMS, depth=12) == "levels"    # < 2 lanes per SM
    assert pick(4096, kernel="simt") == "levels"  # dataflow launches need the tcgen05 kernel


@pytest.mark.parametrize("normalize", [False, True])
def test_ifft_replay_matches_swap_model(normalize):
    """ifft_1d = swap(fft(swap(x))) (+ floor shift by log2 M): the replayed netlist equals the
    integer model on 8 lanes of random 8-point Q4.12 signals, costs exactly the fft's NANDs,
    and fft -> ifft returns the input within the fixed-point rounding of the two passes."""
    from paper_1611_08769_b200.fft import ifft_1d
    lanes, M, F, f = 8, 8, 16, 12
    rng = np.random.default_rng(31)
    vals = rng.uniform(-0.5, 0.5, (lanes, M)) + 1j * rng.uniform(-0.5, 0.5, (lanes, M))
    scheme = GswScheme(EXACT_PARAMS)
    eng = GpuEngine(scheme, dry_run=True, batch_size=lanes)
    sig = input_signal(eng, vals, FixedFormat(F, f))
    out = ifft_1d(sig, normalize=normalize)
    eng.flush()
    store = replay_dry(eng)
    bits = read_dry(eng, store, [h for w in signal_words(out) for h in w.bits])
    got = np.zeros((lanes, 2 * M), dtype=np.int64)
    for wi in range(2 * M):
        u = [sum(((bits[wi * F + k] >> l) & 1) << k for k in range(F)) for l in range(lanes)]
        got[:, wi] = [x - (1 << F) if x >> (F - 1) else x for x in u]
    re = fixedfft.encode_lanes(vals.real, F, f)
    im = fixedfft.encode_lanes(vals.imag, F, f)
    o_im, o_re = fixedfft.fft_1d(im, re, F, f)           # swap in, fft, swap out
    if normalize:
        o_re, o_im = o_re >> 3, o_im >> 3                 # floor division by M = 8
    assert np.array_equal(got, fixedfft.interleave(o_re, o_im))
    ref_eng = GpuEngine(scheme, dry_run=True, batch_size=lanes)
    fft_1d(input_signal(ref_eng, vals, FixedFormat(F, f)))
    assert eng.nand_count == ref_eng.nand_count           # the swaps and the shift are wiring
    if normalize:                                         # round trip through the integer model
        f_re, f_im = fixedfft.fft_1d(re, im, F, f)
        b_im, b_re = fixedfft.fft_1d(f_im, f_re, F, f)
        assert np.abs((b_re >> 3) - re).max() <= 8 and np.abs((b_im >> 3) - im).max() <= 8


def _replay_resident(eng, prog, plan, inputs, n_local):
    """Cleartext model of the lane-resident kernel (tc_nand_resident.cuh) on packed lane bits:
    inputs from the dry-run store, every gate into its local buffer, outputs to their slots."""
    store = replay_dry(eng)          # the level replay's final store: the reference results
    before = {slot: bits for slot, bits in eng.dry_inputs}   # input slots may be reused by outputs
    mask = eng.mask
    loc = [None] * n_local
    ins = [before[int(s)] for s in inputs]
    outs = {}
    for rec in plan:
        x = loc[rec["lidx"]] if rec["lkind"] else ins[rec["lidx"]]
        y = loc[rec["ridx"]] if rec["rkind"] else ins[rec["ridx"]]
        if rec["flags"] & 1:
            x ^= mask
        if rec["flags"] & 2:
            y ^= mask
        loc[rec["dest"]] = mask ^ (x & y)
        if rec["is_out"]:
            outs[int(rec["out_slot"])] = loc[rec["dest"]]
    return store, outs


def test_resident_plan_cfg1_and_random_programs():
    """Lane-resident plans (GpuEngine._resident_plan): the gate benchmark's XOR + AND uses 2
    inputs and 4 local buffers (3 for temporaries, 1 shared by the 2 outputs) and reproduces
    the level replay;
    random small programs (temporaries reused, complemented operands, outputs also read
    later) agree too or are refused when they exceed the kernel's limits."""
    from paper_1611_08769_b200.gates import nor_, not_, or_, xnor_
    scheme = GswScheme(DEFAULT_PARAMS)
    eng = GpuEngine(scheme, dry_run=True, batch_size=64)
    rng = np.random.default_rng(4)
    a, b = (eng.input_bit(int(rng.integers(0, 1 << 62))) for _ in range(2))
    x, y = xor_(a, b), and_(a, b)
    eng.flush()
    prog = eng.dry_programs[-1]
    plan, inputs, n_local = GpuEngine._resident_plan(prog)
    assert (len(plan), len(inputs), n_local) == (6, 2, 4)     # v into t1's buffer, x into y's
    assert plan["is_out"].sum() == 2
    store, outs = _replay_resident(eng, prog, plan, inputs, n_local)
    for h in (x, y):
        assert outs[eng._slot[h.node]] == store[eng._slot[h.node]]
    gates = [not_, and_, or_, xor_, nor_, xnor_]
    done = 0
    scheme0 = GswScheme(DEFAULT0_PARAMS)                   # no depth budget for random programs
    for trial in range(40):
        eng = GpuEngine(scheme0, dry_run=True, batch_size=32)
        pool = [eng.input_bit(int(rng.integers(0, 1 << 31))) for _ in range(int(rng.integers(1, 4)))]
        for _ in range(int(rng.integers(1, 4))):
            g = gates[int(rng.integers(0, len(gates)))]
            p1, p2 = pool[int(rng.integers(0, len(pool)))], pool[int(rng.integers(0, len(pool)))]
            pool.append(g(p1) if g is not_ else g(p1, p2))
        keep = pool[-2:] + [pool[int(rng.integers(0, len(pool)))]]
        del pool
        eng.flush()
        if not eng.dry_programs:
            continue
        prog = eng.dry_programs[-1]
        res = GpuEngine._resident_plan(prog)
        if res is None:                     # over the kernel's gate / input / buffer limits
            continue
        plan, inputs, n_local = res
        store, outs = _replay_resident(eng, prog, plan, inputs, n_local)
        for h in keep:
            if not h.const and eng._slot[h.node] in outs:
                assert outs[eng._slot[h.node]] == store[eng._slot[h.node]]
        done += 1
    assert done >= 10
