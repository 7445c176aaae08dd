"""Shared test helpers: config protocols (BASELINE.json configs) and a cleartext
replay of compiled programs (validates levelisation + slot allocation without a GPU)."""

from __future__ import annotations

import json
import os

import numpy as np

from oracle import fixedfft

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def golden_json(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


def golden_npz(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


# config -> (params name, keygen seed, fmt (F, f), dims, lanes)
FFT_CONFIGS = {
    "cfg0": ("EXACT", 0, (16, 12), 8, 1),
    "cfg2": ("DEFAULT0", 2, (32, 24), 32, 1),
    "cfg3": ("DEFAULT0", 3, (16, 7), (8, 8), 1),
    "cfg4": ("DEFAULT0", 4, (16, 12), 16, 1024),
}


def config_signal(cfg, lane=0):
    """(rng positioned after the plaintext draws, complex values) per make_golden.py."""
    if cfg == "cfg0":
        rng = np.random.default_rng(0)
        return rng, rng.uniform(-1, 1, 8).astype(complex)
    if cfg == "cfg2":
        rng = np.random.default_rng(2)
        re = rng.uniform(-1, 1, 32)
        im = rng.uniform(-1, 1, 32)
        return rng, re + 1j * im
    if cfg == "cfg3":
        rng = np.random.default_rng(3)
        pix = rng.integers(0, 256, (8, 8))
        return rng, (pix / 255.0).ravel().astype(complex)
    if cfg == "cfg4":
        rng = np.random.default_rng(4 + lane)
        re = rng.uniform(-1, 1, 16)
        im = rng.uniform(-1, 1, 16)
        return rng, re + 1j * im
    raise KeyError(cfg)


def model_outputs(cfg, values):
    """Integer-exact oracle outputs (lanes, 2M) for complex input rows (lanes, M)."""
    _, _, (F, f), dims, _ = FFT_CONFIGS[cfg]
    vals = np.atleast_2d(values)
    re = fixedfft.encode_lanes(vals.real, F, f)
    im = fixedfft.encode_lanes(vals.imag, F, f)
    if isinstance(dims, tuple):
        o_re, o_im = fixedfft.fft_2d(re, im, dims[0], dims[1], F, f)
    else:
        o_re, o_im = fixedfft.fft_1d(re, im, F, f)
    return fixedfft.interleave(o_re, o_im)


def replay_dry(engine, n_slots_hint=None):
    """Cleartext replay of every program a dry-run engine compiled.

    Slot contents are packed lane bits (python ints); a NAND reads its operands
    (complemented per flags) and writes ~(a & b).  Inputs are written first, in
    creation order, as the real engine uploads them before the first launch
    that could read them."""
    mask = engine.mask
    store = {}
    for slot, bits in engine.dry_inputs:
        store[slot] = bits
    for prog in engine.dry_programs:
        ops = prog["ops"]
        offs = prog["offsets"]
        for lv in range(len(offs) - 1):
            a, b = int(offs[lv]), int(offs[lv + 1])
            writes = []
            outs = ops["out"][a:b].astype(np.int64)
            reads = np.concatenate([ops["left"][a:b], ops["right"][a:b]]).astype(np.int64)
            assert len(np.unique(outs)) == len(outs), "two gates of one launch write one slot"
            assert not np.intersect1d(outs, reads).size, "a launch writes a slot it also reads"
            for rec in ops[a:b]:
                x = store[int(rec["left"])]
                y = store[int(rec["right"])]
                if rec["flags"] & 1:
                    x ^= mask
                if rec["flags"] & 2:
                    y ^= mask
                writes.append((int(rec["out"]), mask ^ (x & y)))
            for s, v in writes:          # a launch reads before any of its writes land
                store[s] = v
    return store


def read_dry(engine, store, handles):
    out = []
    for h in handles:
        if h.const:
            out.append(engine.mask if h.plain else 0)
        else:
            v = store[engine._slot[h.node]]
            out.append(v ^ engine.mask if h.neg else v)
    return out


def int_word(engine, ints, width):
    """A word of fresh wires holding one two's-complement integer per lane (lanes packed)."""
    from paper_1611_08769_b200 import FixedFormat, FixedWord
    u = [int(v) % (1 << width) for v in ints]
    wires = [engine.input_bit(sum(((x >> b) & 1) << l for l, x in enumerate(u))) for b in range(width)]
    return FixedWord(tuple(wires), FixedFormat(width, 1))


def word_ints(engine, word, signed=True):
    """Per-lane integers of a word (one read-back gather)."""
    masks = engine.read_back_many(list(word.bits))
    width = len(word.bits)
    out = []
    for lane in range(engine.batch_size):
        u = sum(((m >> lane) & 1) << b for b, m in enumerate(masks))
        out.append(u - (1 << width) if signed and u >> (width - 1) else u)
    return out


def wrap(v, width):
    v %= 1 << width
    return v - (1 << width) if v >> (width - 1) else v


REF_PATHS = (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src")


def reference_root():
    """Directory holding the reference package ``fhefft``: the driver's install at
    baseline/_ref (it travels to the GPU box) or the read-only source tree in the build
    container.  None when neither exists."""
    for p in REF_PATHS:
        if os.path.isfile(os.path.join(p, "fhefft", "__init__.py")):
            return p
    return None


def reference_modules():
    """(fhe, engine, fileio, fft, arith, gates) of the reference, or None."""
    import importlib
    import sys
    root = reference_root()
    if root is None:
        return None
    if root not in sys.path:
        sys.path.append(root)
    return tuple(importlib.import_module(f"fhefft.{m}")
                 for m in ("fhe", "engine", "fileio", "fft", "arith", "gates"))


def regfile_gates(prog):
    """fhegpu_rf_gate records + input slots of a compiled program (GpuEngine._regfile_gates)."""
    from paper_1611_08769_b200.engine import GpuEngine
    return GpuEngine._regfile_gates(prog)


def replay_regfile(gates, in_slots, order, slots, fills, n_buf, store, mask, E=4, R=1, W=3, fill_lat=2):
    """Timed model of a register-file launch (one lane per CTA) over lane-packed bits.

    Clock steps: fills are issued in order as soon as the counters allow (landing fill_lat
    steps later), slot b is built when its waits hold (fills landed; near producers' outputs
    in their buffers), its epilogue writes the buffer E steps after the build, a store takes
    its snapshot of the buffer R steps after the epilogue and reaches the store W steps after
    that, unless the next store drains it earlier (the kernel's store warp keeps one store in
    flight).  Hazards the plan leaves uncovered therefore read stale or clobbered data.  Returns
    the store dict (slot -> bits; spills under ('s', k))."""
    from paper_1611_08769_b200._csrc_consts import RF
    n = len(order)
    bufs = [None] * n_buf
    g_store = dict(store)
    built = epi = st = 0
    fill_at = {}                      # fill id -> step its data lands
    fptr = 0
    b_time = {}
    pend_epi = []                     # (time, slot)
    pend_snap = []                    # (time, slot, dest buf)
    pend_write = []                   # (time, slot, key, value)
    vals = {}                         # slot -> (a, b) values read at build
    done_store = set()
    stores_issued = []
    tau = 0
    landed = []                       # (time, fill id)

    def key_of(x):
        return ("s", x & ~RF.STORE_SPILL) if x & RF.STORE_SPILL else int(x)

    while epi < n or pend_write or pend_snap:
        # fills land
        for tm, f in list(landed):
            if tm <= tau:
                landed.remove((tm, f))
                fr = fills[f]
                bufs[int(fr["buf"])] = g_store[key_of(int(fr["src"]))]
                fill_at[f] = tm
        # issue fills whose conditions hold
        while fptr < len(fills):
            fr = fills[fptr]
            if built >= fr["w_built"] and epi >= fr["w_epi"] and st >= fr["w_st"] and \
                    (fptr < RF.RING or built > fills[fptr - RF.RING]["consumer"]):
                landed.append((tau + fill_lat, fptr))
                fptr += 1
            else:
                break
        # epilogue writes
        for tm, s in sorted(pend_epi):
            if tm > tau or s != epi:
                break
            pend_epi.remove((tm, s))
            sl = slots[s]
            if sl["bits"] & (RF.SB_DEST_STORED | RF.SB_HAZARD):       # stores have read their buffers
                for (_, s2, db) in sorted(pend_snap):
                    pend_write.append((tau + W, s2, key_of(int(slots[s2]["store"])), bufs[db]))
                pend_snap.clear()
            a, b = vals.pop(s)
            g = gates[order[s]]
            a ^= mask if g["flags"] & 1 else 0
            b ^= mask if g["flags"] & 2 else 0
            bufs[int(sl["dbuf"])] = ~(a & b) & mask
            if sl["bits"] & RF.SB_STORE:
                # the store warp drains the previous store when it issues a new one (LAG 1)
                for (_, s2, db) in sorted(pend_snap):
                    pend_write.append((tau, s2, key_of(int(slots[s2]["store"])), bufs[db]))
                pend_snap.clear()
                for item in list(pend_write):
                    pend_write.remove(item)
                    g_store[item[2]] = item[3]
                    done_store.add(item[1])
                pend_snap.append((tau + R, s, int(sl["dbuf"])))
            epi += 1
        for item in sorted(pend_snap):
            if item[0] <= tau:
                pend_snap.remove(item)
                _, s2, db = item
                pend_write.append((tau + W, s2, key_of(int(slots[s2]["store"])), bufs[db]))
        for item in sorted(pend_write, key=lambda x: x[0]):
            if item[0] <= tau:
                pend_write.remove(item)
                g_store[item[2]] = item[3]
                done_store.add(item[1])
        # st: every store of slots < st complete
        while st < epi and (not (slots[st]["bits"] & RF.SB_STORE) or st in done_store):
            st += 1
        # build the next slot when its operands are ready
        if built < n and built <= epi + 2:
            sl = slots[built]
            ok = True
            for w in (int(sl["lwait"]), int(sl["rwait"])):
                if w == RF.NONE:
                    continue
                if w & RF.WAIT_FILL:
                    ok &= (w & ~RF.WAIT_FILL) in fill_at
                else:
                    ok &= epi > w
            if ok:
                vals[built] = (bufs[int(sl["lbuf"])], bufs[int(sl["rbuf"])])
                pend_epi.append((tau + E, built))
                built += 1
        tau += 1
        if tau > 50 * n + 1000:
            raise AssertionError(f"model deadlock: built {built} epi {epi} st {st} fill {fptr}")
    return g_store
