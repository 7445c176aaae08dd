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
