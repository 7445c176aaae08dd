"""Circuit templates (CPU): a transform recorded once replays with the same netlist.

GpuEngine.circuit records ``fft_1d`` / ``fft_2d`` once per (call key, input structure) and
replays later calls without running the Python circuit code; the replay is either expanded
into ordinary ops (dry run, mixed programs) or run as a cached program over a private slot
region.  Both must compute what the recorded circuit computes (reference fft.py:137-194)."""

import numpy as np
import pytest

from paper_1611_08769_b200 import (DEFAULT0_PARAMS, EXACT_PARAMS, FixedFormat, GpuEngine, GswScheme, and_,
                                   fft_1d, fft_2d, ifft_1d, input_signal)
from paper_1611_08769_b200.engine import CircuitTemplate
from paper_1611_08769_b200.fft import signal_words
from tests.helpers import FFT_CONFIGS, config_signal, model_outputs, read_dry, replay_dry

PARAMS = {"EXACT": EXACT_PARAMS, "DEFAULT0": DEFAULT0_PARAMS}


def _words(bits, F):
    out = []
    for i in range(0, len(bits), F):
        u = sum((b & 1) << k for k, b in enumerate(bits[i:i + F]))
        out.append(u - (1 << F) if u >> (F - 1) else u)
    return out


def _run(cfg, lanes=1, values=None, scheme=None):
    pname, _, (F, f), dims, _ = FFT_CONFIGS[cfg]
    scheme = scheme or GswScheme(PARAMS[pname])
    eng = GpuEngine(scheme, dry_run=True, batch_size=lanes)
    if values is None:
        values = config_signal(cfg)[1]
    sig = input_signal(eng, values, FixedFormat(F, f), dims=dims if isinstance(dims, tuple) else None)
    out = fft_2d(sig) if isinstance(dims, tuple) else fft_1d(sig)
    return eng, sig, out


@pytest.mark.parametrize("cfg", ["cfg0", "cfg3"])
def test_replay_expands_to_the_recorded_circuit(cfg):
    GpuEngine._TEMPLATES.clear()
    e1, _, out1 = _run(cfg)
    hits1 = e1.template_hits                      # nested calls (fft_2d's row / column fft_1d) replay
    e2, _, out2 = _run(cfg)
    assert e2.template_hits == 1 and hits1 == (0 if cfg == "cfg0" else 7)   # rows 1-7 replay row 0
    assert (e2.nand_count, e2.max_depth, e2.executed_nands) == (e1.nand_count, e1.max_depth, e1.executed_nands)
    F = FFT_CONFIGS[cfg][2][0]
    want = model_outputs(cfg, config_signal(cfg)[1][None])[0].tolist()
    for eng, out in ((e1, out1), (e2, out2)):
        eng.flush()
        store = replay_dry(eng)
        bits = read_dry(eng, store, [h for w in signal_words(out) for h in w.bits])
        assert _words(bits, F) == want
    assert len(e2.dry_programs[0]["ops"]) == len(e1.dry_programs[0]["ops"])


def _replay_region(comp, tpl, in_bits, mask):
    """Cleartext run of a template's private-region program: inputs at slots 0..n_in-1."""
    store = {i: b for i, b in enumerate(in_bits)}
    prog = comp["prog"]
    ops, offs = prog["ops"], prog["offsets"]
    for lv in range(len(offs) - 1):
        writes = []
        for rec in ops[int(offs[lv]):int(offs[lv + 1])]:
            x, y = store[int(rec["left"])], store[int(rec["right"])]
            x ^= mask if rec["flags"] & 1 else 0
            y ^= mask if rec["flags"] & 2 else 0
            writes.append((int(rec["out"]), ~(x & y) & mask))
        for slot, v in writes:
            store[slot] = v
    return {li: store[int(s)] for li, s in zip(tpl.out_internal.tolist(), comp["out_slots"].tolist())}


@pytest.mark.parametrize("cfg,lanes", [("cfg0", 1), ("cfg4", 4)])
def test_region_program_computes_the_transform(cfg, lanes):
    """The cached program a replay runs on the GPU (private slots, inputs copied in, outputs
    copied out) evaluates to the integer model's outputs."""
    GpuEngine._TEMPLATES.clear()
    vals = np.array([config_signal(cfg, l)[1] for l in range(lanes)])
    _run(cfg, lanes, vals)
    eng, sig, out = _run(cfg, lanes, vals)
    (tpl,) = GpuEngine._TEMPLATES.values()
    assert isinstance(tpl, CircuitTemplate) and len(eng._macros) == 1
    comp = eng._template_compile(tpl)
    in_vals = {s: b for s, b in eng.dry_inputs}
    in_nodes = eng._macros[0][1]
    region = _replay_region(comp, tpl, [in_vals[eng._slot[n]] for n in in_nodes], eng.mask)
    bits = []
    for kind, val, neg in tpl.outs.tolist():
        if kind == 0:
            v = eng.mask if val else 0
        else:
            v = region[val] if val >= tpl.n_in else in_vals[eng._slot[in_nodes[val]]]
        bits.append(v ^ eng.mask if neg else v)
    F = FFT_CONFIGS[cfg][2][0]
    want = model_outputs(cfg, vals)
    for lane in range(lanes):
        lane_bits = [(b >> lane) & 1 for b in bits]
        assert _words(lane_bits, F) == want[lane].tolist()


def test_input_structure_is_part_of_the_key():
    """Aliased, complemented or constant input bits record a different netlist: no false hit."""
    GpuEngine._TEMPLATES.clear()
    scheme = GswScheme(EXACT_PARAMS)
    fmt = FixedFormat(16, 12)
    vals = config_signal("cfg0")[1]
    e1 = GpuEngine(scheme, dry_run=True)
    fft_1d(input_signal(e1, vals, fmt))
    e2 = GpuEngine(scheme, dry_run=True)
    sig = input_signal(e2, vals, fmt)
    p0 = sig.points[0]
    bits = list(p0.re.bits)
    bits[3] = e2.constant(1)                        # a public bit
    bits[4] = bits[5]                               # an aliased bit
    from paper_1611_08769_b200.arith import FixedWord
    from paper_1611_08769_b200.fft import ComplexFixed, SignalBuffer
    sig2 = SignalBuffer((ComplexFixed(FixedWord(tuple(bits), fmt), p0.im),) + sig.points[1:], sig.dims)
    fft_1d(sig2)
    assert e2.template_hits == 0 and len(GpuEngine._TEMPLATES) == 2


def test_replay_mixed_with_more_gates_and_ifft():
    """A replay followed by more gates before flush is expanded in place; ifft_1d (swap around
    the cached fft_1d) replays too."""
    GpuEngine._TEMPLATES.clear()
    for _ in range(2):
        eng, sig, out = _run("cfg0")
        x = and_(out.points[0].re.bits[0], out.points[1].re.bits[0])
        inv = ifft_1d(out, normalize=False)
        eng.flush()
        store = replay_dry(eng)
        b0, b1, bx = read_dry(eng, store, [out.points[0].re.bits[0], out.points[1].re.bits[0], x])
        assert bx == b0 & b1
        got = _words(read_dry(eng, store, [h for w in signal_words(inv) for h in w.bits]), 16)
        assert len(got) == 16
    assert eng.template_hits == 2
