"""Circuit templates on the GPU: a replayed transform (cached program over a private slot
region, inputs and outputs bound by device copies) yields the same output ciphertexts as
the recorded circuit, and the reference's decrypted words (fft.py:137-194)."""

import numpy as np
import pytest

from paper_1611_08769_b200 import (DEFAULT0_PARAMS, EXACT_PARAMS, FixedFormat, GpuEngine, GswScheme,
                                   fft_1d, fft_2d, input_signal)
from paper_1611_08769_b200.fft import read_signal_ints, signal_words
from tests.helpers import FFT_CONFIGS, config_signal, golden_npz

pytestmark = pytest.mark.gpu

PARAMS = {"EXACT": EXACT_PARAMS, "DEFAULT0": DEFAULT0_PARAMS}


def _call(scheme, keys, cfg, lanes, eng=None):
    """One API call: encrypt the config's signal(s), transform, flush."""
    pname, seed, (F, f), dims, _ = FFT_CONFIGS[cfg]
    if lanes == 1:
        rng, values = config_signal(cfg)
        eng = eng or GpuEngine(scheme, keys=keys, rng=rng, device_encrypt=True)
        eng.rng = rng
    else:
        rngs, vals = zip(*[config_signal(cfg, l) for l in range(lanes)])
        eng = eng or GpuEngine(scheme, keys=keys, batch_size=lanes, lane_rngs=list(rngs), device_encrypt=True)
        eng.lane_rngs = list(rngs)
        values = np.array(vals)
    sig = input_signal(eng, values, FixedFormat(F, f), dims=dims if isinstance(dims, tuple) else None)
    out = fft_2d(sig) if isinstance(dims, tuple) else fft_1d(sig)
    eng.flush()
    return eng, out


@pytest.mark.parametrize("cfg,lanes", [("cfg0", 1), ("cfg3", 1), ("cfg4", 64)])
def test_replay_equals_recording(cfg, lanes):
    GpuEngine._TEMPLATES.clear()
    pname, seed = FFT_CONFIGS[cfg][0], FFT_CONFIGS[cfg][1]
    scheme = GswScheme(PARAMS[pname])
    keys = scheme.keygen(seed)
    e1, o1 = _call(scheme, keys, cfg, lanes)                 # records (ordinary compile)
    h1 = [h for w in signal_words(o1) for h in w.bits]
    v1 = e1.node_values(h1)
    w1 = read_signal_ints(e1, o1)
    del e1, o1, h1
    e2, o2 = _call(scheme, keys, cfg, lanes)                 # replays (cached region program)
    assert e2.template_hits == 1 and "template" in e2.last_compile
    h2 = [h for w in signal_words(o2) for h in w.bits]
    assert np.array_equal(e2.node_values(h2), v1)
    assert np.array_equal(read_signal_ints(e2, o2), w1)
    want = golden_npz(f"clear_{cfg}.npz")["words"][:lanes]
    assert np.array_equal(w1, want)
    # the same engine again: the region program is reused, inputs rebound
    for _ in range(2):
        _, o3 = _call(scheme, keys, cfg, lanes, eng=e2)
        assert np.array_equal(read_signal_ints(e2, o3), want)
    assert e2.template_hits == 3 and len(e2._regions) == 1


def test_replay_with_unheld_inputs_and_a_new_context():
    """A replay whose input wires nobody holds any more (fft_1d(input_signal(...)) in one
    expression) on a fresh scheme / device context, repeated: inputs are bound before their
    slots are reclaimed, and the store does not grow from call to call."""
    GpuEngine._TEMPLATES.clear()
    want = golden_npz("clear_cfg0.npz")["words"][0].tolist()
    caps = []
    for i in range(5):
        scheme = GswScheme(EXACT_PARAMS) if i < 2 else scheme
        rng, vals = config_signal("cfg0")
        eng = GpuEngine(scheme, keys=scheme.keygen(0), rng=rng, device_encrypt=True) if i < 3 else eng
        eng.rng = rng
        out = fft_1d(input_signal(eng, vals, FixedFormat(16, 12)))
        assert read_signal_ints(eng, out)[0].tolist() == want
        caps.append(eng._n_slots)
        del out
    assert caps[4] == caps[3] == caps[2]
