"""Register-file launches on the GPU (csrc/tc_nand_regfile.cuh): whole per-lane FFT netlists
in one launch, intermediates in shared-memory buffers, equal ciphertext for ciphertext to the
level launches and decrypting to the reference's words (fft.py:137-194)."""

import numpy as np
import pytest

from paper_1611_08769_b200 import (DEFAULT0_PARAMS, FixedFormat, GpuEngine, GswScheme, fft_1d, fft_2d,
                                   input_signal)
from paper_1611_08769_b200.fft import read_signal_ints, signal_words
from tests.helpers import FFT_CONFIGS, config_signal, golden_npz

pytestmark = pytest.mark.gpu


def _run(cfg, lanes, schedule, scheme, keys):
    pname, seed, (F, f), dims, _ = FFT_CONFIGS[cfg]
    if lanes == 1:
        rng, values = config_signal(cfg)
        eng = GpuEngine(scheme, keys=keys, rng=rng, device_encrypt=True, schedule=schedule)
    else:
        rngs, vals = zip(*[config_signal(cfg, l) for l in range(lanes)])
        values = np.array(vals)
        eng = GpuEngine(scheme, keys=keys, batch_size=lanes, lane_rngs=list(rngs), device_encrypt=True,
                        schedule=schedule)
    sig = input_signal(eng, values, FixedFormat(F, f), dims=dims if isinstance(dims, tuple) else None)
    out = fft_2d(sig) if isinstance(dims, tuple) else fft_1d(sig)
    eng.flush()
    hs = [h for w in signal_words(out) for h in w.bits]
    return eng, out, eng.node_values(hs)


@pytest.mark.parametrize("cfg,lanes", [("cfg4", 300), ("cfg4", 17), ("cfg3", 1)])
def test_regfile_equals_level_launches(cfg, lanes):
    GpuEngine._TEMPLATES.clear()
    scheme = GswScheme(DEFAULT0_PARAMS)
    keys = scheme.keygen(FFT_CONFIGS[cfg][1])
    e_rf, o_rf, v_rf = _run(cfg, lanes, "regfile", scheme, keys)
    assert e_rf.last_compile["schedule"] == "regfile" and e_rf.last_program.launches == 1
    words = read_signal_ints(e_rf, o_rf)
    del e_rf, o_rf
    GpuEngine._TEMPLATES.clear()
    e_lv, o_lv, v_lv = _run(cfg, lanes, "levels", scheme, keys)
    assert np.array_equal(v_rf, v_lv)
    assert np.array_equal(words, golden_npz(f"clear_{cfg}.npz")["words"][:lanes])


def test_regfile_is_auto_for_cfg4_and_replays():
    """configs[4] (1024 lanes) runs as one register-file launch under 'auto', first call and
    template replay, and decrypts to the reference's words for every lane."""
    GpuEngine._TEMPLATES.clear()
    scheme = GswScheme(DEFAULT0_PARAMS)
    keys = scheme.keygen(4)
    want = golden_npz("clear_cfg4.npz")["words"]
    for call in range(2):
        eng, out, _ = _run("cfg4", 1024, "auto", scheme, keys)
        assert eng.last_compile["schedule"] == "regfile"
        assert eng.template_hits == call
        assert np.array_equal(read_signal_ints(eng, out), want)
        del eng, out


def test_regfile_operand_reuse_equals_full_rebuild():
    """Slots whose operand equals the one two slots earlier skip the A rebuild / B copy (plan bits
    64 / 128); debug bit 20 rebuilds every operand: identical ciphertexts either way."""
    GpuEngine._TEMPLATES.clear()
    scheme = GswScheme(DEFAULT0_PARAMS)
    keys = scheme.keygen(4)
    vals = {}
    for dbg in (0, 1 << 20):
        scheme.ctx.set_debug(dbg)
        try:
            eng, out, v = _run("cfg4", 20, "regfile", scheme, keys)
            assert eng.last_compile["regfile"]["reuse_l"] > 0 and eng.last_compile["regfile"]["reuse_r"] > 0
            vals[dbg] = v
        finally:
            scheme.ctx.set_debug(0)
        del eng, out
    assert np.array_equal(vals[0], vals[1 << 20])


def test_regfile_host_streaming_equals_device_run():
    """fhegpu_prog_run_host on a register-file program (one launch per streamed chunk, spill
    space outside the streaming regions): the output ciphertexts equal the device run's."""
    GpuEngine._TEMPLATES.clear()
    scheme = GswScheme(DEFAULT0_PARAMS)
    keys = scheme.keygen(4)
    lanes = 300
    rngs, vals = zip(*[config_signal("cfg4", l) for l in range(lanes)])
    eng = GpuEngine(scheme, keys=keys, batch_size=lanes, lane_rngs=list(rngs), device_encrypt=True,
                    schedule="regfile")
    sig = input_signal(eng, np.array(vals), FixedFormat(16, 12))
    out = fft_1d(sig)
    prog = eng.flush()
    assert eng.last_compile["schedule"] == "regfile"
    ins = [h for w in signal_words(sig) for h in w.bits]
    outs = [h for w in signal_words(out) for h in w.bits]
    want = eng.node_values(outs)
    host_in = [eng.node_values([h])[0] for h in ins]
    got = eng.run_host(prog, list(zip(ins, host_in)), outs, chunk_lanes=148)
    assert np.array_equal(np.stack(got), want)
    # the streamed run took the register-file path: one launch per chunk, not 218 level launches
    # (debug bit 15 forces level launches; both must agree)
    scheme.ctx.set_debug(1 << 15)
    try:
        got_lv = eng.run_host(prog, list(zip(ins, host_in)), outs, chunk_lanes=148)
    finally:
        scheme.ctx.set_debug(0)
    assert np.array_equal(np.stack(got_lv), want)
