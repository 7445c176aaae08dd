"""The reference's OWN code driving this package: its server step
(cli.cmd_fft, cli.py:71-87: fileio.read_ciphertext_signal -> fft_1d -> write_ciphertext_signal)
on GpuEngine, and its GswScheme with the INTEGRATION.md section 2 ctypes stub patched in.

The reference is imported from baseline/_ref (the driver's install, present on the GPU box) or
/root/reference (build container); tests skip where neither exists."""

import importlib.util
import os

import numpy as np
import pytest

from paper_1611_08769_b200 import EXACT_PARAMS, GpuEngine, GswScheme
from paper_1611_08769_b200._native import LIB_PATH
from tests.helpers import GOLDEN, ROOT, golden_json, reference_modules

REF = reference_modules()
pytestmark = pytest.mark.skipif(REF is None, reason="reference package not installed")
IN_EFT = os.path.join(GOLDEN, "eft1_exact_in.eft")
OUT_EFT = os.path.join(GOLDEN, "eft1_exact_fft.eft")


def _server_step(engine_factory, out_path):
    """cli.cmd_fft with the engine swapped: everything else is the reference's code."""
    fhe, _, fileio, fft, _, _ = REF
    params = fileio.read_ciphertext_params(IN_EFT)
    scheme = fhe.GswScheme(params)                  # cli.py:74
    engine = engine_factory(scheme)
    signal, fmt = fileio.read_ciphertext_signal(IN_EFT, engine)
    out = fft.fft_2d(signal) if isinstance(signal.dims, tuple) else fft.fft_1d(signal)
    if out_path is not None:
        fileio.write_ciphertext_signal(out_path, params, engine, out, fmt)
    return engine


def test_reference_server_step_records_reference_netlist():
    """CPU (dry run): the reference's reader imports its own Ciphertext(matrix=...) objects
    (import_ct) and its fft_1d records the reference's gate count on GpuEngine."""
    eng = _server_step(lambda s: GpuEngine(s, dry_run=True), None)
    assert eng.nand_count == golden_json("eft1_exact.json")["nand_count"]
    assert eng.scheme.params == EXACT_PARAMS


def test_import_ct_accepts_reference_ciphertexts():
    fhe = REF[0]
    ref_scheme = fhe.GswScheme(fhe.EXACT_PARAMS)
    keys = ref_scheme.keygen(seed=1)
    ct = ref_scheme.encrypt_bit(keys.public_key, 1, np.random.default_rng(3))
    eng = GpuEngine(ref_scheme, dry_run=True)                  # a reference scheme object works too
    h = eng.import_ct(ct)
    assert eng._level[h.node] == ct.level and eng._est[h.node] == ct.noise_est
    want = GswScheme(EXACT_PARAMS)
    from paper_1611_08769_b200 import Ciphertext
    v = Ciphertext(matrix=ct.matrix, params=want.params).v
    np.testing.assert_array_equal(eng._pending_in_val[-1][0], v)
    np.testing.assert_array_equal(Ciphertext(v, params=want.params).matrix, ct.matrix)


@pytest.mark.gpu
def test_reference_server_step_on_gpu_is_byte_identical(tmp_path):
    """The full EFT1 server step of the reference, evaluated on the GPU: the output
    container equals the one the reference's FheEngine wrote, byte for byte."""
    out = tmp_path / "out.eft"
    eng = _server_step(lambda s: GpuEngine(s), out)
    assert out.read_bytes() == open(OUT_EFT, "rb").read()
    assert eng.nand_count == golden_json("eft1_exact.json")["nand_count"]
    assert eng.launches > 0
    # the reference's own fft_1d netlist (EXACT geometry, one signal) ran as one warp-dataflow launch
    assert eng.last_compile["schedule"] == "flow" and eng.last_program.launches == 1


def _stub():
    spec = importlib.util.spec_from_file_location("fhefft_gpu", os.path.join(ROOT, "integration", "fhefft_gpu.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


@pytest.mark.gpu
@pytest.mark.parametrize("preset", ["DEFAULT_PARAMS", "EXACT_PARAMS"])
def test_integration_stub_on_reference_scheme(preset):
    """every patched operator of the reference's GswScheme returns
    the same matrix, level and noise estimate as the unpatched reference."""
    fhe = REF[0]
    params = getattr(fhe, preset)
    ref = fhe.GswScheme(params)
    gpu = fhe.GswScheme(params)
    _stub().attach(gpu, LIB_PATH)
    keys = ref.keygen(seed=5)
    rng = np.random.default_rng(11)
    cts = [ref.encrypt_bit(keys.public_key, b, rng) for b in (0, 1, 1, 0)]
    nb = ref.hom_nand(cts[0], cts[1])                          # a non-fresh operand (swap rule)

    def same(a, b):
        assert np.array_equal(a.matrix, b.matrix) and (a.level, a.noise_est) == (b.level, b.noise_est)

    for x, y in [(cts[0], cts[1]), (cts[1], cts[2]), (cts[2], nb), (nb, cts[3])]:
        same(gpu.hom_nand(x, y), ref.hom_nand(x, y))
        same(gpu.hom_add(x, y), ref.hom_add(x, y))
        same(gpu.hom_mult(x, y), ref.hom_mult(x, y))
    for x in (cts[1], nb):
        same(gpu.hom_not(x), ref.hom_not(x))
        same(gpu.hom_const_mult(x, 7), ref.hom_const_mult(x, 7))
    # truth table through the patched operator (tests/test_fhe.py:74-82 of the reference)
    for a in (0, 1):
        for b in (0, 1):
            out = gpu.hom_nand(cts[0] if a == 0 else cts[1], cts[3] if b == 0 else cts[2])
            assert ref.decrypt_bit(keys.secret_key, out) == 1 - (a & b)
    if preset == "EXACT_PARAMS":                               # 64-deep chain (test_fhe.py:209-218)
        x = cts[1]
        for _ in range(64):
            x = gpu.hom_nand(x, cts[2])
        assert ref.decrypt_bit(keys.secret_key, x) == 1
    else:                                                      # depth check still raises
        deep = gpu.hom_nand(gpu.hom_nand(gpu.hom_nand(cts[1], cts[2]), cts[1]), cts[2])
        with pytest.raises(fhe.NoiseOverflowError):
            gpu.hom_nand(deep, cts[1])
