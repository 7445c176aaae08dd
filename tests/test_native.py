"""C-ABI library: loads without a GPU and exports every symbol include/fhegpu.h declares."""

import os
import re

from paper_1611_08769_b200 import _native
from tests.helpers import ROOT


def _declared():
    text = open(os.path.join(ROOT, "include", "fhegpu.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fhegpu_[a-z_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _native.load_library()
    names = _declared()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
    bound = {n for n, _, _ in _native.SIGNATURES}
    assert set(names) == bound, set(names) ^ bound


def test_library_reports_version_and_errors_without_device():
    lib = _native.load_library()
    assert b"sm_100a" in lib.fhegpu_version()
    assert lib.fhegpu_ctx_kernel(None) == -1
    assert lib.fhegpu_sync(None) != 0
    assert b"null" in lib.fhegpu_last_error()


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _native.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", _native.LIB_PATH],
                          capture_output=True, text=True).stdout
    assert "UTCIMMA" in sass          # tcgen05.mma kind::i8
    assert "STTM" in sass and "LDTM" in sass and "UBLKCP" in sass


def test_argument_validation_happens_before_any_device_call():
    """Bad arguments fail with FHEGPU_EINVAL / FHEGPU_EUNSUP and a message, GPU or not
    (the reference raises ParameterError / UsageError for the same inputs)."""
    import ctypes
    lib = _native.load_library()
    EINVAL, EUNSUP = 1, 4
    h = ctypes.c_void_p()

    def create(n, ell, q, m):
        return lib.fhegpu_ctx_create(ctypes.byref(_native._Params(n, ell, q, m)), 0, ctypes.byref(h))

    assert lib.fhegpu_ctx_create(None, 0, ctypes.byref(h)) == EINVAL
    assert create(0, 29, (1 << 29) - 3, 32) == EUNSUP           # n >= 1
    assert create(16, 29, (1 << 29) - 3, 32) == EUNSUP          # k = n + 1 <= 16
    assert create(8, 29, 1 << 20, 32) == EUNSUP                 # q odd
    assert create(8, 31, (1 << 31) + 1, 32) == EUNSUP           # q < 2^31
    assert create(8, 28, (1 << 29) - 3, 32) == EINVAL           # ell = bitlen(q - 1)
    assert b"ell" in lib.fhegpu_last_error()
    assert lib.fhegpu_bits_create(0, 0, ctypes.byref(h)) == EINVAL   # lanes >= 1
    assert lib.fhegpu_nand_batch(None, None, None, None, 1) == EINVAL
    assert lib.fhegpu_mult_batch(None, None, None, None, 1) == EINVAL
    assert lib.fhegpu_add_batch(None, None, None, None, 1) == EINVAL
    assert lib.fhegpu_const_mult_batch(None, 3, None, None, 1) == EINVAL
    assert lib.fhegpu_prog_run_host(None, None, 1, 1, 0, 0, None, None, 0, None, None) == EINVAL
    assert lib.fhegpu_store_write_packed(None, 0, 1, None) == EINVAL
    assert lib.fhegpu_store_read_packed(None, 0, 1, None) == EINVAL
    assert lib.fhegpu_bits_run(None, None, 0, None, 0) == EINVAL


def test_python_layer_fails_loudly_without_a_device():
    """No CPU fallback: without a CUDA device the product path raises DeviceError."""
    import pytest
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    from paper_1611_08769_b200 import DEFAULT_PARAMS, DeviceError, GpuClearEngine, GswScheme
    with pytest.raises(DeviceError):
        GswScheme(DEFAULT_PARAMS).ctx
    eng = GpuClearEngine(batch_size=4)
    x = eng.input_bit(0b1010)
    with pytest.raises(DeviceError):
        eng.read_back(eng.nand(x, x))


def test_plain_c_consumer_links_against_the_abi():
    """tests/c/abi_kat (built by __graft_entry__.build with gcc) resolves every symbol it uses
    from the in-tree libfhegpu.so -- no Python, no torch."""
    import subprocess
    kat = os.path.join(ROOT, "tests", "c", "abi_kat")
    assert os.path.exists(kat)
    out = subprocess.run(["ldd", kat], capture_output=True, text=True).stdout
    assert "libfhegpu.so" in out and "not found" not in out
