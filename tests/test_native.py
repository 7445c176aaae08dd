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
