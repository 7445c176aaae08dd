"""Drop-in check (CPU, build container only): the REFERENCE's own circuit modules
(fhefft.gates / arith / fft, imported from /root/reference) drive GpuEngine through
the bit-engine protocol unmodified and emit exactly the reference's netlist.
Skipped where the reference is absent (the GPU box)."""

import hashlib
import os
import sys

import numpy as np
import pytest

from paper_1611_08769_b200 import EXACT_PARAMS, GpuEngine, GswScheme
from tests.helpers import golden_json

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference not mounted")


def _ref():
    if REF not in sys.path:
        sys.path.append(REF)
    import fhefft.arith as arith
    import fhefft.fft as fft
    return arith, fft


@pytest.mark.parametrize("cfg", ["cfg0", "cfg4"])
def test_reference_circuits_on_gpu_engine(cfg):
    arith, fft = _ref()
    meta = golden_json(f"trace_{cfg}.json")
    eng = GpuEngine(GswScheme(EXACT_PARAMS), dry_run=True, record_trace=True)
    if cfg == "cfg0":
        x = np.random.default_rng(0).uniform(-1, 1, 8).astype(complex)
        sig = fft.input_signal(eng, x, arith.FixedFormat(16, 12))
    else:
        r = np.random.default_rng(4)
        x = r.uniform(-1, 1, 16) + 1j * r.uniform(-1, 1, 16)
        sig = fft.input_signal(eng, x, arith.FixedFormat(16, 12))
    fft.fft_1d(sig)                      # the reference's driver, butterflies, adders, multipliers
    ops = [t[:4] for t in eng.trace if t[0] in (0, 1)]
    dig = hashlib.sha256(np.asarray(ops, dtype="<i8").tobytes()).hexdigest()[:16]
    assert dig == meta["ops_digest"]
    assert (eng.nand_count, eng.max_depth) == (meta["nand_count"], meta["max_depth"])
