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


def test_resident_slot_order():
    """fhegpu_res_slot_order (host only): every (gate, lane) slot once, each lane's gates in plan
    order, reuse flags only where slot t - 2 is the lane's previous gate with an identical operand;
    the gate benchmark's XOR + AND reuses both operands of its second NAND and the left operand
    of its fourth in every lane, with no operand produced fewer than 5 slots back."""
    import numpy as np

    from paper_1611_08769_b200 import DEFAULT0_PARAMS, DEFAULT_PARAMS, GswScheme
    from paper_1611_08769_b200.engine import GpuEngine
    from paper_1611_08769_b200.gates import and_, nor_, not_, or_, xnor_, xor_

    def check(plan, lanes):
        order = _native.res_slot_order(plan, lanes)
        ow = [(int(c) & 7, (int(c) >> 3) & 3) for c in order]
        assert sorted(ow) == sorted((o, w) for o in range(len(plan)) for w in range(lanes))
        for w in range(lanes):
            assert [o for o, ww in ow if ww == w] == list(range(len(plan)))
        for t, c in enumerate(order):
            o, w = ow[t]
            if c & 96:
                assert t >= 2 and ow[t - 2] == (o - 1, w)
                for bit, kind, idx, prod, m in ((32, "lkind", "lidx", "lprod", 1), (64, "rkind", "ridx", "rprod", 2)):
                    if c & bit:
                        a, b = plan[o], plan[o - 1]
                        assert a[kind] == b[kind] and (a["flags"] & m) == (b["flags"] & m)
                        assert (a[prod] == b[prod]) if a[kind] else (a[idx] == b[idx])
        return order, ow

    eng = GpuEngine(GswScheme(DEFAULT_PARAMS), dry_run=True, batch_size=64)
    a, b = eng.input_bit(1), eng.input_bit(0)
    xor_(a, b), and_(a, b)
    eng.flush()
    plan = GpuEngine._resident_plan(eng.dry_programs[-1])[0]
    order, ow = check(plan, 3)
    assert sum(bool(c & 32) for c in order) == 6 and sum(bool(c & 64) for c in order) == 3
    pos = {s: t for t, s in enumerate(ow)}
    for (o, w), t in pos.items():
        for kind, prod in (("lkind", "lprod"), ("rkind", "rprod")):
            if plan[o][kind]:
                assert t - pos[(int(plan[o][prod]), w)] >= 5
    rng = np.random.default_rng(5)
    gates = [not_, and_, or_, xor_, nor_, xnor_]
    done = 0
    for trial in range(30):
        eng = GpuEngine(GswScheme(DEFAULT0_PARAMS), dry_run=True, batch_size=32)
        pool = [eng.input_bit(int(rng.integers(0, 1 << 31))) for _ in range(int(rng.integers(1, 4)))]
        for _ in range(int(rng.integers(1, 4))):
            g = gates[int(rng.integers(0, len(gates)))]
            p1, p2 = pool[int(rng.integers(0, len(pool)))], pool[int(rng.integers(0, len(pool)))]
            pool.append(g(p1) if g is not_ else g(p1, p2))
        eng.flush()
        res = GpuEngine._resident_plan(eng.dry_programs[-1]) if eng.dry_programs else None
        if res is None:
            continue
        for lanes in (1, 2, 3, 4):
            check(res[0], lanes)
        done += 1
    assert done >= 10
