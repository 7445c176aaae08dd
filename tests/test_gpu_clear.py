"""Bitsliced cleartext engine on the GPU (GpuClearEngine) vs the reference CleartextEngine.

Reference: engine.py:69-121 (protocol, fold rules, lane packing); harness.py:122-198 (the
error experiments it serves).  Goldens: decrypted-output words the reference's own
CleartextEngine produced (tests/golden/clear_cfg*.npz) and its gate counts (trace_cfg*.json).
"""

import numpy as np
import pytest

from paper_1611_08769_b200 import FixedFormat, GpuClearEngine, fft_1d, fft_2d, input_signal
from paper_1611_08769_b200.errors import UsageError
from paper_1611_08769_b200.fft import read_signal_ints
from paper_1611_08769_b200.gates import and_, nor_, not_, or_, xnor_, xor_
from tests.helpers import FFT_CONFIGS, config_signal, golden_json, golden_npz, model_outputs

pytestmark = pytest.mark.gpu


def _fft(eng, cfg, values):
    _, _, (F, f), dims, _ = FFT_CONFIGS[cfg]
    sig = input_signal(eng, values, FixedFormat(F, f), dims=dims if isinstance(dims, tuple) else None)
    return fft_2d(sig) if isinstance(dims, tuple) else fft_1d(sig)


@pytest.mark.parametrize("cfg", ["cfg0", "cfg2", "cfg3", "cfg4"])
def test_fft_configs_equal_reference_cleartext_engine(cfg):
    lanes = FFT_CONFIGS[cfg][4]
    vals = np.array([config_signal(cfg, lane)[1] for lane in range(lanes)])
    eng = GpuClearEngine(batch_size=lanes)
    out = _fft(eng, cfg, vals if lanes > 1 else vals[0])
    got = read_signal_ints(eng, out)
    assert np.array_equal(got, golden_npz(f"clear_{cfg}.npz")["words"])
    tr = golden_json(f"trace_{cfg}.json")
    assert (eng.nand_count, eng.max_depth) == (tr["nand_count"], tr["max_depth"])
    assert eng.launches == tr["max_depth"]                       # one launch per level


def test_many_lanes_against_integer_model():
    """200,003 random 16-point signals (ragged last word) in one pass vs the integer oracle."""
    lanes = 200_003
    rng = np.random.default_rng(42)
    vals = rng.uniform(-1, 1, (lanes, 16)) + 1j * rng.uniform(-1, 1, (lanes, 16))
    eng = GpuClearEngine(batch_size=lanes)
    out = _fft(eng, "cfg4", vals)
    got = read_signal_ints(eng, out)
    assert np.array_equal(got, model_outputs("cfg4", vals))


def test_gates_truth_tables_and_costs():
    """Every gate on all four input pairs as lanes; NAND costs as gates.py:9-34."""
    eng = GpuClearEngine(batch_size=4)
    a, b = eng.input_bit(0b1100), eng.input_bit(0b1010)
    cases = [(not_, (a,), 0b0011, 1), (and_, (a, b), 0b1000, 2), (or_, (a, b), 0b1110, 3),
             (xor_, (a, b), 0b0110, 4), (nor_, (a, b), 0b0001, 4), (xnor_, (a, b), 0b1001, 5)]
    for fn, args, want, cost in cases:
        before = eng.nand_count
        h = fn(*args)
        assert eng.read_back(h) == want, fn.__name__
        assert eng.nand_count - before == cost, fn.__name__


def test_folding_and_constants_like_reference():
    eng = GpuClearEngine(batch_size=3)
    x = eng.input_bit(0b101)
    one, zero = eng.constant(1), eng.constant(0)
    assert eng.read_back(eng.nand(x, one)) == 0b010          # NOT x, gate-free
    assert eng.read_back(eng.nand(zero, x)) == 0b111         # constant 1
    assert eng.read_back(eng.nand(one, one)) == 0
    assert eng.nand_count == 0 and eng.max_depth == 0
    with pytest.raises(UsageError):
        eng.input_bit(0b1000)
    with pytest.raises(UsageError):
        eng.constant(2)
    other = GpuClearEngine(batch_size=3)
    with pytest.raises(UsageError):
        eng.nand(x, other.input_bit(1))


def test_backend_equivalence_random_circuits_and_lanes():
    """Random gate circuits agree bit for bit across GpuClearEngine (many lanes), the GPU
    FHE engine (EXACT) and packed-int cleartext evaluation (tests/test_engine.py:100-123)."""
    from paper_1611_08769_b200 import EXACT_PARAMS, GpuEngine, GswScheme
    scheme = GswScheme(EXACT_PARAMS)
    keys = scheme.keygen(1)
    rng = np.random.default_rng(123)
    ops = [not_, and_, or_, xor_, nor_, xnor_]
    lanes = 77
    for _ in range(3):
        clear = GpuClearEngine(batch_size=lanes)
        fhe = GpuEngine(scheme, keys=keys, rng=np.random.default_rng(5), batch_size=lanes,
                        device_encrypt=True)
        masks = [int(m) for m in rng.integers(0, 2, (6, lanes)) @ (1 << np.arange(lanes, dtype=object))]
        pool_c = [clear.input_bit(m) for m in masks]
        pool_f = [fhe.input_bit(m) for m in masks]
        pool_v = list(masks)                                    # packed-int truth
        full = (1 << lanes) - 1
        py = {not_: lambda a, b: full ^ a, and_: lambda a, b: a & b, or_: lambda a, b: a | b,
              xor_: lambda a, b: a ^ b, nor_: lambda a, b: full ^ (a | b), xnor_: lambda a, b: full ^ (a ^ b)}
        for _ in range(40):
            op = ops[rng.integers(0, len(ops))]
            i, j = rng.integers(0, len(pool_c), 2)
            if op is not_:
                pool_c.append(op(pool_c[i]))
                pool_f.append(op(pool_f[i]))
            else:
                pool_c.append(op(pool_c[i], pool_c[j]))
                pool_f.append(op(pool_f[i], pool_f[j]))
            pool_v.append(py[op](pool_v[i], pool_v[j]))
        assert clear.nand_count == fhe.nand_count <= 200
        assert clear.max_depth == fhe.max_depth
        assert clear.read_back_many(pool_c) == fhe.read_back_many(pool_f) == pool_v


def test_mul_const_matches_mul_fixed_bit_for_bit():
    """tests/test_arith.py:214-223 at scale: a plaintext-constant multiply equals the
    ciphertext-word multiply bit for bit (4096 lanes per constant, bitsliced engine)."""
    from paper_1611_08769_b200 import mul_const, mul_fixed
    from paper_1611_08769_b200.arith import input_word
    rng = np.random.default_rng(7)
    fmt = FixedFormat(32, 16)
    for _ in range(6):
        c = float(rng.uniform(-1, 1))
        xs = list(rng.uniform(-1, 1, 4096))
        eng = GpuClearEngine(batch_size=4096)
        x = input_word(eng, xs, fmt)
        via_const = mul_const(x, c)
        via_ct = mul_fixed(x, input_word(eng, [c] * 4096, fmt))
        assert eng.read_back_many(list(via_const.bits)) == eng.read_back_many(list(via_ct.bits))


def test_random_circuits_tiled_equals_levels_and_clear():
    """Random gate circuits (all gate types, complemented operands; only 6 outputs kept, the
    rest temporaries with many sinks -> SSA, no ring) over 2048 lanes: the tiled dataflow schedule, level launches and the
    bitsliced cleartext engine agree bit for bit (DEFAULT dims, noise-free: default0)."""
    from paper_1611_08769_b200 import DEFAULT0_PARAMS, GpuEngine, GswScheme
    scheme = GswScheme(DEFAULT0_PARAMS)
    keys = scheme.keygen(3)
    lanes = 2048
    rng = np.random.default_rng(11)
    ops = [not_, and_, or_, xor_, nor_, xnor_]
    plan = [(int(rng.integers(0, len(ops))), int(rng.integers(0, 10 ** 6)), int(rng.integers(0, 10 ** 6)))
            for _ in range(30)]
    bits = rng.integers(0, 2, (lanes, 5))
    results = {}
    for name in ("levels", "tiled", "clear"):
        if name == "clear":
            eng = GpuClearEngine(batch_size=lanes)
            pool = eng.input_block(bits)
        else:
            eng = GpuEngine(scheme, keys=keys, rng=np.random.default_rng(1), batch_size=lanes,
                            device_encrypt=True, schedule=name)
            pool = eng.input_block(bits)
        for k, i, j in plan:
            a, b = pool[i % len(pool)], pool[j % len(pool)]
            pool.append(ops[k](a) if ops[k] is not_ else ops[k](a, b))
        keep = pool[-6:]
        del pool, a, b                        # the rest become temporaries of the program
        if name == "tiled":
            prog = eng.flush()
            assert prog.tile_lanes == 128
        results[name] = eng.read_back_many(keep)
        if name != "clear":
            results[name + "_ct"] = eng.node_values([h for h in keep if not h.const])
    assert results["levels"] == results["tiled"] == results["clear"]
    assert np.array_equal(results["levels_ct"], results["tiled_ct"])


@pytest.mark.gpu
def test_random_deep_circuit_queue_equals_levels():
    """A random deep circuit (600 gates of every type, operands drawn with a bias to the
    newest wires -> long dependency chains, plus high-fan-out early wires) over 7 lanes: the
    ready-queue launch, the static dataflow launch and level launches give identical
    ciphertexts and the bitsliced cleartext engine's bits."""
    from paper_1611_08769_b200 import DEFAULT0_PARAMS, GpuEngine, GswScheme
    scheme = GswScheme(DEFAULT0_PARAMS)
    keys = scheme.keygen(5)
    lanes = 7
    rng = np.random.default_rng(23)
    ops = [not_, and_, or_, xor_, nor_, xnor_]
    plan = []
    for n in range(600):
        k = int(rng.integers(0, len(ops)))
        pick = lambda: int(rng.integers(0, 6)) if rng.random() < 0.15 else -1 - int(rng.integers(0, 4))
        plan.append((k, pick(), pick()))
    bits = rng.integers(0, 2, (lanes, 6))
    results = {}
    for name in ("levels", "queue", "dataflow", "clear"):
        if name == "clear":
            eng = GpuClearEngine(batch_size=lanes)
        else:
            eng = GpuEngine(scheme, keys=keys, rng=np.random.default_rng(2), batch_size=lanes,
                            device_encrypt=True, schedule=name)
        pool = eng.input_block(bits)
        for k, i, j in plan:
            a, b = pool[i], pool[j]
            pool.append(ops[k](a) if ops[k] is not_ else ops[k](a, b))
        keep = pool[-8:] + pool[6:10]
        del pool, a, b
        results[name] = eng.read_back_many(keep)
        if name != "clear":
            assert eng.max_depth > 64                       # deep enough for 'auto' to pick the queue
            results[name + "_ct"] = eng.node_values([h for h in keep if not h.const])
    assert results["levels"] == results["queue"] == results["dataflow"] == results["clear"]
    assert np.array_equal(results["levels_ct"], results["queue_ct"])
    assert np.array_equal(results["levels_ct"], results["dataflow_ct"])


@pytest.mark.gpu
@pytest.mark.parametrize("lanes", [1, 2, 5])
def test_resident_tiny_batches(lanes):
    """Lane-resident launches with fewer lanes than one 3-lane group or a partial last group."""
    from paper_1611_08769_b200 import DEFAULT_PARAMS, GpuEngine, GswScheme
    scheme = GswScheme(DEFAULT_PARAMS)
    keys = scheme.keygen(7)
    bits = np.random.default_rng(lanes).integers(0, 2, (lanes, 2))
    eng = GpuEngine(scheme, keys=keys, rng=np.random.default_rng(3), batch_size=lanes, schedule="resident",
                    device_encrypt=True)
    a, b = eng.input_block(bits)
    x, y = xor_(a, b), and_(a, b)
    prog = eng.flush()
    assert prog.launches == 1
    got = eng.read_back_bits([x, y])
    assert (got[0] == (bits[:, 0] ^ bits[:, 1])).all() and (got[1] == (bits[:, 0] & bits[:, 1])).all()


@pytest.mark.gpu
def test_queue_tiny_programs_and_fallback():
    """Queue launches with fewer items than SMs (a 3-gate program, one lane) and a queue
    request on a parameter set without the warp-specialised kernel (EXACT: level launches)."""
    from paper_1611_08769_b200 import DEFAULT0_PARAMS, EXACT_PARAMS, GpuEngine, GswScheme
    for params in (DEFAULT0_PARAMS, EXACT_PARAMS):
        scheme = GswScheme(params)
        keys = scheme.keygen(7)
        for bits in ((0, 1), (1, 1)):
            eng = GpuEngine(scheme, keys=keys, rng=np.random.default_rng(3), schedule="queue",
                            device_encrypt=True)
            a, b = eng.input_bit(bits[0]), eng.input_bit(bits[1])
            y = xor_(and_(a, b), b)
            assert eng.read_back(y) == ((bits[0] & bits[1]) ^ bits[1])
