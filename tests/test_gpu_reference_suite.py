"""The reference's own tests for this path, run against the GPU engines.

Mirrors tests/test_fhe.py:55-218 (scheme), tests/test_arith.py:251-276 (FHE arithmetic) and
tests/test_acceptance.py:33-125 (criteria 1-3) of the reference, with GswScheme.hom_nand on
the tcgen05 kernels, GpuEngine (lazy levelised FHE) and GpuClearEngine (bitsliced cleartext).
Encrypted work is batched as lanes where the reference loops one circuit at a time.
"""

import math
import time

import numpy as np
import pytest

from paper_1611_08769_b200 import (DEFAULT_PARAMS, EXACT_PARAMS, FixedFormat, GpuClearEngine,
                                   GpuEngine, GswScheme, NoiseOverflowError, add, mul_fixed,
                                   mul_integer, sub)
from paper_1611_08769_b200.arith import input_word, read_word
from paper_1611_08769_b200.gates import and_, nor_, not_, or_, xnor_, xor_
from tests.helpers import int_word, word_ints, wrap

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def default():
    s = GswScheme(DEFAULT_PARAMS)
    return s, s.keygen(seed=1)


@pytest.fixture(scope="module")
def exact():
    s = GswScheme(EXACT_PARAMS)
    return s, s.keygen(seed=1)


def test_bit_round_trip_and_nand_truth_table(default):
    s, k = default
    rng = np.random.default_rng(0)
    bits = rng.integers(0, 2, 200)
    assert [s.decrypt_bit(k.secret_key, s.encrypt_bit(k.public_key, int(b), rng)) for b in bits] == list(bits)
    for a in (0, 1):
        for b in (0, 1):
            out = s.hom_nand(s.encrypt_bit(k.public_key, a, rng), s.encrypt_bit(k.public_key, b, rng))
            assert out.level == 1
            assert s.decrypt_bit(k.secret_key, out) == 1 - (a and b)


def test_nand_noise_growth_bounded(default):
    s, k = default
    p = s.params
    rng = np.random.default_rng(1)
    for a, b in ((0, 0), (0, 1), (1, 0), (1, 1)):
        c1, c2 = s.encrypt_bit(k.public_key, a, rng), s.encrypt_bit(k.public_key, b, rng)
        n_in = max(s.measure_noise(k.secret_key, c1), s.measure_noise(k.secret_key, c2))
        n_out = s.measure_noise(k.secret_key, s.hom_nand(c1, c2))
        assert n_out <= (p.n_ct + 1) * n_in + p.m * p.noise_bound


def test_depth_budget_trivial_and_not(default):
    s, k = default
    rng = np.random.default_rng(2)
    ct = s.encrypt_bit(k.public_key, 1, rng)
    for _ in range(s.params.depth_budget):
        ct = s.hom_nand(ct, ct)
    with pytest.raises(NoiseOverflowError):
        s.hom_nand(ct, ct)
    for b in (0, 1):
        t = s.trivial_encrypt_bit(b)
        assert s.decrypt_bit(k.secret_key, t) == b and s.measure_noise(k.secret_key, t) == 0
    ct = s.encrypt_bit(k.public_key, 1, rng)
    inv = s.hom_not(ct)
    assert inv.level == ct.level and s.decrypt_bit(k.secret_key, inv) == 0
    assert s.measure_noise(k.secret_key, inv) == s.measure_noise(k.secret_key, ct)


def test_exact_params_deep_chain(exact):
    s, k = exact
    rng = np.random.default_rng(3)
    ct, expected = s.encrypt_bit(k.public_key, 0, rng), 0
    for _ in range(64):
        ct = s.hom_nand(ct, ct)
        expected = 1 - expected
    assert s.decrypt_bit(k.secret_key, ct) == expected
    assert s.measure_noise(k.secret_key, ct) == 0


def test_criterion_1_fhe_correctness():
    """1000/1000 round trips and 1000/1000 NAND rows exact, DEFAULT params, < 60 s."""
    start = time.perf_counter()
    s = GswScheme(DEFAULT_PARAMS)
    k = s.keygen(seed=10)
    rng = np.random.default_rng(10)
    bits = rng.integers(0, 2, 1000)
    cts = s.encrypt_many(k.public_key, bits, rng)
    from paper_1611_08769_b200 import Ciphertext
    fresh = s.params.m * s.params.noise_bound
    wrap_ct = lambda v: Ciphertext(v, 0, fresh, s.params)            # noqa: E731
    assert sum(s.decrypt_bit(k.secret_key, wrap_ct(v)) == b for v, b in zip(cts, bits)) == 1000
    pairs, want = [], []
    for a, b in ((0, 0), (0, 1), (1, 0), (1, 1)):
        v = s.encrypt_many(k.public_key, [a, b] * 250, rng)
        pairs += [(wrap_ct(v[2 * i]), wrap_ct(v[2 * i + 1])) for i in range(250)]
        want += [1 - (a and b)] * 250
    outs = s.hom_nand_many(pairs)                                         # one launch
    assert sum(s.decrypt_bit(k.secret_key, o) == w for o, w in zip(outs, want)) == 1000
    assert time.perf_counter() - start < 60.0


GATES = [(not_, None, 1), (and_, lambda a, b: a & b, 2), (or_, lambda a, b: a | b, 3),
         (xor_, lambda a, b: a ^ b, 4), (nor_, lambda a, b: 1 - (a | b), 4),
         (xnor_, lambda a, b: 1 - (a ^ b), 5)]


def test_criterion_2_gate_layer():
    """Six gates exhaustive on both GPU backends, NAND costs 1/2/3/4/4/5."""
    s = GswScheme(DEFAULT_PARAMS)
    k = s.keygen(seed=11)
    rng = np.random.default_rng(11)
    for gate, oracle, cost in GATES:
        for a in (0, 1):
            for b in ((0, 1) if oracle else (None,)):
                want = oracle(a, b) if oracle else 1 - a
                for eng in (GpuClearEngine(), GpuEngine(s, keys=k, rng=rng)):
                    args = [eng.input_bit(a)] + ([eng.input_bit(b)] if oracle else [])
                    assert eng.read_back(gate(*args)) == want
                    assert eng.nand_count == cost


def test_criterion_3_arithmetic():
    """Exhaustive 8-bit add/sub and 6-bit multiply (bitsliced); 50 encrypted 8-bit adds and
    20 encrypted 4-bit multiplies -- as lanes of one netlist each -- within the cost bounds."""
    pairs = [(a, b) for a in range(256) for b in range(256)]
    eng = GpuClearEngine(batch_size=len(pairs))
    x, y = int_word(eng, [p[0] for p in pairs], 8), int_word(eng, [p[1] for p in pairs], 8)
    n0 = eng.nand_count
    sums = add(x, y)
    assert eng.nand_count - n0 <= 36 * 8
    assert word_ints(eng, sums, signed=False) == [(a + b) % 256 for a, b in pairs]
    assert word_ints(eng, sub(x, y), signed=False) == [(a - b) % 256 for a, b in pairs]
    mpairs = [(a, b) for a in range(-32, 32) for b in range(-32, 32)]
    eng6 = GpuClearEngine(batch_size=len(mpairs))
    prods = mul_integer(int_word(eng6, [p[0] for p in mpairs], 6), int_word(eng6, [p[1] for p in mpairs], 6))
    assert eng6.nand_count <= 288 * 6 ** 2 * math.log2(6)
    assert word_ints(eng6, prods) == [wrap(a * b, 6) for a, b in mpairs]

    s = GswScheme(EXACT_PARAMS)
    k = s.keygen(seed=12)
    rng = np.random.default_rng(12)
    ab = rng.integers(-128, 128, (50, 2))
    fhe = GpuEngine(s, keys=k, rng=np.random.default_rng(13), batch_size=50, device_encrypt=True)
    out = add(int_word(fhe, ab[:, 0], 8), int_word(fhe, ab[:, 1], 8))
    assert fhe.nand_count <= 36 * 8
    assert word_ints(fhe, out) == [wrap(int(a) + int(b), 8) for a, b in ab]
    mb = rng.integers(-8, 8, (20, 2))
    fhe = GpuEngine(s, keys=k, rng=np.random.default_rng(14), batch_size=20, device_encrypt=True)
    out = mul_integer(int_word(fhe, mb[:, 0], 4), int_word(fhe, mb[:, 1], 4))
    assert fhe.nand_count <= 288 * 4 ** 2 * math.log2(4)
    assert word_ints(fhe, out) == [wrap(int(a) * int(b), 4) for a, b in mb]


def test_fixed_point_sub_and_mul_fhe_equals_clear(exact):
    """tests/test_arith.py:268-279: FHE and cleartext agree on fixed-point sub / mul."""
    s, k = exact
    fmt = FixedFormat(8, 4)
    for ex, ey in ((0.75, 0.5), (-0.5, 0.25)):
        fhe = GpuEngine(s, keys=k, rng=np.random.default_rng(5))
        clear = GpuClearEngine()
        for op in (sub, mul_fixed):
            got_f = read_word(fhe, op(input_word(fhe, ex, fmt), input_word(fhe, ey, fmt)))
            got_c = read_word(clear, op(input_word(clear, ex, fmt), input_word(clear, ey, fmt)))
            assert got_f == got_c
