"""Host scheme layer (CPU): parameters, keys and encryption equal the reference."""

import numpy as np
import pytest

from paper_1611_08769_b200 import (DEFAULT0_PARAMS, DEFAULT_PARAMS, EXACT_PARAMS, Ciphertext,
                                   GswScheme, ParameterError, SchemeParams, decode_gadget_samples)
from paper_1611_08769_b200.errors import NoiseOverflowError
from tests.helpers import golden_json, golden_npz

PRESETS = {"exact": (EXACT_PARAMS, 1), "default": (DEFAULT_PARAMS, 1), "default0": (DEFAULT0_PARAMS, 2)}


@pytest.mark.parametrize("name", sorted(PRESETS))
def test_keys_encryptions_decryptions_match_reference(name):
    params, seed = PRESETS[name]
    kat = golden_npz(f"scheme_{name}.npz")
    meta = golden_json("scheme_kat.json")[name]
    assert params.digest() == meta["digest"]
    s = GswScheme(params)
    keys = s.keygen(seed)
    assert np.array_equal(keys.public_key, kat["pk"])
    assert np.array_equal(keys.secret_key, kat["sk"])
    rng = np.random.default_rng(7)
    cts = [s.encrypt_bit(keys.public_key, b, rng) for b in (0, 1, 1, 0, 1)]
    for i, c in enumerate(cts):
        assert np.array_equal(c.v, kat[f"ct{i}"])
        assert c.noise_est == meta["fresh_noise_est"] and c.level == 0
    assert [s.decrypt_bit(keys.secret_key, c) for c in cts] == meta["bits"]
    rows = np.stack([kat[k][params.n * params.ell + (params.q // 2).bit_length() - 1]
                     for k in ("n01", "n12", "x", "y", "nt")])
    got = s.decrypt_bits_from_rows(keys.secret_key, rows).tolist()
    assert got == [meta[k] for k in ("n01", "n12", "x", "y", "nt")]
    assert np.array_equal(s.trivial_encrypt_bit(1).v, kat["triv1"])


def test_matrix_round_trip():
    s = GswScheme(EXACT_PARAMS)
    keys = s.keygen(4)
    c = s.encrypt_bit(keys.public_key, 1, np.random.default_rng(0))
    m = c.matrix
    assert m.shape == (51, 51) and set(np.unique(m)) <= {0.0, 1.0}
    assert np.array_equal(Ciphertext.from_matrix(m, EXACT_PARAMS).v, c.v)


def test_params_validation_like_reference():
    with pytest.raises(ParameterError):
        SchemeParams(n=4, q=2**20, noise_bound=1, depth_budget=1)
    with pytest.raises(ParameterError):
        SchemeParams(n=4, q=2**20 - 1, noise_bound=2, depth_budget=3)
    p = SchemeParams(n=1, q=127, noise_bound=0, depth_budget=10**12)
    assert p.n_ct == 14 and DEFAULT_PARAMS.ell == 29 and DEFAULT_PARAMS.n_ct == 261


def test_gadget_decoder_extremes():
    q, bound = 2**29 - 3, (2**29 - 3) // 8
    for mu in (0, 1, 2**28, 2**29 - 4):
        for sign in (1, -1):
            xs = [((mu << j) + sign * (bound - 1)) % q for j in range(29)]
            assert decode_gadget_samples(xs, q, bound) == mu


def test_depth_budget_error_message():
    from paper_1611_08769_b200 import GpuEngine
    s = GswScheme(DEFAULT_PARAMS)
    eng = GpuEngine(s, dry_run=True)
    x = eng.input_bit(1)
    for _ in range(3):
        x = eng.nand(x, x)
    with pytest.raises(NoiseOverflowError, match="NAND at level 4 would exceed depth budget 3"):
        eng.nand(x, x)


@pytest.mark.parametrize("name", ["exact", "default"])
def test_ring_op_levels_and_noise_like_reference(name):
    """hom_add / hom_const_mult / hom_mult bookkeeping (fhe.py:352-379) vs the reference's
    recorded levels and noise estimates (host logic only; no device)."""
    from tests.helpers import golden_json
    meta = golden_json("ring_kat.json")[name]
    params = EXACT_PARAMS if name == "exact" else DEFAULT_PARAMS
    s = GswScheme(params)
    z = np.zeros((params.n_ct, params.k), dtype=np.uint32)
    fresh = Ciphertext(z, 0, meta["fresh_noise"], params)
    nb = Ciphertext(z, meta["nb_level"], meta["nb_noise"], params)
    r = meta["results"]
    assert list(s.add_meta(fresh, fresh)) == [r["add01"]["level"], r["add01"]["noise_est"]]
    assert list(s.add_meta(nb, fresh)) == [r["add_nb"]["level"], r["add_nb"]["noise_est"]]
    for key, a, b in (("mult03", fresh, fresh), ("mult_b_nb", fresh, nb), ("mult_nb_b", nb, fresh)):
        _, _, level, est = s.mult_meta(a, b)
        assert (level, est) == (r[key]["level"], r[key]["noise_est"]), key
    for i in range(len(meta["k_vals"])):
        src = fresh if i % 2 else nb
        assert r[f"cmult{i}"]["level"] == src.level
        assert r[f"cmult{i}"]["noise_est"] == min(params.n_ct * src.noise_est, params.q)


def test_wrong_key_raises_noise_overflow():
    """tests/test_fhe.py:175-184: decrypting with another key trips the noise check."""
    s = GswScheme(DEFAULT_PARAMS)
    keys, other = s.keygen(seed=1), s.keygen(seed=999)
    rng = np.random.default_rng(7)
    observed = 0
    for _ in range(16):
        ct = s.encrypt_bit(keys.public_key, 1, rng)
        try:
            s.decrypt_bit(other.secret_key, ct)
        except NoiseOverflowError:
            observed += 1
    assert observed >= 8
