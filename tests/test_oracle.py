"""The CPU oracle against the reference's own outputs (golden vectors made by
tests/golden/make_golden.py, which ran /root/reference)."""

import numpy as np
import pytest

from oracle import digest, fixedfft, gsw
from tests.helpers import FFT_CONFIGS, config_signal, golden_json, golden_npz, model_outputs

PRESETS = {"exact": (gsw.EXACT, 1), "default": (gsw.DEFAULT, 1), "default0": (gsw.DEFAULT0, 2)}


@pytest.mark.parametrize("name", sorted(PRESETS))
def test_oracle_scheme_known_answers(name):
    p, seed = PRESETS[name]
    kat = golden_npz(f"scheme_{name}.npz")
    meta = golden_json("scheme_kat.json")[name]
    pk, sk = gsw.keygen(p, seed)
    assert np.array_equal(pk, kat["pk"]) and np.array_equal(sk, kat["sk"])
    rng = np.random.default_rng(7)
    cts = [gsw.encrypt_compact(p, pk, b, rng) for b in (0, 1, 1, 0, 1)]
    for i, c in enumerate(cts):
        assert np.array_equal(c, kat[f"ct{i}"]), f"encryption {i}"
    assert [gsw.decrypt_bit_compact(p, sk, c) for c in cts] == meta["bits"]
    # compact NAND / NOT == the reference's values, including the swap the noise rule makes
    e = [meta["fresh_noise_est"]] * 5
    n01 = gsw.hom_nand_compact(p, cts[0], cts[1])
    n12 = gsw.hom_nand_compact(p, cts[1], cts[2])
    e_n = gsw.noise_after_nand(p, e[0], e[1])
    left, right = (n01, cts[3]) if e_n >= e[3] else (cts[3], n01)
    x = gsw.hom_nand_compact(p, left, right)
    left, right = (cts[4], n12) if e[4] >= e_n else (n12, cts[4])
    y = gsw.hom_nand_compact(p, left, right)
    nt = gsw.hom_not_compact(p, y)
    for nm, v in (("n01", n01), ("n12", n12), ("x", x), ("y", y), ("nt", nt)):
        assert np.array_equal(v, kat[nm]), nm
        assert gsw.decrypt_bit_compact(p, sk, v) == meta[nm]
    assert np.array_equal(gsw.hom_not_compact(p, nt), y)
    assert np.array_equal(kat["triv0"], np.zeros_like(kat["triv1"]))
    assert np.array_equal(kat["triv1"], gsw.gadget(p))


@pytest.mark.parametrize("p", [gsw.EXACT, gsw.DEFAULT], ids=["exact", "default"])
def test_compact_identity_equals_reference_matrix_algorithm(p):
    """hom_nand_compact == recompose(flatten(I - C1 C2)) of the literal reference algorithm."""
    pk, sk = gsw.keygen(p, 3)
    rng = np.random.default_rng(11)
    vs = [gsw.encrypt_compact(p, pk, int(b), rng) for b in rng.integers(0, 2, 6)]
    vs.append(gsw.hom_nand_compact(p, vs[0], vs[1]))          # non-fresh operands too
    vs.append(gsw.hom_not_compact(p, vs[2]))
    for i in range(len(vs)):
        for j in range(len(vs)):
            if (i + j) % 3:
                continue
            c1 = gsw.bits_of(vs[i], p).astype(np.float64)
            c2 = gsw.bits_of(vs[j], p).astype(np.float64)
            ref = gsw.hom_nand_matrix(p, c1, c2)
            assert np.array_equal(gsw.recompose(ref, p), gsw.hom_nand_compact(p, vs[i], vs[j]))
        ref_not = gsw.hom_not_matrix(p, gsw.bits_of(vs[i], p).astype(np.float64))
        assert np.array_equal(gsw.recompose(ref_not, p), gsw.hom_not_compact(p, vs[i]))


def test_bulk_draws_equal_sequential_draws():
    """encrypt_many's bulk integers(0,2,(c,N,m)) == c sequential (N,m) draws (fhe.py:229)."""
    p = gsw.DEFAULT
    r1 = np.random.default_rng(5)
    seq = np.stack([r1.integers(0, 2, (p.n_ct, p.m)) for _ in range(3)])
    r2 = np.random.default_rng(5)
    bulk = r2.integers(0, 2, (3, p.n_ct, p.m))
    assert np.array_equal(seq, bulk)
    assert r1.integers(0, 1 << 30) == r2.integers(0, 1 << 30)


def test_oracle_replays_cfg0_gate_by_gate():
    """Oracle encryptions + compact gates over the reference's cfg0 trace reproduce the
    reference's per-gate ciphertext digests (all 30,772 hom_nand/hom_not outputs)."""
    p = gsw.EXACT
    tr = golden_npz("trace_cfg0.npz")
    cts = golden_json("cts_cfg0.json")
    gd = golden_npz("cts_cfg0.npz")
    pk, _ = gsw.keygen(p, 0)
    rng, x = config_signal("cfg0")
    n_in = len(tr["inputs"])
    F, f = 16, 12
    re = fixedfft.encode_lanes(x.real[None], F, f)[0] % (1 << F)
    im = fixedfft.encode_lanes(x.imag[None], F, f)[0] % (1 << F)
    bits = []
    for pt in range(8):
        for word in (re[pt], im[pt]):
            bits.extend((int(word) >> b) & 1 for b in range(F))
    assert len(bits) == n_in
    wires = {}
    in_digests = []
    for w, bit in zip(tr["inputs"], bits):
        wires[int(w)] = gsw.encrypt_compact(p, pk, bit, rng)
        in_digests.append(digest.digest_compact(wires[int(w)]))
    assert digest.chain_digest(in_digests) == cts["inputs_chain"]
    ref_gate = [bytes(r).hex() for r in gd["gate_digests"].view(np.uint8).reshape(-1, 8)]
    got = []
    for (kind, l, r, o) in tr["ops"].tolist():
        if kind == 0:
            v = gsw.hom_nand_compact(p, wires[l], wires[r])
        else:
            v = gsw.hom_not_compact(p, wires[l])
        wires[o] = v
        got.append(digest.digest_compact(v))
    assert got[:200] == ref_gate[:200]
    assert digest.chain_digest(got) == cts["gates_chain"]


@pytest.mark.parametrize("cfg", ["cfg0", "cfg2", "cfg3", "cfg4"])
def test_integer_fft_model_matches_reference_cleartext_engine(cfg):
    want = golden_npz(f"clear_{cfg}.npz")["words"]
    lanes = FFT_CONFIGS[cfg][4]
    vals = np.array([config_signal(cfg, lane)[1] for lane in range(lanes)])
    assert np.array_equal(model_outputs(cfg, vals), want)


def test_integer_model_matches_reference_fhe_outputs():
    """cfg0's decrypted FHE outputs (real reference run) equal the model's words."""
    got = model_outputs("cfg0", config_signal("cfg0")[1][None])[0]
    assert got.tolist() == golden_json("cts_cfg0.json")["output_words"]


def _ring_cases(p, z):
    """(result name, op, operands in the order the reference call passed them)."""
    return [("add01", "add", z["ct0"], z["ct1"]), ("add23", "add", z["ct2"], z["ct3"]),
             ("add_nb", "add", z["nb"], z["b0"]), ("mult03", "mult", z["ct0"], z["ct3"]),
             ("mult_b_nb", "mult", z["b1"], z["nb"]), ("mult_nb_b", "mult", z["nb"], z["b0"])]


@pytest.mark.parametrize("name", ["exact", "default"])
def test_oracle_ring_ops_known_answers(name):
    """hom_add / hom_const_mult / hom_mult (fhe.py:352-379): the compact identities and the
    restated matrix algorithm both reproduce the reference's ciphertexts bit for bit."""
    meta = golden_json("ring_kat.json")[name]
    z = golden_npz(f"ring_{name}.npz")
    p = gsw.EXACT if name == "exact" else gsw.DEFAULT
    for res, op, a, b in _ring_cases(p, z):
        if op == "add":
            got = gsw.hom_add_compact(p, a, b)
            mat = gsw.hom_add_matrix(p, gsw.bits_of(a, p).astype(float), gsw.bits_of(b, p).astype(float))
        else:
            left, right = a, b
            # the reference swaps when the right operand is noisier (fhe.py:374-375)
            if res == "mult_b_nb" and meta["nb_noise"] > meta["fresh_noise"]:
                left, right = b, a
            got = gsw.hom_mult_compact(p, left, right)
            mat = gsw.hom_mult_matrix(p, gsw.bits_of(left, p).astype(float), gsw.bits_of(right, p).astype(float))
        assert np.array_equal(got, z[res]), res
        assert np.array_equal(gsw.bits_of(got, p), mat), res
    for i, k in enumerate(meta["k_vals"]):
        src = z["ct2"] if i % 2 else z["nb"]
        got = gsw.hom_const_mult_compact(p, src, k)
        assert np.array_equal(got, z[f"cmult{i}"]), k
        mat = gsw.hom_const_mult_matrix(p, gsw.bits_of(src, p).astype(float), k)
        assert np.array_equal(gsw.bits_of(got, p), mat), k
