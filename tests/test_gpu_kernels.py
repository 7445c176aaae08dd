"""GPU kernel parity: tcgen05 and SIMT level kernels vs the CPU oracle (bit-exact)."""

import numpy as np
import pytest

from oracle import gsw
from paper_1611_08769_b200 import DEFAULT_PARAMS, EXACT_PARAMS, GswScheme, SchemeParams
from paper_1611_08769_b200 import _native
from tests.helpers import golden_json, golden_npz

pytestmark = pytest.mark.gpu

ORACLE = {EXACT_PARAMS: gsw.EXACT, DEFAULT_PARAMS: gsw.DEFAULT}


def _ctx(params, kernel):
    s = GswScheme(params)
    ctx = s.ctx
    ctx.set_kernel(kernel)
    return s, ctx


def _random_cts(p, count, rng, extremes=True):
    v = rng.integers(0, p.q, (count, p.n_ct, p.k), dtype=np.int64)
    if extremes and count >= 4:
        v[0] = 0                      # all-zero (C = 0)
        v[1] = p.q - 1                # all bits set below q
        v[2] = gsw.gadget(gsw.Params(p.n, p.q, p.m, p.noise_bound, p.depth_budget))  # trivial 1
        v[3] = rng.integers(0, 2, v[3].shape)
    return v.astype(np.uint32)


def _oracle_nand(p, a, b, ca, cb):
    op = ORACLE[p]
    a = gsw.hom_not_compact(op, a) if ca else a.astype(np.int64)
    b = gsw.hom_not_compact(op, b) if cb else b.astype(np.int64)
    return gsw.hom_nand_compact(op, a, b)


@pytest.mark.parametrize("params", [DEFAULT_PARAMS, EXACT_PARAMS], ids=["default", "exact"])
@pytest.mark.parametrize("kernel,dbg", [(_native.KERNEL_TCGEN05, 0), (_native.KERNEL_TCGEN05, 2),
                                        (_native.KERNEL_TCGEN05, 4), (_native.KERNEL_TCGEN05, 6),
                                        (_native.KERNEL_SIMT, 0)],
                         ids=["tc-ws", "tc-ws-generic-epilogue", "tc-v2", "tc-v2-generic", "simt"])
def test_level_kernel_random_operands(params, kernel, dbg):
    """A 2-level program over random operands, all complement combinations, many lanes."""
    s, ctx = _ctx(params, kernel)
    ctx.set_debug(dbg)
    rng = np.random.default_rng(1234)
    lanes, n_in = 3, 8
    vals = _random_cts(params, n_in * lanes, rng)
    ctx.reserve(64 * lanes)
    ctx.write(np.arange(n_in * lanes, dtype=np.uint64), vals)
    ops = []
    flags_cycle = [0, 1, 2, 3]
    for i in range(n_in):                     # level 1: slots 8..15
        ops.append((i, (i * 3 + 1) % n_in, 8 + i, flags_cycle[i % 4]))
    lvl1 = len(ops)
    for i in range(6):                        # level 2 reads level-1 outputs and inputs
        ops.append((8 + i, (i + 5) % n_in if i % 2 else 8 + (i + 1) % 8, 16 + i, flags_cycle[(i + 1) % 4]))
    table = np.array(ops, dtype=np.uint32).view(_native.OP_DTYPE).reshape(-1)
    prog = ctx.program(table, [0, lvl1, len(ops)])
    prog.run(lanes)
    ctx.sync()
    v = vals.reshape(n_in, lanes, params.n_ct, params.k)
    store = {i: v[i] for i in range(n_in)}
    for (l, r, o, f) in ops:
        store[o] = np.stack([_oracle_nand(params, store[l][ln], store[r][ln], f & 1, f & 2)
                             for ln in range(lanes)])
    for o in sorted({op[2] for op in ops}):
        got = ctx.read(o * lanes + np.arange(lanes, dtype=np.uint64))
        assert np.array_equal(got.astype(np.int64), store[o]), f"slot {o}"


@pytest.mark.parametrize("params", [DEFAULT_PARAMS, EXACT_PARAMS], ids=["default", "exact"])
def test_nand_batch_and_not_batch_vs_oracle(params):
    s = GswScheme(params)
    rng = np.random.default_rng(99)
    a = _random_cts(params, 37, rng)
    b = _random_cts(params, 37, rng)
    got = s.ctx.nand_batch(a, b)
    for i in range(37):
        assert np.array_equal(got[i].astype(np.int64), _oracle_nand(params, a[i], b[i], 0, 0))
    nt = s.ctx.not_batch(a)
    for i in range(37):
        assert np.array_equal(nt[i].astype(np.int64), gsw.hom_not_compact(ORACLE[params], a[i]))


@pytest.mark.parametrize("name,params", [("default", DEFAULT_PARAMS), ("exact", EXACT_PARAMS)])
def test_scheme_hom_nand_reproduces_reference_ciphertexts(name, params):
    """GswScheme.hom_nand/hom_not on the GPU == the reference's ciphertexts (golden KAT)."""
    kat = golden_npz(f"scheme_{name}.npz")
    meta = golden_json("scheme_kat.json")[name]
    s = GswScheme(params)
    from paper_1611_08769_b200 import Ciphertext
    fresh = meta["fresh_noise_est"]
    cts = [Ciphertext(kat[f"ct{i}"], 0, fresh, params) for i in range(5)]
    n01 = s.hom_nand(cts[0], cts[1])
    n12 = s.hom_nand(cts[1], cts[2])
    x = s.hom_nand(n01, cts[3])
    y = s.hom_nand(cts[4], n12)
    nt = s.hom_not(y)
    for nm, c in (("n01", n01), ("n12", n12), ("x", x), ("y", y), ("nt", nt)):
        assert np.array_equal(c.v, kat[nm]), nm
    assert [n01.level, n12.level, x.level, y.level, nt.level] == meta["levels"]
    assert [n01.noise_est, n12.noise_est, x.noise_est, y.noise_est, nt.noise_est] == meta["noise_est"]
    batch = s.hom_nand_many([(cts[0], cts[1]), (n01, cts[3])])
    assert np.array_equal(batch[1].v, kat["x"])


def test_generic_params_use_simt_kernel():
    p = SchemeParams(n=3, q=2**13 - 1, m=8, noise_bound=0, depth_budget=10**9)
    s = GswScheme(p)
    assert s.ctx.kernel == "simt"
    rng = np.random.default_rng(5)
    a = rng.integers(0, p.q, (5, p.n_ct, p.k)).astype(np.uint32)
    b = rng.integers(0, p.q, (5, p.n_ct, p.k)).astype(np.uint32)
    op = gsw.Params(p.n, p.q, p.m, p.noise_bound, p.depth_budget)
    got = s.ctx.nand_batch(a, b)
    for i in range(5):
        assert np.array_equal(got[i].astype(np.int64), gsw.hom_nand_compact(op, a[i], b[i]))


def test_default_kernel_is_tcgen05_on_b200():
    assert GswScheme(DEFAULT_PARAMS).ctx.kernel == "tcgen05"
    assert GswScheme(EXACT_PARAMS).ctx.kernel == "tcgen05"


@pytest.mark.parametrize("pinned,packed", [(False, False), (True, False), (True, True), (False, True)],
                         ids=["pageable", "pinned", "pinned-packed", "pageable-packed"])
def test_run_host_streaming_matches_oracle(pinned, packed):
    """fhegpu_prog_run_host: XOR + AND compiled once at batch 1, then 1000 host lanes
    streamed in chunks of 96 (11 chunks: 3 regions reused, ragged last chunk)."""
    import torch
    from paper_1611_08769_b200 import Ciphertext, GpuEngine, and_, xor_
    p = DEFAULT_PARAMS
    op = ORACLE[p]
    s = GswScheme(p)
    keys = s.keygen(1)
    rng = np.random.default_rng(77)
    eng = GpuEngine(s, keys=keys, rng=rng, batch_size=1)
    seed_ct = s.encrypt_many(keys.public_key, [0, 1], rng)
    a = eng.input_values(seed_ct[0:1], noise_est=64)
    b = eng.input_values(seed_ct[1:2], noise_est=64)
    x, y = xor_(a, b), and_(a, b)
    prog = eng.flush()
    lanes = 1000
    bits = rng.integers(0, 2, (lanes, 2))
    va = s.encrypt_many(keys.public_key, bits[:, 0], rng).astype(np.uint32)
    vb = s.encrypt_many(keys.public_key, bits[:, 1], rng).astype(np.uint32)
    from paper_1611_08769_b200.fileio import pack_compact, unpack_compact
    ha, hb = (pack_compact(va, p), pack_compact(vb, p)) if packed else (va, vb)
    if pinned:
        ins = [torch.from_numpy(h.view(np.uint8 if packed else np.int32)).pin_memory() for h in (ha, hb)]
        outs = [torch.empty_like(ins[0]).pin_memory() for _ in range(2)]
        eng.run_host(prog, [(a, ins[0]), (b, ins[1])], [x, y], chunk_lanes=96, out=outs, packed=packed)
        ox, oy = (o.numpy() for o in outs)
    else:
        ox, oy = eng.run_host(prog, [(a, ha), (b, hb)], [x, y], chunk_lanes=96, packed=packed)
    if packed:                                # the reference's serialised bytes, bit-exact
        assert ox.shape == (lanes, (p.n_ct ** 2 + 7) // 8)
        ox, oy = unpack_compact(ox, p), unpack_compact(oy, p)
    else:
        ox, oy = ox.view(np.uint32), oy.view(np.uint32)
    for lane in list(range(0, lanes, 97)) + [lanes - 1]:
        A, B = va[lane].astype(np.int64), vb[lane].astype(np.int64)
        n1 = gsw.hom_nand_compact(op, A, B)
        want_x = gsw.hom_nand_compact(op, gsw.hom_nand_compact(op, n1, A), gsw.hom_nand_compact(op, n1, B))
        n2 = gsw.hom_nand_compact(op, A, B)
        want_y = gsw.hom_nand_compact(op, n2, n2)           # not_ = NAND(x, x) (gates.py)
        assert np.array_equal(ox[lane], want_x.astype(np.uint32)), lane
        assert np.array_equal(oy[lane], want_y.astype(np.uint32)), lane
    dec_x = [s.decrypt_bit(keys.secret_key, Ciphertext(ox[l], 3, 0, p)) for l in range(0, lanes, 7)]
    assert dec_x == list(bits[::7, 0] ^ bits[::7, 1])


@pytest.mark.parametrize("params", [DEFAULT_PARAMS, EXACT_PARAMS], ids=["default", "exact"])
def test_store_packed_io_matches_reference_serialisation(params):
    """fhegpu_store_{write,read}_packed == fileio.pack_compact / unpack_compact (EFT1 rows)."""
    from paper_1611_08769_b200.fileio import pack_compact
    s = GswScheme(params)
    ctx = s.ctx
    rng = np.random.default_rng(5)
    v = _random_cts(params, 300, rng)
    packed = np.ascontiguousarray(pack_compact(v, params))
    ctx.reserve(700)
    ctx.write_packed(17, len(v), packed.ctypes.data)
    assert np.array_equal(ctx.read(np.arange(17, 17 + len(v), dtype=np.uint64)), v)
    ctx.write(np.arange(400, 400 + len(v), dtype=np.uint64), v)
    back = np.empty_like(packed)
    ctx.read_packed(400, len(v), back.ctypes.data)
    assert np.array_equal(back, packed)


@pytest.mark.parametrize("name,params", [("default", DEFAULT_PARAMS), ("exact", EXACT_PARAMS)])
def test_ring_ops_reproduce_reference_ciphertexts(name, params):
    """GPU hom_add / hom_const_mult / hom_mult == the reference's ciphertexts (fhe.py:352-379)."""
    from paper_1611_08769_b200 import Ciphertext
    meta = golden_json("ring_kat.json")[name]
    z = golden_npz(f"ring_{name}.npz")
    s = GswScheme(params)
    fresh = lambda v: Ciphertext(v, 0, meta["fresh_noise"], params)          # noqa: E731
    ct = [fresh(z[f"ct{i}"]) for i in range(4)]
    b0, b1 = fresh(z["b0"]), fresh(z["b1"])
    nb = Ciphertext(z["nb"], meta["nb_level"], meta["nb_noise"], params)
    got = {"add01": s.hom_add(ct[0], ct[1]), "add23": s.hom_add(ct[2], ct[3]),
           "add_nb": s.hom_add(nb, b0), "mult03": s.hom_mult(ct[0], ct[3]),
           "mult_b_nb": s.hom_mult(b1, nb), "mult_nb_b": s.hom_mult(nb, b0)}
    for i, k in enumerate(meta["k_vals"]):
        got[f"cmult{i}"] = s.hom_const_mult(ct[2] if i % 2 else nb, k)
    for key, c in got.items():
        assert np.array_equal(c.v, z[key]), key
        assert (c.level, c.noise_est) == (meta["results"][key]["level"], meta["results"][key]["noise_est"]), key


def test_ring_ops_match_ring_oracle_like_reference_tests():
    """The reference's own ring tests (tests/test_fhe.py:134-172), on the GPU operators."""
    s = GswScheme(DEFAULT_PARAMS)
    keys = s.keygen(1)
    pk, sk = keys.public_key, keys.secret_key
    rng = np.random.default_rng(3)
    q = DEFAULT_PARAMS.q
    assert s.decrypt_value(sk, s.hom_add(s.encrypt_value(pk, 3, rng), s.encrypt_value(pk, 5, rng))) == 8
    m1, m2 = rng.integers(0, q, 40), rng.integers(0, q, 40)
    outs = s.hom_add_many([(s.encrypt_value(pk, int(a), rng), s.encrypt_value(pk, int(b), rng))
                           for a, b in zip(m1, m2)])
    assert [s.decrypt_value(sk, c) for c in outs] == [int((a + b) % q) for a, b in zip(m1, m2)]
    ct = s.encrypt_value(pk, 12345, rng)
    assert s.decrypt_value(sk, s.hom_const_mult(ct, 0)) == 0
    for _ in range(10):
        m, k = int(rng.integers(0, q)), int(rng.integers(0, q))
        out = s.hom_const_mult(s.encrypt_value(pk, m, rng), k)
        assert s.decrypt_value(sk, out) == (m * k) % q
    m1, m2 = rng.integers(0, 2 ** 15, 40), rng.integers(0, 2 ** 15, 40)
    outs = s.hom_mult_many([(s.encrypt_value(pk, int(a), rng), s.encrypt_value(pk, int(b), rng))
                            for a, b in zip(m1, m2)])
    assert [s.decrypt_value(sk, c) for c in outs] == [int((a * b) % q) for a, b in zip(m1, m2)]


def test_plain_c_abi_reproduces_reference_nand():
    """C program over the C ABI (no Python in the loop): hom_nand of two reference
    ciphertexts equals the reference's output; hom_not twice is the identity."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = subprocess.run([os.path.join(root, "tests", "c", "abi_kat"),
                          os.path.join(root, "tests", "golden", "kat_default_nand.bin")],
                         capture_output=True, text=True, timeout=120)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "== reference" in res.stdout


@pytest.mark.parametrize("n,q", [(3, 2 ** 13 - 1), (5, 2 ** 20 + 7), (8, 2 ** 31 - 1)])
def test_engine_fft_on_other_parameter_sets(n, q):
    """Any valid SchemeParams runs through the engine (the CUDA-core kernel where no tcgen05
    instance exists: N = 12, 126, 279 here): a noise-free 4-point Q8.8 FFT over 8 lanes
    decrypts to the integer model's words."""
    from paper_1611_08769_b200 import FixedFormat, GpuEngine, fft_1d, input_signal
    from paper_1611_08769_b200.fft import read_signal_ints
    from oracle import fixedfft
    p = SchemeParams(n=n, q=q, m=8, noise_bound=0, depth_budget=10 ** 9)
    s = GswScheme(p)
    keys = s.keygen(2)
    rng = np.random.default_rng(9)
    vals = rng.uniform(-1, 1, (8, 4)) + 1j * rng.uniform(-1, 1, (8, 4))
    eng = GpuEngine(s, keys=keys, rng=rng, batch_size=8, device_encrypt=(p.n_ct * p.m) % 2 == 0)
    out = fft_1d(input_signal(eng, vals, FixedFormat(16, 8)))
    got = read_signal_ints(eng, out)
    re = fixedfft.encode_lanes(vals.real, 16, 8)
    im = fixedfft.encode_lanes(vals.imag, 16, 8)
    want = fixedfft.interleave(*fixedfft.fft_1d(re, im, 16, 8))
    assert np.array_equal(got, want)
