"""Generate the golden vectors under tests/golden/ by RUNNING THE REFERENCE.

Run only in the build container, where the reference package is importable
from /root/reference/pkg/src (it does not exist on the GPU box; the committed
outputs travel instead):

    python tests/golden/make_golden.py scheme        # scheme known answers
    python tests/golden/make_golden.py trace cfg0    # op sequences (any cfg)
    python tests/golden/make_golden.py cts cfg0      # per-gate ciphertext digests
    python tests/golden/make_golden.py clear cfg4    # decrypted outputs (cleartext engine)
    python tests/golden/make_golden.py ring          # Z_q ring ops (hom_add / const_mult / mult)

The reference is instrumented, never modified: the methods of one
``GswScheme`` instance are wrapped so that every ciphertext the reference
produces gets a wire number (creation order) and, optionally, a digest of its
compact form (``oracle/digest.py``).  Operand order is recorded AFTER the
reference's own swap rule (``fhe.py:336-337``), i.e. the order in which the
reference multiplied.

Config protocols (BASELINE.json configs 0..4):
  cfg0  EXACT,    keygen(0), rng=default_rng(0), x=rng.uniform(-1,1,8) real, Q4.12, fft_1d
  cfg1  DEFAULT,  keygen(1), rng=default_rng(1), bits=rng.integers(0,2,(2^20,2)),
        encrypt a,b pair-major with rng; per pair xor_(a,b) then and_(a,b)
  cfg2  default0, keygen(2), rng=default_rng(2), re,im=rng.uniform(-1,1,32) each, Q8.24, fft_1d
  cfg3  default0, keygen(3), rng=default_rng(3), pix=rng.integers(0,256,(8,8)), x=pix/255,
        Q9.7, fft_2d (row-major 8x8)
  cfg4  default0, keygen(4), lane i: rng_i=default_rng(4+i), re,im=rng_i.uniform(-1,1,16),
        Q4.12, fft_1d, 1024 lanes
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))
sys.path.insert(0, "/root/reference/pkg/src")

from fhefft import arith, fft, gates  # noqa: E402
from fhefft.engine import CleartextEngine, FheEngine  # noqa: E402
from fhefft.fhe import DEFAULT_PARAMS, EXACT_PARAMS, GswScheme, SchemeParams  # noqa: E402

from oracle.digest import chain_digest, compact_from_matrix, digest_compact  # noqa: E402

DEFAULT0 = SchemeParams(n=8, q=2**29 - 3, m=32, noise_bound=0, depth_budget=10**9)
PAIRS_FULL = 1 << 20


class Tap:
    """Numbers (and optionally hashes) every ciphertext a scheme instance makes."""

    def __init__(self, scheme: GswScheme, hash_cts: bool):
        self.scheme = scheme
        self.hash_cts = hash_cts
        self.n_wires = 0
        self.inputs = []        # wire ids of fresh encryptions, in draw order
        self.input_digests = []
        self.ops = []           # (kind 0=nand 1=not, left, right, out)
        self.levels = []
        self.digests = []
        p = scheme.params
        self._k, self._ell = p.n + 1, p.ell
        enc, nand, neg = scheme.encrypt_bit, scheme.hom_nand, scheme.hom_not

        def encrypt_bit(pk, bit, rng):
            ct = enc(pk, bit, rng)
            ct._wire = self._new()
            self.inputs.append(ct._wire)
            if hash_cts:
                self.input_digests.append(self._dig(ct))
            return ct

        def hom_nand(c1, c2):
            swapped = c2.noise_est > c1.noise_est      # the rule of fhe.py:336
            left, right = (c2, c1) if swapped else (c1, c2)
            out = nand(c1, c2)
            out._wire = self._new()
            self.ops.append((0, left._wire, right._wire, out._wire))
            self.levels.append(out.level)
            if hash_cts:
                self.digests.append(self._dig(out))
            return out

        def hom_not(c):
            out = neg(c)
            out._wire = self._new()
            self.ops.append((1, c._wire, c._wire, out._wire))
            self.levels.append(out.level)
            if hash_cts:
                self.digests.append(self._dig(out))
            return out

        scheme.encrypt_bit = encrypt_bit
        scheme.hom_nand = hom_nand
        scheme.hom_not = hom_not

    def _new(self):
        w = self.n_wires
        self.n_wires += 1
        return w

    def _dig(self, ct):
        return digest_compact(compact_from_matrix(ct.matrix, self._k, self._ell))


def _out_wires(words):
    """Wire id of every output bit (-1 const 0, -2 const 1)."""
    out = []
    for w in words:
        for h in w.bits:
            if h.const:
                out.append(-2 if h.plain else -1)
            else:
                out.append(h.ct._wire)
    return out


def _signal_words(sig):
    words = []
    for pt in sig.points:
        words.extend([pt.re, pt.im])
    return words


def _word_ints(engine, words, lanes=1):
    """Raw two's-complement integer of every word (per lane)."""
    res = np.zeros((lanes, len(words)), dtype=np.int64)
    for wi, w in enumerate(words):
        masks = [engine.read_back(h) for h in w.bits]
        for lane in range(lanes):
            bits = [(m >> lane) & 1 for m in masks]
            res[lane, wi] = arith.bits_to_int(bits, signed=True)
    return res


def cfg_signal(cfg: str, lane: int = 0):
    """(params, keygen seed, rng, values, fmt, dims) per the protocol above."""
    if cfg == "cfg0":
        rng = np.random.default_rng(0)
        x = rng.uniform(-1, 1, 8).astype(complex)
        return EXACT_PARAMS, 0, rng, x, arith.FixedFormat(16, 12), 8
    if cfg == "cfg2":
        rng = np.random.default_rng(2)
        re = rng.uniform(-1, 1, 32)
        im = rng.uniform(-1, 1, 32)
        return DEFAULT0, 2, rng, re + 1j * im, arith.FixedFormat(32, 24), 32
    if cfg == "cfg3":
        rng = np.random.default_rng(3)
        pix = rng.integers(0, 256, (8, 8))
        x = (pix / 255.0).ravel().astype(complex)
        return DEFAULT0, 3, rng, x, arith.FixedFormat(16, 7), (8, 8)
    if cfg == "cfg4":
        rng = np.random.default_rng(4 + lane)
        re = rng.uniform(-1, 1, 16)
        im = rng.uniform(-1, 1, 16)
        return DEFAULT0, 4, rng, re + 1j * im, arith.FixedFormat(16, 12), 16
    raise SystemExit(f"unknown fft config {cfg}")


def run_fft(cfg: str, params_override=None, hash_cts=False):
    params, seed, rng, x, fmt, dims = cfg_signal(cfg)
    if params_override is not None:
        params = params_override
    scheme = GswScheme(params)
    keys = scheme.keygen(seed=seed)
    tap = Tap(scheme, hash_cts)
    eng = FheEngine(scheme, keys=keys, rng=rng)
    sig = fft.input_signal(eng, x, fmt, dims=dims)
    out = fft.fft_2d(sig) if isinstance(dims, tuple) else fft.fft_1d(sig)
    words = _signal_words(out)
    return tap, eng, keys, words, x, fmt


def save_json(name, obj):
    with open(os.path.join(HERE, name), "w") as fh:
        json.dump(obj, fh, indent=1, sort_keys=True)
        fh.write("\n")


def ops_digest(ops):
    arr = np.asarray(ops, dtype="<i8")
    import hashlib
    return hashlib.sha256(arr.tobytes()).hexdigest()[:16]


# -- commands ------------------------------------------------------------------

def cmd_trace(cfg):
    """Op sequence of one signal (noise-free params => no swaps, so EXACT gives
    the same sequence as default0 at a fraction of the cost)."""
    t0 = time.time()
    if cfg == "cfg1":
        return cmd_trace_pairs()
    tap, eng, keys, words, x, fmt = run_fft(cfg, params_override=EXACT_PARAMS)
    ops = np.asarray(tap.ops, dtype=np.int64)
    rec = {
        "cfg": cfg,
        "nand_count": eng.nand_count,
        "max_depth": eng.max_depth,
        "n_inputs": len(tap.inputs),
        "n_ops": len(tap.ops),
        "n_not": int((ops[:, 0] == 1).sum()),
        "ops_digest": ops_digest(tap.ops),
        "levels_digest": ops_digest(tap.levels),
        "outputs": _out_wires(words),
        "inputs_first": tap.inputs[0],
        "inputs_contiguous": tap.inputs == list(range(tap.inputs[0], tap.inputs[0] + len(tap.inputs))),
        "seconds": round(time.time() - t0, 1),
    }
    save_json(f"trace_{cfg}.json", rec)
    if cfg == "cfg0":
        np.savez_compressed(os.path.join(HERE, f"trace_{cfg}.npz"),
                            ops=ops.astype(np.int32),
                            levels=np.asarray(tap.levels, dtype=np.int32),
                            inputs=np.asarray(tap.inputs, dtype=np.int32))
    print(json.dumps({k: v for k, v in rec.items() if k != "outputs"}))


def cmd_trace_pairs(n_pairs=4):
    scheme = GswScheme(DEFAULT_PARAMS)
    keys = scheme.keygen(seed=1)
    tap = Tap(scheme, hash_cts=False)
    rng = np.random.default_rng(1)
    bits = rng.integers(0, 2, (PAIRS_FULL, 2))
    eng = FheEngine(scheme, keys=keys, rng=rng)
    hs = [(eng.input_bit(int(bits[p, 0])), eng.input_bit(int(bits[p, 1]))) for p in range(n_pairs)]
    outs = []
    for a, b in hs:
        outs.append((gates.xor_(a, b), gates.and_(a, b)))
    rec = {"cfg": "cfg1", "pairs": n_pairs, "nand_count": eng.nand_count,
           "max_depth": eng.max_depth, "ops": tap.ops, "levels": tap.levels,
           "outputs": [[x.ct._wire, y.ct._wire] for x, y in outs]}
    save_json("trace_cfg1.json", rec)
    print(json.dumps(rec)[:400])


def cmd_cts(cfg, checkpoint=4096):
    """Per-gate ciphertext digests from a real reference run at the config's params."""
    t0 = time.time()
    if cfg == "cfg1":
        return cmd_cts_pairs()
    tap, eng, keys, words, x, fmt = run_fft(cfg, hash_cts=True)
    ints = _word_ints(eng, words)[0]
    out_w = _out_wires(words)
    wire_dig = {}
    for w, d in zip(tap.inputs, tap.input_digests):
        wire_dig[w] = d
    for (_, _, _, o), d in zip(tap.ops, tap.digests):
        wire_dig[o] = d
    rec = {
        "cfg": cfg,
        "params": [eng.scheme.params.n, eng.scheme.params.q, eng.scheme.params.m,
                   eng.scheme.params.noise_bound, eng.scheme.params.depth_budget],
        "nand_count": eng.nand_count,
        "max_depth": eng.max_depth,
        "n_ops": len(tap.ops),
        "inputs_chain": chain_digest(tap.input_digests),
        "gates_chain": chain_digest(tap.digests),
        "checkpoint_every": checkpoint,
        "gates_checkpoints": [chain_digest(tap.digests[:i]) for i in
                              range(checkpoint, len(tap.digests) + 1, checkpoint)],
        "output_digests": [wire_dig.get(w, "const") for w in out_w],
        "output_words": [int(v) for v in ints],
        "x_re": [float(v.real) for v in np.atleast_1d(x)],
        "x_im": [float(v.imag) for v in np.atleast_1d(x)],
        "pk_digest": digest_compact(keys.public_key.astype(np.uint32)),
        "seconds": round(time.time() - t0, 1),
    }
    save_json(f"cts_{cfg}.json", rec)
    if cfg == "cfg0":
        np.savez_compressed(os.path.join(HERE, "cts_cfg0.npz"),
                            gate_digests=np.array([bytes.fromhex(d) for d in tap.digests]),
                            input_digests=np.array([bytes.fromhex(d) for d in tap.input_digests]))
    print(json.dumps({k: v for k, v in rec.items()
                      if k not in ("gates_checkpoints", "output_digests", "output_words")}))


def cmd_cts_pairs(n_pairs=4096, n_gate_pairs=64):
    """Gate microbenchmark sample: the first n_pairs pairs of the 2^20 protocol."""
    t0 = time.time()
    scheme = GswScheme(DEFAULT_PARAMS)
    keys = scheme.keygen(seed=1)
    tap = Tap(scheme, hash_cts=True)
    rng = np.random.default_rng(1)
    bits = rng.integers(0, 2, (PAIRS_FULL, 2))
    eng = FheEngine(scheme, keys=keys, rng=rng)
    hs = [(eng.input_bit(int(bits[p, 0])), eng.input_bit(int(bits[p, 1]))) for p in range(n_pairs)]
    xor_d, and_d, xor_v, and_v = [], [], [], []
    for a, b in hs:
        x = gates.xor_(a, b)
        y = gates.and_(a, b)
        xor_d.append(tap._dig(x.ct))
        and_d.append(tap._dig(y.ct))
        xor_v.append(eng.read_back(x))
        and_v.append(eng.read_back(y))
    assert xor_v == [int(a ^ b) for a, b in bits[:n_pairs]]
    assert and_v == [int(a & b) for a, b in bits[:n_pairs]]
    rec = {
        "cfg": "cfg1", "pairs": n_pairs, "nand_count": eng.nand_count, "max_depth": eng.max_depth,
        "bits_digest": digest_compact(bits[:n_pairs].astype(np.uint32)),
        "inputs_chain": chain_digest(tap.input_digests),
        "first_gates": tap.digests[:6 * n_gate_pairs],
        "gates_chain": chain_digest(tap.digests),
        "xor_digests": xor_d, "and_digests": and_d,
        "pk_digest": digest_compact(keys.public_key.astype(np.uint32)),
        "seconds": round(time.time() - t0, 1),
    }
    save_json("cts_cfg1.json", rec)
    print(json.dumps({k: rec[k] for k in ("nand_count", "max_depth", "gates_chain", "seconds")}))


def cmd_clear(cfg):
    """Decrypted outputs of every lane from the reference cleartext engine."""
    if cfg == "cfg4":
        lanes = 1024
        vals = []
        for i in range(lanes):
            _, _, _, x, fmt, dims = cfg_signal("cfg4", lane=i)
            vals.append(x)
        vals = np.array(vals)
    else:
        _, _, _, x, fmt, dims = cfg_signal(cfg)
        vals = np.atleast_2d(x)
        lanes = 1
    eng = CleartextEngine(batch_size=lanes)
    sig = fft.input_signal(eng, vals, fmt, dims=dims)
    out = fft.fft_2d(sig) if isinstance(dims, tuple) else fft.fft_1d(sig)
    ints = _word_ints(eng, _signal_words(out), lanes)
    np.savez_compressed(os.path.join(HERE, f"clear_{cfg}.npz"),
                        words=ints.astype(np.int64), nand_count=eng.nand_count,
                        max_depth=eng.max_depth)
    print(cfg, ints.shape, eng.nand_count, eng.max_depth)


def cmd_scheme():
    """Known answers of the scheme layer: keys, encryptions, NAND/NOT, decrypt."""
    out = {}
    for name, params, seed in (("exact", EXACT_PARAMS, 1), ("default", DEFAULT_PARAMS, 1),
                               ("default0", DEFAULT0, 2)):
        scheme = GswScheme(params)
        keys = scheme.keygen(seed=seed)
        rng = np.random.default_rng(7)
        cts = [scheme.encrypt_bit(keys.public_key, b, rng) for b in (0, 1, 1, 0, 1)]
        k, ell = params.n + 1, params.ell
        comp = lambda c: compact_from_matrix(c.matrix, k, ell)  # noqa: E731
        arrays = {"pk": keys.public_key, "sk": keys.secret_key}
        for i, c in enumerate(cts):
            arrays[f"ct{i}"] = comp(c)
        # a small circuit with non-fresh operands (exercises the swap rule when noisy)
        n01 = scheme.hom_nand(cts[0], cts[1])
        n12 = scheme.hom_nand(cts[1], cts[2])
        x = scheme.hom_nand(n01, cts[3])          # noisy => swapped
        y = scheme.hom_nand(cts[4], n12)
        nt = scheme.hom_not(y)
        nn = scheme.hom_not(nt)
        for nm, c in (("n01", n01), ("n12", n12), ("x", x), ("y", y), ("nt", nt), ("nn", nn)):
            arrays[nm] = comp(c)
        triv = [comp(scheme.trivial_encrypt_bit(b)) for b in (0, 1)]
        arrays["triv0"], arrays["triv1"] = triv
        sk = keys.secret_key
        meta = {
            "params": [params.n, params.q, params.m, params.noise_bound, params.depth_budget],
            "digest": params.digest(),
            "bits": [scheme.decrypt_bit(sk, c) for c in cts],
            "n01": scheme.decrypt_bit(sk, n01), "n12": scheme.decrypt_bit(sk, n12),
            "x": scheme.decrypt_bit(sk, x), "y": scheme.decrypt_bit(sk, y),
            "nt": scheme.decrypt_bit(sk, nt),
            "levels": [n01.level, n12.level, x.level, y.level, nt.level],
            "noise_est": [n01.noise_est, n12.noise_est, x.noise_est, y.noise_est, nt.noise_est],
            "fresh_noise_est": cts[0].noise_est,
        }
        out[name] = meta
        np.savez_compressed(os.path.join(HERE, f"scheme_{name}.npz"),
                            **{k2: np.asarray(v) for k2, v in arrays.items()})
    save_json("scheme_kat.json", out)
    print(json.dumps(out)[:600])


def cmd_eft1():
    """EFT1 containers written by the reference: an encrypted 4-point Q8.8 signal (EXACT,
    keygen(1), default_rng(7)) and the container of its fft_1d output (the server step)."""
    from fhefft import fileio
    scheme = GswScheme(EXACT_PARAMS)
    keys = scheme.keygen(seed=1)
    rng = np.random.default_rng(7)
    fmt = arith.FixedFormat(16, 8)
    values = [0.5 + 0.25j, -0.75 + 0.125j, 0.0 + 0.0j, 1.5 - 1.0j]
    eng = FheEngine(scheme, keys=keys, rng=rng)
    sig = fft.input_signal(eng, values, fmt)
    fileio.write_ciphertext_signal(os.path.join(HERE, "eft1_exact_in.eft"), EXACT_PARAMS, eng, sig, fmt)
    server = FheEngine(scheme, public_key=keys.public_key, rng=np.random.default_rng(0))
    loaded, fmt2 = fileio.read_ciphertext_signal(os.path.join(HERE, "eft1_exact_in.eft"), server)
    out = fft.fft_1d(loaded)
    fileio.write_ciphertext_signal(os.path.join(HERE, "eft1_exact_fft.eft"), EXACT_PARAMS, server, out, fmt2)
    client = FheEngine(scheme, keys=keys)
    res, _ = fileio.read_ciphertext_signal(os.path.join(HERE, "eft1_exact_fft.eft"), client)
    words = _word_ints(client, _signal_words(res))[0]
    save_json("eft1_exact.json", {"values_re": [v.real for v in values], "values_im": [v.imag for v in values],
                                  "fft_words": [int(v) for v in words], "nand_count": server.nand_count})
    print("eft1 ok", server.nand_count)


def cmd_ring():
    """Z_q ring operations hom_add / hom_const_mult / hom_mult (fhe.py:352-379) as the
    reference computes them, with fresh and non-fresh (swapped, leveled) operands."""
    out = {}
    for name, params in (("exact", EXACT_PARAMS), ("default", DEFAULT_PARAMS)):
        scheme = GswScheme(params)
        keys = scheme.keygen(seed=5)
        rng = np.random.default_rng(11)
        q = params.q
        msgs = [3, 5, int(rng.integers(0, q)), int(rng.integers(0, 2 ** 7))]
        cts = [scheme.encrypt_value(keys.public_key, m, rng) for m in msgs]
        bits = [scheme.encrypt_bit(keys.public_key, b, rng) for b in (1, 0)]
        nb = scheme.hom_nand(bits[0], bits[1])              # level 1, noisy
        k_vals = [0, 1, 7, q - 1, int(rng.integers(0, q)), -3]
        k, ell = params.n + 1, params.ell
        comp = lambda c: compact_from_matrix(c.matrix, k, ell)  # noqa: E731
        arrays = {f"ct{i}": comp(c) for i, c in enumerate(cts)}
        arrays["b0"], arrays["b1"], arrays["nb"] = comp(bits[0]), comp(bits[1]), comp(nb)
        results = {
            "add01": scheme.hom_add(cts[0], cts[1]),
            "add23": scheme.hom_add(cts[2], cts[3]),
            "add_nb": scheme.hom_add(nb, bits[0]),
            "mult03": scheme.hom_mult(cts[0], cts[3]),
            "mult_b_nb": scheme.hom_mult(bits[1], nb),      # nb noisier => swapped
            "mult_nb_b": scheme.hom_mult(nb, bits[0]),
        }
        for i, kv in enumerate(k_vals):
            results[f"cmult{i}"] = scheme.hom_const_mult(cts[2] if i % 2 else nb, kv)
        meta = {"params": [params.n, q, params.m, params.noise_bound, params.depth_budget],
                "msgs": msgs, "k_vals": k_vals, "nb_level": nb.level, "nb_noise": nb.noise_est,
                "fresh_noise": cts[0].noise_est, "results": {}}
        for nm, c in results.items():
            arrays[nm] = comp(c)
            meta["results"][nm] = {"level": c.level, "noise_est": c.noise_est}
        meta["decrypt"] = {"add01": scheme.decrypt_value(keys.secret_key, results["add01"]),
                           "mult03": scheme.decrypt_value(keys.secret_key, results["mult03"])}
        out[name] = meta
        np.savez_compressed(os.path.join(HERE, f"ring_{name}.npz"),
                            **{k2: np.asarray(v) for k2, v in arrays.items()})
    save_json("ring_kat.json", out)
    print(json.dumps(out)[:400])


if __name__ == "__main__":
    cmd = sys.argv[1]
    if cmd == "scheme":
        cmd_scheme()
    elif cmd == "trace":
        cmd_trace(sys.argv[2])
    elif cmd == "cts":
        cmd_cts(sys.argv[2])
    elif cmd == "clear":
        cmd_clear(sys.argv[2])
    elif cmd == "eft1":
        cmd_eft1()
    elif cmd == "ring":
        cmd_ring()
    else:
        raise SystemExit(__doc__)
