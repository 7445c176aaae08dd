"""GSW matrix scheme, host side, with ciphertexts held in compact form.

Mirrors the public surface of the reference ``fhefft/fhe.py`` (SchemeParams,
DEFAULT_PARAMS, EXACT_PARAMS, KeyPair, Ciphertext, GswScheme with keygen /
encrypt_bit / encrypt_value / trivial_encrypt_bit / decrypt_bit /
decrypt_bit_with_noise / decrypt_value / measure_noise / hom_nand / hom_not)
with the same draws, thresholds, level and noise bookkeeping and error types.

Representation (the B200 design decision): a
reference ciphertext is a flattened N x N 0/1 matrix C = decompose(V) for a
unique V in [0, q)^(N x k), k = n + 1.  We store V (u32, N x k, 9,396 B at
N = 261 instead of the 545 KB float64 matrix) and evaluate

    NAND(C1, C2) = flatten(I - C1 C2)   as   V = (G - bits(V1) V2) mod q
    NOT(C)       = flatten(I - C)       as   V = (G - V) mod q

on the GPU (csrc/fhegpu.cu).  ``Ciphertext.matrix`` rebuilds the reference's
float64 matrix on demand, so both formulations are interchangeable and
bit-identical.  Key generation, encryption and decryption stay on the host
here (numpy, the reference's exact draw order); they are setup, not the
measured path.
"""

from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass, field

import numpy as np

from .errors import NoiseOverflowError, ParameterError

_EXACT_BITS = 52          # fhe.py:37-39: float64 exactness limit the reference enforces


@dataclass(frozen=True)
class SchemeParams:
    """Lattice parameters (fhe.py:46-100): n, q (odd), m, noise_bound, depth_budget."""

    n: int
    q: int
    m: int = 32
    noise_bound: int = 2
    depth_budget: int = 3

    @property
    def ell(self) -> int:
        """Bits per Z_q value, ceil(log2 q) (fhe.py:63-66)."""
        return int(self.q - 1).bit_length()

    @property
    def k(self) -> int:
        """Z_q columns of a compact ciphertext, n + 1."""
        return self.n + 1

    @property
    def n_ct(self) -> int:
        """Ciphertext side N = (n + 1) ell (fhe.py:68-71)."""
        return (self.n + 1) * self.ell

    def __post_init__(self):
        # same checks, same order, same messages as fhe.py:73-95
        if self.n < 1 or self.m < 1:
            raise ParameterError("n and m must be positive")
        if self.q < 8 or self.q % 2 == 0:
            raise ParameterError("q must be an odd integer >= 8")
        if self.noise_bound < 0 or self.depth_budget < 0:
            raise ParameterError("noise_bound and depth_budget must be >= 0")
        if (self.n_ct + 1) << self.ell >= 1 << _EXACT_BITS:
            raise ParameterError(
                f"q={self.q} with n={self.n} exceeds the exact-arithmetic "
                f"limit (need (N+1)*2^ell < 2^{_EXACT_BITS})")
        if self.m * self.q >= 1 << _EXACT_BITS:
            raise ParameterError("m * q too large for exact encryption arithmetic")
        if self.noise_bound > 0:
            margin = math.log2(8 * self.noise_bound) + self.depth_budget * math.log2(self.n_ct + 1)
            if margin >= 200 or self.q <= 8 * self.noise_bound * (self.n_ct + 1) ** self.depth_budget:
                raise ParameterError(
                    f"q={self.q} too small for noise_bound={self.noise_bound} at "
                    f"depth_budget={self.depth_budget}: need q > 8*nb*(N+1)^depth")

    _FIELDS = ("n", "q", "m", "noise_bound", "depth_budget")

    def __eq__(self, other):
        """Equal to any parameter object with the same five fields -- in particular the
        reference's own ``fhefft.fhe.SchemeParams``, which ``fileio.read_ciphertext_signal``
        compares against ``engine.scheme.params`` (fileio.py:172-174)."""
        try:
            return all(getattr(self, f) == getattr(other, f) for f in self._FIELDS)
        except AttributeError:
            return NotImplemented

    def digest(self) -> str:
        """Same text and hash as fhe.py:97-100, so digests interoperate."""
        text = f"{self.n},{self.q},{self.m},{self.noise_bound},{self.depth_budget}"
        return hashlib.sha256(text.encode()).hexdigest()[:16]


DEFAULT_PARAMS = SchemeParams(n=8, q=2**29 - 3, m=32, noise_bound=2, depth_budget=3)      # fhe.py:105
EXACT_PARAMS = SchemeParams(n=2, q=2**16 + 1, m=8, noise_bound=0, depth_budget=10**9)     # fhe.py:110
# DEFAULT dimensions without noise: the set every FFT config runs on;
# DEFAULT's depth budget of 3 cannot evaluate one adder.
DEFAULT0_PARAMS = SchemeParams(n=8, q=2**29 - 3, m=32, noise_bound=0, depth_budget=10**9)


def decode_gadget_samples(xs, q: int, error_bound: int) -> int:
    """Recover mu from x_j = mu 2^j + e_j (mod q), |e_j| <= error_bound (fhe.py:113-134).

    Successive refinement: keep an estimate est / 2^shift of mu; jump to the
    highest row whose wrap count the current estimate still determines, unwind
    it, and repeat until the estimate pins one integer.
    """
    ell = len(xs)
    eb = max(error_bound, 1)
    est, shift = xs[0], 0
    while (1 << shift) <= 2 * eb:
        room = (q // 2 - eb - 1) // eb
        j = min(ell - 1, shift + max(1, room.bit_length() - 1))
        wraps = (2 * ((est << (j - shift)) - xs[j]) + q) // (2 * q)
        est, shift = wraps * q + xs[j], j
        if j == ell - 1:
            break
    return ((est + (1 << (shift - 1))) >> shift) % q


@dataclass(frozen=True)
class KeyPair:
    """Public m x (n+1) matrix A and secret (n+1)-vector s with s[-1] = 1 (fhe.py:137-146)."""

    public_key: np.ndarray
    secret_key: np.ndarray


@dataclass(eq=False, init=False)
class Ciphertext:
    """One bit (or Z_q value) in compact form: V (N x k, u32, values < q).

    ``level`` and ``noise_est`` carry the reference's bookkeeping
    (fhe.py:148-161).  ``matrix`` is the reference's flattened float64 N x N
    0/1 matrix, rebuilt on demand.  Like the reference's constructor,
    ``Ciphertext(matrix=..., level=...)`` builds one from a matrix (``params``
    then required: the compact form needs q and ell).
    """

    v: np.ndarray
    level: int = 0
    noise_est: int = 0
    params: SchemeParams | None = field(default=None, repr=False)

    def __init__(self, v=None, level: int = 0, noise_est: int = 0, params: SchemeParams | None = None,
                 *, matrix=None):
        if (v is None) == (matrix is None):
            raise ValueError("Ciphertext needs exactly one of v (compact) or matrix")
        if matrix is not None:
            if params is None:
                raise ValueError("Ciphertext(matrix=...) needs params to recompose the matrix")
            v = _recompose(np.asarray(matrix), params)
        self.v = v
        self.level = level
        self.noise_est = noise_est
        self.params = params

    @property
    def matrix(self) -> np.ndarray:
        v = np.asarray(self.v, dtype=np.uint32)
        ell = self.params.ell if self.params is not None else _infer_ell(v)
        bits = (v[:, :, None] >> np.arange(ell, dtype=np.uint32)) & 1
        return bits.reshape(v.shape[0], -1).astype(np.float64)

    @classmethod
    def from_matrix(cls, matrix, params: SchemeParams, level: int = 0, noise_est: int = 0):
        """Compact form of a reference ciphertext matrix (any integer-valued N x N)."""
        return cls(_recompose(np.asarray(matrix), params), level, noise_est, params)


def _infer_ell(v):
    raise ValueError("Ciphertext.matrix needs params to know ell")


def _gadget(params: SchemeParams, mu: int = 1) -> np.ndarray:
    """N x k matrix whose flattening encodes mu I_N (fhe.py:200-208)."""
    g = np.zeros((params.n_ct, params.k), dtype=np.int64)
    r = np.arange(params.n_ct)
    g[r, r // params.ell] = [(mu << (x % params.ell)) % params.q for x in r]
    return g


def _recompose(mat: np.ndarray, params: SchemeParams) -> np.ndarray:
    """fhe.py:181-185 over exact integers: sum_j X[., i ell + j] 2^j mod q."""
    x = np.asarray(mat).astype(np.int64)
    w = np.int64(1) << np.arange(params.ell, dtype=np.int64)
    vals = (x.reshape(x.shape[0], params.k, params.ell) * w).sum(axis=2)
    return np.mod(vals, params.q).astype(np.uint32)


def as_params(p) -> SchemeParams:
    """This package's SchemeParams for any object with the five parameter fields (e.g. the
    reference's ``fhefft.fhe.SchemeParams``, which ``cli.cmd_fft`` reads from a container)."""
    if isinstance(p, SchemeParams):
        return p
    try:
        return SchemeParams(**{f: int(getattr(p, f)) for f in SchemeParams._FIELDS})
    except AttributeError as exc:
        raise ParameterError(f"not a parameter set: {p!r}") from exc


class GswScheme:
    """Scheme operations for one parameter set (fhe.py:164-379 surface)."""

    def __init__(self, params: SchemeParams = DEFAULT_PARAMS, device: int = 0):
        params = as_params(params)
        self.params = params
        self.device = device
        self._g = _gadget(params)
        self._g_u32 = self._g.astype(np.uint32)
        self._ctx = None

    # -- device -------------------------------------------------------------------

    @property
    def ctx(self):
        """Device context (lazily created; raises DeviceError without a GPU/library)."""
        if self._ctx is None:
            from ._native import DeviceContext
            self._ctx = DeviceContext(self.params, self.device)
        return self._ctx

    # -- keys and encryption (host; the reference's exact draws) ---------------

    def keygen(self, seed) -> KeyPair:
        """fhe.py:212-225: t (n), B (m x n), err (m) from default_rng(seed)."""
        p = self.params
        rng = np.random.default_rng(seed)
        t = rng.integers(0, p.q, p.n, dtype=np.int64)
        b = rng.integers(0, p.q, (p.m, p.n), dtype=np.int64)
        err = rng.integers(-p.noise_bound, p.noise_bound + 1, p.m, dtype=np.int64)
        body = b.astype(object) @ t.astype(object)         # entries reach q^2: exact ints
        col = np.array([(int(x) + int(e)) % p.q for x, e in zip(body, err)], dtype=np.int64)
        pk = np.concatenate([b, col[:, None]], axis=1)
        sk = np.concatenate([(p.q - t) % p.q, np.array([1], dtype=np.int64)])
        return KeyPair(public_key=pk, secret_key=sk)

    def encrypt_many(self, public_key: np.ndarray, mus, rng, chunk: int = 512) -> np.ndarray:
        """Compact encryptions of plaintexts ``mus`` in order: (count, N, k) u32.

        Draws ``rng.integers(0, 2, (N, m))`` per ciphertext exactly as
        fhe.py:229 does (a bulk draw of shape (count, N, m) advances the
        Generator identically), then V = (R pk + mu G) mod q in exact float64
        like fhe.py:230-232."""
        p = self.params
        mus = np.asarray(mus, dtype=np.int64) % p.q
        out = np.empty((len(mus), p.n_ct, p.k), dtype=np.uint32)
        pkf = np.asarray(public_key).astype(np.float64)
        gf = self._g.astype(np.float64)
        for s in range(0, len(mus), chunk):
            e = min(len(mus), s + chunk)
            r = rng.integers(0, 2, (e - s, p.n_ct, p.m)).astype(np.float64)
            body = r @ pkf + mus[s:e, None, None] * gf
            out[s:e] = np.mod(body, p.q).astype(np.uint32)
        return out

    def _encrypt(self, public_key, mu: int, rng) -> Ciphertext:
        v = self.encrypt_many(public_key, [mu], rng)[0]
        return Ciphertext(v, 0, self.params.m * self.params.noise_bound, self.params)

    def encrypt_bit(self, public_key: np.ndarray, bit: int, rng) -> Ciphertext:
        if bit not in (0, 1):
            raise ValueError(f"bit must be 0 or 1, got {bit!r}")
        return self._encrypt(public_key, bit, rng)

    def encrypt_value(self, public_key: np.ndarray, value: int, rng) -> Ciphertext:
        return self._encrypt(public_key, value % self.params.q, rng)

    def trivial_encrypt_bit(self, bit: int) -> Ciphertext:
        """Noiseless encoding of a public constant: V = bit * G (fhe.py:244-249)."""
        if bit not in (0, 1):
            raise ValueError(f"bit must be 0 or 1, got {bit!r}")
        return Ciphertext((self._g_u32 * np.uint32(bit)).copy(), 0, 0, self.params)

    def fresh_noise(self) -> int:
        return self.params.m * self.params.noise_bound

    # -- decryption (host) ----------------------------------------------------

    def _check_level(self, ct: Ciphertext):
        if ct.level > self.params.depth_budget:
            raise NoiseOverflowError(
                f"ciphertext level {ct.level} exceeds depth budget {self.params.depth_budget}")

    def _powers_of_secret(self, secret_key) -> list[int]:
        p = self.params
        return [(int(secret_key[i]) << j) % p.q for i in range(p.k) for j in range(p.ell)]

    def gadget_rows_many(self, secret_key, v_rows: np.ndarray) -> np.ndarray:
        """x_j for many ciphertexts from their compact gadget block (fhe.py:259-265).

        v_rows: (count, ell, k) -- rows n*ell .. n*ell+ell-1 of V.  Returns (count, ell)."""
        p = self.params
        pw = np.array(self._powers_of_secret(secret_key), dtype=object).reshape(p.k, p.ell)
        bits = ((np.asarray(v_rows, dtype=np.int64)[..., None] >> np.arange(p.ell)) & 1)
        # dot of each C row with powers(s): sum_i sum_b bit_b(V[row, i]) (s_i 2^b mod q)
        acc = np.tensordot(bits.astype(object), pw, axes=([2, 3], [0, 1]))
        return np.mod(acc, p.q).astype(np.int64)

    def decrypt_bits_from_rows(self, secret_key, v_row: np.ndarray) -> np.ndarray:
        """Vectorised decrypt_bit (fhe.py:267-286) from row n*ell + j of each V.

        v_row: (count, k).  Raises NoiseOverflowError like the reference."""
        p = self.params
        pw = self.decrypt_weights(secret_key).astype(np.int64).reshape(p.k, p.ell)
        v = np.asarray(v_row, dtype=np.int64)
        bits = (v[:, :, None] >> np.arange(p.ell, dtype=np.int64)) & 1
        # sum of up to N terms each < q < 2^31 -> < 2^40: exact in int64
        x = np.mod((bits * pw[None]).sum(axis=(1, 2)), p.q)
        x = np.where(x > p.q // 2, x - p.q, x)
        return self.decrypt_bits_from_sums(x)

    def decrypt_weights(self, secret_key) -> np.ndarray:
        """pw[i*ell + b] = (sk_i << b) mod q: the weights of row n*ell + j's bits in the
        reference's <C[row], recompose-weighted sk> (fhe.py:267-286), u32."""
        p = self.params
        return np.array([(int(secret_key[i]) << b) % p.q for i in range(p.k) for b in range(p.ell)],
                        dtype=np.uint32)

    def decrypt_bits_from_sums(self, x: np.ndarray) -> np.ndarray:
        """Bits from centred decryption sums x in (-q/2, q/2] (fhegpu_store_decrypt_rows), with the
        reference's rounding and noise check (fhe.py:278-286)."""
        p = self.params
        x = np.asarray(x, dtype=np.int64)
        j = (p.q // 2).bit_length() - 1
        scale = 1 << j
        mu = (2 * x + scale) // (2 * scale)
        noise = np.abs(x - mu * scale)
        bad = (mu < 0) | (mu > 1) | (noise >= (p.q + 7) // 8)
        if bad.any():
            raise NoiseOverflowError(
                f"noise {int(noise[bad][0])} at or above decryption threshold q/8={p.q / 8:.0f}")
        return mu.astype(np.int64)

    def decrypt_bit_with_noise(self, secret_key, ct: Ciphertext) -> tuple[int, int]:
        p = self.params
        self._check_level(ct)
        j = (p.q // 2).bit_length() - 1
        x = self._gadget_rows(secret_key, ct)[j]
        if x > p.q // 2:
            x -= p.q
        scale = 1 << j
        mu = (2 * x + scale) // (2 * scale)
        noise = abs(x - mu * scale)
        if mu not in (0, 1) or noise >= (p.q + 7) // 8:
            raise NoiseOverflowError(
                f"noise {noise} at or above decryption threshold q/8={p.q / 8:.0f}")
        return mu, noise

    def decrypt_bit(self, secret_key, ct: Ciphertext) -> int:
        return self.decrypt_bit_with_noise(secret_key, ct)[0]

    def _gadget_rows(self, secret_key, ct: Ciphertext) -> list[int]:
        p = self.params
        block = np.asarray(ct.v)[p.n * p.ell:(p.n + 1) * p.ell]
        return [int(x) for x in self.gadget_rows_many(secret_key, block[None])[0]]

    def decrypt_value(self, secret_key, ct: Ciphertext) -> int:
        p = self.params
        self._check_level(ct)
        xs = self._gadget_rows(secret_key, ct)
        mu = decode_gadget_samples(xs, p.q, p.q // 8)
        if self._max_residual(xs, mu) >= (p.q + 7) // 8:
            raise NoiseOverflowError(
                f"noise {self._max_residual(xs, mu)} at or above decryption threshold "
                f"q/8={p.q / 8:.0f}")
        return mu

    def _max_residual(self, xs, mu: int) -> int:
        p = self.params
        worst = 0
        for j, x in enumerate(xs):
            e = (x - ((mu << j) % p.q)) % p.q
            if e > p.q // 2:
                e -= p.q
            worst = max(worst, abs(e))
        return worst

    def measure_noise(self, secret_key, ct: Ciphertext) -> int:
        xs = self._gadget_rows(secret_key, ct)
        return self._max_residual(xs, self.decrypt_value(secret_key, ct))

    # -- homomorphic gates (GPU) -------------------------------------------------

    def nand_meta(self, ct1: Ciphertext, ct2: Ciphertext):
        """Level check, swap and noise estimate of fhe.py:330-339 -> (left, right, level, est)."""
        p = self.params
        level = max(ct1.level, ct2.level) + 1
        if level > p.depth_budget:
            raise NoiseOverflowError(
                f"NAND at level {level} would exceed depth budget {p.depth_budget}")
        if ct2.noise_est > ct1.noise_est:
            ct1, ct2 = ct2, ct1
        est = min(ct1.noise_est + p.n_ct * ct2.noise_est, p.q)
        return ct1, ct2, level, est

    def hom_nand(self, ct1: Ciphertext, ct2: Ciphertext) -> Ciphertext:
        """NOT(b1 AND b2) = flatten(I - C1 C2) evaluated on the GPU (fhe.py:325-341)."""
        left, right, level, est = self.nand_meta(ct1, ct2)
        out = self.ctx.nand_batch(np.asarray(left.v)[None], np.asarray(right.v)[None])[0]
        return Ciphertext(out, level, est, self.params)

    def hom_nand_many(self, pairs) -> list[Ciphertext]:
        """Batched hom_nand: one kernel launch for every (ct1, ct2) pair."""
        metas = [self.nand_meta(a, b) for a, b in pairs]
        if not metas:
            return []
        v1 = np.stack([np.asarray(m[0].v) for m in metas])
        v2 = np.stack([np.asarray(m[1].v) for m in metas])
        outs = self.ctx.nand_batch(v1, v2)
        return [Ciphertext(o, m[2], m[3], self.params) for o, m in zip(outs, metas)]

    def hom_not(self, ct: Ciphertext) -> Ciphertext:
        """flatten(I - C) = (G - V) mod q; level and noise unchanged (fhe.py:343-350)."""
        out = self.ctx.not_batch(np.asarray(ct.v)[None])[0]
        return Ciphertext(out, ct.level, ct.noise_est, self.params)

    # -- Z_q ring operations (fhe.py:352-379), on the GPU ----------------------------------

    def add_meta(self, ct1: Ciphertext, ct2: Ciphertext):
        """fhe.py:354-356: level = max, est = min(e1 + e2, q) -> (level, est)."""
        return max(ct1.level, ct2.level), min(ct1.noise_est + ct2.noise_est, self.params.q)

    def mult_meta(self, ct1: Ciphertext, ct2: Ciphertext):
        """fhe.py:374-379: noisier operand left, est = min(e1 + N e2, q), level = max (no depth
        check, unlike hom_nand) -> (left, right, level, est)."""
        p = self.params
        if ct2.noise_est > ct1.noise_est:
            ct1, ct2 = ct2, ct1
        est = min(ct1.noise_est + p.n_ct * ct2.noise_est, p.q)
        return ct1, ct2, max(ct1.level, ct2.level), est

    def hom_add(self, ct1: Ciphertext, ct2: Ciphertext) -> Ciphertext:
        """Encrypts (m1 + m2) mod q: flatten(C1 + C2) = (V1 + V2) mod q (fhe.py:352-356)."""
        return self.hom_add_many([(ct1, ct2)])[0]

    def hom_add_many(self, pairs) -> list[Ciphertext]:
        if not pairs:
            return []
        out = self.ctx.add_batch(np.stack([np.asarray(a.v) for a, _ in pairs]),
                                 np.stack([np.asarray(b.v) for _, b in pairs]))
        return [Ciphertext(o, *self.add_meta(a, b), self.params) for o, (a, b) in zip(out, pairs)]

    def hom_const_mult(self, ct: Ciphertext, k: int) -> Ciphertext:
        """Encrypts (k m) mod q: flatten(decompose(kG mod q) C) (fhe.py:358-364)."""
        return self.hom_const_mult_many([ct], k)[0]

    def hom_const_mult_many(self, cts, k: int) -> list[Ciphertext]:
        """Every ciphertext times the same public constant k (one launch)."""
        if not cts:
            return []
        p = self.params
        out = self.ctx.const_mult_batch(int(k) % p.q, np.stack([np.asarray(c.v) for c in cts]))
        return [Ciphertext(o, c.level, min(p.n_ct * c.noise_est, p.q), p) for o, c in zip(out, cts)]

    def hom_mult(self, ct1: Ciphertext, ct2: Ciphertext) -> Ciphertext:
        """Encrypts (m1 m2) mod q: flatten(C1 C2) = bits(V1) V2 mod q (fhe.py:366-379)."""
        return self.hom_mult_many([(ct1, ct2)])[0]

    def hom_mult_many(self, pairs) -> list[Ciphertext]:
        metas = [self.mult_meta(a, b) for a, b in pairs]
        if not metas:
            return []
        out = self.ctx.mult_batch(np.stack([np.asarray(m[0].v) for m in metas]),
                                  np.stack([np.asarray(m[1].v) for m in metas]))
        return [Ciphertext(o, m[2], m[3], self.params) for o, m in zip(out, metas)]
