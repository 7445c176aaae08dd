"""CPU restatement of the reference GSW scheme (the hot path's arithmetic).

TEST INFRASTRUCTURE ONLY -- imported by tests/, __graft_entry__.smoke() and
bench.py's CPU legs, never by the product package.

Two formulations live here:

* the reference's own: ciphertexts are N x N 0/1 float64 matrices and a NAND
  is ``flatten(I - C1 @ C2)`` (``fhe.py:325-341``) -- restated literally so that
  ``bench.py --impl reference`` times the reference algorithm on host cores;
* the compact identity the GPU path uses: with V = recompose(C) (N x k, k=n+1,
  values in [0, q)),  NAND = (G - bits(V1) @ V2) mod q  and  NOT = (G - V) mod q,
  where G = recompose(I) is the gadget matrix.  ``tests/test_oracle.py`` checks
  the two formulations agree bit for bit.

Reference root: /root/reference/pkg/src/fhefft.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Params:
    """Mirror of ``SchemeParams`` (fhe.py:46-71)."""

    n: int
    q: int
    m: int
    noise_bound: int
    depth_budget: int

    @property
    def ell(self) -> int:            # fhe.py:42-43, 63-66: ceil(log2 q)
        return (self.q - 1).bit_length()

    @property
    def k(self) -> int:              # blocks per row: n + 1
        return self.n + 1

    @property
    def n_ct(self) -> int:           # fhe.py:68-71
        return self.k * self.ell


EXACT = Params(n=2, q=2**16 + 1, m=8, noise_bound=0, depth_budget=10**9)   # fhe.py:110
DEFAULT = Params(n=8, q=2**29 - 3, m=32, noise_bound=2, depth_budget=3)     # fhe.py:105
DEFAULT0 = Params(n=8, q=2**29 - 3, m=32, noise_bound=0, depth_budget=10**9)


# -- gadget plumbing (fhe.py:175-189, 200-208) ----------------------------------

def gadget(p: Params, mu: int = 1) -> np.ndarray:
    """N x k matrix with (mu * 2^j mod q) at row i*ell+j, column i (fhe.py:200-208)."""
    g = np.zeros((p.n_ct, p.k), dtype=np.int64)
    col = np.arange(p.n_ct) // p.ell
    g[np.arange(p.n_ct), col] = [(mu << (r % p.ell)) % p.q for r in range(p.n_ct)]
    return g


def bits_of(v: np.ndarray, p: Params) -> np.ndarray:
    """decompose (fhe.py:175-179): row-wise LSB-first ell-bit expansion."""
    v = np.asarray(v, dtype=np.int64)
    sh = np.arange(p.ell, dtype=np.int64)
    return ((v[..., None] >> sh) & 1).reshape(v.shape[:-1] + (p.n_ct,))


def recompose(x: np.ndarray, p: Params) -> np.ndarray:
    """fhe.py:181-185: per row and block, sum_j x[., i*ell+j] 2^j mod q (exact ints)."""
    x = np.asarray(x).astype(np.int64)
    w = np.int64(1) << np.arange(p.ell, dtype=np.int64)
    vals = (x.reshape(x.shape[:-1] + (p.k, p.ell)) * w).sum(axis=-1)
    return np.mod(vals, p.q)


def flatten(x: np.ndarray, p: Params) -> np.ndarray:
    """fhe.py:187-189."""
    return bits_of(recompose(x, p), p).astype(np.float64)


# -- keys and encryption (fhe.py:212-249) -----------------------------------------

def keygen(p: Params, seed):
    """fhe.py:212-225: draws t (n), B (m x n), err (m) from default_rng(seed)."""
    rng = np.random.default_rng(seed)
    t = rng.integers(0, p.q, p.n, dtype=np.int64)
    b = rng.integers(0, p.q, (p.m, p.n), dtype=np.int64)
    err = rng.integers(-p.noise_bound, p.noise_bound + 1, p.m, dtype=np.int64)
    col = [(sum(int(b[i, j]) * int(t[j]) for j in range(p.n)) + int(err[i])) % p.q
           for i in range(p.m)]
    pk = np.concatenate([b, np.array(col, dtype=np.int64)[:, None]], axis=1)
    sk = np.concatenate([(p.q - t) % p.q, np.ones(1, dtype=np.int64)])
    return pk, sk


def encrypt_compact(p: Params, pk: np.ndarray, mu: int, rng) -> np.ndarray:
    """fhe.py:227-233 in compact form: V = (R @ pk + mu G) mod q, R ~ {0,1}^(N x m).

    The draw ``rng.integers(0, 2, (N, m))`` is the reference's, so the stream of
    a shared Generator advances exactly as in the reference."""
    r = rng.integers(0, 2, (p.n_ct, p.m))
    return np.mod(r @ pk + gadget(p, mu % p.q), p.q)


def encrypt_matrix(p: Params, pk: np.ndarray, bit: int, rng) -> np.ndarray:
    """The reference's flattened N x N encryption of a bit (fhe.py:235-238)."""
    return bits_of(encrypt_compact(p, pk, bit, rng), p).astype(np.float64)


# -- decryption (fhe.py:191-198, 259-286) ------------------------------------------

def decrypt_bit_compact(p: Params, sk: np.ndarray, v: np.ndarray) -> int:
    """fhe.py:267-286: row n*ell + j of C dotted with powers-of-2(s), j=bitlen(q//2)-1."""
    j = (p.q // 2).bit_length() - 1
    row = bits_of(np.asarray(v)[p.n * p.ell + j], p)          # one row of C
    pw = np.array([(int(sk[i]) << jj) % p.q for i in range(p.k) for jj in range(p.ell)],
                  dtype=object)
    x = int(np.dot(row.astype(object), pw)) % p.q
    if x > p.q // 2:
        x -= p.q
    scale = 1 << j
    mu = (2 * x + scale) // (2 * scale)
    noise = abs(x - mu * scale)
    if mu not in (0, 1) or noise >= (p.q + 7) // 8:
        raise ValueError(f"decryption failed: noise {noise}")
    return mu


# -- homomorphic gates ------------------------------------------------------------------

def hom_nand_matrix(p: Params, c1: np.ndarray, c2: np.ndarray) -> np.ndarray:
    """The reference algorithm, fhe.py:338-340: flatten(I - C1 @ C2) in float64.

    (Level/noise bookkeeping and the operand swap of fhe.py:330-339 are the
    caller's business; c1 is the left operand AFTER the swap.)"""
    prod = c1 @ c2
    return flatten(np.eye(p.n_ct) - prod, p)


def hom_not_matrix(p: Params, c: np.ndarray) -> np.ndarray:
    """fhe.py:343-350: flatten(I - C)."""
    return flatten(np.eye(p.n_ct) - c, p)


def hom_nand_compact(p: Params, v1: np.ndarray, v2: np.ndarray) -> np.ndarray:
    """Compact identity of a1: recompose(I - C1 C2) = (G - C1 V2) mod q, C1 = bits(V1)."""
    c1 = bits_of(v1, p)
    return np.mod(gadget(p) - c1 @ np.asarray(v2, dtype=np.int64), p.q)


def hom_not_compact(p: Params, v: np.ndarray) -> np.ndarray:
    """Compact identity of a3: (G - V) mod q."""
    return np.mod(gadget(p) - np.asarray(v, dtype=np.int64), p.q)


def noise_after_nand(p: Params, e_left: int, e_right: int) -> int:
    """fhe.py:339: est = min(e1 + N e2, q) with e1 the (post-swap) left operand."""
    return min(e_left + p.n_ct * e_right, p.q)


# -- Z_q ring operations -------------------------------------------------------

def hom_add_matrix(p: Params, c1: np.ndarray, c2: np.ndarray) -> np.ndarray:
    """fhe.py:352-356: flatten(C1 + C2)."""
    return flatten(c1 + c2, p)


def hom_const_mult_matrix(p: Params, c: np.ndarray, k: int) -> np.ndarray:
    """fhe.py:358-364: flatten(decompose(scaled_gadget(k mod q) mod q) @ C)."""
    mk = bits_of(gadget(p, k % p.q), p).astype(np.float64)   # decompose(kG mod q)
    return flatten(mk @ c, p)


def hom_mult_matrix(p: Params, c1: np.ndarray, c2: np.ndarray) -> np.ndarray:
    """fhe.py:366-379: flatten(C1 @ C2) (c1 = left operand after the noise swap)."""
    return flatten(c1 @ c2, p)


def hom_add_compact(p: Params, v1: np.ndarray, v2: np.ndarray) -> np.ndarray:
    """recompose(C1 + C2) = (V1 + V2) mod q (recompose is linear; each V < q < 2^ell)."""
    return np.mod(np.asarray(v1, dtype=np.int64) + np.asarray(v2, dtype=np.int64), p.q)


def hom_mult_compact(p: Params, v1: np.ndarray, v2: np.ndarray) -> np.ndarray:
    """recompose(C1 C2) = C1 V2 mod q = NOT(NAND(V1, V2)): (G - (G - P)) mod q = P mod q."""
    return np.mod(bits_of(v1, p) @ np.asarray(v2, dtype=np.int64), p.q)


def hom_const_mult_compact(p: Params, v: np.ndarray, k: int) -> np.ndarray:
    """hom_mult with the left operand V_k = (k G) mod q (the scaled gadget, fhe.py:200-208)."""
    return hom_mult_compact(p, gadget(p, k % p.q), v)
