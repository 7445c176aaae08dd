"""Ciphertext digests shared by the golden-vector generator and the tests.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

A reference ciphertext is the flattened N x N 0/1 matrix ``C`` of
``fhe.py:148-161``.  Since every flattened matrix is ``decompose(V)`` for a
unique V in [0, q)^(N x (n+1)) (``fhe.py:175-189``), the digest is taken over
the compact form V (little-endian u32, row-major N x (n+1)); it identifies the
reference matrix bit for bit while costing 29x fewer bytes to hash.
"""

from __future__ import annotations

import hashlib

import numpy as np


def compact_from_matrix(matrix: np.ndarray, n_blocks: int, ell: int) -> np.ndarray:
    """V[r, i] = sum_j C[r, i*ell + j] * 2^j  -- ``fhe.py:181-185`` without the
    mod, exact because a flattened C holds the bits of values already < q."""
    n_ct = matrix.shape[0]
    bits = np.asarray(matrix).reshape(n_ct, n_blocks, ell).astype(np.uint64)
    weights = np.uint64(1) << np.arange(ell, dtype=np.uint64)
    return (bits * weights).sum(axis=2).astype(np.uint32)


def digest_compact(v: np.ndarray) -> str:
    """First 16 hex chars of SHA-256 over V as little-endian u32, row-major."""
    arr = np.ascontiguousarray(np.asarray(v, dtype="<u4"))
    return hashlib.sha256(arr.tobytes()).hexdigest()[:16]


def chain_digest(gate_digests) -> str:
    """Digest of an ordered sequence of per-gate digests (hex strings)."""
    h = hashlib.sha256()
    for d in gate_digests:
        h.update(bytes.fromhex(d))
    return h.hexdigest()[:16]
