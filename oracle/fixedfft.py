"""Integer-exact model of the reference's fixed-point FFT circuits.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The reference evaluates every word operation as a NAND netlist, but the
netlist computes exact two's-complement arithmetic, so its decrypted outputs
are reproduced here with plain integer arithmetic on numpy int64 lanes:

* ``add``  -- ripple adder, carry out of the top bit dropped (arith.py:158-187): (x + y) mod 2^F
* ``sub``  -- invert y, ripple with carry-in 1 (arith.py:190-193):                (x - y) mod 2^F
* ``mul_const`` -- carry-save column reduction of the sign-extended product
  truncated to hi = F + f columns, bits [f, f+F) kept (arith.py:198-285):
  floor(((x * c) mod 2^hi) / 2^f) mod 2^F, with c = round(c_real * 2^f)
* twiddles -- decode(encode(cos/sin)) of exp(-2 pi i k / size) (fft.py:69-99)
* ``fft_1d`` -- bit reversal then log2 M stages of butterflies (fft.py:113-174)
* ``fft_2d`` -- row transforms then column transforms (fft.py:177-194)

Words are signed ints of width F; every array has a leading lane axis.
"""

from __future__ import annotations

import cmath

import numpy as np


def wrap(v, width: int):
    """Signed two's-complement wrap to ``width`` bits (vectorised)."""
    v = np.asarray(v, dtype=np.int64)
    m = np.int64(1) << np.int64(width)
    half = np.int64(1) << np.int64(width - 1)
    return ((v + half) % m) - half


def encode_int(x: float, total: int, frac: int) -> int:
    """arith.py:63-70: Python round(x * 2^f) (half to even), range checked."""
    ix = round(x * (1 << frac))
    half = 1 << (total - 1)
    if not -half <= ix < half:
        raise ValueError(f"{x} does not fit {total}.{frac}")
    return ix


def encode_lanes(values, total: int, frac: int) -> np.ndarray:
    """Per-lane integer words of real values (arith.py:99-112 without the bits)."""
    vals = np.asarray(values, dtype=np.float64)
    out = np.rint(vals * float(1 << frac)).astype(np.int64)   # rint == round-half-even
    half = 1 << (total - 1)
    if (out < -half).any() or (out >= half).any():
        raise ValueError("value out of fixed-point range")
    return out


def add(x, y, total):
    return wrap(x + y, total)


def sub(x, y, total):
    return wrap(x - y, total)


def mul_const(x, c_int: int, total: int, frac: int):
    hi = total + frac
    if hi > 62 or abs(int(c_int)) >= 1 << (frac + 1):
        raise ValueError("model limited to hi <= 62 and |c| <= 2^f (all twiddles)")
    prod = np.asarray(x, dtype=np.int64) * np.int64(c_int)        # |prod| < 2^(hi-1)
    kept = np.mod(prod, np.int64(1) << np.int64(hi)) >> np.int64(frac)
    return wrap(kept, total)


def twiddle_ints(size: int, k: int, total: int, frac: int):
    """fft.py:84-91 then mul_const's encode_int: integer twiddle (re, im)."""
    w = cmath.exp(-2j * cmath.pi * k / size)
    return encode_int(w.real, total, frac), encode_int(w.imag, total, frac)


def butterfly(xi, xj, w, total, frac):
    """fft.py:126-134 on integer words; xi/xj are (re, im) lane arrays."""
    wre, wim = w
    t_re = sub(mul_const(xj[0], wre, total, frac), mul_const(xj[1], wim, total, frac), total)
    t_im = add(mul_const(xj[0], wim, total, frac), mul_const(xj[1], wre, total, frac), total)
    hi = (add(xi[0], t_re, total), add(xi[1], t_im, total))
    lo = (sub(xi[0], t_re, total), sub(xi[1], t_im, total))
    return hi, lo


def _bitrev(i: int, width: int) -> int:
    r = 0
    for _ in range(width):
        r = (r << 1) | (i & 1)
        i >>= 1
    return r


def fft_1d(re, im, total: int, frac: int):
    """fft.py:137-174.  re/im: int64 arrays (lanes, M).  Returns (re, im)."""
    re = np.asarray(re, dtype=np.int64)
    im = np.asarray(im, dtype=np.int64)
    m = re.shape[1]
    width = m.bit_length() - 1
    pts = [None] * m
    for i in range(m):
        pts[_bitrev(i, width)] = (re[:, i], im[:, i])
    size = 2
    while size <= m:
        half = size // 2
        new = list(pts)
        for start in range(0, m, size):
            for k in range(half):
                i, j = start + k, start + k + half
                new[i], new[j] = butterfly(pts[i], pts[j], twiddle_ints(size, k, total, frac),
                                           total, frac)
        pts = new
        size *= 2
    return (np.stack([p[0] for p in pts], axis=1), np.stack([p[1] for p in pts], axis=1))


def fft_2d(re, im, rows: int, cols: int, total: int, frac: int):
    """fft.py:177-194: every row (cols-point), then every column (rows-point)."""
    re = np.asarray(re, dtype=np.int64).reshape(-1, rows, cols)
    im = np.asarray(im, dtype=np.int64).reshape(-1, rows, cols)
    lanes = re.shape[0]
    r_re = np.empty_like(re)
    r_im = np.empty_like(im)
    for r in range(rows):
        a, b = fft_1d(re[:, r, :], im[:, r, :], total, frac)
        r_re[:, r, :], r_im[:, r, :] = a, b
    o_re = np.empty_like(re)
    o_im = np.empty_like(im)
    for c in range(cols):
        a, b = fft_1d(r_re[:, :, c], r_im[:, :, c], total, frac)
        o_re[:, :, c], o_im[:, :, c] = a, b
    return o_re.reshape(lanes, -1), o_im.reshape(lanes, -1)


def interleave(re, im):
    """(lanes, M) re/im -> (lanes, 2M) in the reference's output order (point, re then im)."""
    out = np.empty((re.shape[0], 2 * re.shape[1]), dtype=np.int64)
    out[:, 0::2] = re
    out[:, 1::2] = im
    return out
