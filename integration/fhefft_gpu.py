"""The ctypes stub a maintainer adds to the reference (``fhefft/_gpu.py``) to route
``GswScheme.hom_nand / hom_not / hom_add / hom_const_mult / hom_mult`` (fhe.py:325-379)
through ``libfhegpu.so`` (include/fhegpu.h).  INTEGRATION.md section 2 quotes it; the test
``tests/test_reference_dropin.py`` patches it onto the reference's own ``GswScheme`` and checks
every operator against the unpatched reference, bit for bit.

Only the reference's public types are used: a ciphertext is ``type(ct)(matrix=..., level=...,
noise_est=...)`` (fhe.py:148-161).  The conversion to the library's compact form is exact:
C = decompose(V), V = recompose(C) (fhe.py:175-189).  Level, noise and swap bookkeeping stay in
Python exactly as the reference writes them.
"""

import ctypes

import numpy as np


class _Params(ctypes.Structure):                    # fhegpu_params
    _fields_ = [("n", ctypes.c_uint32), ("ell", ctypes.c_uint32),
                ("q", ctypes.c_uint32), ("m", ctypes.c_uint32)]


def load(lib_path):
    lib = ctypes.CDLL(lib_path)
    vp, u32p, u64 = ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint32), ctypes.c_uint64
    lib.fhegpu_ctx_create.argtypes = [ctypes.POINTER(_Params), ctypes.c_int, ctypes.POINTER(vp)]
    lib.fhegpu_last_error.restype = ctypes.c_char_p
    for name in ("fhegpu_nand_batch", "fhegpu_mult_batch", "fhegpu_add_batch"):
        getattr(lib, name).argtypes = [vp, u32p, u32p, u32p, u64]
    lib.fhegpu_not_batch.argtypes = [vp, u32p, u32p, u64]
    lib.fhegpu_const_mult_batch.argtypes = [vp, ctypes.c_uint32, u32p, u32p, u64]
    return lib


def attach(scheme, lib_path, device=0):
    """Patch the operators of a reference ``GswScheme`` instance; returns the context."""
    lib = load(lib_path)
    p = scheme.params
    ctx = ctypes.c_void_p()
    if lib.fhegpu_ctx_create(ctypes.byref(_Params(p.n, p.ell, p.q, p.m)), device, ctypes.byref(ctx)):
        raise RuntimeError(lib.fhegpu_last_error().decode())
    k, ell = p.n + 1, p.ell
    w = 1 << np.arange(ell, dtype=np.uint64)
    u32p = ctypes.POINTER(ctypes.c_uint32)

    def to_v(ct):                                     # recompose (fhe.py:181-185)
        bits = np.asarray(ct.matrix).reshape(p.n_ct, k, ell).astype(np.uint64)
        return ((bits * w).sum(-1) % p.q).astype(np.uint32)

    def to_m(v):                                      # decompose (fhe.py:175-179)
        return ((v[:, :, None] >> np.arange(ell, dtype=np.uint32)) & 1).reshape(p.n_ct, -1).astype(np.float64)

    def call(fn, *args):
        if fn(ctx, *args):
            raise RuntimeError(lib.fhegpu_last_error().decode())

    def ptr(a):
        return a.ctypes.data_as(u32p)

    orig_nand = scheme.hom_nand

    def hom_nand(ct1, ct2):                           # fhe.py:325-341
        level = max(ct1.level, ct2.level) + 1
        if level > p.depth_budget:
            return orig_nand(ct1, ct2)                # raises the reference's NoiseOverflowError
        if ct2.noise_est > ct1.noise_est:
            ct1, ct2 = ct2, ct1
        v1, v2 = to_v(ct1), to_v(ct2)
        out = np.empty_like(v1)
        call(lib.fhegpu_nand_batch, ptr(v1), ptr(v2), ptr(out), 1)
        est = min(ct1.noise_est + p.n_ct * ct2.noise_est, p.q)
        return type(ct1)(matrix=to_m(out), level=level, noise_est=est)

    def hom_not(ct):                                  # fhe.py:343-350
        v = to_v(ct)
        out = np.empty_like(v)
        call(lib.fhegpu_not_batch, ptr(v), ptr(out), 1)
        return type(ct)(matrix=to_m(out), level=ct.level, noise_est=ct.noise_est)

    def hom_add(ct1, ct2):                            # fhe.py:352-356
        v1, v2 = to_v(ct1), to_v(ct2)
        out = np.empty_like(v1)
        call(lib.fhegpu_add_batch, ptr(v1), ptr(v2), ptr(out), 1)
        return type(ct1)(matrix=to_m(out), level=max(ct1.level, ct2.level),
                         noise_est=min(ct1.noise_est + ct2.noise_est, p.q))

    def hom_const_mult(ct, kk):                       # fhe.py:358-364
        v = to_v(ct)
        out = np.empty_like(v)
        call(lib.fhegpu_const_mult_batch, ctypes.c_uint32(kk % p.q), ptr(v), ptr(out), 1)
        return type(ct)(matrix=to_m(out), level=ct.level, noise_est=min(p.n_ct * ct.noise_est, p.q))

    def hom_mult(ct1, ct2):                           # fhe.py:366-379
        if ct2.noise_est > ct1.noise_est:
            ct1, ct2 = ct2, ct1
        v1, v2 = to_v(ct1), to_v(ct2)
        out = np.empty_like(v1)
        call(lib.fhegpu_mult_batch, ptr(v1), ptr(v2), ptr(out), 1)
        return type(ct1)(matrix=to_m(out), level=max(ct1.level, ct2.level),
                         noise_est=min(ct1.noise_est + p.n_ct * ct2.noise_est, p.q))

    scheme.hom_nand, scheme.hom_not = hom_nand, hom_not
    scheme.hom_add, scheme.hom_const_mult, scheme.hom_mult = hom_add, hom_const_mult, hom_mult
    return ctx
