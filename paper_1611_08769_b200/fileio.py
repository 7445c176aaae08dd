"""EFT1 encrypted-signal container and parameter files, byte-compatible with the reference.

Reference: fhefft/fileio.py:1-202 (EFT1 = magic, u32 version, u32 header length, UTF-8
JSON header, then every ciphertext's N x N bit matrix packed 8 bits per byte, MSB first,
row-major; points in order, real word then imaginary word, bits LSB first).

The engine keeps ciphertexts in compact form V (N x k); a container stores the reference
matrix C = decompose(V), so reading and writing are pure bit reshuffles (vectorised here):
C[r, i*ell + j] = bit j of V[r, i].  As in the reference, importing a container resets each
ciphertext's noise estimate to 0 (fileio.py:190-191), which later operand swaps depend on.

This is the server-side I/O of the ``fhefft fft`` step (cli.py:71-87): load an encrypted
signal onto the GPU engine, run the FFT netlist, write the encrypted spectrum.
"""

from __future__ import annotations

import json
import math
import struct

import numpy as np

from .arith import FixedFormat, FixedWord
from .errors import ParseError, UsageError
from .fft import ComplexFixed, SignalBuffer
from .scheme import Ciphertext, SchemeParams

MAGIC = b"EFT1"
CONTAINER_VERSION = 1


def params_to_dict(params: SchemeParams) -> dict:
    return {"n": params.n, "q": params.q, "m": params.m,
            "noise_bound": params.noise_bound, "depth_budget": params.depth_budget}


def params_from_dict(d: dict, path=None) -> SchemeParams:
    try:
        return SchemeParams(n=int(d["n"]), q=int(d["q"]), m=int(d["m"]),
                            noise_bound=int(d["noise_bound"]), depth_budget=int(d["depth_budget"]))
    except KeyError as exc:
        raise ParseError(f"missing parameter field {exc}", path=path) from exc


def write_params(path, params: SchemeParams):
    with open(path, "w") as fh:
        json.dump({"format": "fhefft-params-v1", **params_to_dict(params)}, fh, indent=2)
        fh.write("\n")


def read_params(path) -> SchemeParams:
    with open(path) as fh:
        try:
            data = json.load(fh)
        except json.JSONDecodeError as exc:
            raise ParseError(str(exc), path=path, line=exc.lineno) from exc
    return params_from_dict(data, path=path)


# -- compact <-> packed matrix bits ---------------------------------------------------------

def pack_compact(values: np.ndarray, params: SchemeParams) -> np.ndarray:
    """(count, N, k) compact ciphertexts -> (count, ceil(N^2/8)) bytes of the reference matrix."""
    v = np.asarray(values, dtype=np.uint32)
    bits = ((v[..., None] >> np.arange(params.ell, dtype=np.uint32)) & 1).astype(np.uint8)
    flat = bits.reshape(len(v), params.n_ct * params.n_ct)
    return np.packbits(flat, axis=1)


def unpack_compact(packed: np.ndarray, params: SchemeParams) -> np.ndarray:
    """Inverse of pack_compact; entries of C are 0/1 so V = sum_j C[r, i ell + j] 2^j exactly.

    (fhe.py:181-185 with no mod: a stored flattened matrix is already reduced.)"""
    n, ell = params.n_ct, params.ell
    bits = np.unpackbits(np.asarray(packed, dtype=np.uint8), axis=1)[:, :n * n]
    bits = bits.reshape(len(packed), n, params.k, ell)
    # bit j of V[r, i] is C[r, i*ell + j]: repack each ell-bit group LSB first into a u32
    pad = np.zeros(bits.shape[:3] + (32 - ell,), dtype=np.uint8)
    vals = np.packbits(np.concatenate([bits, pad], axis=3), axis=3, bitorder="little")
    vals = vals.view("<u4")[..., 0]
    if (vals >= params.q).any():
        raise ParseError("container holds a matrix that is not a flattened ciphertext")
    return np.ascontiguousarray(vals, dtype=np.uint32)


def encode_container(params: SchemeParams, fmt: FixedFormat, dims, n_points: int,
                     values: np.ndarray, levels) -> bytes:
    """EFT1 bytes exactly as fileio.py:110-137 writes them."""
    header = {
        "kind": "fhefft-signal",
        "params": params_to_dict(params),
        "params_digest": params.digest(),
        "fixed_format": {"total_bits": fmt.total_bits, "frac_bits": fmt.frac_bits},
        "dims": list(dims) if isinstance(dims, tuple) else dims,
        "points": n_points,
        "ct_side": params.n_ct,
        "levels": [int(x) for x in levels],
    }
    head = json.dumps(header).encode()
    return MAGIC + struct.pack("<II", CONTAINER_VERSION, len(head)) + head + \
        pack_compact(values, params).tobytes()


def decode_container(blob: bytes, path=None):
    """(header, params, fmt, compact values (count, N, k), levels) of an EFT1 blob."""
    if blob[:4] != MAGIC:
        raise ParseError("not an encrypted-signal container (bad magic)", path=path, offset=0)
    version, head_len = struct.unpack("<II", blob[4:12])
    if version != CONTAINER_VERSION:
        raise ParseError(f"unsupported container version {version}", path=path, offset=4)
    try:
        header = json.loads(blob[12:12 + head_len])
    except json.JSONDecodeError as exc:
        raise ParseError(f"bad container header: {exc}", path=path, offset=12) from exc
    params = params_from_dict(header["params"], path=path)
    if params.digest() != header["params_digest"]:
        raise ParseError("parameter digest mismatch", path=path)
    fmt = FixedFormat(header["fixed_format"]["total_bits"], header["fixed_format"]["frac_bits"])
    n = header["ct_side"]
    stride = math.ceil(n * n / 8)
    count = header["points"] * 2 * fmt.total_bits
    payload = blob[12 + head_len:]
    if len(payload) != count * stride:
        raise ParseError(f"payload holds {len(payload)} bytes, expected {count * stride}", path=path)
    packed = np.frombuffer(payload, dtype=np.uint8).reshape(count, stride)
    return header, params, fmt, unpack_compact(packed, params), header["levels"]


def read_ciphertext_params(path) -> SchemeParams:
    with open(path, "rb") as fh:
        blob = fh.read()
    if blob[:4] != MAGIC:
        raise ParseError("not an encrypted-signal container (bad magic)", path=path, offset=0)
    _, head_len = struct.unpack("<II", blob[4:12])
    header = json.loads(blob[12:12 + head_len])
    params = params_from_dict(header["params"], path=path)
    if params.digest() != header["params_digest"]:
        raise ParseError("parameter digest mismatch", path=path)
    return params


# -- engine-facing I/O ---------------------------------------------------------------------------

def write_ciphertext_signal(path, params: SchemeParams, engine, signal: SignalBuffer,
                            fmt: FixedFormat, lane: int = 0):
    """Serialise every word bit of a signal (one lane of a batched engine)."""
    handles = [h for pt in signal.points for word in (pt.re, pt.im) for h in word.bits]
    count = len(handles)
    values = np.empty((count, params.n_ct, params.k), dtype=np.uint32)
    levels = [0] * count
    var = [i for i, h in enumerate(handles) if not h.const]
    if var and hasattr(engine, "read_nodes"):
        vals = engine.read_nodes([handles[i].node for i in var], [handles[i].neg for i in var],
                                 lanes=[lane])
        for j, i in enumerate(var):
            values[i] = vals[j, 0]
            levels[i] = engine._level[handles[i].node]
    else:
        for i in var:
            ct = engine.export_ct(handles[i])
            ct = ct[lane] if isinstance(ct, list) else ct
            values[i] = ct.v
            levels[i] = ct.level
    for i, h in enumerate(handles):
        if h.const:                                   # trivial encryption (fhe.py:244-249)
            values[i] = engine.scheme.trivial_encrypt_bit(h.plain).v
    blob = encode_container(params, fmt, signal.dims, len(signal.points), values, levels)
    with open(path, "wb") as fh:
        fh.write(blob)


def read_ciphertext_signal(path, engine):
    """Load a container onto an engine with matching parameters (noise estimates reset to 0)."""
    with open(path, "rb") as fh:
        blob = fh.read()
    header, params, fmt, values, levels = decode_container(blob, path=path)
    if engine.scheme.params != params:
        raise UsageError(f"engine parameters {engine.scheme.params} do not match the file's {params}")
    if engine.batch_size != 1:
        raise UsageError("containers hold one signal; load it on a batch_size=1 engine")
    handles = [engine.import_ct(Ciphertext(values[i], int(levels[i]), 0, params))
               for i in range(len(values))]
    w = fmt.total_bits
    points = []
    for p in range(header["points"]):
        base = 2 * w * p
        points.append(ComplexFixed(FixedWord(tuple(handles[base:base + w]), fmt),
                                   FixedWord(tuple(handles[base + w:base + 2 * w]), fmt)))
    dims = header["dims"]
    return SignalBuffer(tuple(points), tuple(dims) if isinstance(dims, list) else int(dims)), fmt
