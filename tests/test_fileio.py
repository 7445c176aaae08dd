"""EFT1 container parity with the reference's writer (golden files written by fhefft itself)."""

import os

import numpy as np
import pytest

from oracle import gsw
from paper_1611_08769_b200 import EXACT_PARAMS, FixedFormat, GpuEngine, GswScheme, fft_1d
from paper_1611_08769_b200 import fileio
from paper_1611_08769_b200.errors import ParseError
from paper_1611_08769_b200.fft import read_signal_ints
from tests.helpers import GOLDEN, golden_json


def _blob(name):
    with open(os.path.join(GOLDEN, name), "rb") as fh:
        return fh.read()


@pytest.mark.parametrize("name", ["eft1_exact_in.eft", "eft1_exact_fft.eft"])
def test_container_decode_encode_is_byte_identical(name):
    blob = _blob(name)
    header, params, fmt, values, levels = fileio.decode_container(blob)
    assert params == EXACT_PARAMS and fmt == FixedFormat(16, 8)
    again = fileio.encode_container(params, fmt, header["dims"], header["points"], values, levels)
    assert again == blob


def test_input_container_decrypts_to_the_values():
    _, params, fmt, values, _ = fileio.decode_container(_blob("eft1_exact_in.eft"))
    _, sk = gsw.keygen(gsw.EXACT, 1)
    bits = [gsw.decrypt_bit_compact(gsw.EXACT, sk, v) for v in values]
    meta = golden_json("eft1_exact.json")
    want = []
    for re, im in zip(meta["values_re"], meta["values_im"]):
        for x in (re, im):
            u = round(x * 256) % (1 << 16)
            want.extend((u >> b) & 1 for b in range(16))
    assert bits == want


def test_malformed_containers_raise(tmp_path):
    blob = _blob("eft1_exact_in.eft")
    with pytest.raises(ParseError):
        fileio.decode_container(b"NOPE" + blob[4:])
    with pytest.raises(ParseError):
        fileio.decode_container(blob[:-5])


@pytest.mark.gpu
def test_server_fft_step_reproduces_reference_container(tmp_path):
    """cli fft (cli.py:71-87): load EFT1 on the GPU engine, fft_1d, write EFT1 -> the
    reference's output container, byte for byte."""
    scheme = GswScheme(EXACT_PARAMS)
    keys = scheme.keygen(1)
    server = GpuEngine(scheme, public_key=keys.public_key)
    sig, fmt = fileio.read_ciphertext_signal(os.path.join(GOLDEN, "eft1_exact_in.eft"), server)
    out = fft_1d(sig)
    path = tmp_path / "out.eft"
    fileio.write_ciphertext_signal(path, EXACT_PARAMS, server, out, fmt)
    assert path.read_bytes() == _blob("eft1_exact_fft.eft")
    assert server.nand_count == golden_json("eft1_exact.json")["nand_count"]
    client = GpuEngine(scheme, keys=keys)
    res, _ = fileio.read_ciphertext_signal(path, client)
    assert read_signal_ints(client, res)[0].tolist() == golden_json("eft1_exact.json")["fft_words"]
