"""B200-native engine for the encrypted-FFT hot path of arxiv 1611.08769.

Public surface mirrors the reference package ``fhefft`` (fhefft/__init__.py)
for the hot path: scheme (params, keys, compact ciphertexts, homomorphic NAND
/ NOT on the GPU), the bit-engine protocol (``GpuEngine`` in place of
``FheEngine``), gates, fixed-point arithmetic and the FFT entry points.
Gates run in ``csrc/`` (sm_100a CUDA, tcgen05 tensor cores) behind the C ABI
declared in ``include/fhegpu.h``.
"""

from .arith import (FixedFormat, FixedWord, add, bits_to_int, constant_word, decode, encode,
                    encode_int, full_adder, half_adder, input_word, int_to_bits, mul_const,
                    mul_fixed, mul_integer, read_word, sub)
from .clear import GpuClearEngine
from .engine import GateStats, GpuBit, GpuEngine
from .errors import (CapabilityError, DeviceError, FhefftError, NoiseOverflowError,
                     ParameterError, ParseError, RangeError, UsageError)
from .fft import (ComplexFixed, SignalBuffer, TwiddleTable, bit_reverse_permute, butterfly, fft2,
                  fft_1d, fft_2d, ifft_1d, input_signal, read_signal, read_signal_ints)
from .gates import and_, nor_, not_, or_, xnor_, xor_
from .scheme import (DEFAULT0_PARAMS, DEFAULT_PARAMS, EXACT_PARAMS, Ciphertext, GswScheme, KeyPair,
                     SchemeParams, decode_gadget_samples)

# reference name for the FHE bit engine
FheEngine = GpuEngine
CleartextEngine = GpuClearEngine

__all__ = [
    "CapabilityError", "Ciphertext", "CleartextEngine", "GpuClearEngine", "ComplexFixed", "DEFAULT0_PARAMS", "DEFAULT_PARAMS",
    "DeviceError", "EXACT_PARAMS", "FheEngine", "FhefftError", "FixedFormat", "FixedWord",
    "GateStats", "GpuBit", "GpuEngine", "GswScheme", "KeyPair", "NoiseOverflowError",
    "ParameterError", "ParseError", "RangeError", "SchemeParams", "SignalBuffer", "TwiddleTable",
    "UsageError", "add", "and_", "bit_reverse_permute", "bits_to_int", "butterfly",
    "constant_word", "decode", "decode_gadget_samples", "encode", "encode_int", "fft2", "fft_1d",
    "fft_2d", "full_adder", "half_adder", "ifft_1d", "input_signal", "input_word", "int_to_bits",
    "mul_const", "mul_fixed", "mul_integer", "nor_", "not_", "or_", "read_signal",
    "read_signal_ints", "read_word", "sub", "xnor_", "xor_",
]
