"""Bitsliced cleartext engine on the GPU: drop-in for ``fhefft.engine.CleartextEngine``.

Reference: engine.py:69-121.  Same protocol (``batch_size``, ``mask``, ``nand_count``,
``max_depth``, ``stats``, ``constant``, ``input_bit`` with lanes packed in an int,
``nand``, ``read_back`` returning the packed int), same fold rules (engine.py:107-116:
const/const -> const, NAND(x, 0) -> 1, NAND(x, 1) -> NOT x without a gate), same depth
accounting and error messages.  Results are exact bits, identical to the reference.

What changes is where the bits live: gates are only recorded (the levelised netlist of
``GpuEngine``), and on ``flush`` every level runs as one launch of ``bits_level_kernel``
over (gate x 32-lane word) items -- so one pass evaluates the circuit for millions of
independent inputs (the reference's error experiments, harness.py:122-198, at scale).
"""

from __future__ import annotations

import numpy as np

from .engine import GateStats, GpuBit, LevelledNetlist
from .errors import UsageError


class GpuClearEngine(LevelledNetlist):
    """Exact plaintext bit engine with lane packing, evaluated bitsliced on the GPU."""

    def __init__(self, batch_size: int = 1, device: int = 0, keep_all: bool = False):
        if batch_size < 1:
            raise UsageError("batch_size must be >= 1")
        self.batch_size = batch_size
        self.mask = (1 << batch_size) - 1
        self.nand_count = 0
        self.max_depth = 0
        self.device = device
        self.executed_nands = 0
        self.launches = 0
        self.programs_run = 0
        self.last_compile = None
        self._init_netlist(keep_all)
        self._bits = None
        self._capacity = 0
        self._pending_slots: list[int] = []
        self._pending_words: list[np.ndarray] = []
        self.words = (batch_size + 31) // 32

    # -- protocol attributes -----------------------------------------------------------

    @property
    def stats(self) -> GateStats:
        return GateStats(self.nand_count, self.max_depth)

    @property
    def bits(self):
        """Device wire store (created on first use; raises DeviceError without the library)."""
        if self._bits is None:
            from ._native import BitsContext
            self._bits = BitsContext(self.batch_size, self.device)
        return self._bits

    # -- packing -----------------------------------------------------------------------

    def _to_words(self, lanes: int) -> np.ndarray:
        return np.frombuffer(int(lanes).to_bytes(4 * self.words, "little"), dtype="<u4")

    def _from_words(self, words: np.ndarray) -> int:
        return int.from_bytes(np.ascontiguousarray(words, dtype="<u4").tobytes(), "little")

    # -- bit-engine protocol -----------------------------------------------------------

    def constant(self, bit: int) -> GpuBit:
        if bit not in (0, 1):
            raise UsageError(f"constant must be 0 or 1, got {bit!r}")
        return GpuBit(self, -1, 0, True, bit, -1)

    def input_bit(self, lanes: int) -> GpuBit:
        """New variable wire; ``lanes`` packs one bit per lane (0/1 if batch 1)."""
        if not 0 <= lanes <= self.mask:
            raise UsageError(f"lane value {lanes:#x} out of range for "
                             f"batch_size={self.batch_size}")
        return self._input(self._to_words(lanes))

    def input_words(self, words: np.ndarray) -> list:
        """Many wires at once from packed words, shape (wires, ceil(batch/32)) u32."""
        words = np.asarray(words, dtype=np.uint32)
        if words.ndim != 2 or words.shape[1] != self.words:
            raise UsageError(f"expected (wires, {self.words}) packed words")
        tail = self.batch_size % 32
        if tail and (words[:, -1] >> np.uint32(tail)).any():
            raise UsageError(f"lane bits beyond batch_size={self.batch_size}")
        return [self._input(w) for w in words]

    def input_block(self, bits) -> list:
        """Wires from a (lanes, n) 0/1 array: column j becomes wire j (lane l = row l)."""
        bits = np.asarray(bits)
        if bits.ndim != 2 or bits.shape[0] != self.batch_size:
            raise UsageError(f"expected a ({self.batch_size}, n) bit block")
        if ((bits != 0) & (bits != 1)).any():
            raise UsageError("input bits must be 0 or 1")
        pad = np.zeros((self.words * 32, bits.shape[1]), dtype=np.uint8)
        pad[: self.batch_size] = bits
        packed = np.packbits(pad.T.reshape(bits.shape[1], self.words, 32), axis=2, bitorder="little")
        packed = np.ascontiguousarray(packed)          # view as u32 needs a contiguous last axis
        return self.input_words(packed.view("<u4").reshape(bits.shape[1], self.words))

    def _input(self, words: np.ndarray) -> GpuBit:
        node = self._new_node(0, 0)
        slot = self._alloc_slot()
        self._slot[node] = slot
        self._pending_slots.append(slot)
        self._pending_words.append(words)
        return GpuBit(self, node, 0, False, None, self._new_wire())

    def nand(self, a: GpuBit, b: GpuBit) -> GpuBit:
        if a.engine is not self or b.engine is not self:
            raise UsageError("cannot mix handles from different engines")
        if a.const or b.const:
            return self._fold(a, b)
        self.nand_count += 1
        la, lb = self._level[a.node], self._level[b.node]
        depth = (la if la >= lb else lb) + 1
        if depth > self.max_depth:
            self.max_depth = depth
        node = self._new_node(depth, 0)
        self._pending_ops.extend((a.node, a.neg, b.node, b.neg, node))
        self.executed_nands += 1
        return GpuBit(self, node, 0, False, None, self._new_wire())

    def _fold(self, a: GpuBit, b: GpuBit) -> GpuBit:
        """engine.py:107-116: const/const -> const; NAND(x,0) -> 1; NAND(x,1) -> NOT x."""
        if a.const and b.const:
            return self.constant(0 if (a.plain and b.plain) else 1)
        if b.const:
            a, b = b, a
        if a.plain == 0:
            return self.constant(1)
        return GpuBit(self, b.node, b.neg ^ 1, False, None, self._new_wire())

    def map_parallel(self, fn, items):
        return [fn(x) for x in items]

    # -- evaluation ------------------------------------------------------------------------

    def _upload_inputs(self):
        if not self._pending_slots:
            return
        self._ensure_capacity()
        self.bits.write(np.asarray(self._pending_slots, dtype=np.uint64), np.stack(self._pending_words))
        self._pending_slots.clear()
        self._pending_words.clear()

    def _ensure_capacity(self):
        if self._n_slots > self._capacity:
            cap = max(self._n_slots, int(self._capacity * 1.25) + 64)
            self.bits.reserve(cap)
            self._capacity = cap

    def flush(self):
        """Evaluate every pending gate: one launch per level over all (gate, word) items."""
        self._upload_inputs()
        if not self._pending_ops:
            return None
        prog = self._compile()
        self._pending_ops = []
        self.last_compile = prog
        self._ensure_capacity()
        self.bits.run(prog["ops"], prog["offsets"])
        self.programs_run += 1
        self.launches += int((prog["widths"] > 0).sum())
        return prog

    def read_back(self, h: GpuBit) -> int:
        """Packed lane values of a wire (an int in [0, 2**batch_size))."""
        return self.read_back_many([h])[0]

    def read_back_many(self, handles) -> list[int]:
        words = self.read_words(handles)
        return [self._from_words(w) for w in words]

    def read_words(self, handles) -> np.ndarray:
        """Packed words (len(handles), ceil(batch/32)) u32 of many wires, one gather."""
        out = np.zeros((len(handles), self.words), dtype=np.uint32)
        var = []
        for i, h in enumerate(handles):
            if h.engine is not self:
                raise UsageError("handle belongs to a different engine")
            if h.const:
                if h.plain:
                    out[i] = self._to_words(self.mask)
            else:
                var.append(i)
        if var:
            self.flush()
            slots = np.asarray([self._slot[handles[i].node] for i in var], dtype=np.int64)
            if (slots < 0).any():
                raise UsageError("wire was released (no live handle); use keep_all=True")
            comp = np.asarray([handles[i].neg for i in var], dtype=np.uint8)
            out[var] = self.bits.read(slots.astype(np.uint64), comp)
        return out

    def read_bits(self, handles) -> np.ndarray:
        """Lane bits (len(handles), batch_size) uint8 of many wires."""
        w = self.read_words(handles)
        bits = np.unpackbits(w.view(np.uint8).reshape(len(handles), -1), axis=1, bitorder="little")
        return bits[:, : self.batch_size]

    read_back_bits = read_bits          # the fast path fft.read_signal_ints looks for
