"""GPU bit engine: the reference's bit-engine protocol over a levelised netlist.

Drop-in for ``fhefft.engine.FheEngine`` (engine.py:124-214): same attributes
(``batch_size``, ``nand_count``, ``max_depth``, ``stats``), same methods
(``constant``, ``input_bit``, ``nand``, ``read_back``, ``export_ct``,
``import_ct``, ``map_parallel``), same folding rules, operand swap, level and
noise bookkeeping, and the same error classes.  What changes is *when* gates
run: ``nand`` only records the gate.  On ``flush`` (triggered by
``read_back`` / ``export_ct`` or explicitly) every pending gate is grouped by
its level (the reference's ``level`` = NAND depth), ciphertext slots are
assigned by liveness, and each level executes as ONE kernel launch over every
gate of that level and every lane (independent signal) -- never one gate per
launch.

Folded NOTs (NAND(x, const 1) -> hom_not, engine.py:180-187) cost nothing:
a handle is (node, complement flag) and the complement is applied when a
kernel loads the operand, which is bit-identical to the reference's
``flatten(I - C)`` because (G - (G - V) mod q) mod q = V.

Lanes: ``batch_size`` > 1 evaluates the same netlist for that many
independent inputs (like the reference's ``CleartextEngine`` lane packing):
``input_bit`` takes the lane bits packed in an int (bit l = lane l) and
``read_back`` returns them packed the same way.  Lane l draws its encryption
randomness from ``lane_rngs[l]`` (or the single ``rng``, lane-major).
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np

from .errors import CapabilityError, NoiseOverflowError, UsageError
from ._native import RES_OP_DTYPE
from .scheme import Ciphertext, GswScheme, KeyPair

_UPLOAD_BATCH_BYTES = 256 << 20
STREAM_OUT = 8          # fhegpu_op flag (include/fhegpu.h): output not read later in the program
OP_TEMP = 16            # fhegpu_op flag: output read by nothing outside the program


@dataclass(frozen=True)
class GateStats:
    """Snapshot of the gate accounting (engine.py:37-42)."""

    nand_count: int
    max_depth: int


class GpuBit:
    """One circuit wire: a device ciphertext node (+ complement flag) or a public constant."""

    __slots__ = ("engine", "node", "neg", "const", "plain", "wire")

    def __init__(self, engine, node: int, neg: int, const: bool, plain, wire: int):
        self.engine = engine
        self.node = node
        self.neg = neg
        self.const = const
        self.plain = plain
        self.wire = wire
        if node >= 0:
            engine._refs[node] += 1

    def __del__(self):
        if self.node >= 0:
            try:
                self.engine._refs[self.node] -= 1
            except Exception:  # interpreter shutdown
                pass

    @property
    def ct(self):
        """The reference handle's ``.ct``: this wire's ciphertext (flushes)."""
        return None if self.const else self.engine.export_ct(self)


class CircuitTemplate:
    """A recorded circuit call (e.g. one ``fft_1d`` over one word format), replayable on any
    inputs with the same structure without re-running the Python circuit code.

    The netlist of the reference's circuits depends only on the call's static arguments and
    on the input wires' structure (which bits alias which node, complement flags, constants)
    and their level / noise estimates -- never on the encrypted data (fft.py:137-174 calls
    engine.nand in a fixed order; the fold and swap rules of engine.py:168-187 / fhe.py:336
    read only that bookkeeping).  Local node ids: 0..n_in-1 are the distinct input nodes,
    n_in.. the nodes the call created.  ``outs`` rows: (kind, value, neg), kind 0 = public
    constant `value`, 1 = local node `value`."""

    _next_uid = 0

    def __init__(self, n_in, in_levels, in_ests, ops, levels, ests, outs, nand_count, executed,
                 max_level, wires):
        CircuitTemplate._next_uid += 1
        self.uid = CircuitTemplate._next_uid
        self.n_in = n_in
        self.in_levels, self.in_ests = in_levels, in_ests
        self.ops = ops                      # (n_ops, 5) int64: left, lneg, right, rneg, out (local ids)
        self.levels, self.ests = levels, ests
        self.outs = outs
        self.nand_count, self.executed = nand_count, executed
        self.max_level, self.wires = max_level, wires
        out_nodes = outs[outs[:, 0] == 1, 1]
        self.out_internal = np.unique(out_nodes[out_nodes >= n_in])     # local ids, sorted
        self.compiled: dict = {}            # (batch, schedule pref, kernel) -> region compile | None


class LevelledNetlist:
    """Lazy netlist recorder shared by the GPU engines: node tables (level, noise estimate,
    slot, live-handle refcount), pending gates, and the level sort + liveness slot allocation
    that turns them into one launch per level."""

    def _init_netlist(self, keep_all: bool = False):
        self.keep_all = keep_all
        self._wire = 0
        self._level: list[int] = []
        self._est: list[int] = []
        self._slot: list[int] = []
        self._refs: list[int] = []
        self._pending_ops: list[int] = []       # flat: left, lneg, right, rneg, out
        self._free: list[int] = []
        self._n_slots = 0

    def _new_wire(self) -> int:
        w = self._wire
        self._wire += 1
        return w

    def _new_node(self, level: int, est: int) -> int:
        self._level.append(level)
        self._est.append(est)
        self._slot.append(-1)
        self._refs.append(0)
        return len(self._level) - 1

    def _new_nodes(self, levels, ests, slots=None) -> range:
        """Bulk _new_node: len(levels) nodes (ids returned as a range)."""
        n0, n = len(self._level), len(levels)
        self._level.extend(levels)
        self._est.extend(ests)
        self._slot.extend([-1] * n if slots is None else slots)
        self._refs.extend([0] * n)
        return range(n0, n0 + n)

    def _alloc_slots(self, n: int) -> list:
        """n slots: the most recently freed first (as _alloc_slot), then fresh ones."""
        take = min(n, len(self._free))
        out = self._free[len(self._free) - take:][::-1] if take else []
        if take:
            del self._free[len(self._free) - take:]
        if n > take:
            out.extend(range(self._n_slots, self._n_slots + n - take))
            self._n_slots += n - take
        return out

    def _alloc_slot(self) -> int:
        if self._free:
            return self._free.pop()
        s = self._n_slots
        self._n_slots += 1
        return s

    @staticmethod
    def _dataflow_order(ops, order, sorted_level, n_nodes):
        """Within each level, order ops by the position of their latest producer.

        A dataflow launch hands item i to CTA i % G in order; an item whose producer is
        still in flight stalls that CTA's whole pipeline.  Sorting every level by producer
        position makes the early items of level L+1 consume the early (long finished)
        items of level L, so dependency distances approach a full level width."""
        left_n, right_n, out_n = ops[:, 0], ops[:, 2], ops[:, 4]
        pos = np.full(n_nodes, -1, dtype=np.int64)
        starts = np.flatnonzero(np.diff(sorted_level, prepend=sorted_level[:1] - 1))
        ends = np.append(starts[1:], len(order))
        out = np.empty_like(order)
        for s, e in zip(starts.tolist(), ends.tolist()):
            seg = order[s:e]
            key = np.maximum(pos[left_n[seg]], pos[right_n[seg]])
            seg = seg[np.argsort(key, kind="stable")]
            pos[out_n[seg]] = np.arange(s, e)
            out[s:e] = seg
        return out

    def _compile(self, ssa: bool = False, ring_temps: bool = False, pin_old: bool = False):
        """Level-sort the pending gates and assign ciphertext slots by liveness.

        A slot read at level L is released before the launch of level L + 1 at
        the earliest, so no launch ever writes a slot another gate of the same
        launch reads.  Nodes still referenced by a live handle keep their slot.

        ssa=True (dataflow programs, one launch without level boundaries): no slot is
        reused within the program -- slots released by it return to the pool only after
        it -- and ``deps`` gives, per op, the op indices that produced its operands.

        pin_old=True (register-file programs, which read inputs and write outputs in their own
        order): slots of nodes that existed before the program are not reused inside it, the
        program's own temporaries reuse slots as in level launches.

        ring_temps=True (tiled programs): outputs nobody holds after the program
        ("temporaries") get no batch-wide slot; ``temp`` (per op: left, right, out) carries
        their index 0..n_temp-1 instead (-1 elsewhere) for _tile to place in an L2-sized ring.
        """
        ops = np.asarray(self._pending_ops, dtype=np.int64).reshape(-1, 5)
        level = np.asarray(self._level, dtype=np.int64)
        slot = np.asarray(self._slot, dtype=np.int64)
        refs = np.asarray(self._refs, dtype=np.int64)
        n_nodes = len(level)
        op_level = level[ops[:, 4]]
        order = np.argsort(op_level, kind="stable")
        if ssa:
            order = self._dataflow_order(ops, order, op_level[order], n_nodes)
        ops = ops[order]
        op_level = op_level[order]
        left, lneg, right, rneg, out = ops.T
        # last level at which each node is read by a pending gate
        last_use = np.full(n_nodes, -1, dtype=np.int64)
        np.maximum.at(last_use, left, op_level)
        np.maximum.at(last_use, right, op_level)
        # release point of each slot: the level before whose launch it becomes free
        never = np.iinfo(np.int64).max
        free_at = np.full(n_nodes, never, dtype=np.int64)
        if not self.keep_all:
            dead = refs <= 0
            old = (slot >= 0) & dead
            free_at[old] = np.where(last_use[old] >= 0, last_use[old] + 1, 0)
            new_dead = np.zeros(n_nodes, dtype=bool)
            new_dead[out] = True
            new_dead &= dead
            free_at[new_dead] = np.maximum(last_use[new_dead], level[new_dead]) + 1
        temp_id = np.full(n_nodes, -1, dtype=np.int64)
        if ring_temps and not self.keep_all:
            tnodes = out[new_dead[out]]
            temp_id[tnodes] = np.arange(len(tnodes))
        cand = np.nonzero(free_at != never)[0]
        cand = cand[np.argsort(free_at[cand], kind="stable")]
        cand_at = free_at[cand]
        lv_vals, lv_start = np.unique(op_level, return_index=True)
        lv_end = np.append(lv_start[1:], len(op_level))
        ptr = 0
        free = self._free
        deferred = []
        first_lv = int(lv_vals[0]) if len(lv_vals) else 0
        was_slotted = slot >= 0                    # nodes from before this program
        for lv, s, e in zip(lv_vals.tolist(), lv_start.tolist(), lv_end.tolist()):
            hi = int(np.searchsorted(cand_at, lv, side="right"))
            if hi > ptr:
                rel = slot[cand[ptr:hi]]
                if ssa or pin_old:                 # only slots this program never reads
                    untouched = free_at[cand[ptr:hi]] <= first_lv
                    if pin_old and not ssa:
                        untouched |= ~was_slotted[cand[ptr:hi]]
                    free.extend(rel[(rel >= 0) & untouched].tolist())
                    deferred.extend(rel[(rel >= 0) & ~untouched].tolist())
                else:
                    free.extend(rel[rel >= 0].tolist())
                ptr = hi
            outs = out[s:e]
            if ring_temps:
                outs = outs[temp_id[outs] < 0]             # temporaries live in the ring
            cnt = len(outs)
            take = min(cnt, len(free))
            new_slots = np.empty(cnt, dtype=np.int64)
            if take:
                new_slots[:take] = free[len(free) - take:]
                del free[len(free) - take:]
            if cnt > take:
                new_slots[take:] = np.arange(self._n_slots, self._n_slots + cnt - take)
                self._n_slots += cnt - take
            slot[outs] = new_slots
        table = np.empty(len(out), dtype=[("left", "<u4"), ("right", "<u4"),
                                          ("out", "<u4"), ("flags", "<u4")])
        lo = 0 if ring_temps else None              # ring temporaries: placeholder, see _tile
        table["left"] = np.clip(slot[left], lo, None)
        table["right"] = np.clip(slot[right], lo, None)
        table["out"] = np.clip(slot[out], lo, None)
        table["flags"] = lneg | (rneg << 1)
        if ptr < len(cand):                       # released after the last launch
            rel = slot[cand[ptr:]]
            free.extend(rel[rel >= 0].tolist())
        free.extend(deferred)
        released = cand                            # every released node loses its slot
        slot[released] = -1
        self._slot = slot.tolist()
        offsets = np.append(lv_start, len(out)).astype(np.uint64)
        prog = {"ops": table, "offsets": offsets, "levels": lv_vals,
                "widths": np.diff(offsets).astype(np.int64),
                "nodes": np.stack([left, right, out], axis=1),
                "held": np.ones(len(out), dtype=bool) if self.keep_all else ~new_dead[out]}
        if ssa:
            producer = np.full(n_nodes, -1, dtype=np.int64)
            producer[out] = np.arange(len(out))
            prog["deps"] = np.stack([producer[left], producer[right]], axis=1).astype(np.int32)
        if ring_temps:
            prog["temp"] = np.stack([temp_id[left], temp_id[right], temp_id[out]], axis=1)
            prog["n_temp"] = int((temp_id[out] >= 0).sum())
        return prog


class GpuEngine(LevelledNetlist):
    """Lazy, levelised FHE bit engine on one B200."""

    def __init__(self, scheme: GswScheme, keys: KeyPair | None = None, public_key=None,
                 rng=None, threads: int = 1, batch_size: int = 1, lane_rngs=None,
                 cse: bool = False, keep_all: bool = False, record_trace: bool = False,
                 dry_run: bool = False, device_encrypt: bool = False, schedule: str = "auto"):
        if threads < 1:
            raise UsageError("threads must be >= 1")
        if batch_size < 1:
            raise UsageError("batch_size must be >= 1")
        if schedule not in ("auto", "levels", "dataflow", "queue", "tiled", "resident", "regfile", "flow"):
            raise UsageError(f"schedule must be 'auto', 'levels', 'dataflow', 'queue', 'tiled', "
                             f"'resident', 'regfile' or 'flow', got {schedule!r}")
        self.schedule = schedule
        if lane_rngs is not None and len(lane_rngs) != batch_size:
            raise UsageError("need one rng per lane")
        if not isinstance(scheme, GswScheme):
            # the reference's own GswScheme (cli.cmd_fft builds one from the container's
            # params, cli.py:74-75): evaluate on this package's scheme for the same params
            scheme = GswScheme(scheme.params)
        self.scheme = scheme
        self.params = scheme.params
        self.public_key = keys.public_key if keys is not None else public_key
        self.secret_key = keys.secret_key if keys is not None else None
        self.rng = rng if rng is not None else np.random.default_rng()
        self.lane_rngs = lane_rngs
        self.threads = threads
        self.batch_size = batch_size
        self.mask = (1 << batch_size) - 1
        self.nand_count = 0
        self.max_depth = 0
        self.executed_nands = 0
        self.cse = cse
        self.trace = [] if record_trace else None
        self._init_netlist(keep_all)
        self._pending_in_idx: list[np.ndarray] = []
        self._pending_in_val: list[np.ndarray] = []
        self._pending_in_bytes = 0
        self._cse_map: dict | None = {} if cse else None
        self.last_program = None
        self.programs_run = 0
        self.launches = 0
        self._fresh_noise = self.params.m * self.params.noise_bound
        # dry_run: record and compile only (no encryption, no device) -- used to
        # test netlists and slot allocation on machines without a GPU
        self.dry_run = dry_run
        self.dry_inputs: list[tuple[int, int]] = []     # (slot, packed lane bits)
        self.dry_programs: list[dict] = []
        # device_encrypt: fresh encryptions are generated on the GPU (stream-exact with
        # numpy's PCG64); the host only snapshots generator positions and advances them.
        self.device_encrypt = device_encrypt
        self._enc_streams: list[tuple] = []
        self._enc_stream_id: dict = {}
        self._enc_rows: list[np.ndarray] = []     # per chunk: (stream_idx, u32_off, mu, target)
        self._draws_per_ct = self.params.n_ct * self.params.m
        # per-gate bookkeeping reads these (SchemeParams derives them on every access)
        self._n_ct, self._q, self._budget = self.params.n_ct, self.params.q, self.params.depth_budget
        # circuit templates (`circuit`): a replayed call stays one lazy macro until flush
        self._macros: list[tuple] = []      # (template, input nodes, real node per out_internal)
        self._capturing = 0                 # nesting depth of circuit() recordings
        self._regions: dict = {}            # template uid -> (base slot, Program, compile)
        self.template_hits = 0
        self._spill_block = (0, 0)          # (first slot, slots): register-file spill space
        self._loose: list[int] = []         # nodes given a slot outside _compile (inputs, replay outputs)

    # -- protocol attributes -----------------------------------------------------------

    @property
    def stats(self) -> GateStats:
        return GateStats(self.nand_count, self.max_depth)

    @property
    def ctx(self):
        return self.scheme.ctx

    # -- nodes and slots ---------------------------------------------------------------

    def _lane_idx(self, slot: int) -> np.ndarray:
        return slot * self.batch_size + np.arange(self.batch_size, dtype=np.uint64)

    def _ensure_capacity(self):
        need = self._n_slots * self.batch_size
        if self.ctx.capacity < need:
            self.ctx.reserve(max(need, int(self.ctx.capacity * 1.25) + self.batch_size))

    def _queue_upload(self, node: int, values: np.ndarray):
        """values: (lanes, N, k) compact ciphertexts of one node."""
        slot = self._alloc_slot()
        self._slot[node] = slot
        self._loose.append(node)
        self._pending_in_idx.append(self._lane_idx(slot))
        self._pending_in_val.append(np.ascontiguousarray(values, dtype=np.uint32))
        self._pending_in_bytes += values.nbytes
        if self._pending_in_bytes >= _UPLOAD_BATCH_BYTES:
            self._upload_inputs()

    def _upload_inputs(self):
        if self._enc_rows:
            self._ensure_capacity()
            rows = np.concatenate(self._enc_rows, axis=1)
            self.ctx.encrypt(self.public_key, self._enc_streams, rows[0], rows[1], rows[2], rows[3])
            self._enc_rows.clear()
            self._enc_streams.clear()
            self._enc_stream_id.clear()
            self._pending_in_bytes = 0
        if not self._pending_in_idx:
            return
        self._ensure_capacity()
        idx = np.concatenate(self._pending_in_idx)
        vals = np.concatenate([v.reshape(-1, self.params.n_ct * self.params.k)
                               for v in self._pending_in_val])
        self.ctx.write(idx, vals)
        self._pending_in_idx.clear()
        self._pending_in_val.clear()
        self._pending_in_bytes = 0

    # -- bit-engine protocol ----------------------------------------------------------

    def constant(self, bit: int) -> GpuBit:
        if bit not in (0, 1):
            raise UsageError(f"constant must be 0 or 1, got {bit!r}")
        return GpuBit(self, -1, 0, True, bit, -1)

    def input_bit(self, bits: int) -> GpuBit:
        """Encrypt one wire; ``bits`` is 0/1 (batch 1) or the lanes packed in an int."""
        if self.batch_size == 1:
            if bits not in (0, 1):
                raise UsageError(f"input bit must be 0 or 1, got {bits!r}")
        elif not 0 <= bits <= self.mask:
            raise UsageError(f"lane value {bits:#x} out of range for batch_size={self.batch_size}")
        if self.public_key is None and not self.dry_run:
            raise CapabilityError("encrypting inputs needs the public key")
        lanes = self.batch_size
        if self.dry_run:
            node = self._new_node(0, self._fresh_noise)
            slot = self._alloc_slot()
            self._slot[node] = slot
            self.dry_inputs.append((slot, bits))
            wire = self._new_wire()
            if self.trace is not None:
                self.trace.append((2, -1, -1, wire, node, 0))
            return GpuBit(self, node, 0, False, None, wire)
        if self.device_encrypt:
            mus = np.array([(bits >> l) & 1 for l in range(lanes)], dtype=np.int64)
            return self.input_block(mus[:, None])[0]
        if self.lane_rngs is None:
            mus = [(bits >> l) & 1 for l in range(lanes)]
            vals = self.scheme.encrypt_many(self.public_key, mus, self.rng)
        else:
            vals = np.empty((lanes, self.params.n_ct, self.params.k), dtype=np.uint32)
            for l in range(lanes):
                vals[l] = self.scheme.encrypt_many(self.public_key, [(bits >> l) & 1],
                                                   self.lane_rngs[l])[0]
        return self._input_values(vals, 0, self._fresh_noise)

    def input_block(self, bits) -> list:
        """Fresh wires for a (lanes, n) block of plaintext bits, encrypted on the device.

        Draw order: with ``lane_rngs`` lane l's generator encrypts its n bits in order;
        with the single ``rng`` the block is drawn lane-major (lane 0's n inputs, then
        lane 1's, ...) -- e.g. the pair-major a0, b0, a1, b1, ... of the gate benchmark.
        Identical ciphertexts to encrypting one by one with the reference."""
        bits = np.asarray(bits, dtype=np.int64)
        lanes = self.batch_size
        if bits.ndim != 2 or bits.shape[0] != lanes:
            raise UsageError(f"expected a ({lanes}, n) bit block")
        if ((bits != 0) & (bits != 1)).any():
            raise UsageError("input bits must be 0 or 1")
        if self.public_key is None:
            raise CapabilityError("encrypting inputs needs the public key")
        if self._draws_per_ct % 2:
            raise UsageError("device encryption needs N*m even")
        from ._native import pcg64_stream
        if not self._macros and not self._pending_ops:
            self._reclaim()                    # nothing pending can still read a dead wire
        n = bits.shape[1]
        step = self._draws_per_ct
        slot_list = self._alloc_slots(n)
        nodes = self._new_nodes([0] * n, [self._fresh_noise] * n, slot_list)
        slots = np.asarray(slot_list, dtype=np.uint64)
        self._loose.extend(nodes)
        lane_ix = np.arange(lanes, dtype=np.uint64)
        target = (slots[None, :] * np.uint64(lanes) + lane_ix[:, None])        # (lanes, n)
        if self.lane_rngs is None:
            sid = self._stream_id(pcg64_stream(self.rng))
            stream_idx = np.full((lanes, n), sid, dtype=np.uint32)
            off = (np.arange(lanes * n, dtype=np.uint64) * np.uint64(step)).reshape(lanes, n)
            self.rng.bit_generator.advance(lanes * n * step // 2)
        else:
            stream_idx = np.empty((lanes, n), dtype=np.uint32)
            for l, g in enumerate(self.lane_rngs):
                stream_idx[l, :] = self._stream_id(pcg64_stream(g))
                g.bit_generator.advance(n * step // 2)
            off = np.broadcast_to(np.arange(n, dtype=np.uint64) * np.uint64(step), (lanes, n))
        self._enc_rows.append(np.stack([stream_idx.ravel().astype(np.uint64), off.ravel(),
                                        bits.ravel().astype(np.uint64), target.ravel()]))
        self._pending_in_bytes += lanes * n * 32
        if self.trace is None:
            w0 = self._wire
            self._wire += n
            out = [GpuBit(self, node, 0, False, None, w0 + i) for i, node in enumerate(nodes)]
        else:
            out = []
            for node in nodes:
                wire = self._new_wire()
                self.trace.append((2, -1, -1, wire, node, 0))
                out.append(GpuBit(self, node, 0, False, None, wire))
        if self._pending_in_bytes >= _UPLOAD_BATCH_BYTES:
            self._upload_inputs()
        return out

    def _stream_id(self, st: tuple) -> int:
        sid = self._enc_stream_id.get(st)
        if sid is None:
            sid = len(self._enc_streams)
            self._enc_streams.append(st)
            self._enc_stream_id[st] = sid
        return sid

    def input_values(self, values: np.ndarray, level: int = 0, noise_est: int | None = None) -> GpuBit:
        """New wire from precomputed compact ciphertexts, one per lane: (lanes, N, k)."""
        values = np.asarray(values, dtype=np.uint32)
        if values.shape != (self.batch_size, self.params.n_ct, self.params.k):
            raise UsageError(f"expected {(self.batch_size, self.params.n_ct, self.params.k)}, "
                             f"got {values.shape}")
        return self._input_values(values, level, self._fresh_noise if noise_est is None else noise_est)

    def _input_values(self, values, level, est) -> GpuBit:
        node = self._new_node(level, est)
        self._queue_upload(node, values)
        wire = self._new_wire()
        if self.trace is not None:
            self.trace.append((2, -1, -1, wire, node, 0))
        return GpuBit(self, node, 0, False, None, wire)

    def import_ct(self, ct) -> GpuBit:
        """Wire from a Ciphertext (batch 1) or a list of one Ciphertext per lane.

        Accepts this package's compact ``Ciphertext`` and any object with the reference's
        fields ``matrix`` / ``level`` / ``noise_est`` (fhe.py:148-161) -- e.g. the
        ``fhefft.fhe.Ciphertext(matrix=..., level=...)`` that the reference's
        ``fileio.read_ciphertext_signal`` builds (fileio.py:186-191)."""
        cts = ct if isinstance(ct, (list, tuple)) else [ct]
        if len(cts) != self.batch_size:
            raise UsageError(f"import_ct needs {self.batch_size} ciphertexts (one per lane)")
        vals = np.stack([self._compact_of(c) for c in cts])
        node = self._new_node(max(c.level for c in cts), max(c.noise_est for c in cts))
        self._queue_upload(node, vals)
        return GpuBit(self, node, 0, False, None, -1)

    def _compact_of(self, c) -> np.ndarray:
        p = self.params
        v = getattr(c, "v", None)
        if v is None:
            mat = getattr(c, "matrix", None)
            if mat is None:
                raise UsageError(f"cannot import {type(c).__name__}: no compact v or matrix")
            mat = np.asarray(mat)
            if mat.shape != (p.n_ct, p.n_ct):
                raise UsageError(f"ciphertext matrix shape {mat.shape} does not match N={p.n_ct}")
            return Ciphertext.from_matrix(mat, p).v
        v = np.asarray(v, dtype=np.uint32)
        if v.shape != (p.n_ct, p.k):
            raise UsageError(f"compact ciphertext shape {v.shape} does not match {(p.n_ct, p.k)}")
        return v

    def nand(self, a: GpuBit, b: GpuBit) -> GpuBit:
        if a.engine is not self or b.engine is not self:
            raise UsageError("cannot mix handles from different engines")
        if self._macros:
            self._expand_macros()
        if a.const or b.const:
            return self._fold(a, b)
        la, lb = self._level[a.node], self._level[b.node]
        level = (la if la >= lb else lb) + 1
        if level > self._budget:
            raise NoiseOverflowError(
                f"NAND at level {level} would exceed depth budget {self.params.depth_budget}")
        ea, eb = self._est[a.node], self._est[b.node]
        if eb > ea:                                   # fhe.py:336-337: noisier operand left
            a, b, ea, eb = b, a, eb, ea
        est = ea + self._n_ct * eb
        if est > self._q:
            est = self._q
        self.nand_count += 1
        if level > self.max_depth:
            self.max_depth = level
        key = (a.node, a.neg, b.node, b.neg)
        node = self._cse_map.get(key, -1) if self._cse_map is not None else -1
        if node < 0:
            node = self._new_node(level, est)
            self._pending_ops.extend((a.node, a.neg, b.node, b.neg, node))
            self.executed_nands += 1
            if self._cse_map is not None:
                self._cse_map[key] = node
        wire = self._new_wire()
        if self.trace is not None:
            self.trace.append((0, a.wire, b.wire, wire, node, 0))
        return GpuBit(self, node, 0, False, None, wire)

    def _fold(self, a: GpuBit, b: GpuBit) -> GpuBit:
        """engine.py:180-187: const/const -> const; NAND(x,0) -> 1; NAND(x,1) -> NOT x."""
        if a.const and b.const:
            return self.constant(0 if (a.plain and b.plain) else 1)
        if b.const:
            a, b = b, a
        if a.plain == 0:
            return self.constant(1)
        wire = self._new_wire()
        if self.trace is not None:
            self.trace.append((1, b.wire, b.wire, wire, b.node, b.neg ^ 1))
        return GpuBit(self, b.node, b.neg ^ 1, False, None, wire)

    def map_parallel(self, fn, items):
        """Gates only record here; the GPU provides the parallelism at flush."""
        return [fn(x) for x in items]

    # -- read back ------------------------------------------------------------------------

    def _decrypt_row(self) -> int:
        p = self.params
        return p.n * p.ell + (p.q // 2).bit_length() - 1

    def read_back(self, h: GpuBit) -> int:
        if h.engine is not self:
            raise UsageError("handle belongs to a different engine")
        if h.const:
            return h.plain if self.batch_size == 1 else (self.mask if h.plain else 0)
        return int(self.read_back_many([h])[0])

    def read_back_many(self, handles) -> list[int]:
        """Packed lane bits of many wires with one device gather (vectorised decrypt)."""
        bits = self.read_back_bits(handles)
        if self.batch_size == 1:
            return [int(b) for b in bits[:, 0]]
        weights = [1 << l for l in range(self.batch_size)]
        return [sum(w for w, b in zip(weights, row) if b) for row in bits.tolist()]

    def read_back_bits(self, handles) -> np.ndarray:
        """Decrypted bits of many wires, shape (len(handles), lanes), one device gather."""
        lanes = self.batch_size
        out = np.zeros((len(handles), lanes), dtype=np.uint8)
        var = []
        for i, h in enumerate(handles):
            if h.engine is not self:
                raise UsageError("handle belongs to a different engine")
            if h.const:
                out[i] = h.plain
            else:
                var.append(i)
        if not var:
            return out
        if self.secret_key is None:
            raise CapabilityError("read_back needs the secret key")
        self.flush()
        for i in var:
            lvl = self._level[handles[i].node]
            if lvl > self.params.depth_budget:
                raise NoiseOverflowError(
                    f"ciphertext level {lvl} exceeds depth budget {self.params.depth_budget}")
        slots = np.array([self._slot[handles[i].node] for i in var], dtype=np.uint64)
        idx = (slots[:, None] * np.uint64(lanes) + np.arange(lanes, dtype=np.uint64)).ravel()
        comp = np.repeat(np.array([handles[i].neg for i in var], dtype=np.uint8), lanes)
        # the decryption sums on the device (one int per ciphertext crosses PCIe), rounding and
        # the noise check on the host
        x = self.ctx.decrypt_rows(idx, self._decrypt_row(), self.scheme.decrypt_weights(self.secret_key), comp)
        bits = self.scheme.decrypt_bits_from_sums(x).reshape(len(var), lanes)
        out[var] = bits
        return out

    def node_values(self, handles) -> np.ndarray:
        """Compact ciphertexts (n, lanes, N, k) of variable wires (flushes)."""
        return self.read_nodes([h.node for h in handles], [h.neg for h in handles])

    def read_nodes(self, nodes, negs, lanes=None) -> np.ndarray:
        """Compact ciphertexts (n, len(lanes), N, k) of raw (node, complement) pairs."""
        self.flush()
        lanes = np.arange(self.batch_size, dtype=np.uint64) if lanes is None else \
            np.asarray(lanes, dtype=np.uint64)
        slots = np.asarray([self._slot[n] for n in nodes], dtype=np.int64)
        if (slots < 0).any():
            raise UsageError("node has no live ciphertext (released); use keep_all=True")
        idx = (slots.astype(np.uint64)[:, None] * np.uint64(self.batch_size) + lanes).ravel()
        comp = np.repeat(np.asarray(negs, dtype=np.uint8), len(lanes))
        vals = self.ctx.read(idx, comp)
        return vals.reshape(len(nodes), len(lanes), self.params.n_ct, self.params.k)

    def export_ct(self, h: GpuBit):
        """Ciphertext of a wire (constants become trivial ciphertexts); a list per lane if batched."""
        if h.engine is not self:
            raise UsageError("handle belongs to a different engine")
        if h.const:
            ct = self.scheme.trivial_encrypt_bit(h.plain)
            return ct if self.batch_size == 1 else [ct] * self.batch_size
        vals = self.node_values([h])[0]
        lvl, est = self._level[h.node], self._est[h.node]
        cts = [Ciphertext(vals[l], lvl, est, self.params) for l in range(self.batch_size)]
        return cts[0] if self.batch_size == 1 else cts

    # -- circuit templates ------------------------------------------------------------------

    _TEMPLATES: "dict" = {}            # shared by engines: (key, params, input pattern) -> template
    TEMPLATE_CACHE = 512

    def circuit(self, key, fn, in_bits, flatten, rebuild):
        """Run ``fn()`` -- a circuit call over the wires ``in_bits`` whose netlist is a function
        of ``key`` and the inputs' structure alone -- recording it once as a template and
        replaying the template on later calls with the same key (no Python per gate).

        ``flatten(result)`` lists the output wires of a call's return value and
        ``rebuild(handles)`` turns such a list back into one.  Falls back to plain recording
        when a trace or CSE is on."""
        if self.trace is not None or self._cse_map is not None:
            return fn()
        pattern, in_nodes = self._input_pattern(in_bits)
        if pattern is None:
            return fn()
        p = self.params
        full = (key, (p.n, p.q, p.m, p.noise_bound, p.depth_budget), pattern)
        tpl = self._TEMPLATES.get(full)
        if tpl is not None:
            self._TEMPLATES[full] = self._TEMPLATES.pop(full)          # LRU touch
            self.template_hits += 1
            return rebuild(self._apply_template(tpl, in_nodes))
        if self._macros:
            self._expand_macros()
        n0, op0 = len(self._level), len(self._pending_ops)
        nand0, exec0, wire0 = self.nand_count, self.executed_nands, self._wire
        self._capturing += 1
        try:
            result = fn()
            if self._macros:                 # replays of nested calls become ordinary ops
                self._expand_macros()
        finally:
            self._capturing -= 1
        tpl = self._capture(in_nodes, n0, op0, flatten(result), nand0, exec0, wire0)
        if tpl is not None:
            self._TEMPLATES[full] = tpl
            while len(self._TEMPLATES) > self.TEMPLATE_CACHE:
                self._TEMPLATES.pop(next(iter(self._TEMPLATES)))
        return result

    def _input_pattern(self, in_bits):
        """Hashable structure of the input wires -- per bit a public constant's value or
        (distinct-node index in first-use order, complement), plus each distinct node's (level,
        noise estimate) -- and the distinct nodes.  None if a wire is not this engine's."""
        try:
            if any(h.engine is not self for h in in_bits):
                return None, None
        except AttributeError:
            return None, None
        all_nodes = [h.node for h in in_bits]
        if all_nodes and min(all_nodes) < 0:              # public constants among the inputs
            index, nodes, pat = {}, [], []
            for h in in_bits:
                if h.const:
                    pat.append((-1, int(h.plain)))
                    continue
                i = index.get(h.node)
                if i is None:
                    i = index[h.node] = len(nodes)
                    nodes.append(h.node)
                pat.append((i, h.neg))
            info = tuple((self._level[n], self._est[n]) for n in nodes)
            return (tuple(pat), info), nodes
        # the common case (a transform's input words), without a Python tuple per wire
        arr = np.asarray(all_nodes, dtype=np.int64)
        negs = bytes([h.neg for h in in_bits])
        n = len(arr)
        if n > 1 and (np.diff(arr) > 0).all():            # distinct nodes in creation order
            nodes, idx = all_nodes, b""
        else:
            _, first, inv = np.unique(arr, return_index=True, return_inverse=True)
            order = np.argsort(first, kind="stable")
            rank = np.empty(len(order), dtype=np.int64)
            rank[order] = np.arange(len(order))
            idx = rank[inv].astype(np.int32).tobytes()
            nodes = arr[first[order]].tolist()
        info = (tuple(map(self._level.__getitem__, nodes)), tuple(map(self._est.__getitem__, nodes)))
        return (n, idx, negs, info), nodes

    def _capture(self, in_nodes, n0, op0, out_handles, nand0, exec0, wire0):
        """Template of the ops recorded since (n0, op0), or None if the call reached outside
        its inputs (then it is simply not cached)."""
        n_in = len(in_nodes)
        ops = np.asarray(self._pending_ops[op0:], dtype=np.int64).reshape(-1, 5)
        n1 = len(self._level)
        local = {nd: i for i, nd in enumerate(in_nodes)}

        def to_local(arr):
            out = np.empty(arr.shape, dtype=np.int64)
            new = arr >= n0
            out[new] = arr[new] - n0 + n_in
            for j in np.flatnonzero(~new):
                li = local.get(int(arr[j]))
                if li is None:
                    return None
                out[j] = li
            return out

        cols = [to_local(ops[:, c]) for c in (0, 2, 4)]
        if any(c is None for c in cols):
            return None
        lops = np.stack([cols[0], ops[:, 1], cols[1], ops[:, 3], cols[2]], axis=1)
        outs = np.empty((len(out_handles), 3), dtype=np.int64)
        for j, h in enumerate(out_handles):
            if h.const:
                outs[j] = (0, int(h.plain), 0)
                continue
            if h.node >= n0:
                outs[j] = (1, h.node - n0 + n_in, h.neg)
            elif h.node in local:
                outs[j] = (1, local[h.node], h.neg)
            else:
                return None
        levels = np.asarray(self._level[n0:n1], dtype=np.int64)
        ests = np.asarray(self._est[n0:n1], dtype=np.int64)
        return CircuitTemplate(n_in, [self._level[n] for n in in_nodes], [self._est[n] for n in in_nodes],
                               lops, levels, ests, outs, self.nand_count - nand0,
                               self.executed_nands - exec0, int(levels.max()) if len(levels) else 0,
                               self._wire - wire0)

    def _apply_template(self, tpl, in_nodes):
        """Replay: account the gates, create nodes only for the outputs; the call's gates stay
        one pending macro (expanded into ops only if something else joins the program)."""
        self.nand_count += tpl.nand_count
        self.executed_nands += tpl.executed
        if tpl.max_level > self.max_depth:
            self.max_depth = tpl.max_level
        self._wire += tpl.wires
        oi = tpl.out_internal
        if not hasattr(tpl, "out_levels"):            # per template, once
            tpl.out_levels = tpl.levels[oi - tpl.n_in].tolist()
            tpl.out_ests = tpl.ests[oi - tpl.n_in].tolist()
            tpl.out_list = oi.tolist()
            tpl.outs_list = tpl.outs.tolist()
        new = self._new_nodes(tpl.out_levels, tpl.out_ests)
        self._macros.append((tpl, list(in_nodes), list(new)))
        if len(self._macros) > 1 or self._pending_ops or self._capturing:
            self._expand_macros()
        if not hasattr(tpl, "out_fast"):              # per template, once: every output handle an
            pos = {v: i for i, v in enumerate(tpl.out_list)}    # internal node (the usual case)
            fast = all(kind == 1 and val in pos for kind, val, _ in tpl.outs_list)
            tpl.out_fast = [(pos[val], neg) for _, val, neg in tpl.outs_list] if fast else None
        if tpl.out_fast is not None:
            n0 = new[0] if len(new) else 0
            return [GpuBit(self, n0 + i, neg, False, None, -1) for i, neg in tpl.out_fast]
        real = dict(zip(tpl.out_list, new))
        for i, nd in enumerate(in_nodes):
            real[i] = nd
        out = []
        for kind, val, neg in tpl.outs_list:
            out.append(self.constant(val) if kind == 0 else GpuBit(self, real[val], neg, False, None, -1))
        return out

    def _expand_macros(self):
        """Materialise pending template replays as ordinary nodes and ops."""
        macros, self._macros = self._macros, []
        for tpl, in_nodes, out_real in macros:
            n_local = tpl.n_in + len(tpl.levels)
            m = np.empty(n_local, dtype=np.int64)
            m[:tpl.n_in] = in_nodes
            have = np.zeros(n_local, dtype=bool)
            have[:tpl.n_in] = True
            m[tpl.out_internal] = out_real
            have[tpl.out_internal] = True
            fresh = np.flatnonzero(~have)
            base = len(self._level)
            m[fresh] = base + np.arange(len(fresh))
            k = fresh - tpl.n_in
            self._level.extend(tpl.levels[k].tolist())
            self._est.extend(tpl.ests[k].tolist())
            self._slot.extend([-1] * len(fresh))
            self._refs.extend([0] * len(fresh))
            ops = tpl.ops.copy()
            for c in (0, 2, 4):
                ops[:, c] = m[ops[:, c]]
            self._pending_ops.extend(ops.ravel().tolist())

    def _reclaim(self):
        """Free the slots of inputs / replay outputs nobody holds any more (an ordinary compile
        releases dead nodes itself; replays only run cached programs, so they sweep here)."""
        keep = []
        slot, refs, free, keep_all = self._slot, self._refs, self._free, self.keep_all
        for nd in self._loose:
            sl = slot[nd]
            if sl < 0:
                continue
            if refs[nd] <= 0 and not keep_all:
                free.append(sl)
                slot[nd] = -1
            else:
                keep.append(nd)
        self._loose = keep

    def _template_compile(self, tpl):
        """The template compiled once as a self-contained program over private slots
        0..S-1 (inputs at 0..n_in-1, every output kept), or None when the schedule it
        would get here (tiled / resident: shallow programs) needs the engine's own layout."""
        ck = (self.batch_size, self.schedule, None if self.dry_run else self.ctx.kernel)
        if ck in tpl.compiled:
            return tpl.compiled[ck]
        saved = (self._level, self._est, self._slot, self._refs, self._free, self._n_slots,
                 self._pending_ops, self.keep_all)
        n_in = tpl.n_in
        try:
            self._level = list(tpl.in_levels) + tpl.levels.tolist()
            self._est = list(tpl.in_ests) + tpl.ests.tolist()
            n_local = len(self._level)
            self._slot = list(range(n_in)) + [-1] * (n_local - n_in)
            refs = np.zeros(n_local, dtype=np.int64)
            refs[tpl.out_internal] = 1
            refs[tpl.outs[(tpl.outs[:, 0] == 1) & (tpl.outs[:, 1] < n_in), 1]] = 1   # pass-through inputs
            self._refs = refs.tolist()
            self._free, self._n_slots, self.keep_all = [], n_in, False
            self._pending_ops = tpl.ops.ravel().tolist()
            sched = self._pick_schedule()
            comp = None
            if sched not in ("tiled", "resident"):
                prog = self._compile(ssa=sched in ("dataflow", "queue", "flow"), pin_old=sched == "regfile")
                prog["schedule"] = sched
                if sched == "flow":
                    prog["ops"]["flags"] |= np.where(prog["held"], 0, OP_TEMP).astype(np.uint32)
                out_slots = np.asarray(self._slot, dtype=np.int64)[tpl.out_internal]
                comp = {"prog": prog, "n_slots": self._n_slots, "out_slots": out_slots}
                if sched == "regfile":
                    comp["regfile"] = self._regfile_plan(prog)
        finally:
            (self._level, self._est, self._slot, self._refs, self._free, self._n_slots,
             self._pending_ops, self.keep_all) = saved
        tpl.compiled[ck] = comp
        return comp

    def _run_macro(self, macro):
        """Flush of exactly one template replay: bind the inputs into the template's private
        slot region (device copies), run its cached program, copy the held outputs out.
        None when the template has no region program here (then it is expanded)."""
        tpl, in_nodes, out_real = macro
        if self.dry_run or self.keep_all:
            return None
        comp = self._template_compile(tpl)
        if comp is None:
            return None
        lanes = self.batch_size
        reg = self._regions.get(tpl.uid)
        if reg is None:
            base = self._n_slots                       # a private block, never in the free list
            self._n_slots += comp["n_slots"]
            self._ensure_capacity()
            prog = comp["prog"]
            table = prog["ops"].copy()
            for f in ("left", "right", "out"):
                table[f] += np.uint32(base)
            program = self.ctx.program(table, prog["offsets"])
            if prog["schedule"] in ("dataflow", "queue", "flow"):
                program.set_deps(prog["deps"])
            if prog["schedule"] == "queue":
                program.set_queue(True)
            if prog["schedule"] == "flow":
                prog["flow"] = program.set_flow(True)
            if prog["schedule"] == "regfile":
                self._attach_regfile(program, comp["regfile"], base)
            reg = self._regions[tpl.uid] = (base, program)
        base, program = reg
        self._ensure_capacity()
        src = [self._slot[n] for n in in_nodes]
        if min(src) < 0:
            raise UsageError("template input has no live ciphertext")
        self.ctx.copy_slots(src, [base + i for i in range(tpl.n_in)], lanes)
        self._reclaim()                                  # (after the copy: the inputs may be dead)
        program.run(lanes)
        held = [j for j, nd in enumerate(out_real) if self._refs[nd] > 0]
        dst = self._alloc_slots(len(held))
        for j, slot in zip(held, dst):
            self._slot[out_real[j]] = slot
        self._loose.extend(out_real[j] for j in held)
        self._ensure_capacity()
        if held:
            self.ctx.copy_slots([base + int(comp["out_slots"][j]) for j in held], dst, lanes)
        for nd in in_nodes:                              # inputs nobody holds any more
            if self._refs[nd] <= 0 and self._slot[nd] >= 0:
                self._free.append(self._slot[nd])
                self._slot[nd] = -1
        self.last_program = program
        self.last_compile = dict(comp["prog"], template=tpl.uid)
        self.programs_run += 1
        self.launches += program.launches
        return program

    # -- compile + run ------------------------------------------------------------------------

    def flush(self):
        """Evaluate every pending gate: one kernel launch per level over all lanes."""
        if not self.dry_run:
            self._upload_inputs()
        if self._macros:
            if len(self._macros) == 1 and not self._pending_ops:
                program = self._run_macro(self._macros[0])
                if program is not None:
                    self._macros = []
                    return program
            self._expand_macros()
        if not self._pending_ops:
            return None
        sched = self._pick_schedule()
        dataflow = sched in ("dataflow", "queue", "tiled", "flow")
        ring = self.TILE_RING if sched == "tiled" and self._ring_ok() else 0
        # register-file programs read inputs and write outputs in their own order: input slots
        # are not reused inside the program
        prog = self._compile(ssa=dataflow, ring_temps=ring > 0, pin_old=sched == "regfile")
        prog["schedule"] = sched
        if sched == "flow":              # temporaries stay on chip (their store slot is never read)
            prog["ops"]["flags"] |= np.where(prog["held"], 0, OP_TEMP).astype(np.uint32)
        self._pending_ops = []
        if self._cse_map is not None:
            self._cse_map = {}
        self.last_compile = prog
        if self.dry_run:
            self.dry_programs.append(prog)
            return prog
        self._ensure_capacity()
        lanes = self.batch_size
        if sched == "tiled":
            K = self.batch_size // self.TILE_LANES
            t_base = self._n_slots * K                       # ring after every batch-wide slot
            if ring:
                step_items = len(prog["ops"]) * self.TILE_LANES
                slack = max(1, -(-self.TILE_WINDOW // step_items))   # steps covering the window
                skew = self.TILE_SKEW or slack
                # the roots of chunk c wait for the sinks of chunk c - ring (at step c - ring +
                # skew * depth): keep those a window's worth of steps back, out of flight
                ring = max(ring, skew * (len(prog["offsets"]) - 2) + 1 + slack)
                need = self._n_slots * self.batch_size + ring * prog["n_temp"] * self.TILE_LANES
                if self.ctx.capacity < need:
                    self.ctx.reserve(need)
            tops, tdeps = self._tile(prog, K, self.TILE_LANES, self.TILE_SKEW, self.TILE_WINDOW,
                                     ring, t_base)
            program = self.ctx.program(tops, np.array([0, len(tops)], dtype=np.uint64))
            program.set_deps(tdeps)
            program.tile_lanes = lanes = self.TILE_LANES
            program.base = (prog["ops"], prog["offsets"])
        else:
            program = self.ctx.program(prog["ops"], prog["offsets"])
            if dataflow:
                program.set_deps(prog["deps"])
            if sched == "queue":
                program.set_queue(True)
            if sched == "flow":
                prog["flow"] = program.set_flow(True)
            if sched == "resident":
                plan = self._resident_plan(prog)
                if plan is not None:                 # else: the level launches of `program`
                    program.set_resident(*plan)
            if sched == "regfile":
                self._attach_regfile(program, self._regfile_plan(prog), 0)
        program.run(lanes)
        self.last_program = program
        self.last_compile = prog
        self.programs_run += 1
        self.launches += program.launches
        return program

    # register-file launches (csrc/tc_nand_regfile.cuh): shared-memory buffers per CTA, the
    # planner's dependency distance and fill lookahead (csrc/rf_plan.h)
    RF_BUFFERS = int(os.environ.get("FHEGPU_RF_BUFFERS", "20"))
    RF_DIST = int(os.environ.get("FHEGPU_RF_DIST", "5"))
    RF_LOOK = int(os.environ.get("FHEGPU_RF_LOOK", "10"))    # fills >= 8 slots ahead of their readers
    REGFILE_MIN_LANES = 296        # 'auto': deep programs over >= 2 lanes per SM
    REGFILE_MIN_LEVELS = 16
    REGFILE_AUTO = os.environ.get("FHEGPU_REGFILE", "1") != "0"

    @staticmethod
    def _regfile_gates(prog):
        """fhegpu_rf_gate records of a compiled per-lane program (gates in level order) and the
        store slots of its inputs: operand ids are input i -> i (first-use order), the output of
        gate j -> n_in + j."""
        from ._native import RF_GATE_DTYPE
        table, nodes, held = prog["ops"], prog["nodes"], prog["held"]
        n = len(table)
        maxn = int(nodes.max()) + 1 if n else 1
        producer = np.full(maxn, -1, dtype=np.int64)
        producer[nodes[:, 2]] = np.arange(n)
        flat = nodes[:, :2].ravel()
        pflat = producer[flat]
        is_in = pflat < 0
        in_nodes = flat[is_in]
        uniq, first = np.unique(in_nodes, return_index=True)
        by_use = np.argsort(first, kind="stable")
        uniq, first = uniq[by_use], first[by_use]
        in_id = np.full(maxn, -1, dtype=np.int64)
        in_id[uniq] = np.arange(len(uniq))
        slot_flat = np.stack([table["left"], table["right"]], axis=1).ravel()
        in_slots = slot_flat[is_in][first].astype(np.uint32)
        ids = np.where(is_in, in_id[flat], len(uniq) + pflat).reshape(n, 2)
        gates = np.zeros(n, dtype=RF_GATE_DTYPE)
        gates["left"], gates["right"] = ids[:, 0], ids[:, 1]
        gates["flags"] = table["flags"] & 3
        gates["held"] = held.astype(np.uint8)
        gates["out_slot"] = np.where(held, table["out"], 0)
        return gates, in_slots

    def _regfile_plan(self, prog):
        """Schedule + buffer plan of a compiled program (fhegpu_rf_plan), store slots as compiled."""
        from ._native import rf_plan
        gates, in_slots = self._regfile_gates(prog)
        order, slots, fills, n_spill, stats = rf_plan(gates, in_slots, self.RF_BUFFERS, self.RF_DIST, self.RF_LOOK)
        prog["regfile"] = dict(stats, n_spill=n_spill, buffers=self.RF_BUFFERS,
                               ct_per_gate=(stats["fills"] + stats["stores"]) / max(1, len(gates)))
        return slots, fills, n_spill

    def _attach_regfile(self, program, plan, slot_offset: int):
        """Attach a register-file plan to `program`, store slots shifted by `slot_offset` (a
        template's private region); spills go to this engine's spill block."""
        from ._csrc_consts import RF
        slots, fills, n_spill = plan
        if slot_offset:
            slots, fills = slots.copy(), fills.copy()
            st = (slots["bits"] & RF.SB_STORE) != 0
            st &= (slots["store"] & RF.STORE_SPILL) == 0
            slots["store"][st] += np.uint32(slot_offset)
            fs = (fills["src"] & RF.STORE_SPILL) == 0
            fills["src"][fs] += np.uint32(slot_offset)
        lanes = self.batch_size
        grid = min(self.ctx.num_sms(), lanes)
        need = -(-(grid * n_spill) // lanes)          # slots of spill space
        base, have = self._spill_block
        if have < need:
            base, have = self._n_slots, need
            self._n_slots += need
            self._spill_block = (base, have)
            self._ensure_capacity()
        program.set_regfile(slots, fills, self.RF_BUFFERS, n_spill, base * lanes)

    # tiled dataflow: lanes per chunk, and the single-assignment store budget it may use
    TILE_LANES = int(os.environ.get("FHEGPU_TILE_LANES", "128"))
    TILE_SKEW = int(os.environ.get("FHEGPU_TILE_SKEW", "0"))      # 0: pick from the window below
    TILE_WINDOW = 2304        # items between a level and the next of one chunk: more than a CTA
    #                           pipeline holds (148 x ~12 items, ring + buffers + staging)
    TILE_RING = int(os.environ.get("FHEGPU_TILE_RING", "8"))      # chunks of temporaries kept in L2
    TILED_MAX_LEVELS = 32

    def _ring_ok(self) -> bool:
        """Ring temporaries need the program to have at most two sinks (see _tile)."""
        if self.TILE_RING <= 0 or self.keep_all:
            return False
        ops = np.asarray(self._pending_ops, dtype=np.int64).reshape(-1, 5)
        read = np.zeros(len(self._level), dtype=bool)
        read[ops[:, 0]] = True
        read[ops[:, 2]] = True
        return 1 <= int((~read[ops[:, 4]]).sum()) <= 2
    TILED_MAX_BYTES = 100 << 30

    def _pick_schedule(self) -> str:
        """'levels', 'dataflow', 'queue' or 'tiled' for the pending program.

        levels    one launch per netlist level over all lanes (PDL between launches).
        dataflow  the whole program in one launch, operands awaited per item (opt-in: for
                  the reference's deep single-signal netlists it does not beat levels).
        queue     the whole program in one launch over a ready queue: CTAs pop only items
                  whose producers have completed.  'auto' picks it for deep programs over
                  few lanes whose single-assignment store fits QUEUE_MAX_BYTES (configs[2]
                  and [3]: +8% over levels).
        tiled     lanes cut into chunks of TILE_LANES; the program is replicated per chunk
                  and run as ONE dataflow launch in wavefront order (step s = level 0 of chunk
                  s, level 1 of chunk s-1, ...), so a chunk's intermediates are consumed while
                  still in L2.  The DRAM traffic it saves is energy under the board power cap:
                  cfg1 143 -> 158M NAND/s.  'auto' picks it for wide programs
                  whose single-assignment store fits TILED_MAX_BYTES."""
        if self.schedule != "auto":
            return self.schedule
        if self._pick_flow():
            return "flow"
        if self.dry_run or (self.params.k, self.params.ell) != (9, 29):
            return "levels"
        if self.batch_size >= self.RESIDENT_MIN_LANES and self.ctx.kernel == "tcgen05" and self._resident_ok():
            return "resident"
        if self.REGFILE_AUTO and self.batch_size >= self.REGFILE_MIN_LANES and self.ctx.kernel == "tcgen05":
            outs = np.asarray(self._pending_ops[4::5], dtype=np.int64)
            if len(np.unique(np.asarray(self._level, dtype=np.int64)[outs])) >= self.REGFILE_MIN_LEVELS:
                return "regfile"           # deep programs over many lanes: one register-file launch
        C = self.TILE_LANES
        if self.batch_size % C or self.batch_size < 8 * C:
            return "queue" if self._pick_queue() else "levels"
        if self.ctx.kernel != "tcgen05":              # the dataflow launch needs the tcgen05 kernel
            return "levels"
        n_ops = len(self._pending_ops) // 5
        ct_bytes = ((self.params.n_ct * self.params.k + 3) // 4) * 16
        if (self._n_slots + n_ops) * self.batch_size * ct_bytes > self.TILED_MAX_BYTES:
            return "levels"
        if n_ops * self.batch_size >= 1 << 31 or n_ops * (self.batch_size // C) > 1 << 24:
            return "levels"                   # item index range / host-side tiling cost
        outs = np.asarray(self._pending_ops[4::5], dtype=np.int64)
        if len(np.unique(np.asarray(self._level, dtype=np.int64)[outs])) > self.TILED_MAX_LEVELS:
            return "levels"                    # deep programs are dependency-hop bound (4.8)
        return "tiled"

    FLOW_MIN_LEVELS = 16           # 'auto' runs deeper single-lane EXACT programs as one warp-dataflow launch
    FLOW_MAX_OPS = 1 << 22

    def _pick_flow(self) -> bool:
        """Deep single-lane programs at the EXACT geometry (configs[0]): one warp-dataflow launch
        (csrc/flow_nand.cuh) instead of a ~2.5 us launch per level."""
        if self.dry_run or self.batch_size != 1 or (self.params.k, self.params.ell) != (3, 17):
            return False
        if self.params.q > 1 << 17 or self.ctx.kernel == "simt":
            return False
        n_ops = len(self._pending_ops) // 5
        if not 0 < n_ops <= self.FLOW_MAX_OPS:
            return False
        outs = np.asarray(self._pending_ops[4::5], dtype=np.int64)
        return len(np.unique(np.asarray(self._level, dtype=np.int64)[outs])) >= self.FLOW_MIN_LEVELS

    QUEUE_MIN_LEVELS = 64          # 'auto' runs deeper single-signal programs over the ready queue
    QUEUE_MAX_BYTES = 40 << 30     # ... when their single-assignment store fits this

    def _pick_queue(self) -> bool:
        """Deep programs over few lanes (single-signal FFTs, configs[2]/[3]): one ready-queue
        launch instead of a launch per level when its SSA store fits."""
        if self.dry_run or (self.params.k, self.params.ell) != (9, 29) or self.ctx.kernel != "tcgen05":
            return False
        n_ops = len(self._pending_ops) // 5
        ct_bytes = ((self.params.n_ct * self.params.k + 3) // 4) * 16
        if (self._n_slots + n_ops) * self.batch_size * ct_bytes > self.QUEUE_MAX_BYTES:
            return False
        if n_ops * self.batch_size >= 1 << 31:
            return False
        outs = np.asarray(self._pending_ops[4::5], dtype=np.int64)
        return len(np.unique(np.asarray(self._level, dtype=np.int64)[outs])) >= self.QUEUE_MIN_LEVELS

    RES_MAX_OPS, RES_MAX_IN, RES_MAX_LOCAL = 8, 4, 8       # tc_nand_resident.cuh limits
    RESIDENT_MIN_LANES = 1024      # 'auto' runs small per-lane programs over this many lanes resident
    RES_SMEM_LIMIT = 227 * 1024

    @classmethod
    def _resident_layout(cls, nodes, held):
        """Buffer layout of a per-lane program (gates in level order; nodes (n, 3) = left,
        right, out node ids; held: outputs still referenced after the program): per gate the
        producer of each operand (-1: program input), its destination buffer, the input nodes
        in first-use order and the number of buffers.  A buffer is free for gate i once every
        reader of its value is gate i or earlier (a gate's builders read before its epilogue
        writes); outputs and temporaries keep to buffers of their own kind (the kernel orders
        output writes after earlier stores)."""
        n = len(nodes)
        producer = {int(nd): i for i, nd in enumerate(nodes[:, 2])}
        last_read = np.full(n, -1)
        for i in range(n):
            for nd in nodes[i, :2]:
                if int(nd) in producer:
                    last_read[producer[int(nd)]] = i
        prods, dest, inputs, holder, n_local = [], [0] * n, [], {}, 0
        for i in range(n):
            pr = []
            for nd in (int(nodes[i, 0]), int(nodes[i, 1])):
                if nd in producer:
                    pr.append(producer[nd])
                else:
                    pr.append(-1)
                    if nd not in inputs:
                        inputs.append(nd)
            prods.append(pr)
            free = [b for b, j in holder.items() if bool(held[j]) == bool(held[i]) and last_read[j] <= i]
            dest[i] = min(free) if free else n_local
            n_local += 0 if free else 1
            holder[dest[i]] = i
        return prods, dest, inputs, n_local

    @classmethod
    def _resident_fits(cls, n_ops, n_in, n_local) -> bool:
        ct, W = 9408, 3                               # ciphertext bytes; lanes per group (RES_W)
        smem = (W * n_in + W * n_local) * ct + 2 * 13824 + 2 * 2304 + 1024
        return (0 < n_ops <= cls.RES_MAX_OPS and n_in <= cls.RES_MAX_IN and n_local <= cls.RES_MAX_LOCAL
                and smem <= cls.RES_SMEM_LIMIT)

    @classmethod
    def _resident_plan(cls, prog):
        """Per-lane plan of a small level-compiled program for fhegpu_prog_set_resident, or None.

        Gates keep the level order; an operand produced in the program is read from the local
        buffer its producer wrote, other operands are program inputs (their store slots);
        outputs (nodes still held after the program) are stored (`_resident_layout`)."""
        table, nodes, held = prog["ops"], prog["nodes"], prog["held"]
        n = len(table)
        if n == 0 or n > cls.RES_MAX_OPS:
            return None
        prods, dest, in_nodes, n_local = cls._resident_layout(nodes, held)
        if not cls._resident_fits(n, len(in_nodes), n_local):
            return None
        plan = np.zeros(n, dtype=RES_OP_DTYPE)
        in_slots = [0] * len(in_nodes)
        for i in range(n):
            for side, (kind, idx, prod) in enumerate((("lkind", "lidx", "lprod"), ("rkind", "ridx", "rprod"))):
                p = prods[i][side]
                if p >= 0:
                    plan[i][kind], plan[i][idx], plan[i][prod] = 1, dest[p], p
                else:
                    k = in_nodes.index(int(nodes[i, side]))
                    in_slots[k] = int(table[i]["left" if side == 0 else "right"])
                    plan[i][kind], plan[i][idx], plan[i][prod] = 0, k, -1
            plan[i]["dest"], plan[i]["is_out"] = dest[i], int(held[i])
            plan[i]["flags"] = int(table[i]["flags"]) & 3
            plan[i]["out_slot"] = int(table[i]["out"]) if held[i] else 0
        return plan, np.asarray(in_slots, dtype=np.uint32), n_local

    def _resident_ok(self) -> bool:
        """The pending program as a lane-resident launch fits the kernel's limits (checked on
        the node structure before slots are assigned)."""
        n = len(self._pending_ops) // 5
        if n == 0 or n > self.RES_MAX_OPS or self.keep_all:
            return False
        ops = np.asarray(self._pending_ops, dtype=np.int64).reshape(-1, 5)
        order = np.argsort(np.asarray(self._level, dtype=np.int64)[ops[:, 4]], kind="stable")
        ops = ops[order]
        held = np.asarray(self._refs, dtype=np.int64)[ops[:, 4]] > 0
        _, _, in_nodes, n_local = self._resident_layout(ops[:, [0, 2, 4]], held)
        return self._resident_fits(n, len(in_nodes), n_local)

    @staticmethod
    def _tile(prog, K, lanes_per_chunk=1, skew=0, window=2048, ring=0, t_base=0):
        """Replicate an SSA program over K lane chunks: op (c, o) uses slot s*K + c (a batch-wide
        slot s IS chunk-slots s*K + c of batch/K lanes each), wavefront order, remapped deps.

        Wavefront step of op (c, o) = c + skew * level(o): consecutive levels of one chunk are
        `skew` steps (~skew * n_ops * lanes_per_chunk items) apart, which must exceed what is in
        flight on the GPU (~148 CTAs x 7 stages) or consumers stall on their producers.

        ring > 0 (program compiled with ring_temps): temporaries of chunk c live in region
        c % ring of a small ring at chunk-slot t_base (it stays in L2; no write-back of dead
        values).  Write-after-read safety through the RAW machinery: the roots of chunk c (ops
        with no producer in the program; every other op descends from one) also wait for the
        sinks of chunk c - ring (ops whose output nothing in the program reads), whose
        completion implies every read of that chunk's temporaries in the lane is done."""
        ops, deps, offs = prog["ops"], prog["deps"], prog["offsets"].astype(np.int64)
        n = len(ops)
        if skew <= 0:
            skew = max(1, -(-window // max(1, n * lanes_per_chunk)))
        rank = np.repeat(np.arange(len(offs) - 1), np.diff(offs))          # level index per op
        cc = np.repeat(np.arange(K, dtype=np.int64), n)
        oo = np.tile(np.arange(n, dtype=np.int64), K)
        perm = np.lexsort((cc, oo, rank[oo], cc + skew * rank[oo]))        # step, level, op, chunk
        pos = np.empty(K * n, dtype=np.int64)
        pos[perm] = np.arange(K * n)
        c, o = cc[perm], oo[perm]
        tiled = np.empty(K * n, dtype=ops.dtype)
        temp = prog.get("temp") if ring else None
        for i, f in enumerate(("left", "right", "out")):
            v = ops[f][o].astype(np.int64) * K + c
            if temp is not None:
                tid = temp[o, i]
                v = np.where(tid >= 0, t_base + (c % ring) * prog["n_temp"] + tid, v)
            tiled[f] = v
        # outputs no op of the program reads (sinks) are stored L2 evict-first: they stream out
        # and should not push the chunks' temporaries out of L2
        read = np.zeros(n, dtype=bool)
        read[deps[deps >= 0]] = True
        tiled["flags"] = ops["flags"][o] | np.where(read[o], 0, STREAM_OUT).astype(ops["flags"].dtype)
        d = deps[o]
        tdeps = np.where(d >= 0, pos[c[:, None] * n + np.maximum(d, 0)], -1)
        if temp is not None:
            # a root of chunk c (step c) must come after the sinks of chunk c - ring (step
            # c - ring + skew * level): ring > skew * deepest level keeps the order topological
            sinks = np.flatnonzero(~read)
            roots = (deps < 0).all(axis=1)
            assert 1 <= len(sinks) <= 2, "ring temporaries need at most two sinks"
            assert ring > skew * int(rank[sinks].max()), "ring too short for the wavefront skew"
            war = roots[o] & (c >= ring)
            prev = (c[war] - ring) * n
            tdeps[war, 0] = pos[prev + sinks[0]]
            tdeps[war, 1] = pos[prev + sinks[-1]]
        return tiled, tdeps.astype(np.int32)

    def run_host(self, program, inputs, outputs, chunk_lanes: int = 32768, out=None,
                 sync: bool = True, packed: bool = False):
        """Re-run a flushed `program` over lanes held in HOST memory (fhegpu_prog_run_host).

        The netlist is compiled once (flush, at any batch size); here every input wire of
        the program gets a host array of ``lanes`` dense compact ciphertexts (lanes, N, k)
        u32 -- numpy, or torch pinned tensors for overlapped copies -- and every output
        wire a host array of the same shape (allocated when ``out`` is None).  Lanes stream
        through the device store in chunks; copy-in, the level kernels and copy-out overlap,
        so batches larger than HBM work.  Resident values of this engine are overwritten:
        call this after reading back what you need.  Returns the output arrays.

        ``packed=True``: host arrays are (lanes, ceil(N^2/8)) uint8 -- each lane one
        ciphertext serialised exactly as the reference writes it (fileio.pack_compact /
        an EFT1 payload row); unpacking and packing run on the device.
        """
        if program is None:
            raise UsageError("run_host needs a flushed program")
        p = self.params
        shape_tail = ((p.n_ct * p.n_ct + 7) // 8,) if packed else (p.n_ct, p.k)
        dtype = np.uint8 if packed else np.uint32
        in_slots, in_ptrs, lanes = [], [], None
        keep = []
        for h, arr in inputs:
            if h.const or h.neg or self._slot[h.node] < 0:
                raise UsageError("run_host inputs must be resident, non-negated input wires")
            arr = self._host_array(arr, shape_tail, dtype)
            keep.append(arr)
            if lanes is None:
                lanes = len(arr)
            elif len(arr) != lanes:
                raise UsageError("every host input needs the same number of lanes")
            in_slots.append(self._slot[h.node])
            in_ptrs.append(arr.data_ptr() if hasattr(arr, "data_ptr") else arr.ctypes.data)
        if lanes is None:
            raise UsageError("run_host needs at least one input")
        if out is None:
            out = [np.empty((lanes,) + shape_tail, dtype=dtype) for _ in outputs]
        out_slots, out_ptrs = [], []
        for h, arr in zip(outputs, out):
            if h.const or h.neg or self._slot[h.node] < 0:
                raise UsageError("run_host outputs must be resident, non-negated wires")
            arr = self._host_array(arr, shape_tail, dtype)
            if len(arr) != lanes:
                raise UsageError("output buffer lane count differs from the inputs'")
            out_slots.append(self._slot[h.node])
            out_ptrs.append(arr.data_ptr() if hasattr(arr, "data_ptr") else arr.ctypes.data)
        n_slots = max([self._n_slots] + [s + 1 for s in in_slots + out_slots])
        chunk = max(1, min(int(chunk_lanes), lanes))
        regions = min(3, -(-lanes // chunk))
        need = regions * n_slots * chunk
        rf = self.last_compile.get("regfile") if self.last_program is program else None
        if rf:                                        # register-file chunks spill after the regions
            need += self.ctx.num_sms() * rf["n_spill"]
        if self.ctx.capacity < need:
            self.ctx.reserve(need)
        program.level_program().run_host(lanes, chunk, in_slots, in_ptrs, out_slots, out_ptrs,
                                         host_format=1 if packed else 0)
        if sync:
            self.ctx.sync()
        return out

    @staticmethod
    def _host_array(arr, shape_tail, dtype=np.uint32):
        size = np.dtype(dtype).itemsize
        if hasattr(arr, "data_ptr"):                      # torch tensor (ideally pinned)
            if arr.device.type != "cpu" or not arr.is_contiguous() or arr.element_size() != size:
                raise UsageError(f"host tensors must be contiguous {8 * size}-bit CPU tensors")
            if tuple(arr.shape[1:]) != shape_tail:
                raise UsageError(f"host tensor shape {tuple(arr.shape)} is not (lanes,) + {shape_tail}")
            return arr
        if not isinstance(arr, np.ndarray) or arr.dtype != dtype or not arr.flags.c_contiguous:
            raise UsageError(f"host arrays must be C-contiguous {np.dtype(dtype).name}")
        if arr.shape[1:] != shape_tail:
            raise UsageError(f"host array shape {arr.shape} is not (lanes,) + {shape_tail}")
        return arr
