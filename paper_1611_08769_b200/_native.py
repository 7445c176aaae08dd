"""ctypes binding of libfhegpu.so (include/fhegpu.h).

There is deliberately no CPU fallback: if the library is missing or no CUDA
device is present, every entry point raises ``DeviceError``.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from .errors import DeviceError, ParameterError, UsageError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FHEGPU_LIB") or os.path.join(_HERE, "libfhegpu.so")   # FHEGPU_LIB: debug builds

KERNEL_AUTO, KERNEL_SIMT, KERNEL_TCGEN05 = 0, 1, 2
HOST_COMPACT, HOST_PACKED = 0, 1      # fhegpu_prog_run_host host formats
KERNEL_NAMES = {KERNEL_AUTO: "auto", KERNEL_SIMT: "simt", KERNEL_TCGEN05: "tcgen05"}

OP_DTYPE = np.dtype([("left", "<u4"), ("right", "<u4"), ("out", "<u4"), ("flags", "<u4")])
RF_GATE_DTYPE = np.dtype([("left", "<u4"), ("right", "<u4"), ("flags", "u1"), ("held", "u1"), ("pad", "<u2"),
                          ("out_slot", "<u4")])                                          # fhegpu_rf_gate
RF_SLOT_DTYPE = np.dtype([("lbuf", "u1"), ("rbuf", "u1"), ("dbuf", "u1"), ("bits", "u1"), ("lwait", "<u4"),
                          ("rwait", "<u4"), ("store", "<u4")])                             # fhegpu_rf_slot
RF_FILL_DTYPE = np.dtype([("buf", "<u4"), ("src", "<u4"), ("consumer", "<u4"), ("w_built", "<u4"),
                          ("w_epi", "<u4"), ("w_st", "<u4"), ("flags", "<u4"), ("pad", "<u4")])   # fhegpu_rf_fill
RES_OP_DTYPE = np.dtype([("lkind", "u1"), ("lidx", "u1"), ("rkind", "u1"), ("ridx", "u1"),
                         ("dest", "u1"), ("is_out", "u1"), ("flags", "u1"), ("pad", "u1"),
                         ("lprod", "<i2"), ("rprod", "<i2"), ("out_slot", "<u4")])   # fhegpu_res_op


class _Params(ctypes.Structure):
    _fields_ = [("n", ctypes.c_uint32), ("ell", ctypes.c_uint32),
                ("q", ctypes.c_uint32), ("m", ctypes.c_uint32)]


_lib = None

# (name, restype, argtypes) of every symbol include/fhegpu.h declares
_P = ctypes.c_void_p
_U32P = ctypes.POINTER(ctypes.c_uint32)
_U64P = ctypes.POINTER(ctypes.c_uint64)
_U8P = ctypes.POINTER(ctypes.c_uint8)
SIGNATURES = [
    ("fhegpu_last_error", ctypes.c_char_p, []),
    ("fhegpu_version", ctypes.c_char_p, []),
    ("fhegpu_ctx_create", ctypes.c_int, [ctypes.POINTER(_Params), ctypes.c_int, ctypes.POINTER(_P)]),
    ("fhegpu_ctx_destroy", None, [_P]),
    ("fhegpu_ctx_set_stream", ctypes.c_int, [_P, _P]),
    ("fhegpu_ctx_own_stream", _P, [_P]),
    ("fhegpu_ctx_set_kernel", ctypes.c_int, [_P, ctypes.c_int]),
    ("fhegpu_ctx_kernel", ctypes.c_int, [_P]),
    ("fhegpu_ctx_set_debug", ctypes.c_int, [_P, ctypes.c_uint32]),
    ("fhegpu_ctx_set_graphs", ctypes.c_int, [_P, ctypes.c_int]),
    ("fhegpu_ct_words", ctypes.c_uint32, [_P]),
    ("fhegpu_sync", ctypes.c_int, [_P]),
    ("fhegpu_store_reserve", ctypes.c_int, [_P, ctypes.c_uint64]),
    ("fhegpu_store_capacity", ctypes.c_uint64, [_P]),
    ("fhegpu_store_device_ptr", ctypes.c_uint64, [_P]),
    ("fhegpu_store_write", ctypes.c_int, [_P, _U64P, ctypes.c_uint64, _U32P]),
    ("fhegpu_store_read", ctypes.c_int, [_P, _U64P, _U8P, ctypes.c_uint64, _U32P]),
    ("fhegpu_store_read_rows", ctypes.c_int, [_P, _U64P, _U8P, ctypes.c_uint64, ctypes.c_uint32, _U32P]),
    ("fhegpu_store_write_range", ctypes.c_int, [_P, ctypes.c_uint64, ctypes.c_uint64, _P, ctypes.c_int]),
    ("fhegpu_store_read_range", ctypes.c_int, [_P, ctypes.c_uint64, ctypes.c_uint64, _P, ctypes.c_int]),
    ("fhegpu_prog_create", ctypes.c_int, [_P, _P, ctypes.c_uint64, _U64P, ctypes.c_uint32, ctypes.POINTER(_P)]),
    ("fhegpu_prog_run", ctypes.c_int, [_P, _P, ctypes.c_uint32]),
    ("fhegpu_prog_run_range", ctypes.c_int, [_P, _P, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32]),
    ("fhegpu_prog_launches", ctypes.c_uint32, [_P]),
    ("fhegpu_prog_set_deps", ctypes.c_int, [_P, _P, _P]),
    ("fhegpu_prog_set_queue", ctypes.c_int, [_P, _P, ctypes.c_int]),
    ("fhegpu_prog_set_flow", ctypes.c_int, [_P, _P, ctypes.c_int, ctypes.POINTER(ctypes.c_double), _U32P]),
    ("fhegpu_flow_plan", ctypes.c_int, [_P, _P, ctypes.c_uint64, _P, ctypes.c_uint32, ctypes.c_uint32, _P, _P,
                                        ctypes.POINTER(ctypes.c_double)]),
    ("fhegpu_prog_set_resident", ctypes.c_int, [_P, _P, _P, ctypes.c_uint32, _P, ctypes.c_uint32,
                                                ctypes.c_uint32]),
    ("fhegpu_res_slot_order", ctypes.c_int, [_P, ctypes.c_uint32, ctypes.c_uint32, _P]),
    ("fhegpu_ctx_num_sms", ctypes.c_int, [_P]),
    ("fhegpu_rf_plan", ctypes.c_int, [_P, ctypes.c_uint32, _P, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                                      ctypes.c_uint32, _P, _P, _P, ctypes.c_uint32, _U32P, _U32P, _U32P]),
    ("fhegpu_prog_set_regfile", ctypes.c_int, [_P, _P, _P, ctypes.c_uint32, _P, ctypes.c_uint32, ctypes.c_uint32,
                                               ctypes.c_uint32, ctypes.c_uint64]),
    ("fhegpu_store_write_packed", ctypes.c_int, [_P, ctypes.c_uint64, ctypes.c_uint64, _P]),
    ("fhegpu_store_read_packed", ctypes.c_int, [_P, ctypes.c_uint64, ctypes.c_uint64, _P]),
    ("fhegpu_store_copy_slots", ctypes.c_int, [_P, _U32P, _U32P, ctypes.c_uint32, ctypes.c_uint64]),
    ("fhegpu_store_decrypt_rows", ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint8),
                                                 ctypes.c_uint64, ctypes.c_uint32, _U32P,
                                                 ctypes.POINTER(ctypes.c_int32)]),
    ("fhegpu_prog_run_host", ctypes.c_int, [_P, _P, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int,
                                            ctypes.c_uint32, _P, _P, ctypes.c_uint32, _P, _P]),
    ("fhegpu_prog_destroy", None, [_P]),
    ("fhegpu_nand_batch", ctypes.c_int, [_P, _U32P, _U32P, _U32P, ctypes.c_uint64]),
    ("fhegpu_not_batch", ctypes.c_int, [_P, _U32P, _U32P, ctypes.c_uint64]),
    ("fhegpu_bits_create", ctypes.c_int, [ctypes.c_int, ctypes.c_uint64, ctypes.POINTER(ctypes.c_void_p)]),
    ("fhegpu_bits_destroy", None, [_P]),
    ("fhegpu_bits_words", ctypes.c_uint32, [_P]),
    ("fhegpu_bits_reserve", ctypes.c_int, [_P, ctypes.c_uint64]),
    ("fhegpu_bits_write", ctypes.c_int, [_P, _U64P, ctypes.c_uint64, _U32P]),
    ("fhegpu_bits_run", ctypes.c_int, [_P, _P, ctypes.c_uint64, _U64P, ctypes.c_uint32]),
    ("fhegpu_bits_read", ctypes.c_int, [_P, _U64P, _P, ctypes.c_uint64, _U32P]),
    ("fhegpu_add_batch", ctypes.c_int, [_P, _U32P, _U32P, _U32P, ctypes.c_uint64]),
    ("fhegpu_mult_batch", ctypes.c_int, [_P, _U32P, _U32P, _U32P, ctypes.c_uint64]),
    ("fhegpu_const_mult_batch", ctypes.c_int, [_P, ctypes.c_uint32, _U32P, _U32P, ctypes.c_uint64]),
    ("fhegpu_debug_ws_trace", ctypes.c_int, [_U64P]),
    ("fhegpu_debug_flow_trace", ctypes.c_int, [_U32P, ctypes.c_uint32]),
    ("fhegpu_encrypt", ctypes.c_int, [_P, _U32P, _P, ctypes.c_uint32, _U32P, _U64P, _U32P, _U64P,
                                      ctypes.c_uint64]),
]

PCG_DTYPE = np.dtype([("state_lo", "<u8"), ("state_hi", "<u8"), ("inc_lo", "<u8"), ("inc_hi", "<u8")])


def pcg64_stream(rng) -> tuple:
    """(state_lo, state_hi, inc_lo, inc_hi) of a numpy Generator(PCG64) at its current
    position; requires no buffered 32-bit half (has_uint32 == 0)."""
    st = rng.bit_generator.state
    if st.get("bit_generator") != "PCG64":
        raise ParameterError("device encryption reproduces numpy's PCG64 only")
    if st["has_uint32"]:
        raise ParameterError("generator holds a buffered 32-bit half; draw an even number first")
    s, inc = st["state"]["state"], st["state"]["inc"]
    m = (1 << 64) - 1
    return (s & m, s >> 64, inc & m, inc >> 64)


def load_library(path: str = LIB_PATH):
    """Load libfhegpu.so and attach signatures (no device needed)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise DeviceError(f"CUDA library {path} not built; run __graft_entry__.build()")
    try:
        lib = ctypes.CDLL(path)
    except OSError as exc:
        raise DeviceError(f"cannot load {path}: {exc}") from exc
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _check(rc: int, what: str):
    if rc != 0:
        msg = _lib.fhegpu_last_error().decode(errors="replace")
        raise DeviceError(f"{what} failed (code {rc}): {msg}")


def res_slot_order(plan: np.ndarray, lanes: int = 3) -> np.ndarray:
    """Slot order of a lane-resident group (fhegpu_res_slot_order; host only): one byte per slot,
    gate | lane << 3 | 32 (left operand reused) | 64 (right operand reused)."""
    if _lib is None:
        load_library()
    plan = np.ascontiguousarray(plan, dtype=RES_OP_DTYPE)
    order = np.zeros(len(plan) * lanes, dtype=np.uint8)
    _check(_lib.fhegpu_res_slot_order(plan.ctypes.data_as(ctypes.c_void_p), len(plan), int(lanes),
                                      order.ctypes.data_as(ctypes.c_void_p)), "res_slot_order")
    return order


def rf_plan(gates: np.ndarray, in_slots, n_buf: int = 20, min_dist: int = 5, lookahead: int = 4):
    """Register-file plan of a per-lane netlist (fhegpu_rf_plan; host only): returns
    (order, slots, fills, n_spill, stats) -- see include/fhegpu.h."""
    if _lib is None:
        load_library()
    gates = np.ascontiguousarray(gates, dtype=RF_GATE_DTYPE)
    ins = np.ascontiguousarray(np.asarray(in_slots, dtype=np.uint32).reshape(-1))
    n = len(gates)
    order = np.zeros(n, dtype=np.uint32)
    slots = np.zeros(n, dtype=RF_SLOT_DTYPE)
    fills = np.zeros(2 * n + 16, dtype=RF_FILL_DTYPE)
    n_fills, n_spill = ctypes.c_uint32(), ctypes.c_uint32()
    stats = np.zeros(5, dtype=np.uint32)
    _check(_lib.fhegpu_rf_plan(gates.ctypes.data_as(ctypes.c_void_p), n, ins.ctypes.data_as(ctypes.c_void_p),
                               len(ins), int(n_buf), int(min_dist), int(lookahead),
                               order.ctypes.data_as(ctypes.c_void_p), slots.ctypes.data_as(ctypes.c_void_p),
                               fills.ctypes.data_as(ctypes.c_void_p), len(fills), ctypes.byref(n_fills),
                               ctypes.byref(n_spill), _ptr(stats, ctypes.c_uint32)), "rf_plan")
    return order, slots, fills[:n_fills.value].copy(), int(n_spill.value), \
        {"stalls": int(stats[0]), "stores": int(stats[1]), "fills": int(stats[2]), "reuse_l": int(stats[3]),
         "reuse_r": int(stats[4])}


FLOW_WARPS, FLOW_RING = 8, 4      # FHEGPU_FLOW_WARPS / FHEGPU_FLOW_RING (include/fhegpu.h)


def flow_plan(ops: np.ndarray, deps: np.ndarray, level_offsets, n_cta: int):
    """Warp-dataflow schedule of a levelised program (fhegpu_flow_plan; host only): returns
    (entries (n, 8) u32 grouped by worker, worker_off (n_cta * FLOW_WARPS + 1), model cycles)."""
    if _lib is None:
        load_library()
    ops = np.ascontiguousarray(ops, dtype=OP_DTYPE)
    deps = np.ascontiguousarray(deps, dtype=np.int32).reshape(-1)
    offs = np.ascontiguousarray(level_offsets, dtype=np.uint64)
    n = len(ops)
    ents = np.zeros((n, 8), dtype=np.uint32)
    woff = np.zeros(n_cta * FLOW_WARPS + 1, dtype=np.uint32)
    cyc = ctypes.c_double(0.0)
    _check(_lib.fhegpu_flow_plan(ops.ctypes.data_as(ctypes.c_void_p), deps.ctypes.data_as(ctypes.c_void_p), n,
                                 offs.ctypes.data_as(ctypes.c_void_p), len(offs) - 1, int(n_cta),
                                 ents.ctypes.data_as(ctypes.c_void_p), woff.ctypes.data_as(ctypes.c_void_p),
                                 ctypes.byref(cyc)), "flow_plan")
    return ents, woff, cyc.value


def _ptr(arr, ctype):
    return arr.ctypes.data_as(ctypes.POINTER(ctype))


class Program:
    """A levelised netlist resident on the device (fhegpu_prog)."""

    def __init__(self, ctx: "DeviceContext", ops: np.ndarray, level_offsets: np.ndarray):
        self.ctx = ctx
        self.n_ops = int(len(ops))
        self.n_levels = int(len(level_offsets) - 1)
        ops = np.ascontiguousarray(ops, dtype=OP_DTYPE)
        offs = np.ascontiguousarray(level_offsets, dtype=np.uint64)
        h = ctypes.c_void_p()
        _check(_lib.fhegpu_prog_create(ctx.handle, ops.ctypes.data_as(ctypes.c_void_p),
                                       self.n_ops, _ptr(offs, ctypes.c_uint64),
                                       self.n_levels, ctypes.byref(h)), "prog_create")
        self.handle = h
        self.launches = int(_lib.fhegpu_prog_launches(h))
        # tiled programs (GpuEngine schedule 'tiled'): ops are replicated per lane chunk, so
        # every run launches `tile_lanes` lanes whatever the caller's batch; `base` keeps the
        # untiled level program's (ops, offsets) for level-wise uses (host streaming)
        self.tile_lanes = None
        self.base = None
        self._base_prog = None

    def level_program(self) -> "Program":
        """The untiled level program (itself unless tiled)."""
        if self.base is None:
            return self
        if self._base_prog is None:
            self._base_prog = Program(self.ctx, *self.base)
        return self._base_prog

    def run(self, lanes: int = 1, first: int = 0, last: int | None = None):
        if self.tile_lanes is not None:
            if (first, last) != (0, None) and (first, last) != (0, self.n_levels):
                raise UsageError("a tiled program runs whole")
            lanes = self.tile_lanes
        if first == 0 and last is None:
            _check(_lib.fhegpu_prog_run(self.ctx.handle, self.handle, lanes), "prog_run")
            return
        last = self.n_levels if last is None else last
        _check(_lib.fhegpu_prog_run_range(self.ctx.handle, self.handle, lanes, first, last),
               "prog_run")

    def set_deps(self, deps: np.ndarray):
        """Dataflow mode (fhegpu_prog_set_deps): deps (n_ops, 2) int32 producer op indices."""
        deps = np.ascontiguousarray(deps, dtype=np.int32)
        _check(_lib.fhegpu_prog_set_deps(self.ctx.handle, self.handle, deps.ctypes.data_as(ctypes.c_void_p)),
               "prog_set_deps")
        self.launches = int(_lib.fhegpu_prog_launches(self.handle))

    def set_queue(self, enable: bool = True):
        """Ready-queue mode (fhegpu_prog_set_queue): one launch in which CTAs pop only items
        whose producers have completed (needs set_deps first)."""
        _check(_lib.fhegpu_prog_set_queue(self.ctx.handle, self.handle, int(bool(enable))), "prog_set_queue")
        self.launches = int(_lib.fhegpu_prog_launches(self.handle))

    def set_flow(self, enable: bool = True) -> dict:
        """Warp-dataflow mode (fhegpu_prog_set_flow; EXACT geometry, single lane): one launch,
        every warp a worker with a host-scheduled gate list (needs set_deps first).  Returns
        the schedule's model makespan and operand statistics."""
        cyc = ctypes.c_double(0.0)
        stats = (ctypes.c_uint32 * 4)()
        _check(_lib.fhegpu_prog_set_flow(self.ctx.handle, self.handle, int(bool(enable)), ctypes.byref(cyc), stats),
               "prog_set_flow")
        self.launches = int(_lib.fhegpu_prog_launches(self.handle))
        return {"model_cycles": cyc.value, "ring_operands": stats[0], "scratch_operands": stats[1],
                "store_operands": stats[2], "max_gates_per_worker": stats[3]}

    def set_resident(self, plan: np.ndarray, in_slots, n_local: int):
        """Lane-resident mode (fhegpu_prog_set_resident): plan = RES_OP_DTYPE records of the
        per-lane program, in_slots = store slots of its inputs.  An empty plan disables."""
        plan = np.ascontiguousarray(plan, dtype=RES_OP_DTYPE)
        ins = np.ascontiguousarray(np.asarray(in_slots, dtype=np.uint32).reshape(-1))
        _check(_lib.fhegpu_prog_set_resident(self.ctx.handle, self.handle, plan.ctypes.data_as(ctypes.c_void_p),
                                             len(plan), ins.ctypes.data_as(ctypes.c_void_p), len(ins),
                                             int(n_local)), "prog_set_resident")
        self.launches = int(_lib.fhegpu_prog_launches(self.handle))

    def set_regfile(self, slots: np.ndarray, fills: np.ndarray, n_buf: int, n_spill: int, spill_base: int):
        """Register-file mode (fhegpu_prog_set_regfile): a plan from rf_plan; spills of CTA c at
        store ciphertexts spill_base + c * n_spill.  Empty slots disable."""
        slots = np.ascontiguousarray(slots, dtype=RF_SLOT_DTYPE)
        fills = np.ascontiguousarray(fills, dtype=RF_FILL_DTYPE)
        _check(_lib.fhegpu_prog_set_regfile(self.ctx.handle, self.handle, slots.ctypes.data_as(ctypes.c_void_p),
                                            len(slots), fills.ctypes.data_as(ctypes.c_void_p), len(fills),
                                            int(n_buf), int(n_spill), int(spill_base)), "prog_set_regfile")
        self.launches = int(_lib.fhegpu_prog_launches(self.handle))

    def run_host(self, lanes: int, chunk_lanes: int, in_slots, in_ptrs, out_slots, out_ptrs,
                 host_format: int = 0):
        """fhegpu_prog_run_host: stream `lanes` host-resident lanes through the device in
        chunks (copy-in / evaluate / copy-out overlapped).  *_ptrs are host addresses of
        dense (lanes, N, k) u32 arrays (pinned for overlap).  Asynchronous."""
        ni, no = len(in_slots), len(out_slots)
        if len(in_ptrs) != ni or len(out_ptrs) != no:
            raise UsageError("one host buffer per slot")
        isl = (ctypes.c_uint32 * max(1, ni))(*[int(x) for x in in_slots])
        osl = (ctypes.c_uint32 * max(1, no))(*[int(x) for x in out_slots])
        ip = (ctypes.c_void_p * max(1, ni))(*[int(x) for x in in_ptrs])
        op = (ctypes.c_void_p * max(1, no))(*[int(x) for x in out_ptrs])
        _check(_lib.fhegpu_prog_run_host(self.ctx.handle, self.handle, int(lanes), int(chunk_lanes),
                                         int(host_format), ni, isl, ip, no, osl, op), "prog_run_host")

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and _lib is not None:
            _lib.fhegpu_prog_destroy(h)
            self.handle = None


class DeviceContext:
    """One fhegpu_ctx: device store + stream for one parameter set."""

    def __init__(self, params, device: int = 0):
        lib = load_library()
        if params.q >= 1 << 31 or params.k > 16:
            raise ParameterError("GPU library supports q < 2^31 and n <= 15")
        self.params = params
        cp = _Params(params.n, params.ell, params.q, params.m)
        h = ctypes.c_void_p()
        _check(lib.fhegpu_ctx_create(ctypes.byref(cp), device, ctypes.byref(h)), "ctx_create")
        self.handle = h
        self.device = device
        self.ct_words = int(lib.fhegpu_ct_words(h))
        self.words = params.n_ct * params.k

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and _lib is not None:
            _lib.fhegpu_ctx_destroy(h)
            self.handle = None

    # -- configuration --------------------------------------------------------------
    def set_stream(self, stream_ptr: int | None):
        """Launch on this CUDA stream handle (0 = legacy default stream, None = own stream)."""
        if stream_ptr is None:
            stream_ptr = _lib.fhegpu_ctx_own_stream(self.handle) or 0
        _check(_lib.fhegpu_ctx_set_stream(self.handle, ctypes.c_void_p(stream_ptr)), "set_stream")

    def use_torch_stream(self, stream=None):
        """Launch on a torch CUDA stream (default: torch's current stream)."""
        import torch
        st = stream if stream is not None else torch.cuda.current_stream()
        self.set_stream(int(st.cuda_stream))
        return st

    def set_kernel(self, kernel: int):
        _check(_lib.fhegpu_ctx_set_kernel(self.handle, int(kernel)), "set_kernel")

    def num_sms(self) -> int:
        return int(_lib.fhegpu_ctx_num_sms(self.handle))

    @property
    def kernel(self) -> str:
        return KERNEL_NAMES[int(_lib.fhegpu_ctx_kernel(self.handle))]

    def set_graphs(self, enable: bool):
        _check(_lib.fhegpu_ctx_set_graphs(self.handle, 1 if enable else 0), "set_graphs")

    def set_debug(self, dbg: int):
        _check(_lib.fhegpu_ctx_set_debug(self.handle, int(dbg)), "set_debug")

    def sync(self):
        _check(_lib.fhegpu_sync(self.handle), "sync")

    # -- store ----------------------------------------------------------------------
    def reserve(self, n_cts: int):
        _check(_lib.fhegpu_store_reserve(self.handle, int(n_cts)), "store_reserve")

    @property
    def capacity(self) -> int:
        return int(_lib.fhegpu_store_capacity(self.handle))

    @property
    def store_ptr(self) -> int:
        return int(_lib.fhegpu_store_device_ptr(self.handle))

    def write(self, idx, values: np.ndarray):
        idx = np.ascontiguousarray(idx, dtype=np.uint64)
        vals = np.ascontiguousarray(values, dtype=np.uint32).reshape(len(idx), self.words)
        _check(_lib.fhegpu_store_write(self.handle, _ptr(idx, ctypes.c_uint64), len(idx),
                                       _ptr(vals, ctypes.c_uint32)), "store_write")

    def write_range(self, first: int, count: int, host_ptr: int, sync: bool = True):
        """Raw host pointer (e.g. pinned torch tensor) of count dense ciphertexts -> store."""
        _check(_lib.fhegpu_store_write_range(self.handle, first, count, ctypes.c_void_p(host_ptr),
                                             0 if sync else 1), "store_write_range")

    def read_range(self, first: int, count: int, host_ptr: int, sync: bool = True):
        _check(_lib.fhegpu_store_read_range(self.handle, first, count, ctypes.c_void_p(host_ptr),
                                            0 if sync else 1), "store_read_range")

    def write_packed(self, first: int, count: int, host_ptr: int):
        """Store range <- serialised ciphertexts (ceil(N^2/8) bytes each, fileio.pack_compact)."""
        _check(_lib.fhegpu_store_write_packed(self.handle, first, count, ctypes.c_void_p(host_ptr)),
               "store_write_packed")

    def read_packed(self, first: int, count: int, host_ptr: int):
        """Store range -> serialised ciphertexts (ceil(N^2/8) bytes each)."""
        _check(_lib.fhegpu_store_read_packed(self.handle, first, count, ctypes.c_void_p(host_ptr)),
               "store_read_packed")

    def copy_slots(self, src_slots, dst_slots, lanes: int):
        """Whole-slot device copies: slot src[i] -> dst[i] over `lanes` ciphertexts each."""
        src = np.ascontiguousarray(src_slots, dtype=np.uint32)
        dst = np.ascontiguousarray(dst_slots, dtype=np.uint32)
        if src.shape != dst.shape:
            raise ValueError("copy_slots: source and destination counts differ")
        _check(_lib.fhegpu_store_copy_slots(self.handle, _ptr(src, ctypes.c_uint32), _ptr(dst, ctypes.c_uint32),
                                            len(src), int(lanes)), "store_copy_slots")

    def read(self, idx, complement=None) -> np.ndarray:
        idx = np.ascontiguousarray(idx, dtype=np.uint64)
        out = np.empty((len(idx), self.params.n_ct, self.params.k), dtype=np.uint32)
        comp = None if complement is None else np.ascontiguousarray(complement, dtype=np.uint8)
        _check(_lib.fhegpu_store_read(self.handle, _ptr(idx, ctypes.c_uint64),
                                      None if comp is None else _ptr(comp, ctypes.c_uint8),
                                      len(idx), _ptr(out, ctypes.c_uint32)), "store_read")
        return out

    def read_rows(self, idx, row: int, complement=None) -> np.ndarray:
        idx = np.ascontiguousarray(idx, dtype=np.uint64)
        out = np.empty((len(idx), self.params.k), dtype=np.uint32)
        comp = None if complement is None else np.ascontiguousarray(complement, dtype=np.uint8)
        _check(_lib.fhegpu_store_read_rows(self.handle, _ptr(idx, ctypes.c_uint64),
                                           None if comp is None else _ptr(comp, ctypes.c_uint8),
                                           len(idx), int(row), _ptr(out, ctypes.c_uint32)),
               "store_read_rows")
        return out

    def decrypt_rows(self, idx, row: int, pw: np.ndarray, complement=None) -> np.ndarray:
        """Centred decryption sums x (int64) of row `row` of each ciphertext (see the header)."""
        idx = np.ascontiguousarray(idx, dtype=np.uint64)
        pw = np.ascontiguousarray(pw, dtype=np.uint32)
        out = np.empty(len(idx), dtype=np.int32)
        comp = None if complement is None else np.ascontiguousarray(complement, dtype=np.uint8)
        _check(_lib.fhegpu_store_decrypt_rows(self.handle, _ptr(idx, ctypes.c_uint64),
                                              None if comp is None else _ptr(comp, ctypes.c_uint8),
                                              len(idx), int(row), _ptr(pw, ctypes.c_uint32),
                                              _ptr(out, ctypes.c_int32)), "store_decrypt_rows")
        return out.astype(np.int64)

    # -- programs and scheme operators ------------------------------------------------
    def program(self, ops: np.ndarray, level_offsets) -> Program:
        return Program(self, ops, np.asarray(level_offsets))

    def nand_batch(self, v1: np.ndarray, v2: np.ndarray) -> np.ndarray:
        v1 = np.ascontiguousarray(v1, dtype=np.uint32)
        v2 = np.ascontiguousarray(v2, dtype=np.uint32)
        out = np.empty_like(v1)
        _check(_lib.fhegpu_nand_batch(self.handle, _ptr(v1, ctypes.c_uint32), _ptr(v2, ctypes.c_uint32),
                                      _ptr(out, ctypes.c_uint32), len(v1)), "nand_batch")
        return out

    def encrypt(self, public_key, streams, stream_idx, u32_offset, mu, target):
        """Device encryption (fhegpu_encrypt): ciphertext e -> store index target[e]."""
        pk = np.ascontiguousarray(np.asarray(public_key) % self.params.q, dtype=np.uint32)
        st = np.ascontiguousarray(np.array([tuple(x) for x in streams], dtype=PCG_DTYPE))
        idx = np.ascontiguousarray(stream_idx, dtype=np.uint32)
        off = np.ascontiguousarray(u32_offset, dtype=np.uint64)
        mus = np.ascontiguousarray(mu, dtype=np.uint32)
        tgt = np.ascontiguousarray(target, dtype=np.uint64)
        _check(_lib.fhegpu_encrypt(self.handle, _ptr(pk, ctypes.c_uint32), st.ctypes.data_as(ctypes.c_void_p),
                                   len(st), _ptr(idx, ctypes.c_uint32), _ptr(off, ctypes.c_uint64),
                                   _ptr(mus, ctypes.c_uint32), _ptr(tgt, ctypes.c_uint64), len(idx)),
               "encrypt")

    def _binary(self, fn, name, v1, v2):
        v1 = np.ascontiguousarray(v1, dtype=np.uint32)
        v2 = np.ascontiguousarray(v2, dtype=np.uint32)
        if v1.shape != v2.shape:
            raise UsageError(f"{name}: operand batches differ in shape")
        out = np.empty_like(v1)
        _check(fn(self.handle, _ptr(v1, ctypes.c_uint32), _ptr(v2, ctypes.c_uint32),
                  _ptr(out, ctypes.c_uint32), len(v1)), name)
        return out

    def add_batch(self, v1: np.ndarray, v2: np.ndarray) -> np.ndarray:
        """(V1 + V2) mod q per pair (hom_add, fhe.py:352-356)."""
        return self._binary(_lib.fhegpu_add_batch, "add_batch", v1, v2)

    def mult_batch(self, v1: np.ndarray, v2: np.ndarray) -> np.ndarray:
        """bits(V1) V2 mod q per pair (hom_mult, fhe.py:366-379; v1 = left after the swap)."""
        return self._binary(_lib.fhegpu_mult_batch, "mult_batch", v1, v2)

    def const_mult_batch(self, k: int, v: np.ndarray) -> np.ndarray:
        """hom_const_mult (fhe.py:358-364) of every ciphertext by the public constant k."""
        v = np.ascontiguousarray(v, dtype=np.uint32)
        out = np.empty_like(v)
        _check(_lib.fhegpu_const_mult_batch(self.handle, int(k) % self.params.q, _ptr(v, ctypes.c_uint32),
                                            _ptr(out, ctypes.c_uint32), len(v)), "const_mult_batch")
        return out

    def not_batch(self, v: np.ndarray) -> np.ndarray:
        v = np.ascontiguousarray(v, dtype=np.uint32)
        out = np.empty_like(v)
        _check(_lib.fhegpu_not_batch(self.handle, _ptr(v, ctypes.c_uint32), _ptr(out, ctypes.c_uint32),
                                     len(v)), "not_batch")
        return out


class BitsContext:
    """fhegpu_bits: device wire store of the bitsliced cleartext engine (lanes packed 32/word)."""

    def __init__(self, lanes: int, device: int = 0):
        lib = load_library()
        h = ctypes.c_void_p()
        _check(lib.fhegpu_bits_create(int(device), int(lanes), ctypes.byref(h)), "bits_create")
        self.handle = h.value
        self.lanes = int(lanes)
        self.words = int(lib.fhegpu_bits_words(self.handle))

    def reserve(self, wires: int):
        _check(_lib.fhegpu_bits_reserve(self.handle, int(wires)), "bits_reserve")

    def write(self, slots, words: np.ndarray):
        slots = np.ascontiguousarray(slots, dtype=np.uint64)
        words = np.ascontiguousarray(words, dtype=np.uint32)
        if words.shape != (len(slots), self.words):
            raise UsageError(f"expected ({len(slots)}, {self.words}) words")
        _check(_lib.fhegpu_bits_write(self.handle, _ptr(slots, ctypes.c_uint64), len(slots),
                                      _ptr(words, ctypes.c_uint32)), "bits_write")

    def run(self, ops: np.ndarray, level_offsets):
        ops = np.ascontiguousarray(ops)
        offs = np.ascontiguousarray(level_offsets, dtype=np.uint64)
        _check(_lib.fhegpu_bits_run(self.handle, ops.ctypes.data_as(ctypes.c_void_p), len(ops),
                                    _ptr(offs, ctypes.c_uint64), len(offs) - 1), "bits_run")

    def read(self, slots, complement=None) -> np.ndarray:
        slots = np.ascontiguousarray(slots, dtype=np.uint64)
        out = np.empty((len(slots), self.words), dtype=np.uint32)
        comp = None if complement is None else np.ascontiguousarray(complement, dtype=np.uint8)
        _check(_lib.fhegpu_bits_read(self.handle, _ptr(slots, ctypes.c_uint64),
                                     None if comp is None else comp.ctypes.data_as(ctypes.c_void_p),
                                     len(slots), _ptr(out, ctypes.c_uint32)), "bits_read")
        return out

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and _lib is not None:
            _lib.fhegpu_bits_destroy(h)
            self.handle = None
