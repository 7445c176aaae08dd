/*
 * fhegpu.h -- C ABI of the B200 engine for the encrypted-FFT hot path.
 *
 * The reference (arxiv 1611.08769, package `fhefft`, pure Python) has no FFI;
 * its plugin boundary for this path is the duck-typed bit-engine protocol
 * (fhefft/engine.py:69-214) over the scheme operators GswScheme.hom_nand /
 * GswScheme.hom_not (fhefft/fhe.py:325-350).  This library is what a
 * maintainer would bind (ctypes) to replace those two
 * operators and the engine's gate-at-a-time evaluation:
 *
 *   fhegpu_nand_batch   replaces GswScheme.hom_nand   (fhe.py:325-341), batched
 *   fhegpu_not_batch    replaces GswScheme.hom_not    (fhe.py:343-350), batched
 *   fhegpu_{add,mult,const_mult}_batch  replace hom_add / hom_mult / hom_const_mult
 *                       (fhe.py:352-379), batched
 *   fhegpu_prog_*       replaces FheEngine.nand/_fold  (engine.py:168-187) applied
 *                       gate by gate: a whole levelised netlist (every gate of
 *                       every butterfly of every signal) runs as one kernel per level
 *   fhegpu_store_*      replaces the Ciphertext objects the engine keeps alive
 *                       (engine.py:57-66, fhe.py:148-161): device-resident compact
 *                       ciphertexts, read back for export_ct/read_back (engine.py:189-207)
 *
 * Ciphertext representation (bit-identical to the reference matrix): a
 * reference ciphertext is the flattened N x N 0/1 matrix C = decompose(V); the
 * library stores V, an N x k row-major matrix of u32 values in [0, q)
 * (k = n + 1, N = k * ell).  Each ciphertext occupies ct_words u32 (N*k
 * padded to a multiple of 4 so every ciphertext is 16-byte aligned for bulk
 * copies).  NAND:  V = (G - bits(V1) V2) mod q.   NOT:  V = (G - V) mod q.
 *
 * Conventions: every call returns 0 (FHEGPU_OK) or an error code and sets a
 * thread-local message (fhegpu_last_error).  Host arrays are borrowed for the
 * duration of the call.  Device memory is owned by the context.  A context is
 * bound to one device and one stream and is not thread safe.
 */
#ifndef FHEGPU_H
#define FHEGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fhegpu_ctx fhegpu_ctx;
typedef struct fhegpu_prog fhegpu_prog;

typedef struct {
  uint32_t n;    /* lattice dimension (SchemeParams.n); k = n + 1 */
  uint32_t ell;  /* bits per Z_q value = bitlen(q - 1) (SchemeParams.ell) */
  uint32_t q;    /* odd modulus, 8 <= q < 2^31 for this library */
  uint32_t m;    /* public-key rows (SchemeParams.m); used by encryption only */
} fhegpu_params;

/* One netlist gate.  `left` is the operand the reference multiplies on the
 * left AFTER its noise swap (fhe.py:336-337).  Flags bit 0 / bit 1 complement
 * the left / right operand on load: that is how NOT gates (hom_not, produced
 * only by folding NAND(x, 1), engine.py:180-187) are evaluated for free.
 * Flags bit 3 (FHEGPU_OP_STREAM_OUT, a hint): nothing later in the same program reads `out`;
 * its store is marked L2 evict-first so it does not displace the program's temporaries. */
#define FHEGPU_OP_STREAM_OUT 8u
/* Flags bit 4 (FHEGPU_OP_TEMP, a hint): nothing outside the program reads `out` (no read-back,
 * no later program).  Launches that pass operands on chip (warp-dataflow) skip its store;
 * level launches ignore it. */
#define FHEGPU_OP_TEMP 16u
typedef struct {
  uint32_t left;
  uint32_t right;
  uint32_t out;
  uint32_t flags;
} fhegpu_op;

enum {
  FHEGPU_OK = 0,
  FHEGPU_EINVAL = 1,
  FHEGPU_ECUDA = 2,
  FHEGPU_ENOMEM = 3,
  FHEGPU_EUNSUP = 4
};

enum {
  FHEGPU_OP_COMPLEMENT_LEFT = 1u,
  FHEGPU_OP_COMPLEMENT_RIGHT = 2u
};

enum {
  FHEGPU_KERNEL_AUTO = 0,     /* tcgen05 when the parameter set has a build, else SIMT */
  FHEGPU_KERNEL_SIMT = 1,     /* CUDA-core reference kernel (any k <= 16, ell <= 31) */
  FHEGPU_KERNEL_TCGEN05 = 2   /* sm_100a tensor-core kernel (error if unavailable) */
};

const char *fhegpu_last_error(void);
const char *fhegpu_version(void);

/* Context: device, stream, parameter set.  Replaces GswScheme(params) (fhe.py:167-171). */
int fhegpu_ctx_create(const fhegpu_params *params, int device, fhegpu_ctx **out);
void fhegpu_ctx_destroy(fhegpu_ctx *ctx);
int fhegpu_ctx_set_stream(fhegpu_ctx *ctx, void *cuda_stream); /* NULL = legacy default stream */
void *fhegpu_ctx_own_stream(const fhegpu_ctx *ctx);           /* the stream a new context starts on */
int fhegpu_ctx_set_kernel(fhegpu_ctx *ctx, int kernel);        /* FHEGPU_KERNEL_* */
int fhegpu_ctx_kernel(const fhegpu_ctx *ctx);                  /* kernel a level launch will use */
int fhegpu_ctx_num_sms(const fhegpu_ctx *ctx);                 /* SMs = the widest launch's CTAs */
int fhegpu_ctx_set_debug(fhegpu_ctx *ctx, uint32_t dbg);       /* test knobs; 0 in production */
int fhegpu_ctx_set_graphs(fhegpu_ctx *ctx, int enable);        /* replay programs as CUDA graphs (default on) */
uint32_t fhegpu_ct_words(const fhegpu_ctx *ctx);
int fhegpu_sync(fhegpu_ctx *ctx);

/* Device ciphertext store (indices are ciphertext numbers: slot * lanes + lane). */
int fhegpu_store_reserve(fhegpu_ctx *ctx, uint64_t n_cts);     /* grows, keeps contents */
uint64_t fhegpu_store_capacity(const fhegpu_ctx *ctx);
uint64_t fhegpu_store_device_ptr(const fhegpu_ctx *ctx);      /* base address (for device-side producers) */
int fhegpu_store_write(fhegpu_ctx *ctx, const uint64_t *idx, uint64_t count,
                       const uint32_t *host_v /* count x N*k, dense */);
int fhegpu_store_read(fhegpu_ctx *ctx, const uint64_t *idx, const uint8_t *complement,
                      uint64_t count, uint32_t *host_v /* count x N*k */);
/* Only row `row` of V (k words) per ciphertext: what decryption needs (fhe.py:259-286). */
int fhegpu_store_read_rows(fhegpu_ctx *ctx, const uint64_t *idx, const uint8_t *complement,
                           uint64_t count, uint32_t row, uint32_t *host_rows /* count x k */);

/* Batched decryption phase (fhe.py:267-286, the sum before rounding): for each ciphertext,
 * x = sum_{i<k, b<ell} bit_b(V[row][i]) * pw[i*ell + b] mod q, centred to (-q/2, q/2], where
 * pw[i*ell + b] = (sk_i << b) mod q comes from the caller (the secret key never enters the
 * library).  The caller rounds x to the bit and applies the reference's noise check. */
int fhegpu_store_decrypt_rows(fhegpu_ctx *ctx, const uint64_t *idx, const uint8_t *complement,
                              uint64_t count, uint32_t row, const uint32_t *pw, int32_t *host_x);

/* Contiguous ciphertext ranges [first, first + count) <-> dense host rows (N*k u32 each),
 * one strided async copy (pinned host memory reaches full PCIe bandwidth).  async = 0
 * synchronises the context stream before returning. */
int fhegpu_store_write_range(fhegpu_ctx *ctx, uint64_t first, uint64_t count,
                             const uint32_t *host_v, int async);
int fhegpu_store_read_range(fhegpu_ctx *ctx, uint64_t first, uint64_t count, uint32_t *host_v,
                            int async);

/* Device-side copies of whole slots: for i < n, ciphertexts [src_slots[i] * lanes, +lanes)
 * -> [dst_slots[i] * lanes, +lanes).  Destinations must be distinct and must not be a
 * source of another pair.  Used to bind a cached program's private input slots to the
 * wires a caller holds and to hand its outputs back (no counterpart in the reference:
 * its Ciphertext values are immutable Python objects, fhe.py:148-161).  Asynchronous on the
 * context stream. */
int fhegpu_store_copy_slots(fhegpu_ctx *ctx, const uint32_t *src_slots, const uint32_t *dst_slots, uint32_t n,
                            uint64_t lanes);

/* Store range <-> the reference's serialised ciphertexts (FHEGPU_HOST_PACKED rows of
 * ceil(N*N/8) bytes: fileio.py:72-79, one ciphertext of an EFT1 payload).  Synchronous. */
int fhegpu_store_write_packed(fhegpu_ctx *ctx, uint64_t first, uint64_t count, const uint8_t *host_bytes);
int fhegpu_store_read_packed(fhegpu_ctx *ctx, uint64_t first, uint64_t count, uint8_t *host_bytes);

/* Levelised netlist: ops[level_offsets[l] .. level_offsets[l+1]) are the gates of
 * level l; every op of a level reads only slots written by earlier levels. */
int fhegpu_prog_create(fhegpu_ctx *ctx, const fhegpu_op *ops, uint64_t n_ops,
                       const uint64_t *level_offsets, uint32_t n_levels, fhegpu_prog **out);
/* Run every level for `lanes` independent copies of the netlist (ciphertext
 * index = slot * lanes + lane); one kernel launch per level, on the context stream.
 * The first run on a non-default stream also captures the launches into a CUDA graph
 * that later runs replay with one cudaGraphLaunch. */
int fhegpu_prog_run(fhegpu_ctx *ctx, fhegpu_prog *prog, uint32_t lanes);
/* Run levels [first, last) only (profiling / partial evaluation). */
int fhegpu_prog_run_range(fhegpu_ctx *ctx, fhegpu_prog *prog, uint32_t lanes,
                          uint32_t first_level, uint32_t last_level);
/* Host ciphertext formats for fhegpu_prog_run_host. */
enum {
  FHEGPU_HOST_COMPACT = 0, /* dense compact V: N*k u32 per ciphertext (fhe.py:181-185 inverse) */
  FHEGPU_HOST_PACKED = 1   /* the reference's serialised matrix: C = decompose(V) row-major,
                              8 bits per byte MSB first, ceil(N*N/8) bytes per ciphertext --
                              exactly one ciphertext of an EFT1 payload (fileio.py:72-79) */
};
/* Evaluate the program over `lanes` lanes held in HOST memory, streaming them through
 * the device store in chunks of `chunk_lanes` (so a batch may exceed HBM).  host_in[i]
 * holds `lanes` ciphertexts (lane-major, in `host_format`) for the program input in
 * slot in_slots[i]; host_out[i] receives the ciphertexts of slot out_slots[i].  Chunks
 * rotate through 3 store regions (capacity >= 3 * slots * chunk_lanes): the copy-in of
 * chunk c+1, the level kernels of chunk c and the copy-out of chunk c-1 overlap on
 * separate streams (both PCIe directions busy); copies are contiguous into device
 * staging, repacked to store rows on the device.  Asynchronous w.r.t. the host; the
 * context stream observes completion.  Resident store contents are overwritten.
 * Host buffers should be pinned for the copies to overlap.  This is the batched
 * equivalent of a netlist of hom_nand (fhe.py:325-341) over serialised ciphertexts. */
int fhegpu_prog_run_host(fhegpu_ctx *ctx, fhegpu_prog *prog, uint64_t lanes, uint32_t chunk_lanes,
                         int host_format, uint32_t n_in, const uint32_t *in_slots,
                         const void *const *host_in, uint32_t n_out, const uint32_t *out_slots,
                         void *const *host_out);
/* Dataflow mode: deps[2i], deps[2i+1] = index of the op that produced op i's left / right
 * operand in this program (-1: written before the run).  Requires SSA slots (no slot
 * written twice in the program, none overwritten while a reader may still load it) --
 * the engine's dataflow compile guarantees it.  prog_run then evaluates the whole program
 * in ONE launch: each operand load waits for its producer through per-CTA progress
 * counters instead of a kernel boundary per level (narrow, deep netlists such as a single
 * FFT, fft.py:157-194).  Where no tcgen05 kernel applies it falls back to level launches if
 * the level offsets are a valid schedule (no op depends on an op of its own level), and
 * otherwise fails with FHEGPU_EUNSUP instead of running it wrongly. */
int fhegpu_prog_set_deps(fhegpu_ctx *ctx, fhegpu_prog *prog, const int32_t *deps);

/* Opt-in ready-queue execution of a program whose dependencies are set (fhegpu_prog_set_deps):
 * one launch in which CTAs pop only items whose producing items have completed and retire
 * their own items to the consumers' pending counts (pushing consumers that become ready).
 * No static item -> CTA assignment, so no CTA waits on an operand while other work is ready.
 * Same results as level launches (SSA slots required, as for dataflow).  enable = 0 reverts
 * to the static dataflow order.  Replaces the reference's sequential gate loop
 * (engine.py:168-178 driving fhe.py:325-341) like fhegpu_prog_run. */
int fhegpu_prog_set_queue(fhegpu_ctx *ctx, fhegpu_prog *prog, int enable);

/* Opt-in warp-dataflow execution of a single-lane program at a small geometry (k = 3, ell =
 * 17, q <= 2^17: the reference's EXACT preset, fhe.py:110) whose dependencies are set
 * (fhegpu_prog_set_deps): one launch in which every warp runs a host-scheduled list of gates
 * on the CUDA cores and operands pass through shared-memory rings and a tagged scratch array
 * (csrc/flow_nand.cuh).  A single-signal FFT there is bound by its dependency chain (148 levels
 * of <= 360 gates), which level launches pay at ~2.5 us per level.  model_cycles (optional)
 * receives the schedule's modelled makespan, stats (optional, 4 values) the ring / scratch /
 * store operand counts and the longest worker list.  Runs over other lane counts fall back to
 * level launches.  Same results as level launches (SSA slots required, as for dataflow).
 * Replaces the reference's sequential gate loop (engine.py:168-178 driving fhe.py:325-341)
 * like fhegpu_prog_run. */
int fhegpu_prog_set_flow(fhegpu_ctx *ctx, fhegpu_prog *prog, int enable, double *model_cycles,
                         uint32_t *stats);

/* The warp-dataflow schedule on its own (host only, no device): ops in level order, deps as for
 * fhegpu_prog_set_deps, n_cta CTAs of FHEGPU_FLOW_WARPS workers.  entries receives n_ops
 * records of 8 u32 grouped by worker in execution order -- {left index, right index, out slot,
 * gate index, left meta, right meta, position + 1, 0}; an index is a store slot (meta kind 0)
 * or the producing gate's index (kind 1: scratch, kind 2: ring first); meta = kind | complement
 * << 2 | producer's warp << 4 | (producer's position + 1) << 8 -- and worker_off the n_cta *
 * FHEGPU_FLOW_WARPS + 1 list boundaries. */
#define FHEGPU_FLOW_WARPS 8
#define FHEGPU_FLOW_RING 4
int fhegpu_flow_plan(const fhegpu_op *ops, const int32_t *deps, uint64_t n_ops, const uint64_t *level_offsets,
                     uint32_t n_levels, uint32_t n_cta, uint32_t *entries, uint32_t *worker_off,
                     double *model_cycles);

/* One gate of a lane-resident program (fhegpu_prog_set_resident), 16 bytes. */
typedef struct {
  uint8_t lkind, lidx;   /* left operand: kind 0 = program input lidx, 1 = local buffer lidx */
  uint8_t rkind, ridx;   /* right operand, same encoding */
  uint8_t dest;          /* local buffer the gate writes */
  uint8_t is_out;        /* 1: the gate's output is also stored to slot out_slot */
  uint8_t flags;         /* bit 0 / 1: complement the left / right operand (as fhegpu_op) */
  uint8_t pad;
  int16_t lprod, rprod;  /* plan index of the gate that produced a local operand (-1: input) */
  uint32_t out_slot;
} fhegpu_res_op;

/* Opt-in lane-resident execution of a small per-lane program (<= 8 gates, <= 4 inputs, <= 8
 * local buffers; the gates in topological order): one launch in which every CTA runs the whole
 * program for 3 lanes at a time, loading the program inputs (store slots in_slots[]) once and
 * keeping every gate output in a shared-memory buffer of its lane; only is_out gates are stored.
 * The gates of a lane group run in the order of fhegpu_res_slot_order (a gate whose operand
 * equals its lane's previous gate's reuses that operand's tensor-core staging).
 * A local buffer may be reused once every reader of its previous value is the writer or
 * precedes it in the plan; output gates use buffers only outputs use.  Same results as fhegpu_prog_run's level
 * launches (which remain the fallback where no tcgen05 kernel applies); n_ops = 0 disables.
 * Replaces the reference's gate-by-gate evaluation (engine.py:168-178 -> fhe.py:325-341) for
 * independent lanes, e.g. the gate benchmark's XOR + AND (gates.py:9-34). */
int fhegpu_prog_set_resident(fhegpu_ctx *ctx, fhegpu_prog *prog, const fhegpu_res_op *plan, uint32_t n_ops,
                             const uint32_t *in_slots, uint32_t n_in, uint32_t n_local);
/* The order in which a lane-resident launch runs the lanes x n_ops gates of one lane group
 * (host only, no GPU): order[t] = gate | lane << 3 | 32 (left operand reused from slot t - 2) |
 * 64 (right operand reused).  fhegpu_prog_set_resident uses it with lanes = 3; exposed for
 * tests and tools.  lanes <= 4, lanes * n_ops <= 32. */
int fhegpu_res_slot_order(const fhegpu_res_op *plan, uint32_t n_ops, uint32_t lanes, uint8_t *order);
uint32_t fhegpu_prog_launches(const fhegpu_prog *prog);       /* launches one run issues */
/* Register-file launches (tc_nand_regfile.cuh): one lane at a time per CTA runs a whole
 * per-lane netlist with a pool of shared-memory ciphertext buffers as registers -- operands
 * come from buffers, outputs go to buffers; values that do not fit are spilled (stored at
 * their producer) and filled back; program inputs are fills from their store slots; program
 * outputs (held wires) are stored to theirs.  Replaces the level launches of deep programs
 * over many lanes (configs[4]: every butterfly of 1024 signals, fft.py:137-174) and moves
 * ~0.4 instead of 3 ciphertexts per gate through L2/HBM.
 *
 * fhegpu_rf_plan schedules and allocates (host only; see rf_plan.h):
 *   gates     n_gates gates in a topological order; operand ids: input i -> i, the output of
 *             gate j -> n_in + j; flags bit 0 / 1: complement left / right (fused hom_not);
 *             held: the output is a program output, stored to out_slot
 *   in_slots  store slot of each program input
 *   n_buf     shared-memory buffers (<= 20 fit next to the pipeline's operand buffers)
 *   min_dist  preferred slot distance between a gate and its producers (pipeline depth: 5)
 *   lookahead fills are issued this many slots before their first reader
 * outputs: order[slot] = gate, slots[slot], fills[0 .. *n_fills) (fill_cap >= 2 * n_gates),
 * *n_spill = spill slots per CTA. */
typedef struct fhegpu_rf_gate {
  uint32_t left, right;
  uint8_t flags, held;
  uint16_t pad;
  uint32_t out_slot;
} fhegpu_rf_gate;
typedef struct fhegpu_rf_slot {
  uint8_t lbuf, rbuf, dbuf, bits; /* bits: 1/2 complement l/r, 4 store, 8 dest held a stored
                                     value, 16 ... stored by the previous slot, 32 first write
                                     of dest in the lane, 64/128 left/right operand equal to
                                     slot t-2's (A rebuild / B copy skipped) */
  uint32_t lwait, rwait;          /* 0xFFFFFFFF none; bit 31: fill id, else producer slot */
  uint32_t store;                 /* bit 31: spill index, else store slot (with bits & 4) */
} fhegpu_rf_slot;
typedef struct fhegpu_rf_fill {
  uint32_t buf, src;              /* src bit 31: spill index, else store slot */
  uint32_t consumer;              /* first reading slot */
  uint32_t w_built, w_epi, w_st;  /* wait until the kernel's counters reach these slots */
  uint32_t flags, pad;            /* flags bit 0: first use of the buffer in the lane */
} fhegpu_rf_fill;
int fhegpu_rf_plan(const fhegpu_rf_gate *gates, uint32_t n_gates, const uint32_t *in_slots, uint32_t n_in,
                   uint32_t n_buf, uint32_t min_dist, uint32_t lookahead, uint32_t *order,
                   fhegpu_rf_slot *slots, fhegpu_rf_fill *fills, uint32_t fill_cap, uint32_t *n_fills,
                   uint32_t *n_spill,
                   uint32_t *stats /* [5]: stalls, stores, fills, left / right operand reuses; may be NULL */);
/* Attach a plan to a program: fhegpu_prog_run then runs it as ONE register-file launch
 * (tcgen05, k = 9, ell = 29), else level by level.  Spills of CTA c use ciphertexts
 * [spill_base + c * n_spill, + n_spill) of the store (fhegpu_prog_run_host: right after its
 * streaming regions when the store holds them, one launch per chunk).  n_slots = 0 detaches. */
int fhegpu_prog_set_regfile(fhegpu_ctx *ctx, fhegpu_prog *prog, const fhegpu_rf_slot *slots, uint32_t n_slots,
                            const fhegpu_rf_fill *fills, uint32_t n_fills, uint32_t n_buf, uint32_t n_spill,
                            uint64_t spill_base);

void fhegpu_prog_destroy(fhegpu_prog *prog);

/* Scheme operators on host buffers (count independent gates, one launch).
 * v1 is the left operand after the reference's swap.  Replace hom_nand / hom_not. */
int fhegpu_nand_batch(fhegpu_ctx *ctx, const uint32_t *v1, const uint32_t *v2,
                      uint32_t *out, uint64_t count);
int fhegpu_not_batch(fhegpu_ctx *ctx, const uint32_t *v, uint32_t *out, uint64_t count);

/* Z_q ring operators (replace GswScheme.hom_add / hom_const_mult / hom_mult,
 * fhe.py:352-379; level / noise bookkeeping and hom_mult's swap stay host-side):
 *   add:        (V1 + V2) mod q                       = recompose(C1 + C2)
 *   mult:       C1 V2 mod q  (NAND product, complemented) = recompose(C1 C2)
 *   const_mult: mult with left operand (k G) mod q    = recompose(decompose(kG) C)  */
int fhegpu_add_batch(fhegpu_ctx *ctx, const uint32_t *v1, const uint32_t *v2,
                     uint32_t *out, uint64_t count);
int fhegpu_mult_batch(fhegpu_ctx *ctx, const uint32_t *v1, const uint32_t *v2,
                      uint32_t *out, uint64_t count);
int fhegpu_const_mult_batch(fhegpu_ctx *ctx, uint32_t k, const uint32_t *v, uint32_t *out,
                            uint64_t count);

/* Fresh encryption on the device, stream-exact with numpy's Generator(PCG64)
 * (replaces GswScheme._encrypt / encrypt_bit / encrypt_value, fhe.py:227-242).
 * Ciphertext e draws its N x m bits starting u32_offset[e] 32-bit draws after
 * streams[stream_idx[e]] (a numpy PCG64 state with has_uint32 == 0), exactly as
 * rng.integers(0, 2, (N, m)) would, and stores V = (R pk + mu G) mod q at store
 * index target[e].  pk: m x k row-major, entries < q; mu[e] < q. */
typedef struct {
  uint64_t state_lo, state_hi, inc_lo, inc_hi;
} fhegpu_pcg64;

int fhegpu_encrypt(fhegpu_ctx *ctx, const uint32_t *pk, const fhegpu_pcg64 *streams,
                   uint32_t n_streams, const uint32_t *stream_idx, const uint64_t *u32_offset,
                   const uint32_t *mu, const uint64_t *target, uint64_t count);

/* Debug only: timeline probe of the pipelined kernel (64 gates x 16 events, clock64). */
int fhegpu_debug_ws_trace(uint64_t *host_out);
int fhegpu_debug_flow_trace(uint32_t *host_out, uint32_t n_gates);

/* -- Bitsliced cleartext engine (replaces CleartextEngine's evaluation, engine.py:69-121) --
 * A wire is `lanes` plaintext bits packed 32 per u32 word (bit l of word w = lane 32w + l);
 * NAND = ~(a & b) on whole words, complement flags as in fhegpu_op.  Used for the
 * reference's error experiments (harness.py:122-198) at GPU scale.  Slots are wire indices. */
typedef struct fhegpu_bits fhegpu_bits;
int fhegpu_bits_create(int device, uint64_t lanes, fhegpu_bits **out);
void fhegpu_bits_destroy(fhegpu_bits *bits);
uint32_t fhegpu_bits_words(const fhegpu_bits *bits);       /* u32 words per wire */
int fhegpu_bits_reserve(fhegpu_bits *bits, uint64_t wires); /* grows, keeps contents */
int fhegpu_bits_write(fhegpu_bits *bits, const uint64_t *slots, uint64_t count, const uint32_t *words);
/* One launch per level (levels as in fhegpu_prog_create); synchronous. */
int fhegpu_bits_run(fhegpu_bits *bits, const fhegpu_op *ops, uint64_t n_ops,
                    const uint64_t *level_offsets, uint32_t n_levels);
int fhegpu_bits_read(fhegpu_bits *bits, const uint64_t *slots, const uint8_t *complement,
                     uint64_t count, uint32_t *words);

#ifdef __cplusplus
}
#endif

#endif /* FHEGPU_H */
