// flow_nand.cuh -- warp-dataflow launches for small geometries (EXACT: k = 3, ell = 17, N = 51).
//
// A single-signal FFT at the toy parameter set (configs[0]: 28,401 gates, 148 levels of <= 360
// gates, a 612-byte ciphertext) is bound by the latency of its dependency chain, not by
// bandwidth or arithmetic: level launches cost ~2.45 us per level whatever the kernel does
// inside.  Here the whole program is ONE launch in which every warp is a worker that runs a
// host-scheduled list of gates, each gate start to finish on the CUDA cores (7,803 conditional
// adds: one lane per output row, the right operand broadcast from shared memory), and operands
// travel by the shortest path that exists:
//   * ring     each warp keeps its last RING outputs in shared memory; gates scheduled on the
//              same CTA read them there (~100 cycles after the producer's last store);
//   * scratch  every output is also written to a single-assignment scratch array in global
//              memory (L2), which any SM can read (~1,300 cycles producer to consumer);
//   * store    program inputs are read from the ciphertext store; every output is written
//              there too in the store's plain layout (read-back, later programs).
// There are no flags, fences or counters: every 32-bit word of a ring or scratch row carries a
// tag next to its 17-bit value -- the run's epoch (scratch) or the producer's position in its
// worker's list (ring) -- and a consumer polls the rows it needs until every word carries the
// tag it expects.  A word is written by one store instruction, so a row is valid exactly when
// all its tags match, however the stores of different words are ordered or torn; a ring entry
// overwritten before (or while) a late consumer reads it fails the tag check and the consumer
// falls back to the scratch copy, which is never overwritten within a run.
//
// The schedule (flow_plan, host side) is a list schedule over a latency model: gates by
// decreasing length of the chain of consumers below them, each appended to the worker that can
// start it earliest among the least loaded warp of the CTAs that produced its operands and the
// globally earliest-free worker.  Appending in a topological order makes every worker's list
// deadlock-free as long as all workers are resident (one CTA per SM, grid <= SM count).
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <queue>
#include <vector>

#include "../../include/fhegpu.h"
#include "common.cuh"

namespace fhegpu {
namespace flow {

#ifndef FHEGPU_FLOW_RING_BUILD
#define FHEGPU_FLOW_RING_BUILD FHEGPU_FLOW_RING
#endif
constexpr int RING = FHEGPU_FLOW_RING_BUILD;    // outputs each warp keeps in shared memory
#ifndef FHEGPU_FLOW_WARPS_BUILD
#define FHEGPU_FLOW_WARPS_BUILD FHEGPU_FLOW_WARPS
#endif
constexpr int WARPS = FHEGPU_FLOW_WARPS_BUILD;  // workers per CTA
#ifndef FHEGPU_FLOW_SPLIT
#define FHEGPU_FLOW_SPLIT 1
#endif
constexpr int SPLIT = FHEGPU_FLOW_SPLIT;        // warps per worker (2: output rows split between two warps --
                                                // measured slower, 232 vs 213 us: a gate's arithmetic is
                                                // not what its dependency chain waits for)
constexpr uint32_t VBITS = 17;          // value bits of a tagged word (q <= 2^17)
constexpr uint32_t VMASK = (1u << VBITS) - 1u;
constexpr uint32_t TAG_MAX = 32767u;    // tags 1..32767 (15 bits; 0 = never written): the run's
                                        // epoch, or a gate's position + 1 in its worker's list
constexpr uint32_t MAX_GATES = 1u << 24;
constexpr uint32_t NO_STORE = 0xFFFFFFFFu;   // out slot of a temporary (FHEGPU_OP_TEMP): no plain copy

// Operand meta word: bits 0-1 kind, bit 2 complement, bit 3 (left operand only) acquire before the
// right operand, bits 4-7 producer's warp in the CTA,
// bits 8-22 producer's position + 1 in its worker's list (ring operands; <= TAG_MAX).
enum : uint32_t { K_STORE = 0, K_SCRATCH = 1, K_RING = 2 };

// One scheduled gate (32 bytes): a = {left index, right index, out store slot, own scratch
// index}, b = {left meta, right meta, own position + 1, 0}; out slot NO_STORE: a temporary.  An index is a store slot (kind
// store) or the producing gate's scratch index.
struct Entry {
  uint4 a, b;
};

#ifdef __CUDACC__

// (ld/st.relaxed.gpu and weak stores measured the same as volatile accesses: configs[0] 213-215 us)
#define FLOW_LD_G "ld.volatile.global.v4.u32"
#define FLOW_ST_G "st.volatile.global.v4.u32"
__device__ __forceinline__ uint4 ld_volatile_global_v4(const uint4 *p) {
  uint4 v;
  asm volatile(FLOW_LD_G " {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}

__device__ __forceinline__ void st_volatile_global_v4(uint4 *p, const uint4 &v) {
  asm volatile(FLOW_ST_G " [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

__device__ __forceinline__ uint4 ld_volatile_shared_v4(const uint4 *p) {
  uint4 v;
  asm volatile("ld.volatile.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"((uint32_t)__cvta_generic_to_shared(p))
               : "memory");
  return v;
}

__device__ __forceinline__ void st_volatile_shared_v4(uint4 *p, const uint4 &v) {
  asm volatile("st.volatile.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"((uint32_t)__cvta_generic_to_shared(p)),
               "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// Every word of a row carries `tag` above its value bits: XOR with the tag in place, OR the
// four words, and nothing may remain above the value bits (5 instructions per row).
__device__ __forceinline__ bool tags_ok(const uint4 &v, uint32_t tag) {
  const uint32_t e = tag << VBITS;
  return (((v.x ^ e) | (v.y ^ e) | (v.z ^ e) | (v.w ^ e)) >> VBITS) == 0u;
}

// acc += row where word has the mask bit set: one predicate + three predicated adds (left to
// itself the compiler builds an all-ones mask and ANDs every term: 6.5 instead of 4
// instructions per (row, bit)).
__device__ __forceinline__ void cond_add3(uint32_t word, uint32_t mask, const uint4 &row, uint32_t (&acc)[3]) {
  asm("{\n\t.reg .pred p;\n\t.reg .b32 t;\n\t"
      "and.b32 t, %3, %4;\n\t"
      "setp.ne.u32 p, t, 0;\n\t"
      "@p add.u32 %0, %0, %5;\n\t"
      "@p add.u32 %1, %1, %6;\n\t"
      "@p add.u32 %2, %2, %7;\n\t}"
      : "+r"(acc[0]), "+r"(acc[1]), "+r"(acc[2])
      : "r"(word), "r"(mask), "r"(row.x), "r"(row.y), "r"(row.z));
}

// (Packing a row's three 17-bit values into 21-bit fields of one 64-bit word would make it one
// predicate + one add with carry, but ptxas does not predicate a carry chain or a wide
// multiply-add: it selects the operands instead, 5 instructions per (row, bit).  Not kept.)

// Timeline probe (-DFHEGPU_TRACE=1 builds only, tools/probes/flow_trace.py): per gate (index <
// FLOW_TRACE_GATES) {right wait, left wait, compute, total} in SM clocks, {operand paths taken |
// worker << 16, globaltimer (ns, low word) after the right operand, after the left, at the end},
// {clock64 (low word) at the ring store, after the right operand, at the right operand's ring
// flag; SM id}.
#ifndef FHEGPU_TRACE
#define FHEGPU_TRACE 0
#endif
constexpr uint32_t FLOW_TRACE_GATES = FHEGPU_TRACE ? 32768u : 1u;
constexpr int FLOW_TRACE_WORDS = 12;
__device__ uint32_t g_flow_trace[FLOW_TRACE_WORDS * FLOW_TRACE_GATES];

__device__ __forceinline__ bool tags_newer(const uint4 &v, uint32_t tag) {
  return ((v.x >> VBITS) > tag) | ((v.y >> VBITS) > tag) | ((v.z >> VBITS) > tag) | ((v.w >> VBITS) > tag);
}

#ifndef FHEGPU_FLOW_SPIN_LIMIT
#define FHEGPU_FLOW_SPIN_LIMIT (1u << 24)   // polls before a worker gives up (trap, not a hung GPU)
#endif

// Rows first + 32 h (h < NR) of one operand into v[NR][K], complement applied.  Returns (the
// path taken) when every lane of the warp holds valid rows.
template <int K, int ELL, int NR>
__device__ __forceinline__ uint32_t acquire_rows(uint32_t idx, uint32_t meta, const uint32_t *store,
                                                 const uint4 *scratch, const uint4 *ring_base, uint32_t epoch,
                                                 uint32_t ct_words, uint32_t q, int first, uint32_t (&v)[NR][K],
                                                 const uint4 (&pre)[NR], bool use_pre, long long *t_flag = nullptr) {
  constexpr int ROWS = K * ELL;
  const uint32_t kind = meta & 3u;
  bool has[NR];
#pragma unroll
  for (int h = 0; h < NR; ++h) has[h] = first + 32 * h < ROWS;
  uint32_t path = kind == K_STORE ? K_STORE : K_SCRATCH;
  if (kind == K_STORE) {
    const uint32_t *src = store + (uint64_t)idx * ct_words;
#pragma unroll
    for (int h = 0; h < NR; ++h)
#pragma unroll
      for (int c = 0; c < K; ++c) v[h][c] = has[h] ? __ldcg(src + (first + 32 * h) * K + c) : 0u;
  } else {
    const uint4 *g = scratch + (uint64_t)idx * ROWS;
    const uint32_t pos1 = meta >> 8;
    const uint4 *r = ring_base + ((meta >> 4) & 15u) * (RING * ROWS) + ((pos1 - 1u) % RING) * ROWS;
    uint4 x[NR];
#pragma unroll
    for (int h = 0; h < NR; ++h) x[h] = make_uint4(0u, 0u, 0u, 0u);
    uint32_t spins = 0;
    bool hit = false;
    if (kind == K_RING) {
      // Tags of one ring entry only grow (positions of the producing worker, same residue mod
      // RING): all equal to the expected one = the rows are there; any larger = overwritten,
      // take the scratch copy; otherwise the producer has not finished -- keep polling shared
      // memory only (a scratch poll in flight would cost its L2 round trip even on a hit).
      // The poll reads ONE word (the last row's tag word, every lane the same address): warps
      // polling whole entries would take half the shared-memory pipe from those that compute.
      const uint32_t *flag = reinterpret_cast<const uint32_t *>(r + (ROWS - 1)) + 3;
      for (;;) {
        uint32_t f;
        asm volatile("ld.volatile.shared.u32 %0, [%1];"
                     : "=r"(f)
                     : "r"((uint32_t)__cvta_generic_to_shared(flag))
                     : "memory");
        if ((f >> VBITS) < pos1) {
          if (++spins > FHEGPU_FLOW_SPIN_LIMIT) __trap();
          continue;
        }
#if FHEGPU_TRACE
        if (t_flag) *t_flag = clock64();
#endif
        bool ok = true;
#pragma unroll
        for (int h = 0; h < NR; ++h)                // (every load issued before the first check)
          if (has[h]) x[h] = ld_volatile_shared_v4(r + first + 32 * h);
#pragma unroll
        for (int h = 0; h < NR; ++h) ok = ok & (!has[h] | tags_ok(x[h], pos1));
        if (__all_sync(0xffffffffu, ok)) {
          hit = true;
          break;
        }
        bool gone = false;                          // (off the hit path)
#pragma unroll
        for (int h = 0; h < NR; ++h) gone = gone | (has[h] & tags_newer(x[h], pos1));
        if (__any_sync(0xffffffffu, gone)) break;
        if (++spins > FHEGPU_FLOW_SPIN_LIMIT) __trap();
      }
    }
    if (hit) {
      path = K_RING;
    } else {
      for (;;) {
        bool ok = true;
        if (use_pre) {                              // the first poll was issued by the caller
#pragma unroll
          for (int h = 0; h < NR; ++h) x[h] = pre[h];
          use_pre = false;
        } else {
#pragma unroll
          for (int h = 0; h < NR; ++h)              // (both L2 round trips in flight together)
            if (has[h]) x[h] = ld_volatile_global_v4(g + first + 32 * h);
        }
#pragma unroll
        for (int h = 0; h < NR; ++h) ok = ok & (!has[h] | tags_ok(x[h], epoch));
        if (__all_sync(0xffffffffu, ok)) break;
        if (++spins > FHEGPU_FLOW_SPIN_LIMIT) __trap();
      }
    }
#pragma unroll
    for (int h = 0; h < NR; ++h) {
      v[h][0] = x[h].x & VMASK;
      if (K > 1) v[h][1] = x[h].y & VMASK;
      if (K > 2) v[h][2] = x[h].z & VMASK;
    }
  }
  if (meta & 4u) {
#pragma unroll
    for (int h = 0; h < NR; ++h) {
      const int row = first + 32 * h;
#pragma unroll
      for (int c = 0; c < K; ++c) v[h][c] = has[h] ? sub_mod(gadget_ct<ELL>(row, c), v[h][c], q) : 0u;
    }
  }
  return path;
}

// One CTA = WARPS workers of SPLIT warps.  The warps of a worker run the same gate list
// independently: each computes the output rows lane + 32 * (part + SPLIT * h) from its own copy of
// the right operand, so they never synchronise (a consumer's tag check covers all parts).
// ents: every worker's gates in its order; worker_off[w] .. [w+1].
template <int K, int ELL>
__global__ void __launch_bounds__(32 * WARPS * SPLIT, 1)
flow_kernel(uint32_t *__restrict__ store, uint4 *__restrict__ scratch, const uint4 *__restrict__ ents,
            const uint32_t *__restrict__ worker_off, uint32_t epoch, uint32_t q_magic, DevParams p) {
  static_assert(K <= 3 && K * ELL <= 64 && ELL <= (int)VBITS, "flow kernel geometry");
  constexpr int ROWS = K * ELL;
  constexpr int NL = 2 / SPLIT;                     // output (and left operand) rows per lane
  __shared__ uint4 s_ring[WARPS * RING * ROWS];
  __shared__ uint4 s_stage[WARPS * SPLIT * ROWS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int part = warp % SPLIT, wk = warp / SPLIT;
  for (int i = threadIdx.x; i < WARPS * RING * ROWS; i += 32 * WARPS * SPLIT) s_ring[i] = make_uint4(0u, 0u, 0u, 0u);
  __syncthreads();
  const uint32_t worker = blockIdx.x * WARPS + wk;
  const uint32_t e0 = worker_off[worker], e1 = worker_off[worker + 1];
  uint4 *stage = s_stage + warp * ROWS;
  uint4 *my_ring = s_ring + wk * (RING * ROWS);
  const int first = lane + 32 * part;               // my first output row
  uint4 na, nb;
  if (e0 < e1) na = __ldg(ents + 2 * e0), nb = __ldg(ents + 2 * e0 + 1);
  for (uint32_t e = e0; e < e1; ++e) {
    const uint4 A = na, B = nb;
    if (e + 1 < e1) na = __ldg(ents + 2 * (e + 1)), nb = __ldg(ents + 2 * (e + 1) + 1);
    uint32_t a[NL][K], b[2][K];
#if FHEGPU_TRACE
    const long long t0 = clock64();
#endif
    // The left operand's first scratch poll (or its store rows) is requested before the right
    // operand is waited for: when the left one arrived long ago its L2 round trip overlaps the wait
    // instead of following it (151.1 -> 149.8 us).  Taking a left operand that is already in its
    // ring entry before the wait as well measured slower (155.5 us).
    const uint32_t lkind = B.x & 3u;
    uint4 lpre[NL], nopre[2];
    uint32_t path_l = lkind;
    bool left_done = false;
#pragma unroll
    for (int h = 0; h < 2; ++h) nopre[h] = make_uint4(0u, 0u, 0u, 0u);
    if (lkind == K_SCRATCH) {
#pragma unroll
      for (int h = 0; h < NL; ++h) {
        lpre[h] = make_uint4(0u, 0u, 0u, 0u);
        if (first + 32 * h < ROWS) lpre[h] = ld_volatile_global_v4(scratch + (uint64_t)A.x * ROWS + first + 32 * h);
      }
    } else {
#pragma unroll
      for (int h = 0; h < NL; ++h) lpre[h] = make_uint4(0u, 0u, 0u, 0u);
    }
    // (symmetrically: the right operand's first scratch poll goes out before a left operand that
    // is waited for first)
    const bool rpre_on = (B.x & 8u) && (B.y & 3u) == K_SCRATCH;
    if (rpre_on) {
      nopre[0] = ld_volatile_global_v4(scratch + (uint64_t)A.y * ROWS + lane);
      if (lane + 32 < ROWS) nopre[1] = ld_volatile_global_v4(scratch + (uint64_t)A.y * ROWS + lane + 32);
    }
    // meta bit 3 (planner): the left operand is expected first -- take it before waiting for the
    // right one, so that only the later operand's own read follows its arrival
    if (lkind == K_STORE || (B.x & 8u)) {
      path_l = acquire_rows<K, ELL, NL>(A.x, B.x, store, scratch, s_ring, epoch, p.ct_words, p.q, first, a, lpre,
                                        lkind == K_SCRATCH);
      left_done = true;
    }
#if FHEGPU_TRACE
    long long t_flag = 0;
    const uint32_t path_r =
        acquire_rows<K, ELL, 2>(A.y, B.y, store, scratch, s_ring, epoch, p.ct_words, p.q, lane, b, nopre, rpre_on, &t_flag);
#else
    const uint32_t path_r =
        acquire_rows<K, ELL, 2>(A.y, B.y, store, scratch, s_ring, epoch, p.ct_words, p.q, lane, b, nopre, rpre_on);
#endif
#if FHEGPU_TRACE
    const long long t1 = clock64();
    uint32_t gt1;
    asm volatile("mov.u32 %0, %%globaltimer_lo;" : "=r"(gt1));
#endif
    __syncwarp();                                   // the previous gate's readers are done with stage
    stage[lane] = make_uint4(b[0][0], K > 1 ? b[0][1] : 0u, K > 2 ? b[0][2] : 0u, 0u);
    if (lane + 32 < ROWS) stage[lane + 32] = make_uint4(b[1][0], K > 1 ? b[1][1] : 0u, K > 2 ? b[1][2] : 0u, 0u);
    if (!left_done)
      path_l = acquire_rows<K, ELL, NL>(A.x, B.x, store, scratch, s_ring, epoch, p.ct_words, p.q, first, a, lpre,
                                        lkind == K_SCRATCH);
    __syncwarp();
#if FHEGPU_TRACE
    const long long t2 = clock64();
    uint32_t gt2;
    asm volatile("mov.u32 %0, %%globaltimer_lo;" : "=r"(gt2));
#else
    (void)path_r, (void)path_l;
#endif
    uint32_t acc[NL][3];
#pragma unroll
    for (int h = 0; h < NL; ++h) acc[h][0] = acc[h][1] = acc[h][2] = 0u;
#pragma unroll
    for (int w = 0; w < K; ++w) {
#pragma unroll
      for (int bit = 0; bit < ELL; ++bit) {
        const uint4 row = stage[w * ELL + bit];     // broadcast
#pragma unroll
        for (int h = 0; h < NL; ++h) cond_add3(a[h][w], 1u << bit, row, acc[h]);
      }
    }
#if FHEGPU_TRACE
    const long long t3 = clock64();
#endif
#if FHEGPU_TRACE
    long long t_ring = 0;
#endif
    // out = (G - S mod q) mod q;  S < N * q < 2^32: one-correction Barrett with floor(2^32 / q)
    const uint32_t pos1 = B.z;
    const uint32_t rt = pos1 << VBITS, et = epoch << VBITS;
    uint4 *rdst = my_ring + ((pos1 - 1u) % RING) * ROWS;
    uint4 *gdst = scratch + (uint64_t)A.w * ROWS;
    uint32_t *sdst = store + (uint64_t)A.z * p.ct_words;
    uint32_t o[NL][3];
#pragma unroll
    for (int h = 0; h < NL; ++h) {
      const int row = first + 32 * SPLIT * h;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        uint32_t s = c < K ? acc[h][c] : 0u;
        s -= __umulhi(s, q_magic) * p.q;
        if (s >= p.q) s -= p.q;
        o[h][c] = c < K && row < ROWS ? sub_mod(gadget_ct<ELL>(row, c), s, p.q) : 0u;
      }
    }
    // every ring store before the first global store: a consumer on this SM polls the last
    // row's tag, and stores leave the warp in program order
#pragma unroll
    for (int h = 0; h < NL; ++h) {
      const int row = first + 32 * SPLIT * h;
      if (row < ROWS) st_volatile_shared_v4(rdst + row, make_uint4(o[h][0] | rt, o[h][1] | rt, o[h][2] | rt, rt));
    }
#if FHEGPU_TRACE
    t_ring = clock64();
#endif
#pragma unroll
    for (int h = 0; h < NL; ++h) {
      const int row = first + 32 * SPLIT * h;
      if (row < ROWS) st_volatile_global_v4(gdst + row, make_uint4(o[h][0] | et, o[h][1] | et, o[h][2] | et, et));
    }
    if (A.z != NO_STORE) {
#pragma unroll
      for (int h = 0; h < NL; ++h) {
        const int row = first + 32 * SPLIT * h;
        if (row < ROWS) {
#pragma unroll
          for (int c = 0; c < K; ++c) sdst[row * K + c] = o[h][c];
        }
      }
    }
#if FHEGPU_TRACE
    if (lane == 0 && part == SPLIT - 1 && A.w < FLOW_TRACE_GATES) {
      uint32_t gt3;
      asm volatile("mov.u32 %0, %%globaltimer_lo;" : "=r"(gt3));
      uint32_t *tr = g_flow_trace + FLOW_TRACE_WORDS * A.w;
      uint32_t smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      tr[8] = (uint32_t)t_ring, tr[9] = (uint32_t)t1, tr[10] = (uint32_t)t_flag, tr[11] = smid;
      tr[0] = (uint32_t)(t1 - t0), tr[1] = (uint32_t)(t2 - t1), tr[2] = (uint32_t)(t3 - t2);
      tr[3] = (uint32_t)(clock64() - t0);
      tr[4] = path_r | path_l << 4 | (B.y & 3u) << 8 | (B.x & 3u) << 12 | worker << 16;
      tr[5] = gt1, tr[6] = gt2, tr[7] = gt3;
    }
#endif
  }
}

#endif  // __CUDACC__

// ------------------------------------------------------------------------------------------
// Host: list schedule of a levelised program onto n_cta * WARPS workers.
struct FlowPlan {
  std::vector<Entry> ents;            // grouped by worker, in execution order
  std::vector<uint32_t> worker_off;   // n_workers + 1
  double makespan = 0;                // model cycles
  uint32_t ring_operands = 0, scratch_operands = 0, store_operands = 0;
  uint32_t max_gates_per_worker = 0;
};

// Latency model (cycles at ~1.9 GHz; measured orders of magnitude)
// The constants are the trace's medians (tools/probes/flow_trace.py): ~970 cycles of service per
// gate, ~385 from a producer's ring store to a waiting consumer on the same SM holding the
// operand, ~1,060 through L2.  The planner's structure matters more than its constants
// (tools/probes/flow_timing.py with FHEGPU_FLOW_MODEL): workers run their lists in order, so a
// gate queued behind one whose operand is late waits with it.  With these constants configs[0]
// took 151 us; with a remote hop over-estimated at 2,500 the greedy chases locality, and counting
// on more than the producer's last ring entry then costs 213-500 us (no locality preference at
// all: 188 us).  Planning the gates by chain length overall (not level by level): 145 us; telling
// the kernel which operand to take first (meta bit 3): 137 us; planned idle time after each gate
// (pad 1,200-1,600): 132 us; and with that planner 8 workers per CTA instead of 4 (pad 1,600-2,000):
// 125 us (under the locality-chasing plans 8 had been slower than 4).
struct FlowModel {
  double comp = 970;      // a gate on one warp, operands at hand, to its ring store
  double remote = 1060;   // producer's scratch store -> consumer's poll sees it (through L2)
  double local = 385;     // the same through the CTA's shared-memory ring
  uint32_t ring_eff = 1;  // ring entries a consumer can count on (of RING)
  double own = 385;       // an operand from the worker's own ring
  double pad = 1800;      // idle time planned after every gate (slack against late operands; 1,600-2,000: flat)
  FlowModel() {
    if (const char *e = std::getenv("FHEGPU_FLOW_MODEL")) {   // experiments: "comp,remote,local,ring[,own]"
      double c, r, l, o = -1, p = 0;
      unsigned k;
      if (std::sscanf(e, "%lf,%lf,%lf,%u,%lf,%lf", &c, &r, &l, &k, &o, &p) >= 4) {
        comp = c, remote = r, local = l, ring_eff = k;
        own = o >= 0 ? o : l;
        pad = p;
      }
    }
  }
};

// ops: n records {left, right, out, flags} in level order; deps: 2 per op (producing op or -1);
// level_off: n_levels + 1.
inline FlowPlan flow_plan(const OpRec *ops, const int32_t *deps, uint64_t n, const uint64_t *level_off,
                          uint32_t n_levels, uint32_t n_cta, const FlowModel &m = FlowModel()) {
  const uint32_t W = n_cta * WARPS;
  FlowPlan pl;
  // bottom level of every gate (longest chain of consumers below it): the priority in a level
  std::vector<uint32_t> bl(n, 1);
  for (uint64_t i = n; i-- > 0;) {
    for (int s = 0; s < 2; ++s) {
      const int32_t d = deps[2 * i + s];
      if (d >= 0) bl[d] = std::max(bl[d], bl[i] + 1);
    }
  }
  std::vector<uint32_t> order(n);
  for (uint64_t i = 0; i < n; ++i) order[i] = (uint32_t)i;
  // Gates in increasing order of (1 - beta) * level - beta * (chain of consumers below): a
  // topological order for any beta in [0, 1] (along an edge the level grows and the chain
  // shrinks).  beta = 0 is level order (139 us on configs[0]), beta = 1 longest chain first
  // overall; anything from 0.1 to 1 measures 128-133 us (FHEGPU_FLOW_ORDER=beta).
  double beta = 1.0;
  if (const char *oe = std::getenv("FHEGPU_FLOW_ORDER")) beta = std::min(1.0, std::max(0.0, std::atof(oe)));
  {
    std::vector<double> key(n);
    for (uint32_t l = 0; l < n_levels; ++l)
      for (uint64_t i = level_off[l]; i < level_off[l + 1]; ++i) key[i] = (1.0 - beta) * l - beta * bl[i];
    std::stable_sort(order.begin(), order.end(), [&](uint32_t x, uint32_t y) {
      return key[x] < key[y] || (key[x] == key[y] && bl[x] > bl[y]);
    });
  }
  std::vector<double> fin(n, 0.0), free_at(W, 0.0);
  std::vector<uint32_t> wk(n, 0), pos(n, 0), cnt(W, 0);
  using QE = std::pair<double, uint32_t>;
  std::priority_queue<QE, std::vector<QE>, std::greater<QE>> heap;    // (free time, worker), lazy
  for (uint32_t w = 0; w < W; ++w) heap.push({0.0, w});
  std::vector<std::vector<uint32_t>> lists(W);
  auto start_on = [&](uint32_t g, uint32_t w) {
    double r = 0;
    for (int s = 0; s < 2; ++s) {
      const int32_t d = deps[2 * g + s];
      if (d < 0) continue;
      const bool near = wk[d] / WARPS == w / WARPS && cnt[wk[d]] - pos[d] <= m.ring_eff;
      const bool mine = wk[d] == w && near;
      r = std::max(r, fin[d] + (mine ? m.own : near ? m.local : m.remote));
    }
    return std::max(r, free_at[w]);
  };
  for (uint64_t oi = 0; oi < n; ++oi) {
    const uint32_t g = order[oi];
    while (heap.top().first != free_at[heap.top().second]) {
      const uint32_t w = heap.top().second;
      heap.pop();
      heap.push({free_at[w], w});
    }
    uint32_t best_w = heap.top().second;
    double best = start_on(g, best_w);
    for (int s = 0; s < 2; ++s) {
      const int32_t d = deps[2 * g + s];
      if (d < 0) continue;
      const uint32_t c0 = wk[d] / WARPS * WARPS;
      uint32_t lw = c0;
      for (uint32_t w = c0; w < c0 + WARPS; ++w)
        if (free_at[w] < free_at[lw]) lw = w;
      for (uint32_t w : {lw, wk[d]}) {
        const double st = start_on(g, w);
        if (st < best) best = st, best_w = w;
      }
    }
    fin[g] = best + m.comp;
    wk[g] = best_w;
    pos[g] = cnt[best_w]++;
    free_at[best_w] = fin[g] + m.pad;
    heap.push({free_at[best_w], best_w});
    lists[best_w].push_back(g);
    pl.makespan = std::max(pl.makespan, fin[g]);
  }
  pl.worker_off.assign(W + 1, 0);
  for (uint32_t w = 0; w < W; ++w) {
    pl.worker_off[w + 1] = pl.worker_off[w] + (uint32_t)lists[w].size();
    pl.max_gates_per_worker = std::max<uint32_t>(pl.max_gates_per_worker, (uint32_t)lists[w].size());
  }
  const char *lf = std::getenv("FHEGPU_FLOW_LEFT_FIRST");
  const bool left_first_on = !lf || std::atoi(lf) != 0;
  pl.ents.resize(n);
  for (uint32_t w = 0; w < W; ++w) {
    for (uint32_t i = 0; i < lists[w].size(); ++i) {
      const uint32_t g = lists[w][i];
      Entry &e = pl.ents[pl.worker_off[w] + i];
      uint32_t idx[2], meta[2];
      for (int s = 0; s < 2; ++s) {
        const int32_t d = deps[2 * g + s];
        const uint32_t comp = (ops[g].flags >> s) & 1u;
        if (d < 0) {
          idx[s] = s ? ops[g].right : ops[g].left;
          meta[s] = K_STORE | comp << 2;
          ++pl.store_operands;
        } else {
          idx[s] = (uint32_t)d;
          // ring operands: same CTA and not yet overwritten when this gate is reached IF the
          // workers ran in lockstep with the model; the tag check decides at run time
          const bool same_cta = wk[d] / WARPS == w / WARPS;
          const bool ring = same_cta && (wk[d] != w || i - pos[d] <= (uint32_t)RING);
          meta[s] = (ring ? K_RING : K_SCRATCH) | comp << 2 | (wk[d] % WARPS) << 4 | (pos[d] + 1u) << 8;
          ++(ring ? pl.ring_operands : pl.scratch_operands);
        }
      }
      // which operand the model expects first (with the final placement)
      double arrive[2] = {0.0, 0.0};
      for (int s = 0; s < 2; ++s) {
        const int32_t d = deps[2 * g + s];
        if (d >= 0) arrive[s] = fin[d] + (wk[d] == w ? m.own : wk[d] / WARPS == w / WARPS ? m.local : m.remote);
      }
      if (left_first_on && arrive[0] < arrive[1]) meta[0] |= 8u;
      e.a = make_uint4(idx[0], idx[1], (ops[g].flags & FHEGPU_OP_TEMP) ? NO_STORE : ops[g].out, g);
      e.b = make_uint4(meta[0], meta[1], i + 1u, 0u);
    }
  }
  return pl;
}

}  // namespace flow
}  // namespace fhegpu
