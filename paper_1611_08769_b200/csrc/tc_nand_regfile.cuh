// tc_nand_regfile.cuh -- register-file launches: a whole per-lane netlist per CTA, one lane at a
// time, with shared-memory ciphertext buffers as registers (plan: rf_plan.h).
//
// Level launches read both operands of every gate from L2/HBM and write its output back: 3
// ciphertexts (28 KB) per gate, ~1.5 uJ of the ~5 uJ a gate costs above idle at the board's
// power limit.  Here the planner has scheduled the lane program and assigned
// every value a buffer; only program inputs, program outputs and spills cross L2 (~0.4
// ciphertexts per gate for the reference's FFT netlists).
//
// Pipeline roles, TMEM double buffers, MMA sequence, A/B operand construction, tail rows and
// the fold are those of resident_tc_kernel (tc_nand_resident.cuh).  What changes:
//  * the slot table (one entry per gate of the lane program) and the fill list stream from
//    global memory (L2-resident, shared by every CTA), prefetched one slot ahead;
//  * the producer warp issues the plan's fills (bulk copies into buffers) as soon as their
//    conditions hold, on a ring of RF_FILL_RING completion barriers;
//  * progress is published as three shared-memory counters (slots, per CTA, across lanes):
//      built  operands of slots < built have been read      (tail warp, after main_done)
//      epi    outputs of slots < epi are in their buffers    (epilogue, after the tail rows)
//      st     stores of slots < st have completed            (epilogue store thread, on request)
//    and every hazard the planner found is a wait on one of them;
//  * a gate's output is stored (program output or spill) by the epilogue's store thread.
#pragma once

#include "rf_plan.h"
#include "tc_nand_resident.cuh"

namespace fhegpu {
namespace tc {

template <int K, int ELL>
struct GeoRF {
  using R = GeoRes<K, ELL>;
  static constexpr int CT_BYTES = R::CT_BYTES, CT_WORDS = R::CT_WORDS, B_BYTES = R::B_BYTES,
                       TA_BYTES = R::TA_BYTES;
#ifndef FHEGPU_RF_GATE
#define FHEGPU_RF_GATE 1     // a gate warp waits for every slot's conditions on behalf of the builders
#endif
  static constexpr int WARP_ST = R::THREADS / 32;   // + the store warp
  static constexpr int WARP_GATE = WARP_ST + 1;     // + the gate warp (FHEGPU_RF_GATE)
  static constexpr int THREADS = R::THREADS + 32 + (FHEGPU_RF_GATE ? 32 : 0);
  static constexpr int N_OUT = 3;
  static constexpr int RING = (int)rf::RF_FILL_RING;
  static constexpr int N_BARS = 8 + 3 * N_OUT + RING + 4 + 2;
  __host__ __device__ static uint32_t off_b(uint32_t n_buf) { return ((n_buf * CT_BYTES + 127u) / 128u) * 128u; }
  __host__ __device__ static uint32_t off_ta(uint32_t n_buf) { return off_b(n_buf) + 2u * B_BYTES; }
  __host__ __device__ static uint32_t off_bar(uint32_t n_buf) {
    return ((off_ta(n_buf) + 2u * TA_BYTES + 127u) / 128u) * 128u;
  }
  __host__ __device__ static uint32_t smem_bytes(uint32_t n_buf) { return off_bar(n_buf) + N_BARS * 8u + 128u; }
};

// mbarrier phase wait with a bound (trap instead of a hung GPU if a plan ever deadlocks).
__device__ __forceinline__ bool mbar_try(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.b32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

#ifndef FHEGPU_RF_NAP
#define FHEGPU_RF_NAP 32     // ns of back-off per failed wait: the spinning roles leave issue slots to the
                             // builders (cfg4 615.8 -> 604 ms; 20 / 60 / 150 ns measured the same)
#endif
__device__ __forceinline__ void rf_mbar_wait(uint64_t *bar, uint32_t parity) {
  uint32_t spins = 0;
  while (!mbar_try(bar, parity)) {           // try_wait suspends a while per call: ~seconds
    if (++spins > (1u << 22)) __trap();
#if FHEGPU_RF_NAP > 0
    __nanosleep(FHEGPU_RF_NAP);
#endif
  }
}

// Poll a shared-memory counter until it reaches `need` (bounded: trap instead of a hung GPU).
__device__ __forceinline__ void rf_wait_ge(const uint32_t *ctr, uint32_t need) {
  uint32_t spins = 0;
  while (ld_acquire_cta_smem(ctr) < need) {
    if (++spins > FHEGPU_SPIN_LIMIT) __trap();
#if FHEGPU_RF_NAP > 0
    __nanosleep(FHEGPU_RF_NAP);
#endif
  }
}

__device__ __forceinline__ fhegpu_rf_slot rf_load_slot(const fhegpu_rf_slot *s, uint32_t r) {
  const uint4 v = __ldg(reinterpret_cast<const uint4 *>(s) + r);
  fhegpu_rf_slot o;
  o.lbuf = (uint8_t)(v.x & 0xFF);
  o.rbuf = (uint8_t)((v.x >> 8) & 0xFF);
  o.dbuf = (uint8_t)((v.x >> 16) & 0xFF);
  o.bits = (uint8_t)(v.x >> 24);
  o.lwait = v.y;
  o.rwait = v.z;
  o.store = v.w;
  return o;
}

// Per-lane position of slot t, advanced incrementally.
struct RFPos {
  uint32_t it = 0, r = 0, base = 0;   // lane iteration, gate slot in the lane program, it * n_ops
  __device__ __forceinline__ void next(uint32_t n_ops) {
    if (++r == n_ops) {
      r = 0;
      ++it;
      base += n_ops;
    }
  }
};

// Operand waits of a builder (own = left) or B copier (own = right): its own operand's fill
// barrier or near producer's epilogue (epi counter), and ALSO the other operand's fill -- a
// fill is waited on only by its first reading slot, so both roles must wait there: a later
// reader in the other role is ordered after this slot by that role's own program order only.
__device__ __forceinline__ void rf_operand_wait(uint32_t w, uint32_t it, uint32_t base, uint32_t n_fills,
                                                uint64_t *fill_full, const uint32_t *ctr_epi) {
  if (w == rf::NONE) return;
  if (w & rf::WAIT_FILL) {
    const uint32_t q = it * n_fills + (w & ~rf::WAIT_FILL);
    rf_mbar_wait(&fill_full[q % rf::RF_FILL_RING], (q / rf::RF_FILL_RING) & 1u);
  } else {
    rf_wait_ge(ctr_epi, base + w + 1);
  }
}

// A slot whose output buffer last held a stored value (or, in a later lane, may have): its
// epilogue and tail rows wait for the store warp to see those stores read (dest_ok).
__device__ __forceinline__ bool rf_dest_guarded(const fhegpu_rf_slot &si, uint32_t it) {
  return (si.bits & (rf::SB_DEST_STORED | rf::SB_HAZARD)) || ((si.bits & rf::SB_DEST_FIRST) && it > 0);
}

template <int K, int ELL, bool PM, int ENC>
__global__ void __launch_bounds__(GeoRF<K, ELL>::THREADS, 1)
regfile_tc_kernel(uint32_t *__restrict__ store, const fhegpu_rf_slot *__restrict__ slots,
                  const fhegpu_rf_fill *__restrict__ fills, uint32_t n_ops, uint32_t n_fills, uint32_t n_buf,
                  uint32_t lanes, uint32_t *__restrict__ spill, uint32_t n_spill, DevParams p) {
  using R = GeoRes<K, ELL>;
  using F = GeoRF<K, ELL>;
  using G = GeoWS<K, ELL, PM, ENC, false>;       // roles, TMEM columns, MMA descriptors
  extern __shared__ __align__(1024) uint8_t smem[];
  uint32_t *s_buf = reinterpret_cast<uint32_t *>(smem);
  uint8_t *s_b = smem + F::off_b(n_buf);
  uint8_t *s_ta = smem + F::off_ta(n_buf);
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem + F::off_bar(n_buf));
  uint64_t *op_full = bar;                  // [2]
  uint64_t *main_done = bar + 2;            // [2]
  uint64_t *a_free = bar + 4;               // [2]
  uint64_t *d_free = bar + 6;               // [2]
  uint64_t *rows_ready = bar + 8;           // [N_OUT] epilogue rows of slot t written (every epilogue warp)
  uint64_t *tail_ready = bar + 8 + F::N_OUT;  // [N_OUT] tail rows of slot t written
  uint64_t *slot_free = bar + 8 + 2 * F::N_OUT + F::RING;   // [N_OUT] the store warp is done with slot t
  uint64_t *dest_ok = slot_free + F::N_OUT;   // [4] slot t's buffer may be written (store warp)
  uint64_t *go = dest_ok + 4;                 // [2] slot t's A/B buffers are free and its operands present (gate warp)
  uint64_t *fill_full = bar + 8 + 2 * F::N_OUT;   // [RING]
  uint32_t *ctr = reinterpret_cast<uint32_t *>(bar + F::N_BARS);
  uint32_t *ctr_built = ctr, *ctr_epi = ctr + 1, *ctr_st = ctr + 2, *ctr_streq = ctr + 3;
  uint32_t *tmem_slot = ctr + 8;
  uint32_t *s_fcons = ctr + 16;                  // [RF_FILL_RING] consumer slot of the last fills (producer)

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const uint32_t my_lanes = blockIdx.x < lanes ? (lanes - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const uint32_t n_slots = my_lanes * n_ops;
  auto buf = [&](uint32_t b) { return s_buf + b * R::CT_WORDS; };
  auto lane_of = [&](uint32_t it) { return it * gridDim.x + blockIdx.x; };

  if (warp == G::WARP_MMA) tmem_alloc<512>(tmem_slot);
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&op_full[i], R::NB_WARPS + R::NBC_WARPS);
      mbar_init(&main_done[i], 1);
      mbar_init(&a_free[i], 1);
      mbar_init(&d_free[i], R::NE_WARPS);
    }
    for (int i = 0; i < F::N_OUT; ++i) {
      mbar_init(&rows_ready[i], R::NE_WARPS);
      mbar_init(&tail_ready[i], 1);
    }
    for (int i = 0; i < F::N_OUT; ++i) mbar_init(&slot_free[i], 1);
    for (int i = 0; i < 4; ++i) mbar_init(&dest_ok[i], 1);
    for (int i = 0; i < 2; ++i) mbar_init(&go[i], FHEGPU_RF_GATE ? 2 : 1);
    for (int i = 0; i < F::RING; ++i) mbar_init(&fill_full[i], 1);
    for (int i = 0; i < 8; ++i) ctr[i] = 0;
    fence_mbar_init();
  }
  for (uint32_t w = tid; w < 2 * R::B_BYTES / 4; w += R::THREADS) reinterpret_cast<uint32_t *>(s_b)[w] = 0u;
  for (uint32_t w = tid; w < 2 * R::TA_BYTES / 4; w += R::THREADS) reinterpret_cast<uint32_t *>(s_ta)[w] = 0u;
  // ciphertext padding words of every buffer stay zero (the epilogue writes N * K words; fills
  // copy whole padded ciphertexts, whose padding is zero in the store)
  for (uint32_t w = tid; w < n_buf * R::CT_WORDS; w += R::THREADS) s_buf[w] = 0u;
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  asm volatile("griddepcontrol.wait;" ::: "memory");

  if (warp == F::WARP_ST) {
    // ------------------------------ store warp: outputs, spills, progress ------------------------------
    // Per slot, once the epilogue rows and the tail rows are in the buffer: publish epi, store a
    // program output / spill, and allow the next slot's writes (dest_ok) once every store has
    // read its buffer when that slot's buffer held a stored value.  st (store completion) is
    // published as stores drain and on the producer's request (a fill of a recent spill).
    if (lane == 0) {
      uint32_t st_done = 0;
#ifndef FHEGPU_RF_ST_LAG
#define FHEGPU_RF_ST_LAG 1
#endif
      constexpr uint32_t LAG = FHEGPU_RF_ST_LAG;  // stores kept in flight before st advances
      uint32_t st_ring[LAG];
      uint32_t n_st = 0;
#pragma unroll
      for (uint32_t i = 0; i < LAG; ++i) st_ring[i] = 0;
      auto serve = [&](uint32_t upto) {
        if (ld_volatile_smem(ctr_streq) > st_done) {
          bulk_wait_n<0>();
          st_done = upto;
          st_release_cta_smem(ctr_st, upto);
        }
      };
      mbar_arrive(&dest_ok[0]);                     // slot 0
      RFPos pos;
      fhegpu_rf_slot nxt = rf_load_slot(slots, 0);
      for (uint32_t t = 0; t < n_slots; ++t, pos.next(n_ops)) {
        const fhegpu_rf_slot si = nxt;
        nxt = rf_load_slot(slots, pos.r + 1 == n_ops ? 0u : pos.r + 1);
        const uint32_t ob = t % F::N_OUT, ou = t / F::N_OUT;
        uint32_t spins = 0;
        while (!mbar_try(&rows_ready[ob], ou & 1u)) {   // serve requests while waiting
          serve(t);
          if (++spins > (1u << 22)) __trap();
        }
        rf_mbar_wait(&tail_ready[ob], ou & 1u);
        st_release_cta_smem(ctr_epi, t + 1);          // slot t's output is readable in its buffer
        if (si.bits & rf::SB_STORE) {
          const uint32_t ln = lane_of(pos.it);
          uint32_t *dst = (si.store & rf::STORE_SPILL)
                              ? spill + ((uint64_t)blockIdx.x * n_spill + (si.store & ~rf::STORE_SPILL)) *
                                            R::CT_WORDS
                              : store + ((uint64_t)si.store * lanes + ln) * R::CT_WORDS;
          bulk_s2g(dst, buf(si.dbuf), R::CT_BYTES);
#pragma unroll
          for (uint32_t i = LAG - 1; i > 0; --i) st_ring[i] = st_ring[i - 1];
          st_ring[0] = t;
          if (++n_st > LAG) {
            bulk_wait_n<LAG>();                       // stores older than the last LAG are done
            if (st_ring[LAG - 1] > st_done) {
              st_done = st_ring[LAG - 1];
              st_release_cta_smem(ctr_st, st_done);
            }
          }
        }
        mbar_arrive(&slot_free[ob]);
        if (t + 1 < n_slots) {
          const uint32_t it1 = pos.r + 1 == n_ops ? pos.it + 1 : pos.it;
          if (rf_dest_guarded(nxt, it1)) bulk_wait_read_n<0>();   // its buffer's stores have read it
          mbar_arrive(&dest_ok[(t + 1) & 3u]);
        }
        serve(t + 1);
        trace_ev(p, t, 11);
      }
      bulk_wait_all();
    }
#if FHEGPU_RF_GATE
  } else if (warp == F::WARP_GATE) {
    // ------------------------------ gate: every slot's start conditions, once ------------------------------
    // The A builders pace this pipeline, and each of their waits costs ~100-250 cycles of
    // mbarrier / counter latency even when its condition has long held (timeline: 270 + 180
    // cycles per slot).  This warp performs the operand waits (fill barriers, epi counter) ahead
    // of time and arrives on go[t & 1]; the builders and B copiers wait on that one barrier.  (Release/acquire chains are cumulative:
    // what the gate observed is visible to those who observe its arrival.)
    if (lane == 0) {
      RFPos pos;
      fhegpu_rf_slot nxt = rf_load_slot(slots, 0);
      for (uint32_t t = 0; t < n_slots; ++t, pos.next(n_ops)) {
        const uint32_t b = t & 1u, u = t >> 1;
        const fhegpu_rf_slot si = nxt;
        nxt = rf_load_slot(slots, pos.r + 1 == n_ops ? 0u : pos.r + 1);
        // go[b] takes two arrivals per slot: this one (operands present) and the tail warp's
        // after it has read the accumulator of slot t - 2 (buffers free) -- the builders wake on
        // the tail warp's arrival itself.  Slot t - 2's phase must have completed before slot
        // t's first arrival; slots 0 and 1 have no earlier slot: the gate arrives for it.
        if (t >= 2) rf_mbar_wait(&go[b], (u & 1u) ^ 1u);
        rf_operand_wait(si.lwait, pos.it, pos.base, n_fills, fill_full, ctr_epi);
        rf_operand_wait(si.rwait, pos.it, pos.base, n_fills, fill_full, ctr_epi);
        mbar_arrive(&go[b]);
        if (t < 2) mbar_arrive(&go[b]);
      }
    }
#endif
  } else if (warp == G::WARP_PROD) {
    // ------------------------------ producer: the plan's fills, in order ------------------------------
    // The whole warp loads the fill records 32 at a time (the next batch prefetched) and hands
    // them to lane 0 by shuffle: a record fetched per fill would put an L2 round trip on every
    // fill of a burst (a butterfly's operands).
    auto load = [&](uint32_t f, uint4 &a, uint4 &c) {
      if (f < n_fills) {
        a = __ldg(reinterpret_cast<const uint4 *>(fills + f));        // buf, src, consumer, w_built
        c = __ldg(reinterpret_cast<const uint4 *>(fills + f) + 1);    // w_epi, w_st, flags, pad
      } else {
        a = c = make_uint4(0u, 0u, 0u, 0u);
      }
    };
    auto shfl4 = [&](const uint4 &v, uint32_t j) {
      return make_uint4(__shfl_sync(0xffffffffu, v.x, j), __shfl_sync(0xffffffffu, v.y, j),
                        __shfl_sync(0xffffffffu, v.z, j), __shfl_sync(0xffffffffu, v.w, j));
    };
    for (uint32_t it = 0; it < my_lanes; ++it) {
      const uint32_t base = it * n_ops, ln = lane_of(it);
      uint4 a, c;
      load(lane, a, c);
      for (uint32_t f0 = 0; f0 < n_fills; f0 += 32) {
        uint4 na, nc;
        load(f0 + 32 + lane, na, nc);
        const uint32_t cnt = min(32u, n_fills - f0);
        for (uint32_t j = 0; j < cnt; ++j) {
          const uint4 A = shfl4(a, j), C = shfl4(c, j);
          if (lane == 0) {
            const uint32_t f = f0 + j;
            uint32_t need_built = A.w ? base + A.w : 0, need_epi = C.x ? base + C.x : 0;
            uint32_t need_st = C.y ? base + C.y : 0;
            if ((C.z & rf::FF_FIRST) && it > 0)       // the buffer's last occupant is the previous lane's
              need_built = max(need_built, base), need_epi = max(need_epi, base), need_st = max(need_st, base);
            const uint32_t q = it * n_fills + f;
            if (q >= rf::RF_FILL_RING)                // its barrier's previous fill has been waited for
              need_built = max(need_built, s_fcons[q % rf::RF_FILL_RING] + 1);
            s_fcons[q % rf::RF_FILL_RING] = base + A.z;
            rf_wait_ge(ctr_built, need_built);
            rf_wait_ge(ctr_epi, need_epi);
            if (need_st && ld_acquire_cta_smem(ctr_st) < need_st) {
              st_volatile_smem(ctr_streq, need_st);   // ask the store warp to drain its stores
              rf_wait_ge(ctr_st, need_st);
            }
            fence_proxy_async_global();               // completed stores -> this async-proxy load
            const uint32_t *src = (A.y & rf::STORE_SPILL)
                                      ? spill + ((uint64_t)blockIdx.x * n_spill +
                                                 (A.y & ~rf::STORE_SPILL)) * R::CT_WORDS
                                      : store + ((uint64_t)A.y * lanes + ln) * R::CT_WORDS;
            uint64_t *fb = &fill_full[q % rf::RF_FILL_RING];
            mbar_expect_tx(fb, R::CT_BYTES);
            bulk_g2s(buf(A.x), src, R::CT_BYTES, fb);
          }
          __syncwarp();
        }
        a = na, c = nc;
      }
    }
  } else if (warp == G::WARP_MMA) {
    // ------------------------------ MMA issuer (as resident_tc_kernel) ------------------------------
    const uint64_t bdesc0 = smem_desc(smem_u32(s_b), G::LBO, G::SBO);
    const uint64_t tdesc0 = smem_desc(smem_u32(s_ta), G::TA_LBO, 0u);
    for (uint32_t t = 0; t < n_slots; ++t) {
      const uint32_t b = t & 1u, u = t >> 1;
      rf_mbar_wait(&op_full[b], u & 1u);
      if (lane == 0) trace_ev(p, t, 2);
      rf_mbar_wait(&d_free[b], (u & 1u) ^ 1u);
      if (lane == 0) trace_ev(p, t, 3);
      tc_fence_after();
      const uint32_t tb = tmem_base + b * G::BUF_COLS;
      const uint64_t bd_b = bdesc0 + ((b * R::B_BYTES) >> 4);
      const uint64_t td_b = tdesc0 + ((b * R::TA_BYTES) >> 4);
      if (elect_one()) {
#pragma unroll
        for (int mt = 0; mt < G::MT; ++mt) {
#pragma unroll
          for (int s = 0; s < K; ++s)
            mma_i8_ts(tb + mt * G::NPAD, tb + G::D_COLS + mt * 8 * K + 8 * s, bd_b + ((s * 4 * G::LBO) >> 4),
                      G::IDESC, s > 0 ? 1u : 0u);
        }
        if constexpr (G::TAIL > 0) {
#pragma unroll
          for (int s = 0; s < K; ++s)
            mma_i8_ss(tb + G::D_COLS, td_b + ((s * 2 * G::TA_LBO) >> 4), bd_b + ((s * 4 * G::LBO) >> 4),
                      G::IDESC_TAIL, s > 0 ? 1u : 0u);
        }
      }
      __syncwarp();
      if (elect_one()) mma_commit(&main_done[b]);
      __syncwarp();
      if (lane == 0) trace_ev(p, t, 4);
    }
  } else if (warp == G::WARP_TAIL) {
    // ------------------------------ tail rows, into the gate's buffer ------------------------------
    if constexpr (G::TAIL > 0) {
      RFPos pos;
      fhegpu_rf_slot nxt = rf_load_slot(slots, 0);
      for (uint32_t t = 0; t < n_slots; ++t, pos.next(n_ops)) {
        const uint32_t b = t & 1u, u = t >> 1;
        const fhegpu_rf_slot si = nxt;
        nxt = rf_load_slot(slots, pos.r + 1 == n_ops ? 0u : pos.r + 1);
        rf_mbar_wait(&main_done[b], u & 1u);
        if (lane == 0) trace_ev(p, t, 12);
        tc_fence_after();
        uint32_t d[36];
        load_acc36(tmem_base + b * G::BUF_COLS + G::D_COLS, d, false);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
#if FHEGPU_RF_GATE
          mbar_arrive(&go[b]);                        // A(b) / B(b) free for slot t + 2
#else
          mbar_arrive(&a_free[b]);
#endif
          // slot t's MMAs are done, so its operand buffers were read long before (op_full):
          // publish from here -- a release on the MMA warp would sit on its issue path
          st_release_cta_smem(ctr_built, t + 1);
        }
        const uint32_t ob = t % F::N_OUT;
        if (rf_dest_guarded(si, pos.it)) rf_mbar_wait(&dest_ok[t & 3u], (t >> 2) & 1u);
        if (lane == 0) trace_ev(p, t, 13);
        uint32_t *out_st = buf(si.dbuf);
        if (lane < G::TAIL) {
          const int row = G::MMA_ROWS + lane;
          const int rb = row / ELL, rbit = row - rb * ELL;
#pragma unroll
          for (int i = 0; i < K; ++i) out_st[row * K + i] = finish_neg<ELL, PM, ENC>(&d[i * 4], i == rb ? (1u << rbit) : 0u, p);
        }
        fence_proxy_async_smem();
        __syncwarp();
        // tail_ready(t) reuses the entry of slot t - 3: the store warp must be done with it
        if (lane == 0) {
          rf_mbar_wait(&slot_free[ob], ((t / F::N_OUT) & 1u) ^ 1u);
          mbar_arrive(&tail_ready[ob]);
        }
        if (lane == 0) trace_ev(p, t, 14);
      }
    }
  } else if (warp >= R::WARP_BC0 && warp < R::WARP_EPI0) {
    // ------------------------------ B operand copiers ------------------------------
    const int bc = tid - 32 * R::WARP_BC0;
    constexpr int NBT = 32 * (R::NBC_WARPS > 0 ? R::NBC_WARPS : 1);
    constexpr int B_ROWS = (G::KB + NBT - 1) / NBT;
    int b_src[B_ROWS], b_dst[B_ROWS], b_w[B_ROWS], b_j[B_ROWS];
#pragma unroll
    for (int x = 0; x < B_ROWS; ++x) {
      const int kr = bc + x * NBT;
      const int ww = kr >> 5, kk = kr & 31;
      const int j = 8 * (kk & 3) + (kk >> 2);
      b_src[x] = kr < G::KB && j < ELL ? (ww * ELL + j) * K : -1;
      b_dst[x] = (kr >> 3) * G::LBO + (kr & 7) * 16;
      b_w[x] = ww;
      b_j[x] = j;
    }
    RFPos pos;
    fhegpu_rf_slot nxt = rf_load_slot(slots, 0);
    for (uint32_t t = 0; t < n_slots; ++t, pos.next(n_ops)) {
      const uint32_t b = t & 1u, u = t >> 1;
      const fhegpu_rf_slot si = nxt;
      nxt = rf_load_slot(slots, pos.r + 1 == n_ops ? 0u : pos.r + 1);
      if (bc == 0) trace_ev(p, t, 0);
#if FHEGPU_RF_GATE
      rf_mbar_wait(&go[b], u & 1u);                   // B(b) free (MMAs of slot t - 2 done), operands present
#else
      rf_mbar_wait(&a_free[b], (u & 1u) ^ 1u);        // B(b) was last read by the MMAs of slot t - 2
      rf_operand_wait(si.rwait, pos.it, pos.base, n_fills, fill_full, ctr_epi);
      if (si.lwait != rf::NONE && (si.lwait & rf::WAIT_FILL))
        rf_operand_wait(si.lwait, pos.it, pos.base, n_fills, fill_full, ctr_epi);
#endif
      const uint32_t *v2 = buf(si.rbuf);
      const bool comp2 = si.bits & rf::SB_RNEG;
      uint8_t *bb = s_b + b * R::B_BYTES;
      // B(b) still holds slot t-2's right operand: equal operands skip the copy (same lane only)
      const bool reuse = (si.bits & rf::SB_REUSE_R) && pos.r >= 2 && !(p.dbg & (1u << 20));
#pragma unroll
      for (int x = 0; x < (reuse ? 0 : B_ROWS); ++x) {
        if (b_src[x] < 0) continue;
        uint32_t vals[K];
#pragma unroll
        for (int i = 0; i < K; ++i) vals[i] = v2[b_src[x] + i];
        if (comp2) {
#pragma unroll
          for (int i = 0; i < K; ++i) vals[i] = sub_mod(i == b_w[x] ? (1u << b_j[x]) : 0u, vals[i], p.q);
        }
        uint8_t *dst = bb + b_dst[x];
#pragma unroll
        for (int ch = 0; ch < G::NCH; ++ch) {
          uint4 val;
          val.x = 4 * ch + 0 < K ? vals[4 * ch + 0] : 0u;
          val.y = 4 * ch + 1 < K ? vals[4 * ch + 1] : 0u;
          val.z = 4 * ch + 2 < K ? vals[4 * ch + 2] : 0u;
          val.w = 4 * ch + 3 < K ? vals[4 * ch + 3] : 0u;
          *reinterpret_cast<uint4 *>(dst + ch * G::SBO) = val;
        }
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&op_full[b]);
      if (bc == 0) trace_ev(p, t, 1);
    }
  } else if (warp < R::WARP_EPI0) {
    // ------------------------------ A operand builders ------------------------------
    const int bt = tid - 32 * G::WARP_BUILD0;
    const int bw = bt >> 5;
    const int quad = warp & 3;
    const int tile = (bw >> 2) % G::MT;
    const int row = 128 * tile + 32 * quad + lane;
    const uint32_t lane_off = (uint32_t)(32 * quad) << 16;
    const int row_blk = row / ELL, row_bit = row - row_blk * ELL;
    RFPos pos;
    fhegpu_rf_slot nxt = rf_load_slot(slots, 0);
    // (trace builds: dbg bits 8-10 pick the builder warp whose events are recorded)
    const bool tr0 = FHEGPU_TRACE ? bt == 32 * (int)((p.dbg >> 8) & 7u) : bt == 0;
    for (uint32_t t = 0; t < n_slots; ++t, pos.next(n_ops)) {
      const uint32_t b = t & 1u, u = t >> 1;
      const fhegpu_rf_slot si = nxt;
      nxt = rf_load_slot(slots, pos.r + 1 == n_ops ? 0u : pos.r + 1);
      if (tr0) trace_ev(p, t, 5);
#if FHEGPU_RF_GATE
      rf_mbar_wait(&go[b], u & 1u);
      if (tr0) trace_ev(p, t, 7);
#else
      rf_mbar_wait(&a_free[b], (u & 1u) ^ 1u);
      if (tr0) trace_ev(p, t, 7);
      rf_operand_wait(si.lwait, pos.it, pos.base, n_fills, fill_full, ctr_epi);
      if (si.rwait != rf::NONE && (si.rwait & rf::WAIT_FILL))
        rf_operand_wait(si.rwait, pos.it, pos.base, n_fills, fill_full, ctr_epi);
#endif
      if (tr0) trace_ev(p, t, 6);
      tc_fence_after();
      const uint32_t *v1 = buf(si.lbuf);
      const bool comp1 = si.bits & rf::SB_LNEG;
      // A(b) still holds slot t-2's left operand except tile 0's first 6 words, which that slot's
      // M = 64 tail accumulator overwrote (as in resident_tc_kernel), and TA(b) its tail rows
      const bool reuse = (si.bits & rf::SB_REUSE_L) && pos.r >= 2 && !(p.dbg & (1u << 20));
      {
        const uint32_t a_addr = tmem_base + b * G::BUF_COLS + lane_off + G::D_COLS + tile * 8 * K;
        if (reuse) {
          if (tile == 0) build_a_words<K, 0, 6, ENC>(v1, row, row_blk, row_bit, comp1, p.q, a_addr);
        } else {
          build_a_words<K, 0, K, ENC>(v1, row, row_blk, row_bit, comp1, p.q, a_addr);
        }
      }
      if constexpr (G::TAIL > 0) {
        if (bt < G::TAIL * K && !reuse) {
          const int m = bt / K, ww = bt - m * K;
          const int rr = G::MMA_ROWS + m;
          uint32_t v = v1[rr * K + ww];
          if (comp1) v = sub_mod(ww == rr / ELL ? (1u << (rr % ELL)) : 0u, v, p.q);
          uint32_t sp[8];
          spread_word_sr<ENC>(v, sp);
          uint8_t *dst = s_ta + b * R::TA_BYTES + (2 * ww) * G::TA_LBO + m * 16;
          *reinterpret_cast<uint4 *>(dst) = make_uint4(sp[0], sp[1], sp[2], sp[3]);
          *reinterpret_cast<uint4 *>(dst + G::TA_LBO) = make_uint4(sp[4], sp[5], sp[6], sp[7]);
        }
      }
      tmem_wait_st();
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&op_full[b]);
      if (tr0) trace_ev(p, t, 8);
    }
  } else {
    // ------------------------------ epilogue, into the gate's buffer ------------------------------
    // Each warp on its own (no CTA barrier per slot): TMEM -> fold -> rows of the gate's
    // buffer -> rows_ready.  Stores and progress counters belong to the store warp.
    const int et = tid - 32 * R::WARP_EPI0;
    const int ew = et >> 5;
    const int quad = warp & 3;
    const int tile = (ew >> 2) & 1;
    const int row = 128 * tile + 32 * quad + lane;
    const uint32_t lane_off = (uint32_t)(32 * quad) << 16;
    const int row_blk = row / ELL, row_bit = row - row_blk * ELL;
    RFPos pos;
    fhegpu_rf_slot nxt = rf_load_slot(slots, 0);
    for (uint32_t t = 0; t < n_slots; ++t, pos.next(n_ops)) {
      const uint32_t b = t & 1u, u = t >> 1;
      const fhegpu_rf_slot si = nxt;
      nxt = rf_load_slot(slots, pos.r + 1 == n_ops ? 0u : pos.r + 1);
      uint32_t *out_st = buf(si.dbuf);
      rf_mbar_wait(&main_done[b], u & 1u);
      if (et == 0) trace_ev(p, t, 9);
      tc_fence_after();
      const uint32_t dcol = tmem_base + b * G::BUF_COLS + lane_off + tile * G::NPAD;
      uint32_t d[36];
      load_acc36(dcol, d, false);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&d_free[b]);
      // (delaying this fold so that the builders of slot t + 2 run first was measured: 150 ns of
      // sleep here 597 -> 608 ms, 300 ns 750 ms -- the epilogue is as close to the period)
      if (rf_dest_guarded(si, pos.it)) rf_mbar_wait(&dest_ok[t & 3u], (t >> 2) & 1u);
#pragma unroll
      for (int i = 0; i < K; ++i)
        out_st[row * K + i] = finish_neg<ELL, PM, ENC>(&d[i * 4], i == row_blk ? (1u << row_bit) : 0u, p);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {                             // (entry reuse: as tail_ready)
        rf_mbar_wait(&slot_free[t % F::N_OUT], ((t / F::N_OUT) & 1u) ^ 1u);
        mbar_arrive(&rows_ready[t % F::N_OUT]);
      }
      if (et == 0) trace_ev(p, t, 10);
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == G::WARP_MMA) tmem_dealloc<512>(tmem_base);
}

}  // namespace tc
}  // namespace fhegpu
