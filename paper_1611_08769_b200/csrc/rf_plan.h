// rf_plan.h -- host planner for register-file launches (regfile_tc_kernel, tc_nand_regfile.cuh).
//
// A register-file launch runs a whole per-lane netlist (e.g. one 16-point FFT, 108k gates) on
// one lane at a time per CTA, with a pool of shared-memory ciphertext buffers as its registers:
// a gate reads its operands from buffers and the epilogue writes its output into a buffer.
// Values that do not fit are spilled (stored once, at production) and filled back by the
// producer warp's bulk copies; program inputs are fills from their store slots, program outputs
// are stores to theirs.  Level launches move 3 ciphertexts through L2 per gate; a register-file
// schedule of the reference's FFT netlist moves ~0.4.
//
// Planning, once per netlist:
//  1. schedule: list scheduling of the DAG.  A gate may run D slots after its latest producer
//     (the pipeline publishes a gate's output ~5 slots after it starts); among the gates allowed
//     at slot t the one whose latest producer ran last is taken (follows chains: locality),
//     then the longest path to a sink.  Gates reading only program inputs have the lowest
//     priority, so new chains start only when nothing else can run.
//  2. buffers: walk the schedule; a missing operand is filled into a buffer whose last read and
//     write lie >= `look` slots back when one exists (the producer warp can then issue the fill
//     that early): free, else holding a dead value, else the value used furthest in the future
//     (Belady).  An evicted value with later uses that is not already in the store gets a spill
//     store at its producer's epilogue.
//  3. spill slots: interval colouring of [producer slot, last refill's consumer], CTA-private.
//
// Every cross-role hazard becomes a condition on the kernel's progress counters (slots are
// per-lane program positions):
//   built > s : all operands of slot s have been read (builders and B copiers arrived)
//   epi   > s : slot s's output is complete in its buffer (tail rows included)
//   st    > s : every store issued by slots <= s has completed (read and written)
// A fill into buffer b waits for the previous occupant's last read, its write (if nobody read
// it), and its store; a fill of a spilled value waits for that value's store; fill f reuses
// fill-barrier f mod RF_FILL_RING, so it also waits for fill f - RF_FILL_RING's consumer.
// An epilogue writing b after a stored occupant first waits for the store to have read b.
#pragma once

#include <algorithm>
#include <cstdint>
#include <functional>
#include <queue>
#include <string>
#include <vector>

#include "../../include/fhegpu.h"

namespace fhegpu {
namespace rf {

constexpr uint32_t NONE = 0xFFFFFFFFu;
constexpr uint32_t WAIT_FILL = 0x80000000u;   // lwait / rwait: fill id (else producer slot)
constexpr uint32_t STORE_SPILL = 0x80000000u; // store / fill src: spill index (else store slot)
constexpr uint32_t RF_FILL_RING = 16;         // fill-completion mbarriers in the kernel
constexpr uint32_t RF_NEAR = 5;               // producers >= 5 slots back need no wait (pipeline)

// slot bits (fhegpu_rf_slot.bits)
constexpr uint8_t SB_LNEG = 1, SB_RNEG = 2, SB_STORE = 4, SB_DEST_STORED = 8, SB_HAZARD = 16,
                  SB_DEST_FIRST = 32, SB_REUSE_L = 64, SB_REUSE_R = 128;
// fill flags
constexpr uint32_t FF_FIRST = 1;   // first use of the buffer in the lane program

struct Planner {
  // inputs
  const fhegpu_rf_gate *gates = nullptr;
  uint32_t n = 0, n_in = 0, n_buf = 0, dist = 5, look = 4;
  bool reuse = true;                      // prefer operand reuse two slots apart (schedule)
  const uint32_t *in_slots = nullptr;
  // outputs
  std::vector<uint32_t> order;            // slot -> gate
  std::vector<fhegpu_rf_slot> slots;
  std::vector<fhegpu_rf_fill> fills;
  uint32_t n_spill = 0, stalls = 0, n_stores = 0, n_reuse_l = 0, n_reuse_r = 0;
  std::string err;

  uint32_t nv() const { return n_in + n; }

  bool schedule() {
    std::vector<std::vector<uint32_t>> succ(n);
    std::vector<uint32_t> indeg(n, 0);
    for (uint32_t g = 0; g < n; ++g) {
      const uint32_t a = gates[g].left, b = gates[g].right;
      if (a >= nv() || b >= nv()) return fail("operand id out of range at gate " + std::to_string(g));
      uint32_t pa = a >= n_in ? a - n_in : NONE, pb = b >= n_in ? b - n_in : NONE;
      if ((pa != NONE && pa >= g) || (pb != NONE && pb >= g))
        return fail("gates must be in a topological order (gate " + std::to_string(g) + ")");
      if (pa != NONE) succ[pa].push_back(g), ++indeg[g];
      if (pb != NONE && pb != pa) succ[pb].push_back(g), ++indeg[g];
    }
    std::vector<uint32_t> h(n, 1);
    for (uint32_t g = n; g-- > 0;)
      for (uint32_t s : succ[g]) h[g] = std::max(h[g], h[s] + 1);
    std::vector<int64_t> md(n, -1);   // slot of the latest scheduled producer
    // readers of each value by side (operand reuse: slot t's operand equal to slot t-2's lets the
    // kernel skip rebuilding A / copying B -- see tc_nand_regfile.cuh)
    std::vector<std::vector<uint32_t>> lread(nv()), rread(nv());
    for (uint32_t g = 0; g < n; ++g) lread[gates[g].left].push_back(g), rread[gates[g].right].push_back(g);
    std::vector<uint8_t> in_cand(n, 0), done(n, 0);
    // candidates: max (md, h, -g); pending: min allowed slot
    using Cand = std::tuple<int64_t, uint32_t, int64_t>;
    std::priority_queue<Cand> cand;
    using Pend = std::tuple<int64_t, int64_t, int64_t, uint32_t>;   // allowed, -md, -h, g
    std::priority_queue<Pend, std::vector<Pend>, std::greater<Pend>> pend;
    auto push = [&](uint32_t g) {
      const int64_t allowed = md[g] < 0 ? 0 : md[g] + (int64_t)dist;
      pend.emplace(allowed, -md[g], -(int64_t)h[g], g);
    };
    for (uint32_t g = 0; g < n; ++g)
      if (indeg[g] == 0) push(g);
    order.clear();
    order.reserve(n);
    auto same_l = [&](uint32_t a, uint32_t b) {
      return gates[a].left == gates[b].left && ((gates[a].flags ^ gates[b].flags) & 1u) == 0;
    };
    auto same_r = [&](uint32_t a, uint32_t b) {
      return gates[a].right == gates[b].right && ((gates[a].flags ^ gates[b].flags) & 2u) == 0;
    };
    for (int64_t t = 0; (uint32_t)t < n; ++t) {
      while (!pend.empty() && std::get<0>(pend.top()) <= t) {
        const uint32_t g = std::get<3>(pend.top());
        pend.pop();
        cand.emplace(md[g], h[g], -(int64_t)g);
        in_cand[g] = 1;
      }
      while (!cand.empty() && done[(uint32_t)(-std::get<2>(cand.top()))]) cand.pop();   // taken by reuse
      uint32_t g = NONE;
      if (reuse && t >= 2) {                  // an allowed gate sharing slot t-2's operands
        const uint32_t p2 = order[t - 2];
        int best = 0;
        for (int side = 0; side < 2 && best < 3; ++side) {
          const auto &rd = side ? rread[gates[p2].right] : lread[gates[p2].left];
          if (rd.size() > 64) continue;       // (hubs: not worth the scan)
          for (uint32_t c : rd) {
            if (!in_cand[c] || done[c]) continue;
            const int sc = (same_l(c, p2) ? 2 : 0) + (same_r(c, p2) ? 1 : 0);
            if (sc > best) best = sc, g = c;
          }
        }
      }
      if (g != NONE) {
        done[g] = 1;
      } else if (!cand.empty()) {
        g = (uint32_t)(-std::get<2>(cand.top()));
        cand.pop();
        done[g] = 1;
      } else {
        if (pend.empty()) return fail("schedule: no ready gate (cycle?)");
        g = std::get<3>(pend.top());
        pend.pop();
        done[g] = 1;
        ++stalls;
      }
      order.push_back(g);
      for (uint32_t s : succ[g]) {
        md[s] = std::max(md[s], t);
        if (--indeg[s] == 0) push(s);
      }
    }
    return true;
  }

  bool allocate() {
    const uint32_t V = nv();
    std::vector<uint32_t> pos(n);                       // gate -> slot
    for (uint32_t t = 0; t < n; ++t) pos[order[t]] = t;
    // reads of each value, by slot (ascending)
    std::vector<std::vector<uint32_t>> uses(V);
    for (uint32_t t = 0; t < n; ++t) {
      const fhegpu_rf_gate &gt = gates[order[t]];
      uses[gt.left].push_back(t);
      if (gt.right != gt.left) uses[gt.right].push_back(t);
    }
    std::vector<uint32_t> use_ptr(V, 0);
    auto next_use = [&](uint32_t v, uint32_t t) -> uint32_t {   // first read at slot >= t
      uint32_t &p = use_ptr[v];
      while (p < uses[v].size() && uses[v][p] < t) ++p;
      return p < uses[v].size() ? uses[v][p] : NONE;
    };
    auto produced_at = [&](uint32_t v) { return v >= n_in ? pos[v - n_in] : NONE; };
    auto held = [&](uint32_t v) { return v >= n_in && gates[v - n_in].held; };
    std::vector<uint32_t> vbuf(V, NONE);          // buffer holding the value (or being filled)
    std::vector<uint32_t> occ(n_buf, NONE);       // value in each buffer
    std::vector<uint32_t> b_lastread(n_buf, NONE), b_written(n_buf, NONE);   // per residency
    std::vector<uint8_t> b_filled(n_buf, 0), b_used(n_buf, 0);
    std::vector<uint8_t> spill(V, 0);             // stored at production to a spill slot
    std::vector<uint32_t> last_fill_consumer(V, NONE);
    std::vector<uint32_t> pend_fill(V, NONE);     // fill id not yet waited by a reader
    std::vector<uint32_t> res_prod(V, NONE);      // slot that wrote the value into its buffer
    slots.assign(n, fhegpu_rf_slot{});
    fills.clear();
    // store slots known so far (held outputs from the start, spills as they are decided): an
    // output buffer whose stored occupant has a later store in (p, t - 4] needs no dest_ok wait --
    // the store warp drains each store before issuing the next (LAG 1) and is never more than
    // 4 slots behind the epilogue (slot_free), tc_nand_regfile.cuh
    std::vector<uint32_t> fen(n + 1, 0);
    auto fen_add = [&](uint32_t i) { for (++i; i <= n; i += i & (0u - i)) ++fen[i]; };
    auto fen_sum = [&](uint32_t i) {              // stores at slots < i
      uint32_t r = 0;
      for (; i > 0; i -= i & (0u - i)) r += fen[i];
      return r;
    };
    for (uint32_t t = 0; t < n; ++t)
      if (gates[order[t]].held) fen_add(t);
    for (uint32_t t = 0; t < n; ++t) {
      slots[t].lwait = slots[t].rwait = NONE;
      slots[t].store = NONE;
    }
    auto in_store = [&](uint32_t v) { return v < n_in || held(v) || spill[v]; };
    struct Prev { uint32_t v, lastread, written; bool stored; uint8_t used; };
    // A buffer for slot t: for a fill (the gate's missing operand) or for the gate's output.
    // Fill victims prefer "cold" buffers -- last read and written >= `look` slots before t --
    // so the fill's conditions hold `look` slots before its consumer: free, then dead, then the
    // value used furthest in the future (Belady), cold before warm.  Output buffers: a value
    // dying at t (an operand read for the last time, or dead), then free, then Belady.
    auto take = [&](uint32_t t, uint32_t avoid_a, uint32_t avoid_b, bool for_fill) -> std::pair<uint32_t, Prev> {
      uint32_t best = NONE, best_cls = 0xFF;
      uint64_t best_key = 0;
      for (uint32_t b = 0; b < n_buf; ++b) {
        const uint32_t v = occ[b];
        if (v != NONE && (v == avoid_a || v == avoid_b)) continue;
        const uint32_t u = v == NONE ? NONE : next_use(v, t + 1);
        uint32_t cls;
        uint64_t key;                                   // larger is better within a class
        if (for_fill) {
          cls = v == NONE ? 0 : (u == NONE ? 1 : 2);
          const bool cold = (b_lastread[b] == NONE || b_lastread[b] + look <= t) &&
                            (b_written[b] == NONE || b_written[b] + look <= t);
          if (!cold) cls += 3;
        } else {
          cls = v == NONE ? 1 : (u == NONE ? 0 : 2);
        }
        if (v == NONE) key = 0xFFFFFFFFull - (b_written[b] == NONE ? 0 : b_written[b] + 1ull);   // oldest
        else key = u == NONE ? 0 : u;                                                           // furthest
        if (cls < best_cls || (cls == best_cls && key > best_key)) best = b, best_cls = cls, best_key = key;
      }
      if (best == NONE) return {NONE, Prev{}};
      Prev pv{occ[best], b_lastread[best], b_written[best], false, b_used[best]};
      if (pv.v != NONE) {
        const uint32_t u = next_use(pv.v, t + 1);
        if (u != NONE && !in_store(pv.v)) {           // stored at its producer's epilogue
          spill[pv.v] = 1;
          fen_add(produced_at(pv.v));
        }
        pv.stored = pv.v >= n_in && (held(pv.v) || spill[pv.v]) && res_prod[pv.v] != NONE;
        vbuf[pv.v] = NONE;
        occ[best] = NONE;
      }
      return {best, pv};
    };
    auto issue_fill = [&](uint32_t v, uint32_t t, uint32_t other) -> bool {
      auto [b, pv] = take(t, v, other, true);
      if (b == NONE) return fail("regfile: no buffer for a fill at slot " + std::to_string(t));
      fhegpu_rf_fill f{};
      f.buf = b;
      f.consumer = t;
      f.w_built = pv.lastread == NONE ? 0 : pv.lastread + 1;
      f.w_epi = pv.written == NONE ? 0 : pv.written + 1;
      f.w_st = pv.stored ? res_prod[pv.v] + 1 : 0;
      if (v >= n_in && spill[v]) f.w_st = std::max(f.w_st, produced_at(v) + 1);
      const uint32_t fid = (uint32_t)fills.size();
      if (fid >= RF_FILL_RING) f.w_built = std::max(f.w_built, fills[fid - RF_FILL_RING].consumer + 1);
      f.flags = b_used[b] ? 0 : FF_FIRST;
      f.src = v;                                   // value id: resolved to a store location later
      fills.push_back(f);
      occ[b] = v, vbuf[v] = b, b_used[b] = 1;
      b_lastread[b] = NONE, b_written[b] = NONE, b_filled[b] = 1;
      res_prod[v] = NONE;
      pend_fill[v] = fid;
      last_fill_consumer[v] = t;
      return true;
    };
    for (uint32_t t = 0; t < n; ++t) {
      const uint32_t g = order[t];
      const fhegpu_rf_gate &gt = gates[g];
      if (vbuf[gt.left] == NONE && !issue_fill(gt.left, t, gt.right)) return false;
      if (vbuf[gt.right] == NONE && !issue_fill(gt.right, t, gt.left)) return false;
      fhegpu_rf_slot &s = slots[t];
      s.bits = (uint8_t)(gt.flags & 3u);
      if (t >= 2) {
        const fhegpu_rf_gate &g2 = gates[order[t - 2]];
        if (g2.left == gt.left && ((g2.flags ^ gt.flags) & 1u) == 0) s.bits |= SB_REUSE_L, ++n_reuse_l;
        if (g2.right == gt.right && ((g2.flags ^ gt.flags) & 2u) == 0) s.bits |= SB_REUSE_R, ++n_reuse_r;
      }
      for (int side = 0; side < 2; ++side) {
        const uint32_t v = side ? gt.right : gt.left;
        const uint32_t b = vbuf[v];
        if (b == NONE) return fail("regfile: operand not resident (internal)");
        uint32_t w = NONE;
        if (pend_fill[v] != NONE) w = WAIT_FILL | pend_fill[v];
        else if (res_prod[v] != NONE && t - res_prod[v] < RF_NEAR) w = res_prod[v];
        (side ? s.rbuf : s.lbuf) = (uint8_t)b;
        (side ? s.rwait : s.lwait) = w;
        b_lastread[b] = t;
      }
      pend_fill[gt.left] = pend_fill[gt.right] = NONE;
      // destination
      const uint32_t o = n_in + g;
      auto r = take(t, NONE, NONE, false);
      const uint32_t db = r.first;
      const Prev pv = r.second;
      if (db == NONE) return fail("regfile: no destination buffer at slot " + std::to_string(t));
      if (pv.stored) {
        const uint32_t p = res_prod[pv.v];
        if (p + 1 == t) s.bits |= SB_DEST_STORED | SB_HAZARD;
        else if (t < 5 || p + 1 > t - 4 || fen_sum(t - 3) - fen_sum(p + 1) == 0) s.bits |= SB_DEST_STORED;
      }
      if (!b_used[db]) s.bits |= SB_DEST_FIRST;
      s.dbuf = (uint8_t)db;
      occ[db] = o, vbuf[o] = db, b_used[db] = 1;
      b_lastread[db] = NONE, b_written[db] = t, b_filled[db] = 0;
      res_prod[o] = t;
    }
    // stores: program outputs to their slots, spilled values to spill slots (interval colouring)
    std::vector<std::pair<uint32_t, uint32_t>> iv;   // (producer slot, value)
    for (uint32_t v = n_in; v < V; ++v)
      if (spill[v]) iv.emplace_back(pos[v - n_in], v);
    std::sort(iv.begin(), iv.end());
    std::vector<uint32_t> spill_of(V, NONE);
    std::priority_queue<std::pair<uint32_t, uint32_t>, std::vector<std::pair<uint32_t, uint32_t>>,
                        std::greater<std::pair<uint32_t, uint32_t>>> busy;   // (end, spill slot)
    std::vector<uint32_t> free_sp;
    n_spill = 0;
    for (auto [p, v] : iv) {
      while (!busy.empty() && busy.top().first < p) free_sp.push_back(busy.top().second), busy.pop();
      uint32_t k;
      if (!free_sp.empty()) k = free_sp.back(), free_sp.pop_back();
      else k = n_spill++;
      spill_of[v] = k;
      busy.emplace(last_fill_consumer[v] == NONE ? p : last_fill_consumer[v], k);
    }
    n_stores = 0;
    for (uint32_t t = 0; t < n; ++t) {
      const uint32_t v = n_in + order[t];
      if (held(v)) slots[t].store = gates[order[t]].out_slot, slots[t].bits |= SB_STORE, ++n_stores;
      else if (spill[v]) slots[t].store = STORE_SPILL | spill_of[v], slots[t].bits |= SB_STORE, ++n_stores;
    }
    for (auto &f : fills) {
      const uint32_t v = f.src;
      if (v < n_in) f.src = in_slots[v];
      else if (held(v)) f.src = gates[v - n_in].out_slot;
      else f.src = STORE_SPILL | spill_of[v];
    }
    return true;
  }

  bool fail(const std::string &m) {
    err = m;
    return false;
  }

  bool run() {
    if (n_buf < 4 || n_buf > 255) return fail("regfile: 4 <= n_buf <= 255");
    if (n == 0) return fail("regfile: empty program");
    return schedule() && allocate();
  }
};

}  // namespace rf
}  // namespace fhegpu
