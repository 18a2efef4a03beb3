// k_ledger.cu -- reward events -> staleness ledger (DESIGN.md §3.1 W8-W9, §3.3), external
// Consume, metric reduction and dump kernels.
//
// One warp per scenario.  Reward events of the window are put in (t_reward, trajectory id)
// order with a warp rank sort (keys t_complete + R, id), then applied in that order: mark the
// member; once the whole GRPO group is rewarded delete its Reserved entry and cascade
// earlier Reserved entries into the hole, then Occupy the earliest empty slot
// (P:366).  Slot searches are warp ballots over 32 slots at a time.
#pragma once
#include <cassert>
#include "sf_internal.cuh"

namespace sf {

#ifndef SF_LEDGER_WARPS
#define SF_LEDGER_WARPS 4
#endif
constexpr int kLedgerWarps = SF_LEDGER_WARPS;

__device__ __forceinline__ long long ring_base(const ScenConst &C, int B, int b) {
  return C.led_off + (long long)(b % (C.eta + 1)) * B;
}

// lowest slot index in [0, B) of ring buffer b satisfying pred (warp ballot), or -1
template <typename Pred>
__device__ __forceinline__ int first_slot(int B, Pred pred) {
  for (int s0 = 0; s0 < B; s0 += 32) {
    const int sl = s0 + (int)lane_id();
    const bool h = sl < B && pred(sl);
    const unsigned m = __ballot_sync(0xffffffffu, h);
    if (m) return s0 + __ffs(m) - 1;
  }
  return -1;
}

// Lowest Empty slot of ring r (-1 if none), from the Empty-slot bitmap: one load per 32 words.
__device__ __forceinline__ int first_empty(const GParams &P, const Dev &D, const ScenConst &C, int r) {
  const int bw = (P.B + 31) >> 5;
  const unsigned *e = D.led_emp + (long long)(C.ring_off + r) * bw;
  for (int w0 = 0; w0 < bw; w0 += 32) {
    const int w = w0 + (int)lane_id();
    unsigned word = w < bw ? e[w] : 0u;
    if (w == bw - 1 && (P.B & 31)) word &= (1u << (P.B & 31)) - 1u;
    const unsigned m = __ballot_sync(0xffffffffu, word != 0u);
    if (m) {
      const int l = __ffs(m) - 1;
      return ((w0 + l) << 5) + __ffs(__shfl_sync(0xffffffffu, word, l)) - 1;
    }
  }
  return -1;
}

// Remove group g's Reserved entry at its ledger position and run the delete-and-relocate
// cascade (reading A13); (hb, hs) returns the final hole.
static __device__ void delete_relocate(const GParams &P, const Dev &D, const ScenConst &C, int g, int cu, int &hb,
                                       int &hs, long long &m_reloc, int &err) {
  const unsigned lane = lane_id();
  const int B = P.B, eta = C.eta;
  hb = D.led_b[C.grp_off + g];
  hs = D.led_s[C.grp_off + g];
  {
    const long long base = ring_base(C, B, hb);
    if (D.led_st[base + hs] != E_RESERVED || D.led_g[base + hs] != g) { err = ERR_LEDGER; return; }
    __syncwarp();
    if (lane == 0) {
      D.led_st[base + hs] = E_EMPTY; D.led_g[base + hs] = -1; D.led_v[base + hs] = -1;
      emp_mark(P, D, C, hb % (eta + 1), hs, true);
      D.led_nres[C.ring_off + hb % (eta + 1)] -= 1;
    }
    __syncwarp();
  }
  for (;;) {
    int fb = -1, fs = -1;
    for (int bb = cu; bb < hb; ++bb) {
      if (D.led_nres[C.ring_off + bb % (eta + 1)] == 0) continue;
      const long long base = ring_base(C, B, bb);
      const int hole = hb;
      const int sl = first_slot(B, [&](int x) {        // both loads issued together (bitwise &)
        return (D.led_st[base + x] == E_RESERVED) & (D.led_v[base + x] + eta >= hole);
      });
      if (sl >= 0) { fb = bb; fs = sl; break; }
    }
    if (fb < 0) break;
    const long long src = ring_base(C, B, fb) + fs, dst = ring_base(C, B, hb) + hs;
    const int mg = D.led_g[src], mv = D.led_v[src];
    __syncwarp();
    if (lane == 0) {
      D.led_st[dst] = E_RESERVED; D.led_g[dst] = mg; D.led_v[dst] = mv;
      D.led_st[src] = E_EMPTY; D.led_g[src] = -1; D.led_v[src] = -1;
      emp_mark(P, D, C, hb % (eta + 1), hs, false);
      emp_mark(P, D, C, fb % (eta + 1), fs, true);
      D.led_nres[C.ring_off + hb % (eta + 1)] += 1;
      D.led_nres[C.ring_off + fb % (eta + 1)] -= 1;
      D.led_b[C.grp_off + mg] = hb;
      D.led_s[C.grp_off + mg] = hs;
    }
    __syncwarp();
    hb = fb;
    hs = fs;
    ++m_reloc;
  }
}

static __device__ void complete_group(const GParams &P, const Dev &D, const ScenConst &C, ScenState &SS, int g, int cu,
                               long long &m_reloc, long long &m_occ, int &err) {
  const unsigned lane = lane_id();
  const int B = P.B, eta = C.eta;
  const int vg = D.gv[C.grp_off + g];
  int hb, hs;
  delete_relocate(P, D, C, g, cu, hb, hs, m_reloc, err);
  if (err) return;
  // Occupy: earliest buffer >= cu with an empty slot, lowest slot
  int ob = -1, os = -1;
  for (int b = cu; b <= cu + eta; ++b) {
    const int r = C.ring_off + b % (eta + 1);
    if (B - D.led_nres[r] - D.led_nocc[r] <= 0) continue;
    os = first_empty(P, D, C, b % (eta + 1));
    if (os >= 0) { ob = b; break; }
  }
  if (ob < 0) { err = ERR_LEDGER; return; }
  if (ob < vg || ob > vg + eta) { err = ERR_STALENESS; atomicAdd(&SS.m[M_VIOLATIONS], lane == 0 ? 1ULL : 0ULL); }
  __syncwarp();
  if (lane == 0) {
    const long long dst = ring_base(C, B, ob) + os;
    D.led_st[dst] = E_OCCUPIED; D.led_g[dst] = g; D.led_v[dst] = vg;
    emp_mark(P, D, C, ob % (eta + 1), os, false);
    D.led_nocc[C.ring_off + ob % (eta + 1)] += 1;
    D.led_b[C.grp_off + g] = ob;
    D.led_s[C.grp_off + g] = os;
  }
  __syncwarp();
  ++m_occ;
}

// Filtering (P:413 (2), reading R-FILTER): the hole at (hb, hs) takes the Occupied entry of the
// earliest later buffer (lowest slot) with version <= hb, repeated with the hole each move leaves.
static __device__ void fill_forward(const GParams &P, const Dev &D, const ScenConst &C, int cu, int hb, int hs,
                                    long long &m_reloc) {
  const unsigned lane = lane_id();
  const int B = P.B, eta = C.eta;
  for (;;) {
    int fb = -1, fs = -1;
    for (int bb = hb + 1; bb <= cu + eta; ++bb) {
      if (D.led_nocc[C.ring_off + bb % (eta + 1)] == 0) continue;
      const long long base = ring_base(C, B, bb);
      const int hole = hb;
      const int sl = first_slot(B, [&](int x) { return (D.led_st[base + x] == E_OCCUPIED) & (D.led_v[base + x] <= hole); });
      if (sl >= 0) { fb = bb; fs = sl; break; }
    }
    if (fb < 0) break;
    const long long src = ring_base(C, B, fb) + fs, dst = ring_base(C, B, hb) + hs;
    const int mg = D.led_g[src], mv = D.led_v[src];
    __syncwarp();
    if (lane == 0) {
      D.led_st[dst] = E_OCCUPIED; D.led_g[dst] = mg; D.led_v[dst] = mv;
      D.led_st[src] = E_EMPTY; D.led_g[src] = -1; D.led_v[src] = -1;
      emp_mark(P, D, C, hb % (eta + 1), hs, false);
      emp_mark(P, D, C, fb % (eta + 1), fs, true);
      D.led_nocc[C.ring_off + hb % (eta + 1)] += 1;
      D.led_nocc[C.ring_off + fb % (eta + 1)] -= 1;
      D.led_b[C.grp_off + mg] = hb;
      D.led_s[C.grp_off + mg] = hs;
    }
    __syncwarp();
    hb = fb;
    hs = fs;
    ++m_reloc;
  }
}

// Drop a tracked group (filtering, P:413 (2), reading R-FILTER): abort its ledger entry (Reserved:
// delete-and-relocate; Occupied: emptied), move later Occupied entries forward into the hole, and
// Abort every member not yet consumed; the group leaves the live-group count.
static __device__ void filter_group(const GParams &P, const Dev &D, const ScenConst &C, ScenState &SS, int g, int cu,
                                    CmdLog &cl, long long &m_reloc, int &err) {
  const unsigned lane = lane_id();
  int hb = D.led_b[C.grp_off + g], hs = D.led_s[C.grp_off + g];
  const long long at = ring_base(C, P.B, hb) + hs;
  if (D.led_st[at] == E_RESERVED) {
    delete_relocate(P, D, C, g, cu, hb, hs, m_reloc, err);
    if (err) return;
  } else {
    if (D.led_st[at] != E_OCCUPIED || D.led_g[at] != g) { err = ERR_LEDGER; return; }
    __syncwarp();
    if (lane == 0) {
      D.led_st[at] = E_EMPTY; D.led_g[at] = -1; D.led_v[at] = -1;
      emp_mark(P, D, C, hb % (C.eta + 1), hs, true);
      D.led_nocc[C.ring_off + hb % (C.eta + 1)] -= 1;
    }
    __syncwarp();
  }
  fill_forward(P, D, C, cu, hb, hs, m_reloc);
  for (int m = 0; m < P.G; ++m) abort_member(P, D, C, cl, g * P.G + m, true);
  if (lane == 0) {
    D.cvbuf[C.grp_off + g] = -2;                  // retired without consumption
    SS.live -= 1;
  }
  __syncwarp();
}

constexpr int kEvStage = 512;     // reward events staged per warp in shared memory (a power of two)

struct EvStage {
  long long t[kEvStage];
  int id[kEvStage];
  int ioff[kMaxInst + 1];         // start of each instance's events in the window's event order
};

// (t, id) < (t', id'): the order in which reward events reach the ledger (W8)
__device__ __forceinline__ bool ev_less(long long ta, int ia, long long tb, int ib) {
  return (ta < tb) | ((ta == tb) & (ia < ib));
}

// bitonic sort of n <= kEvStage staged events by (t, id), in shared memory (padded to a power of two
// with (+inf, +inf); keys are distinct); O(N log^2 N / 32) compare-exchanges per lane
__device__ __forceinline__ void ev_sort_smem(EvStage &es, int n) {
  int N = 1;
  while (N < n) N <<= 1;
  for (int e = n + (int)lane_id(); e < N; e += 32) { es.t[e] = 0x7fffffffffffffffLL; es.id[e] = 0x7fffffff; }
  __syncwarp();
  for (int k = 2; k <= N; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = lane_id(); i < N; i += 32) {
        const int p = i ^ j;
        if (p > i) {
          const long long ta = es.t[i], tb = es.t[p];
          const int ia = es.id[i], ib = es.id[p];
          const bool up = (i & k) == 0;
          if (ev_less(tb, ib, ta, ia) == up) { es.t[i] = tb; es.t[p] = ta; es.id[i] = ib; es.id[p] = ia; }
        }
      }
      __syncwarp();
    }
}

// the same network over event ids in global scratch (n > kEvStage, rare), keyed by
// (D.t_complete[id], id); padding ids are -1 (= +inf)
__device__ __forceinline__ void ev_sort_global(const Dev &D, const ScenConst &C, int *ids, int n) {
  int N = 1;
  while (N < n) N <<= 1;
  for (int e = n + (int)lane_id(); e < N; e += 32) ids[e] = -1;
  __syncwarp();
  auto key_t = [&](int id) { return id < 0 ? 0x7fffffffffffffffLL : D.t_complete[C.traj_off + id]; };
  for (int k = 2; k <= N; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = lane_id(); i < N; i += 32) {
        const int p = i ^ j;
        if (p > i) {
          const int ia = ids[i], ib = ids[p];
          const long long ta = key_t(ia), tb = key_t(ib);
          const bool up = (i & k) == 0;
          const bool b_lt_a = ev_less(tb, ib < 0 ? 0x7fffffff : ib, ta, ia < 0 ? 0x7fffffff : ia);
          if (b_lt_a == up) { ids[i] = ib; ids[p] = ia; }
        }
      }
      __syncwarp();
    }
}

// One window of W8-W9 for scenario s, executed by one warp (es: that warp's staging).
// C = D.sc[s] (passed in, loaded by the caller before its wait).
__device__ __forceinline__ void ledger_scenario(const GParams &P, const Dev &D, int s, EvStage &es, const ScenConst C) {
  const unsigned lane = lane_id();
  ScenState &SS = D.ss[s];
  const int err0 = SS.err;    // checked after the event-count loads below (reads + staging only)
  const long long t_end = SS.t + P.delta;
  // Pending reward events: the carry list D.ev_id[ev_off, ev_off + SS.ev_n) (not yet due in an
  // earlier window) followed by this window's completions in the instances' segments (D.iev,
  // written by k_advance without atomics), instance by instance.
  const int n_carry = SS.ev_n;
  int n = n_carry;
  for (int i0 = 0; i0 < C.I; i0 += 32) {
    const int i = i0 + (int)lane;
    const int ni = i < C.I ? D.iev_n[C.inst_off + i] : 0;
    const int off = n + warp_excl_scan(ni);
    if (i < C.I) es.ioff[i] = off;
    n = __shfl_sync(0xffffffffu, off + ni, 31);
  }
  if (lane == 0) es.ioff[C.I] = n;
  __syncwarp();
  if (err0) return;
  auto seg_of = [&](int e) {                      // instance whose segment holds event e >= n_carry
    int lo = 0, hi = C.I - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (es.ioff[mid] <= e) lo = mid; else hi = mid - 1;
    }
    return lo;
  };
  const bool big = n > kEvStage;                  // rare: the events do not fit the staging
  int *gids = D.mlq + C.mlq_off;                  // big: ids sorted in the MLQ scratch (>= 3 cap ints)
  for (int e = lane; e < n; e += 32) {
    int id;
    if (e < n_carry) id = D.ev_id[C.ev_off + e];
    else { const int i = seg_of(e); id = D.iev[C.list_off + (long long)i * C.cap + (e - es.ioff[i])]; }
    if (big) gids[e] = id;
    else { es.id[e] = id; es.t[e] = D.t_complete[C.traj_off + id]; }
  }
  __syncwarp();
  for (int i = lane; i < C.I; i += 32) D.iev_n[C.inst_off + i] = 0;
#ifdef SF_CHECK
  assert(n >= 0 && n <= C.cap);
#endif
  const int cu = SS.cu;
  int err = 0;
  long long m_reloc = 0, m_occ = 0;
  CmdLog cl{SS.cmd_hash, SS.cmd_n, SS.window, 0};
  int np = 0;
  // sort by (t_reward, id) = (t_complete + R, id) (W8)
  if (big) ev_sort_global(D, C, gids, n);
  else ev_sort_smem(es, n);
  auto ev_id = [&](int k) { return big ? gids[k] : es.id[k]; };
  // apply in order, 32 events per batch: the members' reward counters are loaded in parallel and
  // same-group events inside a batch are counted with __match_any_sync
  for (int k0 = 0; k0 < n; k0 += 32) {
    const int k = k0 + (int)lane;
    const bool valid = k < n;
    const int id = valid ? ev_id(k) : 0;
    const long long te = valid ? (big ? D.t_complete[C.traj_off + id] : es.t[k]) : 0;
    const bool ok = valid && te + P.R <= t_end;
    const int g = grp_of(P, id);
    const unsigned okm = __ballot_sync(0xffffffffu, ok);
    // redundancy: the reward of an aborted member is ignored, and inside this batch the
    // members of a group past its Gr-th reward are aborted when the group completes
    bool eff = ok;
    if (P.abortable && ok) eff = D.loc[C.traj_off + id] != L_ABORTED;
    const int nrw = eff ? D.n_rew[C.grp_off + g] : 0;
    const unsigned same = __match_any_sync(0xffffffffu, eff ? g : -1 - (int)lane);
    const int nr = nrw + 1 + __popc(same & lanemask_lt());
    if (eff && (same >> lane) == 1u) D.n_rew[C.grp_off + g] = min(nrw + __popc(same), P.Gr);   // last of its group
    if (P.red && eff && nr <= P.Gr) D.loc[C.traj_off + id] = L_REWARDED;
    unsigned cm = __ballot_sync(0xffffffffu, eff && nr == P.Gr);
    __syncwarp();
    while (cm) {
      const int l = __ffs(cm) - 1;
      cm &= cm - 1;
      const int gc = __shfl_sync(0xffffffffu, g, l);
      if (P.red)                                      // group-level redundancy: Abort the others
        for (int m = 0; m < P.G; ++m) abort_member(P, D, C, cl, gc * P.G + m);
      if (P.filt && D.gfilt[C.grp_off + gc]) filter_group(P, D, C, SS, gc, cu, cl, m_reloc, err);
      else complete_group(P, D, C, SS, gc, cu, m_reloc, m_occ, err);
      if (err) break;
    }
    np += __popc(okm);
    if (err || okm != __ballot_sync(0xffffffffu, valid)) break;   // sorted: the rest are later
  }
  __syncwarp();
  // the events not yet due are carried to the next window, in order
  for (int k = np + (int)lane; k < n; k += 32) D.ev_id[C.ev_off + k - np] = ev_id(k);
  __syncwarp();
  // Deadlock watchdog (the oracle's rule, DESIGN.md §4 R-WATCHDOG): no progress in this
  // window (cumulative progress metrics unchanged), nothing pending at its end, groups unconsumed
  if (P.wd > 0 && P.atw > 0 && !err) {
    bool pend = false;
    for (int i = lane; i < C.I; i += 32) {
      const long long gi = C.inst_off + i;
      pend |= D.ist[gi] != I_IDLE || D.ipullpend[gi] != 0 || D.iintkind[gi] != INT_NONE || D.iabort[gi] != 0 ||
              D.iarr_n[gi] != 0;
    }
    pend = __any_sync(0xffffffffu, pend) || SS.trainer_busy || n - np > 0;
    const long long sig = (long long)(SS.m[M_TICKS] + SS.m[M_ROUTES] + SS.m[M_INTERRUPTS] + SS.m[M_PULLS] +
                                      SS.m[M_COMPLETIONS] + SS.m[M_OCCUPIED] + m_occ + SS.m[M_BATCHES] +
                                      SS.m[M_PUBLISHES] + SS.m[M_INGESTED] + SS.m[M_ABORTS] + cl.aborts);
    const bool work_left = SS.live > 0 || SS.n_ingested < SS.n_pool;
    __syncwarp();
    if (lane == 0) {
      if (sig == SS.wd_sig && !pend && work_left) {
        if (++SS.wd_idle >= P.wd) err = ERR_DEADLOCK;
      } else {
        SS.wd_idle = 0;
      }
      SS.wd_sig = sig;
    }
    err = __shfl_sync(0xffffffffu, err, 0);
  }
  if (lane == 0) {
    SS.ev_n = n - np;
    SS.cmd_hash = cl.hash; SS.cmd_n = cl.cmd_n;
    SS.t = t_end;                                       // W9
    SS.window += 1;
    if (err) SS.err = err;
    metric_add(SS, M_WINDOWS, 1);
    metric_add(SS, M_RELOCATIONS, m_reloc);
    metric_add(SS, M_OCCUPIED, m_occ);
    metric_add(SS, M_ABORTS, cl.aborts);
  }
}

}  // namespace sf
