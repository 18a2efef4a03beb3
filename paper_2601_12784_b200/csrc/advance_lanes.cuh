// advance_lanes.cuh -- decode advance with one LANE per rollout instance (
// §3.1 W6-W7, boundary procedure §3.2 B1-B8).
//
// A warp advances 32 consecutive instances (one per lane) through the window.  Each instance is an
// independent little state machine (W7), so the natural B200 mapping for thousands of small
// instances is one per thread: a lane walks its instance boundary by boundary while the warp's
// other lanes walk theirs.  The instance's run slots live in shared memory in a padded
// slot-major layout (row s = slot s of all 32 lanes, stride 33: rows and columns are
// bank-conflict free), four int32 columns per slot:
//   done  -- the window-relative decode-step count at whose end the slot's trajectory completes
//            (tc + remaining at admission; the slot's remaining length is done - tc), -1 dead,
//            <= -2: completed at boundary -2-done of this window (event not yet emitted)
//   fin   -- p + T (context at completion), rid -- trajectory id, rT -- target T
// so a decode step is a scalar update per lane (tc += 1, kv += k5 n, next step time), and a
// completion test is "tc == min_done" -- no per-slot work on a quiet step.  Slots are appended in
// admission order (LIFO preemption takes the highest live slot) and compacted back into the
// instance's HBM run list at the window end.  Completion events are emitted at the window end (or
// when kCB completion boundaries have accumulated); the ledger sorts events by (t, id), so their
// order in the segment is irrelevant.  Instances whose run + wait + arrivals exceed kLS take the
// warp-per-instance path of advance.cuh after the lane loop.
#pragma once
#include "advance.cuh"

namespace sf {

#ifndef SF_LANES
#define SF_LANES 8                     // measured on C5: 8 -> 121.9, 16 -> 113.9, 32 -> 102.7 G/s
#endif
constexpr int kLanes = SF_LANES;       // instances per warp (lanes kLanes..31 help in the cooperative
                                       // passes only): fewer than 32 leaves more warps per scheduler
constexpr int kLS = 84;                // run slots per lane (instance) in shared memory
constexpr int kLP = kLanes + 1;        // padded row stride (odd: rows and columns conflict free)
constexpr int kAS = 8;                 // staged arrivals per lane
constexpr int kCB = 8;                 // completion boundaries buffered per lane before an emit
constexpr int kDeadSlot = -1;

struct LaneSmem {
  int done[kLS * kLP];
  int fin[kLS * kLP];
  int rid[kLS * kLP];
  int rT[kLS * kLP];
  long long cb_t[kCB * kLanes];        // completion boundary times (lane-major per index)
  long long a_t[kAS * kLanes];         // delivery window (B6): t_arr, id of arrivals [a_base, +kAS)
  int a_id[kAS * kLanes];
  int b_id[kAS * kLanes], b_ctx[kAS * kLanes], b_T[kAS * kLanes], b_gen[kAS * kLanes];   // admission window (B7)
  int mind[32];                        // per-lane min live done at window start
};

struct LaneInst {
  // instance state (as InstState) + lane bookkeeping
  int st, pullv, pullpend, intkind, intk, cc, v, whead, wn, arr_n, arr_head, abortn, abortarr, evn;
  long long nb, until, kv, prefill, t_cmd;
  long long ticks, iters, tokens;
  int comps, preempts;
  int nlive, tail, tc, min_done, run_n0, ncb, a_base, b_base, arr_ring0;
  bool blocked, head_ok;
  int head_id, head_gen, head_T, head_ctx;
  int cn_n;
  long long cn;
  long long cur_b;                     // the boundary being processed (between the two phases)
  bool cur_tick, cur_pull, need_scan;
  int sc_cnt, sc_min;                  // cooperative completion scan result for this lane
  long long sc_rel;
#ifdef SF_TIMING
  int n_stage, n_headld;               // arrival-window refills, wait heads read from HBM
#endif
};

#define LS_AT(arr, s) (arr)[(s) * kLP + (int)lane_id()]

// delivery window: (t_arr, id) of arrivals [k0, k0 + kAS) of this lane's instance (one HBM round trip)
__device__ __forceinline__ void lane_stage_arrivals(const GParams &P, const Dev &D, const ScenConst &C, long long lb,
                                                    LaneInst &x, LaneSmem &sm, int k0) {
  const int lane = (int)lane_id();
  x.a_base = k0;
#ifdef SF_TIMING
  ++x.n_stage;
#endif
#pragma unroll
  for (int a = 0; a < kAS; ++a) {
    const int k = k0 + a;
    long long t = kInf;
    int id = 0;
    if (k < x.arr_n) { t = D.arr_t[lb + k]; id = D.arr_id[lb + k]; }
    sm.a_t[a * kLanes + lane] = t;
    sm.a_id[a * kLanes + lane] = id;
  }
}

// admission window: (id, gen, T, p + gen) of arrivals [k0, k0 + kAS) (two HBM round trips for kAS
// admissions instead of two per admission)
__device__ __forceinline__ void lane_stage_admissions(const GParams &P, const Dev &D, const ScenConst &C, long long lb,
                                                      LaneInst &x, LaneSmem &sm, int k0) {
  const int lane = (int)lane_id();
  x.b_base = k0;
#ifdef SF_TIMING
  ++x.n_stage;
#endif
  int ids[kAS];
#pragma unroll
  for (int a = 0; a < kAS; ++a) ids[a] = k0 + a < x.arr_n ? D.arr_id[lb + k0 + a] : -1;
#pragma unroll
  for (int a = 0; a < kAS; ++a) {
    int g = 0, T = 0, p = 0;
    if (ids[a] >= 0) {
      const long long j = C.traj_off + ids[a];
      g = D.gen[j]; T = D.T[j]; p = D.prompt[C.grp_off + grp_of(P, ids[a])];
    }
    sm.b_id[a * kLanes + lane] = ids[a];
    sm.b_gen[a * kLanes + lane] = g;
    sm.b_T[a * kLanes + lane] = T;
    sm.b_ctx[a * kLanes + lane] = p + g;
  }
}

__device__ __forceinline__ long long lane_arr_time(const GParams &P, const Dev &D, const ScenConst &C, long long lb,
                                                   LaneInst &x, LaneSmem &sm, int k) {
  if (k >= x.arr_n) return kInf;
  if (k >= x.a_base + kAS) lane_stage_arrivals(P, D, C, lb, x, sm, k);
  return sm.a_t[(k - x.a_base) * kLanes + (int)lane_id()];
}

// emit the completion events buffered in the lane's slots (D.gen, D.loc, D.t_complete, event
// segment), making those slots dead
__device__ __forceinline__ void lane_emit_events(const Dev &D, const ScenConst &C, long long lb, LaneInst &x,
                                                 LaneSmem &sm) {
  if (x.ncb == 0) return;
  const int lane = (int)lane_id();
  for (int s = 0; s < x.tail; ++s) {
    const int d = LS_AT(sm.done, s);
    if (d <= -2) {
      const int id = LS_AT(sm.rid, s);
      const long long j = C.traj_off + id;
      D.gen[j] = LS_AT(sm.rT, s);
      D.loc[j] = L_DONE;
      D.t_complete[j] = sm.cb_t[(-2 - d) * kLanes + lane];      // reward due at b + R
      D.iev[lb + x.evn] = id;
      ++x.evn;
      LS_AT(sm.done, s) = kDeadSlot;
    }
  }
  x.ncb = 0;
}

__device__ __forceinline__ int lane_min_done(const LaneInst &x, const LaneSmem &sm) {
  int m = 0x7fffffff;
  for (int s = 0; s < x.tail; ++s) {
    const int d = LS_AT(sm.done, s);
    if (d >= 0) m = min(m, d);
  }
  return m;
}

// one boundary of this lane's instance at time b (B1-B8; the order and effects of
// advance_reg in advance.cuh, with slots in shared memory), in two phases around the warp's
// cooperative completion scan: phase A = B1 and the start of B2 (returns in x.need_scan whether
// slots complete at this step), phase B = the rest.
__device__ __forceinline__ void lane_boundary_a(const GParams &P, const Dev &D, const ScenConst &C, long long lb,
                                                LaneInst &x, LaneSmem &sm, long long b) {
  const int cap = C.cap;
  const long long k5 = P.k5;
  x.t_cmd = kInf;
  x.cur_b = b;
  const bool tick_end = (x.st == I_TICK);
  const bool pull_done = (x.st == I_PULL);
  x.cur_tick = tick_end;
  x.cur_pull = pull_done;
  x.need_scan = false;
  // B1: pending interrupts leave without this step's token; KV released (A17, A18)
  if (!pull_done && x.intkind != INT_NONE) {
    if (x.intkind == INT_ALL) {
      for (int s = 0; s < x.tail; ++s)
        if (LS_AT(sm.done, s) >= 0) LS_AT(sm.done, s) = kDeadSlot;
      x.nlive = 0; x.wn = 0; x.kv = 0; x.min_done = 0x7fffffff;
    } else {
      x.wn -= x.intk;                                    // wait tail (A7)
    }
    if (x.wn == 0) x.head_ok = false;
    x.blocked = false;
    x.intkind = INT_NONE;
  }
  // B1 (Abort): aborted run / wait members leave for good, their KV released (reading R-ABORT)
  if (x.abortn > 0) {
    long long release = 0;
    int nab = 0;
    for (int s = 0; s < x.tail; ++s) {
      const int d = LS_AT(sm.done, s);
      if (d < 0) continue;
      const int id = LS_AT(sm.rid, s);
      if (D.loc[C.traj_off + id] == L_ABORTED) {
        const int rem = d - x.tc;
        release += k5 * (long long)(LS_AT(sm.fin, s) - rem);          // p + gen
        D.gen[C.traj_off + id] = LS_AT(sm.rT, s) - rem;                // progress kept
        LS_AT(sm.done, s) = kDeadSlot;
        ++nab;
      }
    }
    if (nab) {
      x.kv -= release;
      x.nlive -= nab;
      x.min_done = lane_min_done(x, sm);
    }
    // wait ring: drop aborted members, FIFO order kept
    int out = 0;
    for (int k = 0; k < x.wn; ++k) {
      int pos = x.whead + k;
      if (pos >= cap) pos -= cap;
      const int id = D.wait_id[lb + pos];
      if (D.loc[C.traj_off + id] != L_ABORTED) {
        int o = x.whead + out;
        if (o >= cap) o -= cap;
        D.wait_id[lb + o] = id;
        ++out;
      }
    }
    x.wn = out;
    x.abortn = 0;
    x.head_ok = false;
    x.blocked = false;
    x.arr_ring0 = -1;                                    // ring positions moved: stop mapping arrivals
  }
  if (tick_end) {
    // B2: one token for every running trajectory; B3's completions are the slots due at this step
    x.tc += 1;
    x.kv += k5 * x.nlive;
    x.tokens += x.nlive;
    if (x.tc == x.min_done) {
      if (x.ncb == kCB) lane_emit_events(D, C, lb, x, sm);
      x.need_scan = true;
    }
  }
}

// the warp scans the slot columns of every lane that has completions at its current step: mark
// the due slots completed (boundary index ncb), sum their released KV, count them, and find the
// new earliest completion among the rest
__device__ __forceinline__ void lanes_complete_scan(const GParams &P, LaneInst &x, LaneSmem &sm) {
  const int lane = (int)lane_id();
  unsigned m = __ballot_sync(0xffffffffu, x.need_scan);
  while (m) {
    const int l = __ffs(m) - 1;
    m &= m - 1;
    const int tcl = __shfl_sync(0xffffffffu, x.tc, l);
    const int tl = __shfl_sync(0xffffffffu, x.tail, l);
    const int mark = -2 - __shfl_sync(0xffffffffu, x.ncb, l);
    long long rel = 0;
    int cnt = 0, mn = 0x7fffffff;
#pragma unroll
    for (int c = 0; c < (kLS + 31) / 32; ++c) {
      const int sl = c * 32 + lane;
      const int d = sl < tl ? sm.done[sl * kLP + l] : kDeadSlot;
      const bool hit = d == tcl;
      if (hit) {
        sm.done[sl * kLP + l] = mark;
        rel += (long long)sm.fin[sl * kLP + l];
      }
      if (d >= 0 && !hit) mn = min(mn, d);
      cnt += __popc(__ballot_sync(0xffffffffu, hit));
    }
    rel = warp_sum(rel);
    mn = warp_min(mn);
    if (lane == l) { x.sc_rel = rel * P.k5; x.sc_cnt = cnt; x.sc_min = mn; }
  }
  __syncwarp();
}

__device__ __forceinline__ void lane_boundary_b(const GParams &P, const Dev &D, const ScenConst &C, long long lb,
                                                LaneInst &x, LaneSmem &sm) {
  const int cap = C.cap;
  const long long k5 = P.k5;
  const long long b = x.cur_b;
  if (x.cur_tick) {
    if (x.need_scan) {
      sm.cb_t[x.ncb * kLanes + (int)lane_id()] = b;
      ++x.ncb;
      x.kv -= x.sc_rel;
      x.nlive -= x.sc_cnt;
      x.cc += x.sc_cnt;
      x.comps += x.sc_cnt;
      x.min_done = x.sc_min;
      x.blocked = false;
    }
    x.st = I_IDLE;
  } else if (x.cur_pull) {
    x.v = x.pullv; x.cc = 0; x.st = I_IDLE;
  }
  // B4: preemption while KV exceeds M: newest admitted (highest live slot) -> wait front (A21)
  if (x.kv > P.M) {
    while (x.kv > P.M && x.nlive > 0) {
      int s = x.tail - 1;
      while (LS_AT(sm.done, s) < 0) --s;
      const int d = LS_AT(sm.done, s);
      const int rem = d - x.tc;
      const int id = LS_AT(sm.rid, s);
      const int Tj = LS_AT(sm.rT, s);
      const long long j = C.traj_off + id;
      const int g_ = Tj - rem;
      const long long ctx = LS_AT(sm.fin, s) - rem;        // p + gen
      x.kv -= k5 * ctx;
      x.whead = x.whead == 0 ? cap - 1 : x.whead - 1;
      D.gen[j] = g_;
      D.loc[j] = L_WAIT;
      D.n_preempt[j] += 1;
      D.wait_id[lb + x.whead] = id;
      LS_AT(sm.done, s) = kDeadSlot;
      if (d == x.min_done) x.min_done = lane_min_done(x, sm);
      --x.nlive;
      ++x.wn;
      ++x.preempts;
      x.head_ok = true; x.head_id = id; x.head_gen = g_; x.head_T = Tj; x.head_ctx = (int)ctx;
      x.arr_ring0 = -1;        // the front push may reuse ring slots of admitted arrivals: stop mapping
    }
    x.blocked = true;                                     // the last victim (the head) cannot re-fit now
  }
  // B5: a pending Pull blocks generation for q
  if (x.pullpend) {
    x.pullpend = 0;
    x.st = I_PULL;
    x.until = b + P.q;
    return;
  }
  // B6: arrivals with t_arr <= b join the wait tail in (t_arr, id) order
  long long na = lane_arr_time(P, D, C, lb, x, sm, x.arr_head);
  if (na <= b) {
    if (x.wn == 0) { x.head_ok = false; x.blocked = false; }
    do {
      const int id = sm.a_id[(x.arr_head - x.a_base) * kLanes + (int)lane_id()];
      if (x.abortarr > 0 && D.loc[C.traj_off + id] == L_ABORTED) {   // aborted in transit: dropped
        --x.abortarr;
        x.arr_ring0 = -1;
      } else {
        int pos = x.whead + x.wn;
        if (pos >= cap) pos -= cap;
        if (x.arr_head == 0) x.arr_ring0 = pos;
        D.wait_id[lb + pos] = id;
        D.loc[C.traj_off + id] = L_WAIT;
        ++x.wn;
      }
      ++x.arr_head;
      na = lane_arr_time(P, D, C, lb, x, sm, x.arr_head);
    } while (na <= b);
  }
  // B7: FIFO admission while the head fits the KV budget
  if (x.wn > 0 && !x.blocked) {
    while (x.wn > 0) {
      if (!x.head_ok) {
        // the head is arrival k of this window when its ring position is arr_ring0 + k
        int k = -1;
        if (x.arr_ring0 >= 0) {
          k = x.whead - x.arr_ring0;
          if (k < 0) k += cap;
          if (k >= x.arr_head) k = -1;
        }
        if (k >= 0) {
          if (k < x.b_base || k >= x.b_base + kAS) lane_stage_admissions(P, D, C, lb, x, sm, k);
          const int o = (k - x.b_base) * kLanes + (int)lane_id();
          x.head_id = sm.b_id[o]; x.head_gen = sm.b_gen[o]; x.head_T = sm.b_T[o]; x.head_ctx = sm.b_ctx[o];
        } else {
#ifdef SF_TIMING
          ++x.n_headld;
#endif
          x.head_id = D.wait_id[lb + x.whead];
          const long long j = C.traj_off + x.head_id;
          x.head_gen = D.gen[j];
          x.head_T = D.T[j];
          x.head_ctx = D.prompt[C.grp_off + grp_of(P, x.head_id)] + x.head_gen;
        }
        x.head_ok = true;
      }
      if (x.kv + k5 * x.head_ctx > P.M) { x.blocked = true; break; }
      if (x.tail == kLS) {
        // compact the slots (completed-but-unemitted events first), order kept
        lane_emit_events(D, C, lb, x, sm);
        int o = 0;
        for (int s = 0; s < x.tail; ++s) {
          const int d = LS_AT(sm.done, s);
          if (d >= 0) {
            if (o != s) {
              LS_AT(sm.done, o) = d; LS_AT(sm.fin, o) = LS_AT(sm.fin, s);
              LS_AT(sm.rid, o) = LS_AT(sm.rid, s); LS_AT(sm.rT, o) = LS_AT(sm.rT, s);
            }
            ++o;
          }
        }
        x.tail = o;
        x.run_n0 = 0;                                     // the HBM list no longer mirrors the slots
      }
      const int s = x.tail++;
      const int dn = x.tc + (x.head_T - x.head_gen);
      LS_AT(sm.done, s) = dn;
      LS_AT(sm.fin, s) = x.head_ctx - x.head_gen + x.head_T;
      LS_AT(sm.rid, s) = x.head_id;
      LS_AT(sm.rT, s) = x.head_T;
      x.min_done = min(x.min_done, dn);
      D.loc[C.traj_off + x.head_id] = L_RUN;
      x.kv += k5 * x.head_ctx;
      x.prefill += x.head_ctx;
      ++x.nlive;
      x.whead = x.whead + 1 == cap ? 0 : x.whead + 1;
      --x.wn;
      x.head_ok = false;
    }
  }
  // B8: next decode step, Eq 7 + prefill stall (A20)
  if (x.nlive > 0) {
    if (x.nlive != x.cn_n) { x.cn_n = x.nlive; x.cn = max(P.k2, (long long)P.k3i * x.nlive) + P.k4; }
    x.nb = b + (long long)P.k1i * (int)x.kv + x.cn + (long long)P.kpi * (int)x.prefill;
    x.prefill = 0;
    x.st = I_TICK;
    x.iters += x.nlive;
    ++x.ticks;
  } else {
    x.st = I_IDLE;
  }
}

// One window of W6-W7 for the 32 instances gi0 + lane (lanes past n_inst_total idle).  Instances that
// do not fit kLS slots are advanced by the whole warp afterwards (advance_instance, advance.cuh).
__device__ __forceinline__ void advance_lanes(const GParams &P, const Dev &D, int gi0, int n_inst_total, LaneSmem &sm,
                                              AdvStage &stage) {
  const int lane = (int)lane_id();
  const int gi = gi0 + lane;
  const bool have = lane < kLanes && gi < n_inst_total;
#ifdef SF_TIMING
  const long long ta = clock64();
  long long tb = 0, tc_ = 0, td = 0;
  int n_iter = 0;
#endif
  const int s = have ? D.inst_scen[gi] : 0;
  const ScenConst C = D.sc[s];                           // constant: its load overlaps the waits
  // wait for this lane's scenario's previous window (its HBM run list is final) ...
  if (P.pdl && have) while (ld_acquire(&D.f_led[s]) < P.epoch - 1) __nanosleep(64);
  __syncwarp();
  const int i = gi - C.inst_off;
  const long long lb = C.list_off + (long long)i * C.cap;
  LaneInst x;
  x.nlive = have ? D.irun_n[gi] : 0;                     // run list: written only by the advance
  const int itick0 = have ? D.itick[gi] : 0;             // remaining = run_done - itick
  // ... stage the run lists into the slot columns (coalesced per instance), overlapping the wait
  // for the coordinators below
  {
    // four instances per round: their loads are issued together (no dependence between them)
    const int want_n = (have && x.nlive <= kLS) ? x.nlive : 0;
    for (int l0 = 0; l0 < kLanes; l0 += 4) {
      int rv[4][(kLS + 31) / 32], fv[4][(kLS + 31) / 32], iv[4][(kLS + 31) / 32], tv[4][(kLS + 31) / 32];
      int rn[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        rn[u] = __shfl_sync(0xffffffffu, want_n, l0 + u);
        const long long lbl = __shfl_sync(0xffffffffu, lb, l0 + u);
        const int itl = __shfl_sync(0xffffffffu, itick0, l0 + u);
#pragma unroll
        for (int c = 0; c < (kLS + 31) / 32; ++c) {
          const int sl = c * 32 + lane;
          rv[u][c] = 0x7fffffff; fv[u][c] = 0; iv[u][c] = 0; tv[u][c] = 0;
          if (sl < rn[u]) {
            rv[u][c] = D.run_done[lbl + sl] - itl; fv[u][c] = D.run_fin[lbl + sl];
            iv[u][c] = D.run_id[lbl + sl]; tv[u][c] = D.run_T[lbl + sl];
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int l = l0 + u;
        int mn = 0x7fffffff;
#pragma unroll
        for (int c = 0; c < (kLS + 31) / 32; ++c) {
          const int sl = c * 32 + lane;
          if (sl < rn[u]) {
            sm.done[sl * kLP + l] = rv[u][c]; sm.fin[sl * kLP + l] = fv[u][c];
            sm.rid[sl * kLP + l] = iv[u][c]; sm.rT[sl * kLP + l] = tv[u][c];
            mn = min(mn, rv[u][c]);
          }
        }
        mn = warp_min(mn);
        if (lane == 0) sm.mind[l] = mn;
      }
    }
  }
#ifdef SF_TIMING
  tb = clock64();
#endif
  // this lane's scenario's coordinator is done (PDL)
  if (P.pdl && have) while (ld_acquire(&D.f_coord[s]) < P.epoch) __nanosleep(64);
  __syncwarp();
  if (have) (void)ld_acquire(&D.f_coord[s]);
#ifdef SF_TIMING
  tc_ = clock64();
#endif
  ScenState &SS = D.ss[s];
  const int err0 = have ? SS.err : 1;
  const long long t = SS.t, t_end = t + P.delta;
  if (have) {
    x.st = D.ist[gi]; x.nb = D.inb[gi]; x.until = D.iuntil[gi];
    x.pullv = D.ipullv[gi]; x.pullpend = D.ipullpend[gi];
    x.intkind = D.iintkind[gi]; x.intk = D.iintk[gi];
    x.kv = D.ikv[gi]; x.prefill = D.iprefill[gi]; x.cc = D.ic[gi]; x.v = D.iv[gi];
    x.whead = D.iwhead[gi]; x.wn = D.iwn[gi];
    x.arr_n = D.iarr_n[gi];
    x.abortn = D.iabort[gi]; x.abortarr = D.iabort_arr[gi]; x.evn = D.iev_n[gi];
  } else {
    x.st = I_IDLE; x.nb = x.until = x.kv = x.prefill = 0;
    x.pullv = x.pullpend = x.intkind = x.intk = x.cc = x.v = x.whead = x.wn = x.arr_n = 0;
    x.abortn = x.abortarr = x.evn = 0;
  }
  const bool lane_path = have && !err0 && x.nlive + x.wn + x.arr_n <= kLS;
  const bool warp_path = have && !err0 && !lane_path;
  x.arr_head = 0;
  x.ticks = x.iters = x.tokens = 0;
  x.comps = x.preempts = 0;
  x.tail = x.nlive;
  x.run_n0 = x.nlive;
  x.tc = 0;
  x.min_done = lane_path ? sm.mind[lane] : 0x7fffffff;
  x.ncb = 0;
  x.a_base = 0;
  x.arr_ring0 = -1;
  x.blocked = false; x.head_ok = false;
  x.head_id = x.head_gen = x.head_T = x.head_ctx = 0;
  x.cn_n = x.nlive;                                      // Eq 7's max(k2, k3 n) + k4 for the running n
  x.cn = max(P.k2, (long long)P.k3i * x.nlive) + P.k4;
#ifdef SF_TIMING
  x.n_stage = x.n_headld = 0;
#endif
  // W6: commands to an idle instance apply at a boundary at t
  x.t_cmd = (x.st == I_IDLE && (x.pullpend || x.intkind != INT_NONE || x.abortn > 0)) ? t : kInf;
  x.b_base = -kAS;
  if (lane_path && x.arr_n > 0) {
    lane_stage_arrivals(P, D, C, lb, x, sm, 0);
    lane_stage_admissions(P, D, C, lb, x, sm, 0);
  }

  bool active = lane_path;
  while (__any_sync(0xffffffffu, active)) {
#ifdef SF_TIMING
    ++n_iter;
#endif
    bool go = false;
    x.need_scan = false;
    if (active && x.st == I_TICK && x.intkind == INT_NONE && x.abortn == 0 && !x.pullpend &&
        !(x.wn > 0 && !x.blocked)) {
      // quiet decode steps, lane-locally: a step end with no pending command, no completion
      // (tc + 1 < min_done), no preemption (kv + k5 n <= M), no arrival due and nothing admissible
      // only credits the step (B2) and starts the next one (B8) -- as advance_reg's quiet loop
      const long long na = lane_arr_time(P, D, C, lb, x, sm, x.arr_head);
      const long long k5n = (long long)P.k5 * x.nlive;
      while (x.nb <= t_end && x.tc + 1 < x.min_done && x.kv + k5n <= P.M && na > x.nb) {
        x.tc += 1;
        x.kv += k5n;
        x.tokens += x.nlive;
        x.nb += (long long)P.k1i * (int)x.kv + x.cn;
        x.iters += x.nlive;
        ++x.ticks;
      }
    }
    if (active) {
      long long b;
      if (x.st == I_TICK) b = x.nb;
      else if (x.st == I_PULL) b = x.until;
      else b = min(x.t_cmd, lane_arr_time(P, D, C, lb, x, sm, x.arr_head));
      if (b > t_end) active = false;                     // kInf > t_end
      else { lane_boundary_a(P, D, C, lb, x, sm, b); go = true; }
    }
    lanes_complete_scan(P, x, sm);
    if (go) lane_boundary_b(P, D, C, lb, x, sm);
  }
#ifdef SF_TIMING
  td = clock64();
#endif
  // completion events (cooperatively, one lane's slot column at a time): D.gen = T, D.loc, D.t_complete
  // (reward due at b + R) and the instance's event segment
  {
    unsigned m = __ballot_sync(0xffffffffu, lane_path && x.ncb > 0);
    while (m) {
      const int l = __ffs(m) - 1;
      m &= m - 1;
      const int tl = __shfl_sync(0xffffffffu, x.tail, l);
      const long long lbl = __shfl_sync(0xffffffffu, lb, l);
      const long long toff = __shfl_sync(0xffffffffu, C.traj_off, l);
      int ev = __shfl_sync(0xffffffffu, x.evn, l);
#pragma unroll
      for (int c = 0; c < (kLS + 31) / 32; ++c) {
        const int sl = c * 32 + lane;
        const int d = sl < tl ? sm.done[sl * kLP + l] : kDeadSlot;
        const bool e = d <= -2;
        const unsigned em = __ballot_sync(0xffffffffu, e);
        if (e) {
          const int id = sm.rid[sl * kLP + l];
          const long long j = toff + id;
          D.gen[j] = sm.rT[sl * kLP + l];
          D.loc[j] = L_DONE;
          D.t_complete[j] = sm.cb_t[(-2 - d) * kLanes + l];
          D.iev[lbl + ev + __popc(em & lanemask_lt())] = id;
          sm.done[sl * kLP + l] = kDeadSlot;
        }
        ev += __popc(em);
      }
      if (lane == l) { x.evn = ev; x.ncb = 0; }
    }
  }
  // write the run lists back compacted, in admission order (remaining = done - tc), one lane's
  // column at a time with coalesced stores
  int pos_mine = 0;
  {
    unsigned m = __ballot_sync(0xffffffffu, lane_path);
    while (m) {
      const int l = __ffs(m) - 1;
      m &= m - 1;
      const int tl = __shfl_sync(0xffffffffu, x.tail, l);
      const int itl = __shfl_sync(0xffffffffu, itick0, l);
      const int n0 = __shfl_sync(0xffffffffu, x.run_n0, l);
      const long long lbl = __shfl_sync(0xffffffffu, lb, l);
      int pos = 0;
      for (int c = 0; c * 32 < tl; ++c) {
        const int sl = c * 32 + lane;
        const int d = sl < tl ? sm.done[sl * kLP + l] : kDeadSlot;
        const bool lv = d >= 0;
        const unsigned lm = __ballot_sync(0xffffffffu, lv);
        if (lv) {
          const int p = pos + __popc(lm & lanemask_lt());
          if (p != sl || sl >= n0) {                      // run_done of an unmoved entry is unchanged
            D.run_done[lbl + p] = itl + d;
            D.run_id[lbl + p] = sm.rid[sl * kLP + l];
            D.run_T[lbl + p] = sm.rT[sl * kLP + l];
            D.run_fin[lbl + p] = sm.fin[sl * kLP + l];
          }
        }
        pos += __popc(lm);
      }
      if (lane == l) pos_mine = pos;
    }
  }
  if (lane_path) {
    const int pos = pos_mine;
    // keep undelivered arrivals (held while pulling / later than the window) at the list front
    const int remain = x.arr_n - x.arr_head;
    if (x.arr_head > 0)
      for (int k = 0; k < remain; ++k) {
        D.arr_t[lb + k] = D.arr_t[lb + x.arr_head + k];
        D.arr_id[lb + k] = D.arr_id[lb + x.arr_head + k];
      }
    D.ist[gi] = x.st; D.inb[gi] = x.nb; D.iuntil[gi] = x.until;
    D.ipullpend[gi] = x.pullpend; D.iintkind[gi] = x.intkind;
    D.ikv[gi] = x.kv; D.iprefill[gi] = x.prefill; D.ic[gi] = x.cc; D.iv[gi] = x.v;
    D.irun_n[gi] = pos; D.iwhead[gi] = x.whead; D.iwn[gi] = x.wn; D.iarr_n[gi] = remain;
    D.iev_n[gi] = x.evn;
    D.itick[gi] = itick0 + x.tc;
    if (x.abortn != D.iabort[gi]) D.iabort[gi] = x.abortn;
    if (x.abortarr != D.iabort_arr[gi]) D.iabort_arr[gi] = x.abortarr;
    metric_add(SS, M_TICKS, x.ticks);
    metric_add(SS, M_TRAJ_ITERS, x.iters);
    metric_add(SS, M_TOKENS, x.tokens);
    metric_add(SS, M_COMPLETIONS, x.comps);
    metric_add(SS, M_PREEMPTIONS, x.preempts);
#ifdef SF_TIMING
    if (D.dbg2) {                  // lane layout: loop, stage, wait, tail cycles, iterations, ticks, comps, arrivals
      long long *r = D.dbg2 + 8LL * gi;
      r[0] = td - tc_; r[1] = tb - ta; r[2] = tc_ - tb; r[3] = clock64() - td; r[4] = n_iter; r[5] = x.n_stage;
      r[6] = x.n_headld; r[7] = x.arr_n;
    }
#endif
  }
  // the instances that do not fit the lane slots: one at a time with the whole warp
  unsigned big = __ballot_sync(0xffffffffu, warp_path);
  while (big) {
    const int l = __ffs(big) - 1;
    big &= big - 1;
    const int gl = gi0 + l;
    const int sl = __shfl_sync(0xffffffffu, s, l);
    advance_instance(P, D, gl, stage, sl, D.sc[sl]);
  }
}

#undef LS_AT

}  // namespace sf
