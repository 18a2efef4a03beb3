// k_advance.cu -- decode advance of every rollout instance through one window
// (DESIGN.md §3.1 W6-W7, boundary procedure §3.2 B1-B8).
//
// One warp per instance; instances are independent inside a window (W7), which is the data
// parallelism of the step.  Fast path (every instance whose run+wait+arrivals fit 32*kR): the
// instance's run list is staged ONCE per window from HBM into registers -- lane l holds run
// slots l, l+32, ... with a warp-uniform live bitmask per register row -- and every decode
// step of the window decrements the remaining-length counters in registers (one token per
// running trajectory), detects completions with __ballot_sync, and reduces the
// released KV with warp shuffles only when something completed.  Slot order = admission order,
// so completions leave holes (compacted lazily through shared memory) and LIFO preemption
// takes the highest live slot.  The list is written back compacted at the window end.
// Fallback path: the same procedure streaming the run list through global memory.
#pragma once
#include <cassert>
#include "sf_internal.cuh"

namespace sf {

constexpr long long kInf = 0x7fffffffffffffffLL;
constexpr int kR = 4;                      // register rows -> 128 run slots per instance
#ifndef SF_ADV_WARPS
#define SF_ADV_WARPS 8
#endif
constexpr int kWarpsPerBlock = SF_ADV_WARPS;

struct InstState {
  int st, pullv, pullpend, intkind, intk, cc, v, run_n, whead, wn, arr_n, arr_head;
  int abortn, abortarr;                     // pending Aborts: run/wait members, undelivered arrivals
  int evn;                                  // completion events in this instance's segment (D.iev)
  int itick;                                // decode steps ended (run_done - itick = remaining)
  long long nb, until, kv, prefill, t_cmd;
  long long ticks, iters, tokens, comps, preempts;
};

// completion of run entry (id, T, fin = p + T) at boundary b; event slot e of the instance segment
__device__ __forceinline__ void emit_completion(const Dev &D, const ScenConst &C, long long lb, int id, int Tj, int fin,
                                                long long b, int e, long long k5, long long &release) {
  const long long j = C.traj_off + id;
  release += k5 * (long long)fin;
  D.gen[j] = Tj;
  D.loc[j] = L_DONE;
  D.t_complete[j] = b;                      // reward due at b + R
  D.iev[lb + e] = id;
}

// B1 (Abort, reading R-ABORT): drop the aborted members from the wait ring, FIFO order kept
// (in-place forward compaction, 32 entries per step).  Returns the new queue length.
__device__ __forceinline__ int compact_wait_aborted(const Dev &D, const ScenConst &C, long long lb, int whead, int wn) {
  const int cap = C.cap;
  int out = 0;
  for (int k0 = 0; k0 < wn; k0 += 32) {
    const int k = k0 + (int)lane_id();
    int id = 0;
    bool keep = false;
    if (k < wn) {
      int pos = whead + k;
      if (pos >= cap) pos -= cap;
      id = D.wait_id[lb + pos];
      keep = D.loc[C.traj_off + id] != L_ABORTED;
    }
    const unsigned km = __ballot_sync(0xffffffffu, keep);
    __syncwarp();
    if (keep) {
      int pos = whead + out + __popc(km & lanemask_lt());
      if (pos >= cap) pos -= cap;
      D.wait_id[lb + pos] = id;
    }
    out += __popc(km);
    __syncwarp();
  }
  return out;
}

// ------------------------------------------------------------------ register-resident path
// Each live slot holds dn = the window's decode-step count at whose end it completes (its remaining
// length is dn - tc, tc = steps ended so far in the window; run_done - itick in HBM), so a decode
// step touches no slot: it completes the slots with dn == tc, and only when tc reaches the
// warp-uniform minimum mind.  Dead / empty slots hold a sentinel (kDead); a window has far fewer than kDead
// steps.  Every live slot also keeps its trajectory's target T and final context p + T in
// registers, so completions and preemptions need no memory loads; completion events are
// buffered in shared memory and reserved in the scenario's event list with one atomic per
// flush.  Up to 32 pending arrivals are prefetched (id, gen, T, prompt) into lanes so that
// admitting them reads registers.  `blocked` records that the wait head did not fit the KV
// budget and no KV was released since (KV only grows on a quiet step), so quiet steps skip B7.
constexpr int kDead = 1 << 30;
constexpr int kEvBuf = 32 * kR;           // completion events buffered per warp

struct AdvStage {
  int4 compact[32 * kR];                  // (rem, id, T, p + T) during slot compaction
  int ev[kEvBuf];
};

// append n buffered completion events to this instance's segment (single writer: no atomics)
__device__ __forceinline__ void flush_events(const Dev &D, long long lb, InstState &x, const int *ev, int &n) {
  if (n == 0) return;
  for (int k = lane_id(); k < n; k += 32) D.iev[lb + x.evn + k] = ev[k];
  __syncwarp();
  x.evn += n;
  n = 0;
}

// An instance's run list and step count as loaded before its coordinator has finished: only the
// advance writes them, so once the scenario's previous window is complete (f_led) they are final,
// and a warp can load them while its coordinator still runs (k_advance, PDL).
struct RunPre {
  int run_n, itick;
  int dn[kR], id[kR], T[kR], fin[kR];
};

__device__ __forceinline__ void preload_run(const Dev &D, const ScenConst &C, int gi, RunPre &r) {
  const int lane = (int)lane_id();
  const long long lb = C.list_off + (long long)(gi - C.inst_off) * C.cap;
  r.run_n = D.irun_n[gi];
  r.itick = D.itick[gi];
#pragma unroll
  for (int q = 0; q < kR; ++q) {
    const int s = q * 32 + lane;
    r.dn[q] = kDead; r.id[q] = 0; r.T[q] = 0; r.fin[q] = 0;
    if (s < r.run_n) {
      r.dn[q] = D.run_done[lb + s] - r.itick; r.id[q] = D.run_id[lb + s]; r.T[q] = D.run_T[lb + s];
      r.fin[q] = D.run_fin[lb + s];
    }
  }
}

static __device__ void advance_reg(const GParams &P, const Dev &D, const ScenConst &C, ScenState &SS, InstState &x,
                                   long long lb, long long t_end, AdvStage &sm, const RunPre *pre) {
  const unsigned lane = lane_id();
  const int cap = C.cap;
  const long long k5 = P.k5;
  int rem[kR], rid[kR], tq[kR], fin[kR];     // dn (completion step, see above), id, target T, final context p + T
  unsigned live[kR];
  const int it0 = x.itick;
  int tc = 0;                                // decode steps ended in this window
  int n_orig = x.run_n;                      // slots [0, n_orig) mirror HBM until a compaction
#pragma unroll
  for (int q = 0; q < kR; ++q) {
    const int s = q * 32 + (int)lane;
    if (pre) { rem[q] = pre->dn[q]; rid[q] = pre->id[q]; tq[q] = pre->T[q]; fin[q] = pre->fin[q]; }
    else {
      rem[q] = kDead; rid[q] = 0; tq[q] = 0; fin[q] = 0;
      if (s < x.run_n) { rem[q] = D.run_done[lb + s] - it0; rid[q] = D.run_id[lb + s]; tq[q] = D.run_T[lb + s]; fin[q] = D.run_fin[lb + s]; }
    }
    live[q] = __ballot_sync(0xffffffffu, s < x.run_n);
  }
  auto min_dn = [&]() {                      // earliest completion step among the live slots
    int m = kDead;
#pragma unroll
    for (int q = 0; q < kR; ++q) m = min(m, rem[q]);
    return warp_min(m);
  };
  int mind = min_dn();
  // Arrivals are read through two 32-wide register windows, each refilled with one coalesced
  // load per 32 arrivals: window 6 (id, t_arr) for delivery in B6, window 7 (id, gen, T, prompt)
  // for admission in B7.  Lane k of a window holds arrival base + k.
  int b6 = 0, a6_id = 0, b7 = 0, a7_id = 0, a7_gen = 0, a7_T = 0, a7_p = 0;
  long long a6_t = kInf;
  auto load6 = [&](int base) {
    b6 = base;
    const int k = base + (int)lane;
    a6_id = 0; a6_t = kInf;
    if (k < x.arr_n) { a6_id = D.arr_id[lb + k]; a6_t = D.arr_t[lb + k]; }
  };
  auto load7 = [&](int base) {
    b7 = base;
    const int k = base + (int)lane;
    a7_id = 0; a7_gen = 0; a7_T = 0; a7_p = 0;
    if (k < x.arr_n) {
      a7_id = D.arr_id[lb + k];
      const long long j = C.traj_off + a7_id;
      a7_gen = D.gen[j]; a7_T = D.T[j]; a7_p = D.prompt[C.grp_off + grp_of(P, a7_id)];
    }
  };
  if (x.arr_n > 0) { load6(0); load7(0); }      // (load6(0) is also issued speculatively in advance_instance)
  int arr_ring0 = -1;                       // wait-ring position of arrival 0 once appended
  int nlive = x.run_n, tail = x.run_n, n_ev = 0;
  // arrival k's time (k only grows): window 6, refilled when k leaves it
  auto arr_time = [&](int k) -> long long {
    if (k >= x.arr_n) return kInf;
    if (k >= b6 + 32) load6(k);
    return __shfl_sync(0xffffffffu, a6_t, k - b6);
  };
  long long next_arr = arr_time(x.arr_head);
  bool head_ok = false, blocked = false;
  int head_id = 0, head_gen = 0, head_T = 0;
  long long head_ctx = 0;
  int cn_n = -1;
  long long cn = 0;                                   // max(k2, k3 n) + k4 for n = cn_n

  for (;;) {
    long long b;
    if (x.st == I_TICK) b = x.nb;
    else if (x.st == I_PULL) b = x.until;
    else b = min(x.t_cmd, next_arr);
    if (b > t_end) break;                             // kInf > t_end
    x.t_cmd = kInf;
    const bool tick_end = (x.st == I_TICK);
    const bool pull_done = (x.st == I_PULL);
    // B1: pending interrupts leave without this step's token; KV released (A17, A18)
    if (!pull_done && x.intkind != INT_NONE) {
      if (x.intkind == INT_ALL) {
#pragma unroll
        for (int q = 0; q < kR; ++q) { live[q] = 0u; rem[q] = kDead; }
        nlive = 0; tail = 0; x.wn = 0; x.kv = 0; mind = kDead;
      } else {
        x.wn -= x.intk;                                  // wait tail (A7)
      }
      if (x.wn == 0) head_ok = false;
      blocked = false;
      x.intkind = INT_NONE;
    }
    // B1 (Abort): aborted run / wait members leave for good, their KV released (reading R-ABORT)
    if (x.abortn > 0) {
      long long release = 0;
      int nab = 0;
#pragma unroll
      for (int q = 0; q < kR; ++q) {
        const bool a = ((live[q] >> lane) & 1u) && D.loc[C.traj_off + rid[q]] == L_ABORTED;
        const unsigned am = __ballot_sync(0xffffffffu, a);
        if (a) {
          release += k5 * (long long)(fin[q] - (rem[q] - tc));                    // p + gen
          D.gen[C.traj_off + rid[q]] = tq[q] - (rem[q] - tc);                    // progress kept
          rem[q] = kDead;
        }
        live[q] &= ~am;
        nab += __popc(am);
      }
      if (nab) {
        x.kv -= warp_sum(release);
        nlive -= nab;
        mind = min_dn();
        int t = 0;
#pragma unroll
        for (int q = 0; q < kR; ++q)
          if (live[q]) t = q * 32 + 32 - __clz(live[q]);
        tail = t;
      }
      x.wn = compact_wait_aborted(D, C, lb, x.whead, x.wn);
      x.abortn = 0;
      head_ok = false;
      blocked = false;
      arr_ring0 = -1;                                  // ring positions moved: stop mapping arrivals
    }
    if (tick_end) {
      // B2 + B3 in registers: one token per running trajectory, ballot the completions
      const int n0 = nlive;
      unsigned d[kR], dany = 0;
      ++tc;
      if (tc == mind) {
#pragma unroll
        for (int q = 0; q < kR; ++q) {
          d[q] = __ballot_sync(0xffffffffu, rem[q] == tc);
          dany |= d[q];
        }
      }
      x.kv += k5 * n0;
      x.tokens += n0;
      if (dany) {
        int ncomp = 0;
#pragma unroll
        for (int q = 0; q < kR; ++q) ncomp += __popc(d[q]);
        if (n_ev + ncomp > kEvBuf) flush_events(D, lb, x, sm.ev, n_ev);
        long long release = 0;
        int before = n_ev;
#pragma unroll
        for (int q = 0; q < kR; ++q) {
          if ((d[q] >> lane) & 1u) {
            const long long j = C.traj_off + rid[q];
            release += k5 * (long long)fin[q];
            D.gen[j] = tq[q];
            D.loc[j] = L_DONE;
            D.t_complete[j] = b;                         // reward due at b + R
            sm.ev[before + __popc(d[q] & lanemask_lt())] = rid[q];
            rem[q] = kDead;
          }
          before += __popc(d[q]);
          live[q] &= ~d[q];
        }
        n_ev = before;
        release = warp_sum(release);
        x.kv -= release;
        nlive -= ncomp;
        x.cc += ncomp;
        x.comps += ncomp;
        int t = 0;
#pragma unroll
        for (int q = 0; q < kR; ++q)
          if (live[q]) t = q * 32 + 32 - __clz(live[q]);
        tail = t;
        blocked = false;
        mind = min_dn();
        __syncwarp();
      }
      x.st = I_IDLE;
    } else if (pull_done) {
      x.v = x.pullv; x.cc = 0; x.st = I_IDLE;
    }
    // B4: preemption while KV exceeds M: newest admitted (highest live slot) -> wait front (A21)
    if (x.kv > P.M) {
      while (x.kv > P.M && nlive > 0) {
        int hq = 0;
#pragma unroll
        for (int q = 0; q < kR; ++q)
          if (live[q]) hq = q;
        unsigned hm = 0;
        int r_ = 0, i_ = 0, t_ = 0, f_ = 0;
#pragma unroll
        for (int q = 0; q < kR; ++q)
          if (q == hq) { hm = live[q]; r_ = rem[q]; i_ = rid[q]; t_ = tq[q]; f_ = fin[q]; }
        const int hl = 31 - __clz(hm);
        const int dv = __shfl_sync(0xffffffffu, r_, hl);
        const int r = dv - tc;                         // remaining
        const int id = __shfl_sync(0xffffffffu, i_, hl);
        const int Tj = __shfl_sync(0xffffffffu, t_, hl);
        const int fj = __shfl_sync(0xffffffffu, f_, hl);
        const long long j = C.traj_off + id;
        const int g_ = Tj - r;
        const long long ctx = fj - r;                  // p + gen
        x.kv -= k5 * ctx;
        x.whead = x.whead == 0 ? cap - 1 : x.whead - 1;
        if (lane == 0) {
          D.gen[j] = g_;
          D.loc[j] = L_WAIT;
          D.n_preempt[j] += 1;
          D.wait_id[lb + x.whead] = id;
        }
#pragma unroll
        for (int q = 0; q < kR; ++q)
          if (q == hq) {
            live[q] &= ~(1u << hl);
            if ((int)lane == hl) rem[q] = kDead;
          }
        --nlive;
        tail = hq * 32 + hl;
        if (dv == mind) mind = min_dn();
        ++x.wn;
        ++x.preempts;
        head_ok = true; head_id = id; head_gen = g_; head_T = Tj; head_ctx = ctx;
        arr_ring0 = -1;      // the front push may reuse ring slots of admitted arrivals: stop mapping
      }
      blocked = true;                                 // the last victim (the head) cannot re-fit now
    }
    // B5: a pending Pull blocks generation for q
    if (x.pullpend) {
      x.pullpend = 0;
      x.st = I_PULL;
      x.until = b + P.q;
      continue;
    }
    // B6: arrivals with t_arr <= b join the wait tail in (t_arr, id) order
    if (next_arr <= b) {
      if (x.wn == 0) { head_ok = false; blocked = false; }
      do {
        if (x.arr_head >= b6 + 32) load6(x.arr_head);
        const int id = __shfl_sync(0xffffffffu, a6_id, x.arr_head - b6);
        if (x.abortarr > 0 && D.loc[C.traj_off + id] == L_ABORTED) {   // aborted in transit: dropped
          --x.abortarr;
          arr_ring0 = -1;
        } else {
          int pos = x.whead + x.wn;
          if (pos >= cap) pos -= cap;
          if (x.arr_head == 0) arr_ring0 = pos;
          if (lane == 0) { D.wait_id[lb + pos] = id; D.loc[C.traj_off + id] = L_WAIT; }
          ++x.wn;
        }
        ++x.arr_head;
        next_arr = arr_time(x.arr_head);
      } while (next_arr <= b);
      __syncwarp();
    }
    // B7: FIFO admission while the head fits the KV budget
    if (x.wn > 0 && !blocked) {
      while (x.wn > 0) {
        if (!head_ok) {
          // the head is arrival k of this window when its ring position is arr_ring0 + k
          int k = -1;
          if (arr_ring0 >= 0) {
            k = x.whead - arr_ring0;
            if (k < 0) k += cap;
            if (k >= x.arr_head || k < b7) k = -1;
          }
          if (k >= 0) {
            if (k >= b7 + 32) load7(k);
            head_id = __shfl_sync(0xffffffffu, a7_id, k - b7);
            head_gen = __shfl_sync(0xffffffffu, a7_gen, k - b7);
            head_T = __shfl_sync(0xffffffffu, a7_T, k - b7);
            head_ctx = __shfl_sync(0xffffffffu, a7_p, k - b7) + head_gen;
          } else {
            head_id = D.wait_id[lb + x.whead];
            const long long j = C.traj_off + head_id;
            head_gen = D.gen[j];
            head_T = D.T[j];
            head_ctx = D.prompt[C.grp_off + grp_of(P, head_id)] + head_gen;
          }
          head_ok = true;
        }
        if (x.kv + k5 * head_ctx > P.M) { blocked = true; break; }
        if (tail == 32 * kR) {
          // stable compaction of the live slots through shared memory
#pragma unroll
          for (int q = 0; q < kR; ++q) {
            int before = 0;
#pragma unroll
            for (int qq = 0; qq < kR; ++qq)
              if (qq < q) before += __popc(live[qq]);
            if ((live[q] >> lane) & 1u)
              sm.compact[before + __popc(live[q] & lanemask_lt())] = make_int4(rem[q], rid[q], tq[q], fin[q]);
          }
          __syncwarp();
#pragma unroll
          for (int q = 0; q < kR; ++q) {
            const int s = q * 32 + (int)lane;
            rem[q] = kDead;
            if (s < nlive) { const int4 e = sm.compact[s]; rem[q] = e.x; rid[q] = e.y; tq[q] = e.z; fin[q] = e.w; }
            live[q] = __ballot_sync(0xffffffffu, s < nlive);
          }
          __syncwarp();
          tail = nlive;
          n_orig = 0;
        }
        const int s = tail++;
        const int sq = s >> 5, sl = s & 31;
        n_orig = min(n_orig, s);                       // a reused slot no longer mirrors HBM
#pragma unroll
        for (int q = 0; q < kR; ++q)
          if (q == sq) {
            if ((int)lane == sl) {
              rem[q] = tc + head_T - head_gen; rid[q] = head_id;
              tq[q] = head_T; fin[q] = (int)(head_ctx - head_gen) + head_T;
            }
            live[q] |= 1u << sl;
          }
        mind = min(mind, tc + head_T - head_gen);
        if (lane == 0) D.loc[C.traj_off + head_id] = L_RUN;
        x.kv += k5 * head_ctx;
        x.prefill += head_ctx;
        ++nlive;
        x.whead = x.whead + 1 == cap ? 0 : x.whead + 1;
        --x.wn;
        head_ok = false;
      }
    }
    // B8: next decode step, Eq 7 + prefill stall (A20)
    if (nlive > 0) {
      if (nlive != cn_n) { cn_n = nlive; cn = max(P.k2, (long long)P.k3i * nlive) + P.k4; }
      x.nb = b + (long long)P.k1i * (int)x.kv + cn + (long long)P.kpi * (int)x.prefill;
      x.prefill = 0;
      x.st = I_TICK;
      x.iters += nlive;
      ++x.ticks;
    } else {
      x.st = I_IDLE;
      continue;
    }
    // Quiet decode steps: the next boundary is a step end with no pending command, no
    // completion (tc + 1 < mind), no preemption (kv + k5 n <= M), no arrival due, and no
    // admission possible (B7 just left the head blocked or the queue empty).  Such a boundary
    // only credits the step (B2) and starts the next one (B8).
    if (x.intkind == INT_NONE && !x.pullpend) {
      const int k5n = (int)(k5 * nlive);
      if (P.skip) {
        // f1: jump over the whole run of quiet steps in closed form.  With
        // kv0 = kv at the current step start and c1 = k1 kv0 + cn, the j-th quiet boundary is
        //   b_j = nb + g(j-1),  g(x) = c1 x + q1 x (x+1) / 2,  q1 = k1 k5n   (Eq 7, kv growing k5 n per step)
        // and boundary j is quiet iff j <= minrem - 1, kv0 + j k5n <= M, b_j <= t_end and
        // b_j < next arrival.  m = the largest such j: g is increasing, so x = m - 1 is the floor
        // root of g(x) = t_lim - nb, estimated in fp64 and then fixed by exact integer checks (int64
        // when the products provably fit, else int128).
        const int mr = mind - tc;                               // the earliest remaining length
        long long m_hi = (long long)mr - 1;
        m_hi = min(m_hi, (long long)((unsigned)(P.M - x.kv) / (unsigned)k5n));   // M - kv < 2^30
        const long long t_lim = min(t_end, next_arr - 1);
        long long m = 0;
        __int128 gm = 0;                                        // g(m): b_{m+1} = nb + g(m)
#ifdef SF_SKIP_BSEARCH
        {                                                       // A/B reference: binary search
          const __int128 c1 = (__int128)P.k1i * x.kv + cn, q1 = (__int128)P.k1i * k5n;
          auto g = [&](long long xx) -> __int128 { return c1 * xx + q1 * (((__int128)xx * (xx + 1)) >> 1); };
          long long lo = 0, hi = max(m_hi, 0LL);
          while (lo < hi) {
            const long long mid = (lo + hi + 1) >> 1;
            if ((__int128)x.nb + g(mid - 1) <= t_lim) lo = mid; else hi = mid - 1;
          }
          m = lo;
          gm = g(m);
        }
#else
        if (m_hi > 0 && x.nb <= t_lim) {
          const long long R = t_lim - x.nb;
          const double c1d = (double)P.k1i * (double)x.kv + (double)cn, q1d = (double)P.k1i * (double)k5n;
          const double A = 0.5 * q1d, Bq = c1d + A, Rd = (double)R;
          // stable root of A x^2 + Bq x = R; only an estimate (the exact checks below fix it), so fp32
          const float xe = __fdividef((float)(2.0 * Rd), (float)Bq + sqrtf((float)(Bq * Bq + 4.0 * A * Rd)));
          long long xx = (long long)fminf(fmaxf(floorf(xe), 0.f), (float)(m_hi - 1));
          if (c1d < 0x1p40 && q1d < 0x1p23 && m_hi < (1LL << 19)) {
            // every product below stays under 2^61: exact in int64
            const long long c1 = (long long)P.k1i * x.kv + cn, q1 = (long long)P.k1i * k5n;
            auto g = [&](long long t) -> long long { return c1 * t + q1 * ((t * (t + 1)) >> 1); };
            while (xx + 1 <= m_hi - 1 && g(xx + 1) <= R) ++xx;
            while (xx >= 0 && g(xx) > R) --xx;
            m = xx + 1;
            if (m > 0) gm = g(m);
          } else {
            const __int128 c1 = (__int128)P.k1i * x.kv + cn, q1 = (__int128)P.k1i * k5n;
            auto g = [&](long long t) -> __int128 { return c1 * t + q1 * (((__int128)t * (t + 1)) >> 1); };
            while (xx + 1 <= m_hi - 1 && g(xx + 1) <= R) ++xx;
            while (xx >= 0 && g(xx) > R) --xx;
            m = xx + 1;
            if (m > 0) gm = g(m);
          }
        }
#endif
        if (m > 0) {
          tc += (int)m;
          x.nb = (long long)((__int128)x.nb + gm);                   // b_{m+1} = nb + g(m)
          x.kv += m * k5n;
          x.tokens += m * nlive;
          x.iters += m * nlive;
          x.ticks += m;
        }
      } else {
        for (;;) {
          const long long bq = x.nb;
          if (bq > t_end || x.kv + k5n > P.M || next_arr <= bq || tc + 1 >= mind) break;
          ++tc;
          x.kv += k5n;
          x.tokens += nlive;
          x.nb = bq + (long long)P.k1i * (int)x.kv + cn;
          x.iters += nlive;
          ++x.ticks;
        }
      }
    }
  }
  flush_events(D, lb, x, sm.ev, n_ev);
#ifdef SF_CHECK_ADV
  assert(x.evn <= C.cap);
  assert(nlive >= 0 && nlive <= 32 * kR && x.wn >= 0 && x.wn <= cap && x.kv >= 0 && x.kv <= P.M);
#pragma unroll
  for (int q = 0; q < kR; ++q) assert(!((live[q] >> lane) & 1u) || (rem[q] - tc > 0 && rem[q] - tc <= tq[q]));
#endif
  // write the run list back compacted, in admission order; an entry that kept its slot since the
  // window start is unchanged in HBM (run_done is absolute) and is not rewritten
  int before = 0;
#pragma unroll
  for (int q = 0; q < kR; ++q) {
    if ((live[q] >> lane) & 1u) {
      const int pos = before + __popc(live[q] & lanemask_lt());
      if (pos != q * 32 + (int)lane || pos >= n_orig) {
        D.run_done[lb + pos] = it0 + rem[q];                 // = itick after the window + remaining
        D.run_id[lb + pos] = rid[q];
        D.run_T[lb + pos] = tq[q];
        D.run_fin[lb + pos] = fin[q];
      }
    }
    before += __popc(live[q]);
  }
  x.run_n = nlive;
  x.itick = it0 + tc;
}

// ------------------------------------------------------------------ global-memory path
static __device__ void advance_global(const GParams &P, const Dev &D, const ScenConst &C, ScenState &SS, InstState &x,
                               long long lb, long long t_end) {
  const unsigned lane = lane_id();
  const int cap = C.cap;
  const long long k5 = P.k5;
  for (;;) {
    long long b;
    if (x.st == I_TICK) b = x.nb;
    else if (x.st == I_PULL) b = x.until;
    else b = min(x.t_cmd, x.arr_head < x.arr_n ? D.arr_t[lb + x.arr_head] : kInf);
    if (b == kInf || b > t_end) break;
    x.t_cmd = kInf;
    const bool tick_end = (x.st == I_TICK);
    const bool pull_done = (x.st == I_PULL);
    if (!pull_done && x.intkind != INT_NONE) {
      if (x.intkind == INT_ALL) { x.run_n = 0; x.wn = 0; x.kv = 0; }
      else x.wn -= x.intk;
      x.intkind = INT_NONE;
    }
    if (x.abortn > 0) {                              // B1 (Abort), reading R-ABORT
      int out = 0;
      long long release = 0;
      for (int base = 0; base < x.run_n; base += 32) {
        const int k = base + (int)lane;
        int rem = 0, id = 0, Tk = 0, fk = 0;
        bool ab = false;
        if (k < x.run_n) {
          rem = D.run_done[lb + k]; id = D.run_id[lb + k]; Tk = D.run_T[lb + k]; fk = D.run_fin[lb + k];
          ab = D.loc[C.traj_off + id] == L_ABORTED;
          if (ab) {
            const int r = rem - x.itick;                                             // remaining
            release += k5 * (long long)(fk - r);                                     // p + gen
            D.gen[C.traj_off + id] = Tk - r;
          }
        }
        const bool keep = k < x.run_n && !ab;
        const unsigned mk = __ballot_sync(0xffffffffu, keep);
        __syncwarp();
        if (keep) {
          const int pos = out + __popc(mk & lanemask_lt());
          D.run_done[lb + pos] = rem; D.run_id[lb + pos] = id; D.run_T[lb + pos] = Tk; D.run_fin[lb + pos] = fk;
        }
        out += __popc(mk);
        __syncwarp();
      }
      x.kv -= warp_sum(release);
      x.run_n = out;
      x.wn = compact_wait_aborted(D, C, lb, x.whead, x.wn);
      x.abortn = 0;
    }
    if (tick_end) {
      // one token each: the step count advances; an entry completes when its run_done is reached.
      // Only the 4-byte run_done is read per entry; entries move (and are rewritten) only behind a
      // completion
      const int n0 = x.run_n;
      x.itick += 1;
      int out = 0, ncomp = 0;
      long long release = 0;
      for (int base = 0; base < n0; base += 32) {
        const int k = base + (int)lane;
        const bool valid = k < n0;
        const int dn = valid ? D.run_done[lb + k] : 0;
        const bool done = valid && dn == x.itick;
        const bool keep = valid && !done;
        const unsigned mk = __ballot_sync(0xffffffffu, keep);
        const unsigned md = __ballot_sync(0xffffffffu, done);
        const int pos = out + __popc(mk & lanemask_lt());
        int id = 0, Tk = 0, fk = 0;
        if (done || (keep && pos != k)) { id = D.run_id[lb + k]; Tk = D.run_T[lb + k]; fk = D.run_fin[lb + k]; }
        __syncwarp();
        if (keep && pos != k) { D.run_done[lb + pos] = dn; D.run_id[lb + pos] = id; D.run_T[lb + pos] = Tk; D.run_fin[lb + pos] = fk; }
        if (done) emit_completion(D, C, lb, id, Tk, fk, b, x.evn + ncomp + __popc(md & lanemask_lt()), k5, release);
        out += __popc(mk);
        ncomp += __popc(md);
      }
      if (ncomp) release = warp_sum(release);
      x.kv += k5 * n0 - release;
      x.tokens += n0;
      x.run_n = out;
      x.evn += ncomp;
      x.cc += ncomp;
      x.comps += ncomp;
      x.st = I_IDLE;
      __syncwarp();
    }
    if (pull_done) { x.v = x.pullv; x.cc = 0; x.st = I_IDLE; }
    while (x.kv > P.M && x.run_n > 0) {
      const int k = x.run_n - 1;
      const int id = D.run_id[lb + k];
      const long long j = C.traj_off + id;
      const int rk = D.run_done[lb + k] - x.itick;      // remaining
      const int g_ = D.run_T[lb + k] - rk;
      x.kv -= k5 * (long long)(D.run_fin[lb + k] - rk);                         // p + gen
      x.whead = x.whead == 0 ? cap - 1 : x.whead - 1;
      if (lane == 0) {
        D.gen[j] = g_;
        D.loc[j] = L_WAIT;
        D.n_preempt[j] += 1;
        D.wait_id[lb + x.whead] = id;
      }
      ++x.wn;
      --x.run_n;
      ++x.preempts;
    }
    if (x.pullpend) {
      x.pullpend = 0;
      x.st = I_PULL;
      x.until = b + P.q;
      __syncwarp();
      continue;
    }
    while (x.arr_head < x.arr_n && D.arr_t[lb + x.arr_head] <= b) {
      const int id = D.arr_id[lb + x.arr_head];
      if (x.abortarr > 0 && D.loc[C.traj_off + id] == L_ABORTED) {   // aborted in transit: dropped
        --x.abortarr;
        ++x.arr_head;
        continue;
      }
      int pos = x.whead + x.wn;
      if (pos >= cap) pos -= cap;
      if (lane == 0) { D.wait_id[lb + pos] = id; D.loc[C.traj_off + id] = L_WAIT; }
      ++x.wn;
      ++x.arr_head;
    }
    __syncwarp();
    while (x.wn > 0) {
      const int id = D.wait_id[lb + x.whead];
      const long long j = C.traj_off + id;
      const int gj = D.gen[j];
      const long long ctx = D.prompt[C.grp_off + grp_of(P, id)] + gj;
      if (x.kv + k5 * ctx > P.M) break;
      if (lane == 0) {
        const int Tj = D.T[j];
        D.run_id[lb + x.run_n] = id;
        D.run_done[lb + x.run_n] = x.itick + (Tj - gj);
        D.run_T[lb + x.run_n] = Tj;
        D.run_fin[lb + x.run_n] = (int)(ctx - gj) + Tj;
        D.loc[j] = L_RUN;
      }
      x.kv += k5 * ctx;
      x.prefill += ctx;
      ++x.run_n;
      x.whead = x.whead + 1 == cap ? 0 : x.whead + 1;
      --x.wn;
    }
    __syncwarp();
    if (x.run_n > 0) {
      x.nb = b + tick_latency(P, x.kv, x.run_n, x.prefill);
      x.prefill = 0;
      x.st = I_TICK;
      x.iters += x.run_n;
      ++x.ticks;
    } else {
      x.st = I_IDLE;
    }
  }
}

// One window of W6-W7 for global instance gi, executed by one warp (stage: 32*kR int2 of smem).
// s = D.inst_scen[gi] and C = D.sc[s] are passed in so that a caller can load them (never written
// by a window) before waiting on the coordinator's flag.
// The instance's window-start fields (written by the previous window's advance and by this
// window's coordinator): valid once the coordinator of this window is done.
__device__ __forceinline__ void load_inst_state(const Dev &D, int gi, InstState &x) {
  x.st = D.ist[gi]; x.nb = D.inb[gi]; x.until = D.iuntil[gi];
  x.pullv = D.ipullv[gi]; x.pullpend = D.ipullpend[gi];
  x.intkind = D.iintkind[gi]; x.intk = D.iintk[gi];
  x.kv = D.ikv[gi]; x.prefill = D.iprefill[gi]; x.cc = D.ic[gi]; x.v = D.iv[gi];
  x.whead = D.iwhead[gi]; x.wn = D.iwn[gi];
  x.arr_n = D.iarr_n[gi]; x.arr_head = 0;
  x.abortn = D.iabort[gi]; x.abortarr = D.iabort_arr[gi]; x.evn = D.iev_n[gi];
}

// xs: the fields already loaded by load_inst_state (a caller that prefetches them while the
// warp's previous instance is processed), else loaded here.
__device__ __forceinline__ void advance_instance(const GParams &P, const Dev &D, int gi, AdvStage &stage, int s,
                                                 const ScenConst C, const RunPre *pre = nullptr,
                                                 const InstState *xs = nullptr) {
  const unsigned lane = lane_id();
#ifdef SF_TIMING
  const long long t0_adv = clock64();
#endif
  // the instance's own fields depend only on gi: issue them with the scenario lookups, not after
  InstState x;
  if (xs) x = *xs;
  else load_inst_state(D, gi, x);
  if (pre) { x.run_n = pre->run_n; x.itick = pre->itick; }
  else { x.run_n = D.irun_n[gi]; x.itick = D.itick[gi]; }
  ScenState &SS = D.ss[s];
  const int err0 = SS.err;    // checked below, before the first write
  const int i = gi - C.inst_off;
  const long long t = SS.t, t_end = t + P.delta;
  const long long lb = C.list_off + (long long)i * C.cap;

  x.ticks = x.iters = x.tokens = x.comps = x.preempts = 0;
  // W6: commands to an idle instance apply at a boundary at t
  x.t_cmd = (x.st == I_IDLE && (x.pullpend || x.intkind != INT_NONE || x.abortn > 0)) ? t : kInf;

  if (err0) return;
  if (x.run_n + x.wn + x.arr_n <= 32 * kR) advance_reg(P, D, C, SS, x, lb, t_end, stage, pre && pre->run_n <= 32 * kR ? pre : nullptr);
  else advance_global(P, D, C, SS, x, lb, t_end);

  // keep undelivered arrivals (held while pulling / later than the window) at the list front
  const int remain = x.arr_n - x.arr_head;
  if (x.arr_head > 0 && remain > 0) {
    for (int k0 = 0; k0 < remain; k0 += 32) {
      const int k = k0 + (int)lane;
      long long ta = 0;
      int ia = 0;
      if (k < remain) { ta = D.arr_t[lb + x.arr_head + k]; ia = D.arr_id[lb + x.arr_head + k]; }
      __syncwarp();
      if (k < remain) { D.arr_t[lb + k] = ta; D.arr_id[lb + k] = ia; }
      __syncwarp();
    }
  }
  if (lane == 0) {
    D.ist[gi] = x.st; D.inb[gi] = x.nb; D.iuntil[gi] = x.until;
    D.ipullpend[gi] = x.pullpend; D.iintkind[gi] = x.intkind;
    D.ikv[gi] = x.kv; D.iprefill[gi] = x.prefill; D.ic[gi] = x.cc; D.iv[gi] = x.v;
    D.irun_n[gi] = x.run_n; D.iwhead[gi] = x.whead; D.iwn[gi] = x.wn; D.iarr_n[gi] = remain;
    D.iev_n[gi] = x.evn;
    D.itick[gi] = x.itick;
    if (x.abortn != D.iabort[gi]) D.iabort[gi] = x.abortn;
    if (x.abortarr != D.iabort_arr[gi]) D.iabort_arr[gi] = x.abortarr;
    metric_add(SS, M_TICKS, x.ticks);
    metric_add(SS, M_TRAJ_ITERS, x.iters);
    metric_add(SS, M_TOKENS, x.tokens);
    metric_add(SS, M_COMPLETIONS, x.comps);
    metric_add(SS, M_PREEMPTIONS, x.preempts);
#ifdef SF_TIMING
    if (D.dbg2) {
      long long *r = D.dbg2 + 8LL * gi;
      r[0] = clock64() - t0_adv; r[1] = x.ticks; r[2] = x.comps; r[3] = x.arr_n; r[4] = x.preempts;
      r[5] = x.run_n; r[6] = x.wn; r[7] = x.iters;
    }
#endif
  }
}

}  // namespace sf
