// k_coord.cu -- window begin + rollout coordinator (DESIGN.md §3.1 W0-W5).
//
// One warp per scenario.  The coordinator is inherently sequential over routed trajectories
// (each Route mutates the snapshot and the ledger, Alg 2), so parallelism is
// across scenarios (warps) and, inside one decision, across instances: lane l owns instances
// l, l+32, ... (KS instances per lane, KS = ceil(I/32) chosen at launch so that small-I
// scenarios keep few registers and high occupancy).  Candidate tests, Eq 3 gains and the
// waterfall argmax are lane-parallel with deterministic (value, lowest id) warp reductions;
// fp64 uses only correctly rounded __d*_rn operations so decisions equal the oracle's bit for
// bit.  Latency: MLQ items are prefetched 32 at a time (one lane each) and route records are
// staged in shared memory, where each instance's arrivals are ordered by (t_arr, id).
#pragma once
#include "sf_internal.cuh"

namespace sf {

#ifndef SF_COORD_WARPS
#define SF_COORD_WARPS 2   // 2-warp blocks: a finished scenario's slot is reused sooner (A/B: 4 -> 2
#endif                     // warps per block, window -0.6 %; 1 warp: -0.3 %)
constexpr int kCoordWarps = SF_COORD_WARPS;   // scenarios per block
#ifndef SF_COORD_MINB
#define SF_COORD_MINB (16 / SF_COORD_WARPS)  // 1-slot variant: 16 warps per SM = 128 registers, no spills (measured)
#endif
constexpr int kArrStage = 128; // route records staged per warp in shared memory

template <int KS>
struct InstRegs {
  int v[KS];
  long long kv[KS];
  int n[KS];
  int w[KS];
};

struct Cyc {                   // lane-uniform per-cycle scalars
  long long t;
  int cu, ps, eta, I, G, B;
  int n_v, n_vl, vl_head, n_ingested, min_live_g;
  int min_v;                   // smallest version in the versioned MLQ (its first item's)
  long long window;
  unsigned long long hash;
  int cmd_n;
  int reserves;
  int mlq_err;
  int use_bits;
  int red_w;                   // lanes holding instances (power of 2 >= min(I, 32)): reduction width
#ifdef SF_TIMING_ROUTE
  long long rt[6], rt_last;    // SF_TIMING_ROUTE builds: cycles per routing sub-step (tools/route_steps.py)
#endif
};

#ifdef SF_TIMING_ROUTE
#define SF_RT(k) do { if (tentative < 0) { const long long _n = clock64(); c.rt[k] += _n - c.rt_last; c.rt_last = _n; } } while (0)
#else
#define SF_RT(k) do { } while (0)
#endif

constexpr int kEmptyWords = 160;   // ledger empty-slot bitmap held in smem when (eta+1)*B <= 5120

constexpr int kRepG = 4;        // route_group_batch: lane-replicated waterfall for I <= kRepG
constexpr int kGMax = 16;       // group-batched routing for G <= kGMax (route_group_batch)

struct Stage {                 // per-warp shared-memory staging
  double tab[kGMax][32];       // route_group_batch: Eq 3 gain of lane's instance after j more routes
  unsigned empty[kEmptyWords]; // bit s of ring r: slot s of ring buffer r is Empty (valid if use_bits)
  int sfree[kMaxEta + 1];
  int sfree_tmp[kMaxEta + 1];
  int vcnt[kMaxEta + 2];
  long long arr_t[kArrStage];
  int arr_id[kArrStage];
  short arr_inst[kArrStage];
  int n_arr;
};

// verify(v) on the per-warp free counts sfree[d] of buffers cu + d, d in [0, eta].
__device__ __forceinline__ bool verify_free(const int *sfree, int v, int cu, int eta) {
  for (int b = v + eta; b >= max(v, cu); --b)
    if (sfree[b - cu] > 0) return true;
  return false;
}

// verify(v) for every v = cu - eta + d, d in [0, eta], as a bitmask: bit d is set iff one of
// the buffers cu .. cu + d has a free slot (the reserve range [max(v, cu), v + eta] = [cu, cu+d]).
// Versions below cu - eta can never verify.
// One ballot (all lanes): bit d of the result is set from the lowest d with a free slot up to eta.
__device__ __forceinline__ unsigned verify_mask(const int *sfree, int eta) {
  const int lane = (int)lane_id();
  const unsigned m = __ballot_sync(0xffffffffu, lane <= eta && sfree[lane] > 0);
  const unsigned low = m & (0u - m);
  return low ? (((2u << eta) - 1u) & ~(low - 1u)) : 0u;
}

__device__ __forceinline__ void log_cmd(const GParams &P, const Dev &D, const ScenConst &C, Cyc &c, int kind,
                                        int inst, int traj) {
  c.hash += record_hash(c.cmd_n, c.window, kind, inst, traj);
  if (c.cmd_n < P.cmdlog_cap && lane_id() == 0) {
    long long *r = D.cmdlog + C.cmd_off + 4LL * c.cmd_n;
    r[0] = c.window; r[1] = kind; r[2] = inst; r[3] = traj;
  }
  c.cmd_n++;
}

// Materialise the versioned part of the MLQ (Alg 2 line 2): TS-resident trajectories
// of versioned groups (TS bitmap, scanned over the live id window) in (v, id) ascending order
// into D.mlq[mlq_off ...].  Versions lie in [max(0, cu - eta), ps]; items are bucketed stably by
// version with packed (v - vlo) << 27 | id keys.  Returns the count; *min_v = smallest version
// present (INT_MAX if none, -1 if an item's version is out of range: protocol bug).
static __device__ int build_mlq(const GParams &P, const Dev &D, const ScenConst &C, const Cyc &c, Stage &sg, int *min_v) {
  const unsigned lane = lane_id();
  const int w_lo = (c.min_live_g * c.G) >> 5;
  const int w_hi = (c.n_ingested * c.G + 31) >> 5;
  int *tmp = D.mlq + C.mlq_off + C.cap;
  int *out = D.mlq + C.mlq_off;
  int n_tmp = 0;
  // only the chunks of 32 words whose summary bit is set (D.tsv_sum), in ascending order; a chunk
  // found all-zero has its summary bit cleared (bits are set only by tsv_mark)
  if (w_lo < w_hi) {
    const int c_lo = w_lo >> 5, c_hi = (w_hi - 1) >> 5;          // chunks [c_lo, c_hi]
#pragma unroll 1
    for (int s0 = c_lo >> 5; s0 <= (c_hi >> 5); s0 += 32) {
      const int sw = s0 + (int)lane;
      unsigned sm = sw <= (c_hi >> 5) ? D.tsv_sum[C.sum_off + sw] : 0u;
      if (sw == (c_lo >> 5)) sm &= ~0u << (c_lo & 31);
      if (sw == (c_hi >> 5) && (c_hi & 31) != 31) sm &= (2u << (c_hi & 31)) - 1u;
      unsigned lanes = __ballot_sync(0xffffffffu, sm != 0u);
      while (lanes) {
        const int L = __ffs(lanes) - 1;
        lanes &= lanes - 1;
        unsigned bits = __shfl_sync(0xffffffffu, sm, L);
        while (bits) {
          const int b = __ffs(bits) - 1;
          bits &= bits - 1;
          const int ch = ((s0 + L) << 5) + b;
          const int w = (ch << 5) + (int)lane;
          const unsigned raw = D.tsv_bits[C.bits_off + w];     // the chunk lies inside the scenario's words
          unsigned word = (w >= w_lo && w < w_hi) ? raw : 0u;
          if (!__any_sync(0xffffffffu, raw != 0u)) {
            if (lane == 0) atomicAnd(&D.tsv_sum[C.sum_off + (ch >> 5)], ~(1u << (ch & 31)));
            continue;
          }
          const int cnt = __popc(word);
          const int off = warp_excl_scan(cnt);
          const int tot = __shfl_sync(0xffffffffu, off + cnt, 31);
          int pos = n_tmp + off;
          while (word) {
            const int bb = __ffs(word) - 1;
            word &= word - 1;
            tmp[pos++] = (w << 5) + bb;
          }
          n_tmp += tot;
        }
      }
    }
  }
  *min_v = 0x7fffffff;
  if (n_tmp == 0) return 0;
  __syncwarp();
  const int vlo = max(0, c.cu - c.eta);
  const int nv = c.ps - vlo + 1;
  if ((int)lane < kMaxEta + 2) sg.vcnt[lane] = 0;
  __syncwarp();
  bool bad = false;
#pragma unroll 1
  for (int k0 = 0; k0 < n_tmp; k0 += 32) {
    const int k = k0 + (int)lane;
    if (k < n_tmp) {
      const int id = tmp[k];
      const int d = D.gv[C.grp_off + grp_of(P, id)] - vlo;
      if (d < 0 || d >= nv) bad = true;
      else { tmp[k] = (d << 27) | id; atomicAdd(&sg.vcnt[d], 1); }
    }
  }
  __syncwarp();
  if (__any_sync(0xffffffffu, bad)) { *min_v = -1; return 0; }
  {
    // bucket bases: exclusive prefix of the counts over d < nv (nv <= kMaxEta + 1 <= 32), in place;
    // the smallest version present
    const int cnt = (int)lane < nv ? sg.vcnt[lane] : 0;
    const int ex = warp_excl_scan(cnt);
    const unsigned nz = __ballot_sync(0xffffffffu, cnt > 0);
    if (nz) *min_v = vlo + __ffs(nz) - 1;
    __syncwarp();
    if ((int)lane < nv) sg.vcnt[lane] = ex;
    __syncwarp();
  }
#pragma unroll 1
  for (int k0 = 0; k0 < n_tmp; k0 += 32) {
    // stable scatter: rank among the chunk's lanes with the same bucket, then each bucket's base
    // advances by its count (added by the bucket's highest lane)
    const int k = k0 + (int)lane;
    const int key = k < n_tmp ? tmp[k] : -1;
    const int dk = key >= 0 ? (key >> 27) : -1;
    const unsigned same = __match_any_sync(0xffffffffu, dk);
    if (dk >= 0) out[sg.vcnt[dk] + __popc(same & lanemask_lt())] = key & 0x7ffffff;
    __syncwarp();
    if (dk >= 0 && (same >> lane) == 1u) sg.vcnt[dk] += __popc(same);
    __syncwarp();
  }
  __syncwarp();
  return n_tmp;
}


// The waterfall's reduction (route_pass): over the lanes' best (key = version << 7 | instance, d),
// key 0x7fffffff = none, the lowest version, then the highest d, then the lowest instance; returns
// that key in every lane (0x7fffffff: no candidate).  For wide warps (>= SF_REDUX_MIN lanes hold
// instances) four single-instruction redux.sync reductions: the version, then the two halves of d's
// order-preserving bit pattern among the lanes still in, then the key; narrow ones butterfly
// shuffles over red_w lanes.  d is never -0.0 (a difference of two positive T values, or 0.0), so
// the bit-pattern order is the double order.
#ifndef SF_REDUX_MIN
#define SF_REDUX_MIN 8
#endif
__device__ __forceinline__ int waterfall_reduce(int bk, double bd, int red_w) {
  if (red_w >= SF_REDUX_MIN) {
    const unsigned vk = (unsigned)bk >> 7;
    const unsigned vmin = __reduce_min_sync(0xffffffffu, vk);
    if (vmin == (0x7fffffffu >> 7)) return 0x7fffffff;
    const unsigned long long b = (unsigned long long)__double_as_longlong(bd);
    const unsigned long long u = (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
    bool in = vk == vmin;
    const unsigned hmax = __reduce_max_sync(0xffffffffu, in ? (unsigned)(u >> 32) : 0u);
    in = in && (unsigned)(u >> 32) == hmax;
    const unsigned lmax = __reduce_max_sync(0xffffffffu, in ? (unsigned)u : 0u);
    in = in && (unsigned)u == lmax;
    return (int)__reduce_min_sync(0xffffffffu, in ? (unsigned)bk : 0xffffffffu);
  }
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    if (o >= red_w) break;
    const int ok = __shfl_xor_sync(0xffffffffu, bk, o);
    const double od = __shfl_xor_sync(0xffffffffu, bd, o);
    const bool better = ((ok >> 7) < (bk >> 7)) | (((ok >> 7) == (bk >> 7)) & ((od > bd) | ((od == bd) & (ok < bk))));
    bk = better ? ok : bk;
    bd = better ? od : bd;
  }
  return __shfl_sync(0xffffffffu, bk, 0);
}

// Group-batched routing (one instance per lane, KS == 1).  After the first member of a
// versionless group is routed (which fixed v_g and Reserved), its remaining members are the next
// MLQ items (consecutive ids, same l = p since gen = 0, same candidate set {i : S[i].v >= v_g},
// same threshold).  Each decision changes only the chosen instance's state, so every lane
// precomputes its instance's Eq 3 gain after j = 0..nrem-1 further routes of this group (the
// same operation trees as the one-at-a-time pass: dT = T(n+1, kv+k5 l) - T(n, kv), 0 once
// gamma fails), and the nrem decisions become reductions over those tables -- no divisions on
// the sequential chain.  Returns the members routed; *stopped if a member found no instance.
static __device__ int route_group_batch(const GParams &P, const Dev &D, const ScenConst &C, Cyc &c, InstRegs<1> &S,
                                 double &Tcur, int &acc_delta, int &arrn, Stage &sg, int id0, int vg, int l,
                                 int nrem, double thr, int tentative, int &routed, bool &hit, bool &stopped) {
  const unsigned lane = lane_id();
  const bool cnd = (int)lane < c.I && S.v[0] >= vg;
  const long long k5l = (long long)P.k5 * l;
  {
    // gain after j further routes here: gamma holds for the (j+1)-th route iff the lane's instance
    // has no waiting work and kv + (j+1) k5 l <= M (kv only grows, so once false it stays false);
    // then T(n+j+1, kv+(j+1) k5 l) - T(n+j, kv+j k5 l).  The divisions are independent of each
    // other (branch-free div_int_rn), so they are issued together.
    const bool ok0 = cnd && S.w[0] == 0;
    double prev = Tcur;
#pragma unroll 4
    for (int j = 0; j < kGMax; ++j) {
      if (j >= nrem) break;
      const long long kvj = S.kv[0] + (long long)(j + 1) * k5l;
      const bool gj = ok0 && kvj <= P.M;
      const double Tn = gj ? throughput_d(P, S.n[0] + j + 1, kvj) : 0.0;
      sg.tab[j][lane] = gj ? __dsub_rn(Tn, prev) : 0.0;
      prev = Tn;
    }
  }
  __syncwarp();
  int jr = 0, done = 0, my_sel = 0, my_slot = 0;       // the group's lane-th route: instance, arrival slot
  const long long cmd0 = c.cmd_n;
  if (c.I <= kRepG) {
    // few instances: every lane evaluates the waterfall over all of them from the gain table
    // (broadcast shared-memory reads, per-instance route counts replicated), so the decision needs
    // no shuffle round; same order (version asc, dT desc, instance asc) as the reduction below
    int pr[kRepG], jq[kRepG];
#pragma unroll
    for (int q = 0; q < kRepG; ++q) {
      const int vq = __shfl_sync(0xffffffffu, S.v[0], q);
      pr[q] = (q < c.I && vq >= vg) ? vq : 0x7fffffff;
      jq[q] = 0;
    }
    for (; done < nrem; ++done) {
      int bp = 0x7fffffff, sel = -1;
      double bd = 0.0;
#pragma unroll
      for (int q = 0; q < kRepG; ++q) {
        const double d = pr[q] != 0x7fffffff ? sg.tab[jq[q]][q] : 0.0;
        const bool take = (d >= thr) & ((pr[q] < bp) | ((pr[q] == bp) & (d > bd)));
        bp = take ? pr[q] : bp;
        sel = take ? q : sel;
        bd = take ? d : bd;
      }
      if (sel < 0) { stopped = true; break; }
      if (tentative >= 0 && sel == tentative) { hit = true; return done + 1; }
      const int aslot = __shfl_sync(0xffffffffu, arrn, sel);
      if ((int)lane == sel) { ++jr; ++arrn; ++acc_delta; }
#pragma unroll
      for (int q = 0; q < kRepG; ++q) jq[q] += (int)(q == sel);
      if ((int)lane == done) { my_sel = sel; my_slot = aslot; }
    }
  } else
  for (; done < nrem; ++done) {
    const double my = cnd ? sg.tab[jr][lane] : 0.0;
    // waterfall as one reduction (see route_pass): lowest version with dT >= thr, then highest dT,
    // then lowest id
    int sel = -1;
    const int bk = waterfall_reduce((cnd && my >= thr) ? ((S.v[0] << 7) | (int)lane) : 0x7fffffff, my, c.red_w);
    if (bk != 0x7fffffff) sel = bk & 127;
    if (sel < 0) { stopped = true; break; }
    if (tentative >= 0 && sel == tentative) { hit = true; return done + 1; }
    const int aslot = __shfl_sync(0xffffffffu, arrn, sel);
    if ((int)lane == sel) { ++jr; ++arrn; ++acc_delta; }
    if ((int)lane == done) { my_sel = sel; my_slot = aslot; }   // issued after the loop
  }
  if (tentative < 0 && done > 0) {
    // the group's routes, lane-parallel (nothing in the loop reads what they write); versionless
    // members were never interrupted, so t_ready = t (A18).  Their Route records are consecutive
    // commands: checksum terms lane-parallel too.
    const bool mine = (int)lane < done;
    const long long idx = cmd0 + lane;
    const int id = id0 + 1 + (int)lane;
    if (mine) {
      const long long j = C.traj_off + id;
      D.loc[j] = L_TRANSIT;
      D.tinst[j] = (short)my_sel;
      atomicAdd(&D.n_routes[j], 1);
      D.arr_id[C.list_off + (long long)my_sel * C.cap + my_slot] = id;
      D.arr_t[C.list_off + (long long)my_sel * C.cap + my_slot] = c.t + P.r;
      const int r = routed + (int)lane;
      if (r < kArrStage) {
        sg.arr_t[r] = c.t + P.r;
        sg.arr_id[r] = id;
        sg.arr_inst[r] = (short)my_sel;
      }
    }
    routed += done;
    const unsigned long long h = mine ? record_hash(idx, c.window, CMD_ROUTE, my_sel, id) : 0ULL;
    if (mine && idx < P.cmdlog_cap) {
      long long *r = D.cmdlog + C.cmd_off + 4LL * idx;
      r[0] = c.window; r[1] = CMD_ROUTE; r[2] = my_sel; r[3] = id;
    }
    c.hash += warp_sum(h);
    c.cmd_n += done;
  }
  // the snapshot after jr routes to this lane's instance (Eq 3's S')
  for (int j = 0; j < jr; ++j) {
    if (S.w[0] == 0 && S.kv[0] + k5l <= P.M) { S.n[0] += 1; S.kv[0] += k5l; }
    else S.w[0] += 1;
  }
  if (jr) Tcur = throughput_d(P, S.n[0], S.kv[0]);
  __syncwarp();
  return done;
}

// Versioned MLQ items with few instances (I <= kRep, one instance per lane, Alg 2 waterfall):
// lane a holds prefetched item k0 + a plus, for every instance q, its version and its item's Eq 3
// gain and Eq 2 value there if routed (dT[q], Tn[q]).  A decision is the waterfall evaluated
// lane-locally in the item's lane and broadcast; the chosen instance's snapshot entry is read from
// its owner lane (shuffles), the owner applies the route, and every lane recomputes only its own
// item's gain on the chosen instance (operation trees as in the one-at-a-time pass, so the
// decisions are the same bit for bit).  Items are consumed in MLQ order until one is not routed
// (*stop) or, in an Alg 3 trial, one is routed to the tentative instance (*hit).  Returns the
// items decided (routed, plus the failing one if *stop).  Command records are hashed lane-parallel
// after the loop.
constexpr int kRep = 4;
static __device__ int route_versioned_rep(const GParams &P, const Dev &D, const ScenConst &C, Cyc &c, InstRegs<1> &S,
                                          double &Tcur, int &acc_delta, int &arrn, Stage &sg, int tentative, int nbv,
                                          int p_id, int p_vg, int p_l, long long p_ready, double p_thr, int &routed,
                                          bool &stop, bool &hit) {
  const unsigned lane = lane_id();
  const int I = c.I;
  int pr[kRep];                                         // waterfall priority: version, or INT_MAX if not a candidate
  double dT[kRep], Tn[kRep];
  unsigned cmask = 0;                                   // check_routable for a versioned item: v_i >= v_g
  const long long k5l = (long long)P.k5 * p_l;
  const int k5l_i = (int)k5l;                           // <= M < 2^30 (A27); kv < 2^31 (throughput_d)
#pragma unroll
  for (int q = 0; q < kRep; ++q) {
    const int rvq = __shfl_sync(0xffffffffu, S.v[0], q);
    const int nq = __shfl_sync(0xffffffffu, S.n[0], q);
    const int wq = __shfl_sync(0xffffffffu, S.w[0], q);
    const long long kvq = __shfl_sync(0xffffffffu, S.kv[0], q);
    const double Tq = __shfl_sync(0xffffffffu, Tcur, q);
    const bool cq = q < I && rvq >= p_vg;
    cmask |= (unsigned)cq << q;
    pr[q] = cq ? rvq : 0x7fffffff;
    dT[q] = 0.0;
    Tn[q] = 0.0;
    if (cq && wq == 0 && kvq + k5l <= P.M) {                                           // gamma (Eq 3)
      Tn[q] = throughput_d(P, nq + 1, kvq + k5l);
      dT[q] = __dsub_rn(Tn[q], Tq);
    }
  }
  int *const arr_id0 = D.arr_id + C.list_off;
  long long *const arr_t0 = D.arr_t + C.list_off;
  int a = 0, my_sel = 0, my_slot = 0;                   // this lane's item: instance and arrival slot
  SF_RT(0);
  for (; a < nbv; ++a) {
    // waterfall in this lane (meaningful in lane a): lowest version with dT >= thr, highest dT, lowest id
    // (a non-candidate has pr = INT_MAX and dT = 0, so it never beats the initial bd = 0)
    int bp = 0x7fffffff, bq = -1;
    double bd = 0.0, bt = 0.0;
#pragma unroll
    for (int q = 0; q < kRep; ++q) {
      const bool take = (dT[q] >= p_thr) & ((pr[q] < bp) | ((pr[q] == bp) & (dT[q] > bd)));
      bp = take ? pr[q] : bp;
      bq = take ? q : bq;
      bd = take ? dT[q] : bd;
      bt = take ? Tn[q] : bt;
    }
    const int sel = __shfl_sync(0xffffffffu, bq, a);
    if (sel < 0) { stop = true; break; }                 // no candidate / none clears thr
    if (tentative >= 0 && sel == tentative) { hit = true; return a + 1; }
    SF_RT(1);
    // the chosen instance's snapshot entry, from its owner lane; lane a's T(n+1, kv+k5 l) there
    const int k5la = __shfl_sync(0xffffffffu, k5l_i, a);
    const double tb = __shfl_sync(0xffffffffu, bt, a);
    int ns = __shfl_sync(0xffffffffu, S.n[0], sel);
    int ws = __shfl_sync(0xffffffffu, S.w[0], sel);
    int kvs = __shfl_sync(0xffffffffu, (int)S.kv[0], sel);
    double Ts = __shfl_sync(0xffffffffu, Tcur, sel);
    const int aslot = __shfl_sync(0xffffffffu, arrn, sel);
    const bool gamma = ws == 0 && (long long)kvs + k5la <= P.M;   // Step 5: Eq 3's S'
    if (gamma) { ns += 1; kvs += k5la; Ts = tb; } else { ws += 1; }
    if ((int)lane == sel) { S.n[0] = ns; S.w[0] = ws; S.kv[0] = kvs; Tcur = Ts; arrn += 1; acc_delta += 1; }
    SF_RT(2);
    double ds = 0.0, tn = 0.0;
    if (((cmask >> sel) & 1u) && ws == 0 && (long long)kvs + k5l_i <= P.M) {
      tn = throughput_nz(P, ns + 1, kvs + k5l_i);
      ds = __dsub_rn(tn, Ts);
    }
#pragma unroll
    for (int q = 0; q < kRep; ++q)
      if (q == sel) { dT[q] = ds; Tn[q] = tn; }
    SF_RT(3);
    if ((int)lane == a) { my_sel = sel; my_slot = aslot; }
    SF_RT(5);
  }
  if (tentative < 0 && a > 0) {
    // issue Route(sel, id) for items 0 .. a-1, lane-parallel (nothing in the loop reads what these
    // write): t_arr = t_ready + r (A18); then their command records (lane = position in the
    // command stream after cmd_n)
    const bool mine = (int)lane < a;
    if (mine) {
      const long long j = C.traj_off + p_id;
      const long long t_arr = max(c.t, p_ready) + P.r;
      D.loc[j] = L_TRANSIT;
      D.tinst[j] = (short)my_sel;
      atomicAdd(&D.n_routes[j], 1);
      const int ao = my_sel * C.cap + my_slot;            // < I (eta+1) B G < 2^31 (sf_create)
      arr_id0[ao] = p_id;
      arr_t0[ao] = t_arr;
      const int r = routed + (int)lane;
      if (r < kArrStage) {
        sg.arr_t[r] = t_arr;
        sg.arr_id[r] = p_id;
        sg.arr_inst[r] = (short)my_sel;
      }
      atomicAnd(&D.tsv_bits[C.bits_off + (p_id >> 5)], ~(1u << (p_id & 31)));
    }
    routed += a;
    const long long idx = c.cmd_n + lane;
    const unsigned long long h = mine ? record_hash(idx, c.window, CMD_ROUTE, my_sel, p_id) : 0ULL;
    if (mine && idx < P.cmdlog_cap) {
      long long *r = D.cmdlog + C.cmd_off + 4LL * idx;
      r[0] = c.window; r[1] = CMD_ROUTE; r[2] = my_sel; r[3] = p_id;
    }
    c.hash += warp_sum(h);
    c.cmd_n += a;
  }
  __syncwarp();
  return stop ? a + 1 : a;
}

// One routing pass (Alg 2, or vanilla §6.5) over the MLQ = [versioned n_v items] ++
// [versionless groups vl_head..n_ingested).  tentative >= 0: Alg 3 trial for that instance on
// scratch state, returns 1 as soon as a route targets it (early exit allowed).
// Otherwise issues Route commands and Reserves on the live ledger; returns routes issued.
// TRIAL (compile time): an Alg 3 trial (tentative_in >= 0) or the real pass (tentative_in ignored,
// -1): each instantiation drops the other's code -- the trial all writes, the pass the early exits.
template <int KS, bool TRIAL>
__device__ int route_pass(const GParams &P, const Dev &D, const ScenConst &C, Cyc &c, InstRegs<KS> &S,
                          int *sfree, int acc_delta[KS], int arrn[KS], Stage &sg, bool vanilla, int tentative_in) {
  const int tentative = TRIAL ? tentative_in : -1;
  if (TRIAL) __builtin_assume(tentative >= 0);
  const unsigned lane = lane_id();
  const int total = c.n_v + c.n_vl;
  int pass_group = -1, pass_vg = -1, routed = 0;
  unsigned vmask = verify_mask(sfree, c.eta);
  const int vbase = c.cu - c.eta;
  double Tcur[KS];                                   // Eq 2 of each owned instance's current S
  double Tn[KS];                                     // Eq 2 after routing the current item here (gamma)
#pragma unroll
  for (int q = 0; q < KS; ++q) Tcur[q] = throughput_d(P, S.n[q], S.kv[q]);
  int k = 0;
  bool stop = false;
  int knext = 0;
  {
    // the MLQ's first item has no candidate instance: stop before any prefetch.  It is
    // the lowest-version versioned item (candidates: v_i >= min_v) or, without versioned items, the
    // first member of a versionless group (candidates: verify(v_i), the bitmask vmask)
    bool any = false;
#pragma unroll
    for (int q = 0; q < KS; ++q) {
      const int i = (int)lane + 32 * q;
      any |= i < c.I && (c.n_v > 0 ? S.v[q] >= c.min_v
                                   : (S.v[q] >= vbase && ((vmask >> (S.v[q] - vbase)) & 1u)));
    }
    if (total > 0 && !__any_sync(0xffffffffu, any)) { stop = true; knext = total; }
  }
#ifdef SF_TIMING_ROUTE
  c.rt_last = clock64();
#endif
  while (knext < total && !stop) {
    const int k0 = knext;
    // prefetch 32 MLQ items: lane a holds item k0 + a, with its Eq 4 threshold mu * ideal(l)
    // (Alg 2 line P:1175) computed here, lane-parallel, off the decision chain
    int p_id = 0, p_vg = -1, p_l = 0;
    long long p_ready = 0;
    double p_thr = 0.0;
    {
      const int kk = k0 + (int)lane;
      if (kk < total) {
        p_id = kk < c.n_v ? D.mlq[C.mlq_off + kk] : c.vl_head * c.G + (kk - c.n_v);
        const int g = grp_of(P, p_id);
        p_vg = D.gv[C.grp_off + g];
        p_l = D.prompt[C.grp_off + g] + D.gen[C.traj_off + p_id];
        if (tentative < 0) p_ready = D.ready[C.traj_off + p_id];
        if (!vanilla) p_thr = __dmul_rn(P.mu, ideal_gain_d(P, p_l));
      }
    }
    const int nb = min(32, total - k0);
    int a = 0;
    SF_RT(0);
    if constexpr (KS == 1) {
#ifndef SF_NO_REP
      if (!vanilla && c.I <= kRep && k0 < c.n_v) {
#else
      if (false) {
#endif
        const int nbv = min(nb, c.n_v - k0);
        bool hit = false;
        const int done = route_versioned_rep(P, D, C, c, S, Tcur[0], acc_delta[0], arrn[0], sg, tentative, nbv, p_id,
                                             p_vg, p_l, p_ready, p_thr, routed, stop, hit);
        if (hit) return 1;
        if (stop) { k = k0 + done - 1; break; }
        knext = k0 + done;
        continue;
      }
    }
    for (; a < nb; ++a) {
      k = k0 + a;
      const int id = __shfl_sync(0xffffffffu, p_id, a);
      const int g = grp_of(P, id);
      int vg = __shfl_sync(0xffffffffu, p_vg, a);
      if (vg < 0 && g == pass_group) vg = pass_vg;
      const bool first_member = vg < 0;
      const int l = __shfl_sync(0xffffffffu, p_l, a);
      // Step 1: candidates (check_routable)
      bool cand[KS];
      bool any = false;
#pragma unroll
      for (int q = 0; q < KS; ++q) {
        const int i = (int)lane + 32 * q;
        cand[q] = i < c.I && (vg < 0 ? (S.v[q] >= vbase && ((vmask >> (S.v[q] - vbase)) & 1u)) : S.v[q] >= vg);
        any |= cand[q];
      }
      if (!__any_sync(0xffffffffu, any)) { stop = true; break; }
      const double thr_a = __shfl_sync(0xffffffffu, p_thr, a);
      int sel = -1;
      SF_RT(1);
      if (vanilla) {
        // fewest trajectories, lowest id
        long long best = 0x7fffffffffffffffLL;
#pragma unroll
        for (int q = 0; q < KS; ++q) {
          if (!cand[q]) continue;
          const long long key = ((long long)(S.n[q] + S.w[q]) << 8) | (lane + 32 * q);
          best = min(best, key);
        }
        for (int o = 1; o < c.red_w; o <<= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
        best = __shfl_sync(0xffffffffu, best, 0);
        sel = (int)(best & 0xff);
      } else {
        // Steps 2-4: waterfall over version groups.  The first group (by
        // ascending version) whose best dT clears thr = mu * ideal is the lowest version holding
        // ANY candidate with dT >= thr, and that group's argmax (highest dT, lowest id) is such a
        // candidate.  So one reduction on (version asc, dT desc, id asc) over the candidates with
        // dT >= thr gives the waterfall's choice (no candidate: withhold).
        const double thr = thr_a;
        int bk = 0x7fffffff;                               // version << 7 | instance
        double bd = 0.0;
#pragma unroll
        for (int q = 0; q < KS; ++q) {
          Tn[q] = 0.0;
          double d = 0.0;
          {
            // gamma (Eq 3); the division is issued for every owned instance (branch-free, the KS
            // divisions overlap) and its result kept only where gamma holds.  kv + k5 l <= M < 2^31.
            const long long kvl = S.kv[q] + (long long)P.k5 * l;
            const bool gam = cand[q] & (S.w[q] == 0) & (kvl <= P.M);
            const double t = throughput_nz(P, S.n[q] + 1, gam ? (int)kvl : 0);
            Tn[q] = gam ? t : 0.0;
            d = gam ? __dsub_rn(t, Tcur[q]) : 0.0;
          }
          const int key = (S.v[q] << 7) | ((int)lane + 32 * q);
          // branch-free (bitwise predicates + selects): data-dependent short-circuit branches
          // would diverge the warp on the decision chain
          const bool take = cand[q] & (d >= thr) & (((key >> 7) < (bk >> 7)) | (((key >> 7) == (bk >> 7)) & (d > bd)));
          bk = take ? key : bk;
          bd = take ? d : bd;
        }
        bk = waterfall_reduce(bk, bd, c.red_w);
        if (bk != 0x7fffffff) sel = bk & 127;               // accept (reading A4)
      }
      SF_RT(2);
      if (sel < 0) { stop = true; break; }
      // Step 5: route -- update S (Eq 3), Reserve if the group has no version yet.
      const int owner = sel & 31, qs = sel >> 5;
      int sv = 0, sw = 0;
      long long skv = 0;
#pragma unroll
      for (int q = 0; q < KS; ++q)
        if (q == qs) { sv = S.v[q]; sw = S.w[q]; skv = S.kv[q]; }
      sv = __shfl_sync(0xffffffffu, sv, owner);
      sw = __shfl_sync(0xffffffffu, sw, owner);
      skv = __shfl_sync(0xffffffffu, skv, owner);
      if (vg < 0) {
        vg = sv;
        int b = -1;
        for (int bb = vg + c.eta; bb >= max(vg, c.cu); --bb)
          if (sfree[bb - c.cu] > 0) { b = bb; break; }
        __syncwarp();
        if (lane == 0) sfree[b - c.cu] -= 1;
        __syncwarp();
        vmask = verify_mask(sfree, c.eta);
        if (tentative < 0) {
          // latest empty slot = highest index in ring buffer b
          const int ring = b % (c.eta + 1);
          const long long base = C.led_off + (long long)ring * c.B;
          int slot = -1;
          if (c.use_bits) {
            const int bw = (c.B + 31) >> 5;
            for (int w0 = bw - 1; w0 >= 0 && slot < 0; w0 -= 32) {
              const int w = w0 - (int)lane;
              const unsigned word = w >= 0 ? sg.empty[ring * bw + w] : 0u;
              const unsigned m = __ballot_sync(0xffffffffu, word != 0u);
              if (m) {
                const int l = __ffs(m) - 1;
                const unsigned ww = __shfl_sync(0xffffffffu, word, l);
                slot = ((w0 - l) << 5) + 31 - __clz(ww);
              }
            }
            __syncwarp();
            if (lane == 0) sg.empty[ring * bw + (slot >> 5)] &= ~(1u << (slot & 31));
          } else {
            for (int top = c.B - 1; top >= 0 && slot < 0; top -= 32) {
              const int sl = top - (int)lane;
              const bool e = sl >= 0 && D.led_st[base + sl] == E_EMPTY;
              const unsigned m = __ballot_sync(0xffffffffu, e);
              if (m) slot = top - (__ffs(m) - 1);
            }
          }
          if (lane == 0) {
            D.led_st[base + slot] = E_RESERVED;
            emp_mark(P, D, C, ring, slot, false);
            D.led_g[base + slot] = g;
            D.led_v[base + slot] = vg;
            D.led_b[C.grp_off + g] = b;
            D.led_s[C.grp_off + g] = slot;
            atomicAdd(&D.led_nres[C.ring_off + ring], 1);
            D.gv[C.grp_off + g] = vg;
          }
          __syncwarp();
          c.reserves += 1;
        }
        pass_group = g;
        pass_vg = vg;
      }
      const bool gamma = (skv + (long long)P.k5 * l <= P.M) && (sw == 0);
      if ((int)lane == owner) {
#pragma unroll
        for (int q = 0; q < KS; ++q)
          if (q == qs) {
            if (gamma) {
              S.n[q] += 1; S.kv[q] += (long long)P.k5 * l;
              Tcur[q] = vanilla ? throughput_d(P, S.n[q], S.kv[q]) : Tn[q];   // = T(n+1, kv+k5 l) (Eq 3's S')
            }
            else S.w[q] += 1;
          }
      }
      if (tentative >= 0 && sel == tentative) return 1;
      SF_RT(3);
      if (tentative < 0) {
      // issue Route(sel, id): t_arr = t_ready + r (A18)
      int aslot = 0;
#pragma unroll
      for (int q = 0; q < KS; ++q)
        if (q == qs) aslot = arrn[q];
      aslot = __shfl_sync(0xffffffffu, aslot, owner);
      if ((int)lane == owner) {
#pragma unroll
        for (int q = 0; q < KS; ++q)
          if (q == qs) { arrn[q] += 1; acc_delta[q] += 1; }
      }
      const long long rdy = __shfl_sync(0xffffffffu, p_ready, a);
      if (lane == 0) {
        const long long j = C.traj_off + id;
        const long long t_arr = max(c.t, rdy) + P.r;
        D.loc[j] = L_TRANSIT;
        D.tinst[j] = (short)sel;
        atomicAdd(&D.n_routes[j], 1);
        D.arr_id[C.list_off + (long long)sel * C.cap + aslot] = id;
        D.arr_t[C.list_off + (long long)sel * C.cap + aslot] = t_arr;
        if (routed < kArrStage) {
          sg.arr_t[routed] = t_arr;
          sg.arr_id[routed] = id;
          sg.arr_inst[routed] = (short)sel;
        }
        if (k < c.n_v) atomicAnd(&D.tsv_bits[C.bits_off + (id >> 5)], ~(1u << (id & 31)));
      }
      log_cmd(P, D, C, c, CMD_ROUTE, sel, id);
      ++routed;
      }
      SF_RT(4);
      // the rest of a versionless group (waterfall only), decided from precomputed gains
      if constexpr (KS == 1) {
        if (first_member && !vanilla && c.G > 1 && c.G <= kGMax && k >= c.n_v) {
          const int nrem = min(c.G - 1, total - (k + 1));
          if (nrem > 0) {
            bool hit = false, stopped = false;
            const int r = route_group_batch(P, D, C, c, S, Tcur[0], acc_delta[0], arrn[0], sg, id, vg, l, nrem,
                                            thr_a, tentative, routed, hit, stopped);
            if (hit) return 1;
            a += r;
            if (stopped) { k = k0 + a + 1; stop = true; break; }
          }
        }
      }
      SF_RT(5);
    }
    knext = k0 + a;
  }
  if (tentative >= 0) return 0;
  if (!stop) k = total;
  // TS bookkeeping for the versionless range (reading A11)
  if (k >= total) {
    c.vl_head = c.n_ingested;
  } else if (k >= c.n_v) {
    const int id = c.vl_head * c.G + (k - c.n_v);
    const int g = grp_of(P, id);
    if (g == pass_group) {
      // group versioned in this pass but only partly routed: its other members join the
      // versioned part of the TS
      for (int m = id + (int)lane; m < (g + 1) * c.G; m += 32) tsv_mark(D, C, m);
      c.vl_head = g + 1;
    } else {
      c.vl_head = g;
    }
  }
  __syncwarp();
  return routed;
}

// Interrupt (Table 1 row P:573; Alg 1 lines 6-8 / 10-11): victims of instance i are its run list
// (admission order) then its wait deque entries [w_lo, w_hi) (front -> back order).
static __device__ int interrupt_victims(const GParams &P, const Dev &D, const ScenConst &C, Cyc &c, int i, bool run_too,
                                 int w_lo, int w_hi) {
  const unsigned lane = lane_id();
  const long long gi = C.inst_off + i;
  const long long lb = C.list_off + (long long)i * C.cap;
  const long long apply_t = D.ist[gi] == I_TICK ? D.inb[gi] : c.t;
  const int nrun = run_too ? D.irun_n[gi] : 0;
  const int itk = D.itick[gi];                       // remaining = run_done - itick
  const int whead = D.iwhead[gi];
  const int nvict = nrun + (w_hi - w_lo);
  for (int k0 = 0; k0 < nvict; k0 += 32) {
    const int k = k0 + (int)lane;
    int id = -1;
    if (k < nvict) {
      if (k < nrun) {
        id = D.run_id[lb + k];
        const long long j = C.traj_off + id;
        D.gen[j] = D.T[j] - (D.run_done[lb + k] - itk);   // partial progress kept
      } else {
        int pos = whead + w_lo + (k - nrun);
        if (pos >= C.cap) pos -= C.cap;
        id = D.wait_id[lb + pos];
      }
      const long long j = C.traj_off + id;
      D.loc[j] = L_TS;
      D.ready[j] = apply_t;
      atomicAdd(&D.n_interrupt[j], 1);
      tsv_mark(D, C, id);
    }
    // one Interrupt record per victim, consecutive commands: lane k's record is the k-th
    const int nk = min(32, nvict - k0);
    const bool mine = (int)lane < nk;
    const long long idx = c.cmd_n + lane;
    const unsigned long long h = mine ? record_hash(idx, c.window, CMD_INTERRUPT, i, id) : 0ULL;
    if (mine && idx < P.cmdlog_cap) {
      long long *r = D.cmdlog + C.cmd_off + 4LL * idx;
      r[0] = c.window; r[1] = CMD_INTERRUPT; r[2] = i; r[3] = id;
    }
    c.hash += warp_sum(h);
    c.cmd_n += nk;
  }
  __syncwarp();
  return nvict;
}

// Order every instance's arrivals by (t_arr, id) (B6).  All route records of the cycle are
// staged in shared memory (when they fit): each record's rank among the records of its own
// instance is its position in that instance's arrival list.  Otherwise rank-sort one instance
// at a time through global memory and the free MLQ scratch.
static __device__ void order_arrivals_all(const GParams &P, const Dev &D, const ScenConst &C, const Stage &sg, int n_routed) {
  for (int e = lane_id(); e < n_routed; e += 32) {
    const int ie = sg.arr_id[e];
    const long long te = sg.arr_t[e];
    const int inst = sg.arr_inst[e];
    int rank = 0;
#pragma unroll 4
    for (int f = 0; f < n_routed; ++f) {                 // branch-free compare (no divergence)
      const long long tf = sg.arr_t[f];
      rank += (int)((sg.arr_inst[f] == inst) & ((tf < te) | ((tf == te) & (sg.arr_id[f] < ie))));
    }
    const long long lb = C.list_off + (long long)inst * C.cap;
    D.arr_id[lb + rank] = ie;
    D.arr_t[lb + rank] = te;
  }
  __syncwarp();
}

static __device__ void order_arrivals_global(const GParams &P, const Dev &D, const ScenConst &C, const Cyc &c, int i, int n) {
  // t_arr was stored with each route; rank every arrival against 32-wide coalesced chunks of the
  // list broadcast by shuffles, scatter (id, t) to the scratch, copy back in order.
  const unsigned lane = lane_id();
  const long long lb = C.list_off + (long long)i * C.cap;
  int *tid = D.mlq + C.mlq_off;                                  // [0, cap): ids
  long long *tt = (long long *)(D.mlq + ((C.mlq_off + C.cap + 1) & ~1LL));   // times, 8-byte aligned (3 cap + 2)
  for (int e0 = 0; e0 < n; e0 += 32) {
    const int e = e0 + (int)lane;
    const long long te = e < n ? D.arr_t[lb + e] : 0;
    const int ie = e < n ? D.arr_id[lb + e] : 0;
    int rank = 0;
    for (int f0 = 0; f0 < n; f0 += 32) {
      const int f = f0 + (int)lane;
      const long long tf = f < n ? D.arr_t[lb + f] : 0x7fffffffffffffffLL;
      const int jf = f < n ? D.arr_id[lb + f] : 0x7fffffff;
      const int nb = min(32, n - f0);
      for (int b = 0; b < nb; ++b) {
        const long long tb = __shfl_sync(0xffffffffu, tf, b);
        const int jb = __shfl_sync(0xffffffffu, jf, b);
        rank += (tb < te) || (tb == te && jb < ie);
      }
    }
    if (e < n) { tid[rank] = ie; tt[rank] = te; }
  }
  __syncwarp();
  for (int e = lane; e < n; e += 32) {
    D.arr_id[lb + e] = tid[e];
    D.arr_t[lb + e] = tt[e];
  }
  __syncwarp();
}

// One window of W0-W5 for scenario s, executed by one warp (sg: that warp's staging).
// C = D.sc[s], passed in so that a caller can load it (it is never written by a window) before
// waiting on the previous window's flag.
template <int KS>
__device__ __forceinline__ void coord_scenario(const GParams &P, const Dev &D, int s, Stage &sg, const ScenConst C) {
  const unsigned lane = lane_id();
  ScenState &SS = D.ss[s];
  const int err0 = SS.err;    // checked after the first loads below (all reads), not before them

  int *sfree = sg.sfree;
#ifdef SF_TIMING
  const long long t0_clk = clock64();
  long long ck[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#define SF_CK(k) ck[k] = clock64() - t0_clk
#else
#define SF_CK(k)
#endif

  Cyc c;
  c.t = SS.t; c.cu = SS.cu; c.ps = SS.ps; c.eta = C.eta; c.I = C.I; c.G = P.G; c.B = P.B;
  c.vl_head = SS.vl_head; c.n_ingested = SS.n_ingested; c.window = SS.window; c.min_live_g = SS.min_live_g;
  c.hash = SS.cmd_hash; c.cmd_n = SS.cmd_n; c.reserves = 0; c.mlq_err = 0; c.n_v = 0; c.n_vl = 0;
  c.use_bits = 0;
#ifdef SF_TIMING_ROUTE
  for (int q = 0; q < 6; ++q) c.rt[q] = 0;
#endif
  c.red_w = 1;
  while (c.red_w < min(C.I, 32)) c.red_w <<= 1;
  int live = SS.live, err = 0;
  int dbg_tent = 0;
  long long m_pub = 0, m_batches = 0, m_ingested = 0, m_valid = 0, m_invalid = 0, m_viol = 0;
  long long m_routes = 0, m_interrupts = 0, m_pulls = 0, m_reserves = 0, m_aborts = 0;
  const int nring = C.eta + 1;

  // ---------------- one memory round trip for W0, the oldest-live scan, W2 and the ledger view:
  // every load below depends only on C and SS, so all are issued before any of them is used.  A
  // Consume in W0 empties one ring (patched below) and, with redundancy, may Abort members on
  // instances (W2's fields are then reloaded).
  int nres_r = 0, nocc_r = 0;                           // lane r <= eta: counts of ring r
  if ((int)lane <= C.eta) { nres_r = D.led_nres[C.ring_off + lane]; nocc_r = D.led_nocc[C.ring_off + lane]; }
  int cvb = -1;
  {
    const int g = c.min_live_g + (int)lane;
    if (g < c.n_ingested) cvb = D.cvbuf[C.grp_off + g];
  }
  InstRegs<KS> S;
  bool ok = true;
  int err_eq1 = 0;
  auto load_w2 = [&]() {
    ok = true;
    err_eq1 = 0;
#pragma unroll
    for (int q = 0; q < KS; ++q) {
      const int i = lane + 32 * q;
      S.v[q] = 0; S.kv[q] = 0; S.n[q] = 0; S.w[q] = 0;
      if (i < C.I) {
        const long long gi = C.inst_off + i;
        const int kind = D.iintkind[gi], pp = D.ipullpend[gi], an = D.iarr_n[gi], st = D.ist[gi], ab = D.iabort[gi];
        const int pv = D.ipv[gi], v = D.iv[gi], acc = D.iacc[gi], rn = D.irun_n[gi], wn = D.iwn[gi], cc = D.ic[gi];
        const long long kv = D.ikv[gi];
        // bitwise, not short-circuit: the loads stay independent
        const bool quiescent = (kind == INT_NONE) & (pp == 0) & (an == 0) & (st != I_PULL) & (ab == 0);
        const bool eq1 = (pv == v) & (acc == rn + wn + cc);
        if (quiescent & !eq1) err_eq1 = ERR_EQ1;
        ok &= quiescent & eq1;
        S.v[q] = v; S.kv[q] = kv; S.n[q] = rn; S.w[q] = wn;
      }
    }
  };
  load_w2();
  const int bw = (P.B + 31) >> 5;
  c.use_bits = nring * bw <= kEmptyWords;
  const int nw = nring * bw;
  // the ledger's Empty-slot bitmap (D.led_emp, same word layout as sg.empty): word u * 32 + lane
  unsigned ew[kEmptyWords / 32];
#pragma unroll
  for (int u = 0; u < kEmptyWords / 32; ++u) {
    const int w = u * 32 + (int)lane;
    ew[u] = c.use_bits && w < nw ? D.led_emp[(long long)C.ring_off * bw + w] : 0u;
  }
  if (err0) return;
  int consumed_ring = -1;

  // ---------------- W0: auto trainer (reading A24): publish if due, then Consume if Ready
  if (P.atw > 0) {
    int busy = SS.trainer_busy;
    if (busy && SS.publish_at <= c.t) {
      c.ps += 1;
      m_pub = 1;
      busy = 0;
    }
    const int ring = c.cu % nring;
    if (!busy && __shfl_sync(0xffffffffu, nocc_r, ring) >= P.Br) {   // Ready (App C: >= B Occupied)
      CmdLog cl{c.hash, c.cmd_n, c.window, 0};
      const int retired = consume_buffer(P, D, C, SS, ring, c.cu, cl, err, nullptr);
      c.hash = cl.hash; c.cmd_n = cl.cmd_n; m_aborts = cl.aborts;
      if (lane == 0) {
        D.led_nocc[C.ring_off + ring] = 0;
        D.led_nres[C.ring_off + ring] = 0;
        SS.batch_n += 1;
        SS.publish_at = c.t + (long long)P.atw * P.delta;
      }
      if ((int)lane == ring) { nres_r = 0; nocc_r = 0; }
      consumed_ring = ring;
      live -= retired;
      busy = 1;
      c.cu += 1;
      m_batches = 1;
    }
    __syncwarp();
    if (lane == 0) SS.trainer_busy = busy;
    err = warp_max(err);
  }
  if (consumed_ring >= 0) {
    // the consumed ring is now all Empty; Aborted surplus members changed instance fields
#pragma unroll
    for (int u = 0; u < kEmptyWords / 32; ++u) {
      const int w = u * 32 + (int)lane;
      if (w >= consumed_ring * bw && w < (consumed_ring + 1) * bw) ew[u] = ~0u;
    }
    if (P.red && m_aborts > 0) load_w2();
  }
  // oldest live group (bounds the TS bitmap scan): skip consumed groups
  {
    bool first = consumed_ring < 0;                     // the prefetched first 32 groups are current
    for (;;) {
      const int g = c.min_live_g + (int)lane;
      int cv = cvb;
      if (!first) cv = g < c.n_ingested ? D.cvbuf[C.grp_off + g] : -1;
      first = false;
      const bool consumed = g < c.n_ingested && cv != -1;   // consumed or aborted
      const unsigned m = __ballot_sync(0xffffffffu, !consumed);
      if (m) { c.min_live_g += __ffs(m) - 1; break; }
      c.min_live_g += 32;
    }
  }
  // ---------------- W1: TS ingest up to (eta+1)*B live groups (A23)
  {
    const int n_pool = SS.n_pool;
    const int room = (C.eta + 1) * P.B - live;
    const int k = min(room, n_pool - c.n_ingested);
    if (k > 0) {
      const long long j0 = C.traj_off + (long long)c.n_ingested * P.G;
      for (long long a = lane; a < (long long)k * P.G; a += 32) D.loc[j0 + a] = L_TS;
      c.n_ingested += k;
      live += k;
      m_ingested = k;
    }
  }
  __syncwarp();
  // ---------------- W2: snapshot + Eq 1 (reading R-EQ1) on the fields loaded above
  int free_l = 0;
  {
    const int ring = (c.cu + lane) % nring;
    const int nr = __shfl_sync(0xffffffffu, nres_r, ring), no = __shfl_sync(0xffffffffu, nocc_r, ring);
    if ((int)lane <= C.eta) free_l = P.B - nr - no;
  }
  if (err_eq1) err = ERR_EQ1;
  err = warp_max(err);
  if (err == ERR_EQ1) m_viol += 1;
  const bool valid = __all_sync(0xffffffffu, ok) && !err;

  if (valid) {
    m_valid = 1;
    // working snapshot S in registers; ledger free counts of buffers cu..cu+eta in smem
    int acc_delta[KS], arrn[KS];
#pragma unroll
    for (int q = 0; q < KS; ++q) {
      acc_delta[q] = 0;
      arrn[q] = 0;
    }
    if ((int)lane <= C.eta) sfree[lane] = free_l;
    if (c.use_bits) {
      // ledger Empty-slot bitmap into shared memory (loaded above), bits >= B of each ring's last
      // word cleared (the Reserve search takes the highest set bit)
      const unsigned tail = (P.B & 31) ? (1u << (P.B & 31)) - 1u : ~0u;
#pragma unroll
      for (int u = 0; u < kEmptyWords / 32; ++u) {
        const int w = u * 32 + (int)lane;
        if (w < nw) sg.empty[w] = (w % bw == bw - 1) ? (ew[u] & tail) : ew[u];
      }
    }
    __syncwarp();
    const bool vanilla_route = !(C.strategy & 1), vanilla_sync = !(C.strategy & 2), sf_mig = (C.strategy & 4) != 0;
    int min_v = 0x7fffffff;
    c.n_v = build_mlq(P, D, C, c, sg, &min_v);
    if (min_v < 0) c.mlq_err = 1;
    c.min_v = min_v;
    c.n_vl = (c.n_ingested - c.vl_head) * c.G;

    SF_CK(0);
    // ---------------- W3: synchronization (Alg 3; vanilla P:788)
    unsigned selmask[KS];
#pragma unroll
    for (int q = 0; q < KS; ++q) {
      const int i = lane + 32 * q;
      bool elig = false;
      if (i < C.I) {
        if (vanilla_sync) elig = S.v[q] < c.ps;
        else elig = c.ps > S.v[q] && !((c.n_vl > 0 && verify_free(sfree, S.v[q], c.cu, c.eta)) ||
                                       (c.n_v > 0 && min_v <= S.v[q]));
      }
      selmask[q] = __ballot_sync(0xffffffffu, elig);
    }
    if (!vanilla_sync) {
#pragma unroll
      for (int q = 0; q < KS; ++q) {
        unsigned m = selmask[q], keep = 0;
        while (m) {
          const int li = __ffs(m) - 1;
          m &= m - 1;
          const int i = li + 32 * q;
          InstRegs<KS> T = S;
          if ((int)lane == li) T.v[q] = c.ps;             // S_temp[i].inst_version <- ps
          if ((int)lane <= C.eta) sg.sfree_tmp[lane] = sfree[lane];
          __syncwarp();
          int dummy_a[KS], dummy_b[KS];
#pragma unroll
          for (int qq = 0; qq < KS; ++qq) { dummy_a[qq] = 0; dummy_b[qq] = 0; }
          Cyc ct = c;
          ++dbg_tent;
          if (route_pass<KS, true>(P, D, C, ct, T, sg.sfree_tmp, dummy_a, dummy_b, sg, vanilla_route, i)) keep |= 1u << li;
        }
        selmask[q] = keep;
      }
    }
    // apply: Interrupt(i, run u wait) + Pull(i) for each selected i ascending (Alg 1 lines 3-8)
#pragma unroll
    for (int q = 0; q < KS; ++q) {
      unsigned m = selmask[q];
      while (m) {
        const int li = __ffs(m) - 1;
        m &= m - 1;
        const int i = li + 32 * q;
        const long long gi = C.inst_off + i;
        const int nv = interrupt_victims(P, D, C, c, i, true, 0, D.iwn[gi]);
        if (nv > 0 && lane == 0) { D.iintkind[gi] = INT_ALL; D.iintk[gi] = 0; }
        m_interrupts += nv;
        log_cmd(P, D, C, c, CMD_PULL, i, -1);
        m_pulls += 1;
        if (lane == 0) {
          D.ipullpend[gi] = 1;
          D.ipullv[gi] = c.ps;                 // version delivered = ps at issue (A19)
          D.ipv[gi] = c.ps;                    // Table 1 Pull row
          D.iacc[gi] = 0;
        }
        if ((int)lane == li) { S.v[q] = c.ps; S.kv[q] = 0; S.n[q] = 0; S.w[q] = 0; acc_delta[q] = 0; }
        __syncwarp();
      }
    }
    SF_CK(1);
    // ---------------- W4: migration (Alg 4), StaleFlow only (vanilla: none)
    if (sf_mig) {
      int k1[KS];
      double Tq[KS];
#pragma unroll
      for (int q = 0; q < KS; ++q) {
        const int i = lane + 32 * q;
        k1[q] = (i < C.I && S.w[q] > P.phi_wait) ? S.w[q] - P.phi_wait : 0;
        Tq[q] = throughput_d(P, S.n[q], S.kv[q]);
      }
      // argmax / argmin of Eq 2 with lowest-id ties (A9)
      double tmax = -1.0, tmin = 0.0;
      int imax = 0x7fffffff, imin = 0x7fffffff;
#pragma unroll
      for (int q = 0; q < KS; ++q) {
        const int i = lane + 32 * q;
        if (i >= C.I) continue;
        if (imax == 0x7fffffff || Tq[q] > tmax) { tmax = Tq[q]; imax = i; }
        if (imin == 0x7fffffff || Tq[q] < tmin) { tmin = Tq[q]; imin = i; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double oa = __shfl_xor_sync(0xffffffffu, tmax, o);
        const int oi = __shfl_xor_sync(0xffffffffu, imax, o);
        const bool bx = (oi != 0x7fffffff) & ((imax == 0x7fffffff) | (oa > tmax) | ((oa == tmax) & (oi < imax)));
        tmax = bx ? oa : tmax;
        imax = bx ? oi : imax;
        const double ob = __shfl_xor_sync(0xffffffffu, tmin, o);
        const int oj = __shfl_xor_sync(0xffffffffu, imin, o);
        const bool bn = (oj != 0x7fffffff) & ((imin == 0x7fffffff) | (ob < tmin) | ((ob == tmin) & (oj < imin)));
        tmin = bn ? ob : tmin;
        imin = bn ? oj : imin;
      }
      int case2 = -1;
      if (tmin > 0.0 && __ddiv_rn(tmax, tmin) > P.phi_tp) case2 = imax;      // A5, A6, A8
      // case 1 (ascending i), then case 2
#pragma unroll
      for (int q = 0; q < KS; ++q) {
        unsigned m = __ballot_sync(0xffffffffu, k1[q] > 0);
        while (m) {
          const int li = __ffs(m) - 1;
          m &= m - 1;
          const int i = li + 32 * q;
          const long long gi = C.inst_off + i;
          const int kk = __shfl_sync(0xffffffffu, k1[q], li);
          const int wn = D.iwn[gi];
          const int nv = interrupt_victims(P, D, C, c, i, false, wn - kk, wn);
          m_interrupts += nv;
          if (lane == 0) { D.iintkind[gi] = INT_WAIT_TAIL; D.iintk[gi] = kk; D.iacc[gi] -= nv; }
          if ((int)lane == li) S.w[q] -= kk;
          __syncwarp();
        }
      }
      if (case2 >= 0) {
        const int i = case2, q2 = i >> 5, li = i & 31;
        const long long gi = C.inst_off + i;
        int kk = 0;
#pragma unroll
        for (int qq = 0; qq < KS; ++qq)
          if (qq == q2) kk = k1[qq];
        kk = __shfl_sync(0xffffffffu, kk, li);
        const int wn = D.iwn[gi];
        const int nv = interrupt_victims(P, D, C, c, i, true, 0, wn - kk);
        m_interrupts += nv;
        if (lane == 0) { D.iintkind[gi] = INT_ALL; D.iintk[gi] = 0; D.iacc[gi] -= nv; }
        if ((int)lane == li) {
#pragma unroll
          for (int qq = 0; qq < KS; ++qq)
            if (qq == q2) { S.kv[qq] = 0; S.n[qq] = 0; S.w[qq] = 0; }
        }
        __syncwarp();
      }
    }
    SF_CK(2);
    // ---------------- W5: routing (Alg 2) over the TS incl. interrupted trajectories
    // (the versioned MLQ changes only if W3/W4 interrupted something: otherwise the first build stands)
    if (m_interrupts > 0) {
      c.n_v = build_mlq(P, D, C, c, sg, &min_v);
      if (min_v < 0) c.mlq_err = 1;
      c.min_v = min_v;
    }
    SF_CK(3);
#ifdef SF_TIMING
    const long long t_rp = clock64();
#endif
    const int nr = route_pass<KS, false>(P, D, C, c, S, sfree, acc_delta, arrn, sg, vanilla_route, -1);
#ifdef SF_TIMING
    dbg_tent = (int)(clock64() - t_rp);          // (slot 7) cycles in the real routing pass
#endif
    m_routes = nr;
    m_reserves = c.reserves;
    SF_CK(4);
    // write back per-instance route effects (Table 1 Route row)
#pragma unroll
    for (int q = 0; q < KS; ++q) {
      const int i = lane + 32 * q;
      if (i < C.I && (acc_delta[q] || arrn[q])) {
        const long long gi = C.inst_off + i;
        D.iacc[gi] += acc_delta[q];
        D.iarr_n[gi] = arrn[q];
      }
    }
    __syncwarp();
    // order each instance's arrivals by (t_arr, id) for B6
    if (nr <= kArrStage) {
      if (nr > 1) order_arrivals_all(P, D, C, sg, nr);
      else if (nr == 1 && lane == 0) {
        const long long lb = C.list_off + (long long)sg.arr_inst[0] * C.cap;
        D.arr_t[lb] = sg.arr_t[0];
      }
    } else {
      for (int i = 0; i < C.I; ++i) {
        int n = 0;
#pragma unroll
        for (int q = 0; q < KS; ++q)
          if ((int)lane + 32 * q == i) n = arrn[q];
        n = __shfl_sync(0xffffffffu, n, i & 31);
        if (n > 0) order_arrivals_global(P, D, C, c, i, n);
      }
    }
    SF_CK(5);
  } else {
    m_invalid = 1;
  }
  __syncwarp();
  if (lane == 0) {
    SS.ps = c.ps; SS.cu = c.cu; SS.live = live; SS.n_ingested = c.n_ingested; SS.vl_head = c.vl_head;
    SS.min_live_g = c.min_live_g;
    SS.cmd_hash = c.hash; SS.cmd_n = c.cmd_n;
    if (c.mlq_err) err = ERR_LEDGER;
    if (err) SS.err = err;
    metric_add(SS, M_PUBLISHES, m_pub);
    metric_add(SS, M_BATCHES, m_batches);
    metric_add(SS, M_INGESTED, m_ingested);
    metric_add(SS, M_VALID_SNAP, m_valid);
    metric_add(SS, M_INVALID_SNAP, m_invalid);
    metric_add(SS, M_VIOLATIONS, m_viol);
    metric_add(SS, M_ROUTES, m_routes);
    metric_add(SS, M_INTERRUPTS, m_interrupts);
    metric_add(SS, M_PULLS, m_pulls);
    metric_add(SS, M_RESERVES, m_reserves);
    metric_add(SS, M_ABORTS, m_aborts);
#ifdef SF_TIMING
    if (D.dbg) {
      D.dbg[8 * s + 0] = clock64() - t0_clk;
      D.dbg[8 * s + 1] = m_routes;
#ifdef SF_TIMING_ROUTE
      for (int q = 0; q < 6; ++q) D.dbg[8 * s + 2 + q] = c.rt[q];
#else
      for (int q = 0; q < 6; ++q) D.dbg[8 * s + 2 + q] = ck[q];
#endif
    }
#endif
  }
}

// The coordinator instantiated for scenario s's own instance count, up to the kernel's KS: in a
// mixed family (C4: I = 8 .. 128) a small scenario does not run the 4-instances-per-lane code.
template <int KS>
__device__ __forceinline__ void coord_scenario_fit(const GParams &P, const Dev &D, int s, Stage &sg, const ScenConst C) {
  if (KS == 1 || C.I <= 32) coord_scenario<1>(P, D, s, sg, C);
  else if (KS == 2 || C.I <= 64) coord_scenario<KS == 1 ? 1 : 2>(P, D, s, sg, C);
  else coord_scenario<KS>(P, D, s, sg, C);
}

}  // namespace sf
