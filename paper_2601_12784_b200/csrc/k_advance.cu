// k_advance.cu -- decode advance of every rollout instance through one window
// (DESIGN.md §3.1 W6-W7, boundary procedure §3.2 B1-B8).
//
// One warp per instance; instances are independent inside a window (W7), which is the data
// parallelism of the step.  Per decode step the warp streams the instance's run list
// (`run_rem`, int32 remaining tokens; `run_id` only for compaction) with coalesced lane-
// contiguous loads, decrements every counter (one token per running trajectory),
// detects completions with __ballot_sync, compacts the survivors in place (stable, so the run
// list stays in admission order for LIFO preemption), and reduces the released KV with warp
// shuffles.  Everything per-instance (KV, counts, next step time) stays in registers across
// all steps of the window.
#include "sf_internal.cuh"

namespace sf {

constexpr long long kInf = 0x7fffffffffffffffLL;

__global__ void __launch_bounds__(256) k_advance(GParams P, Dev D, int n_inst_total) {
  const int gi = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (gi >= n_inst_total) return;
  const unsigned lane = lane_id();
  const int s = D.inst_scen[gi];
  const ScenConst C = D.sc[s];
  ScenState &SS = D.ss[s];
  if (SS.err) return;
  const int i = gi - C.inst_off;
  const long long t = SS.t, t_end = t + P.delta;
  const long long lb = C.list_off + (long long)i * C.cap;
  const int cap = C.cap;
  const int G = P.G;
  const long long k5 = P.k5;

  int st = D.ist[gi];
  long long nb = D.inb[gi], until = D.iuntil[gi];
  int pullv = D.ipullv[gi], pullpend = D.ipullpend[gi];
  int intkind = D.iintkind[gi], intk = D.iintk[gi];
  long long kv = D.ikv[gi], prefill = D.iprefill[gi];
  int cc = D.ic[gi], v = D.iv[gi];
  int run_n = D.irun_n[gi], whead = D.iwhead[gi], wn = D.iwn[gi];
  const int arr_n = D.iarr_n[gi];
  int arr_head = 0;
  long long ticks = 0, iters = 0, tokens = 0, comps = 0, preempts = 0;
  // W6: commands to an idle instance apply at a boundary at t
  long long t_cmd = (st == I_IDLE && (pullpend || intkind != INT_NONE)) ? t : kInf;

  for (;;) {
    long long b;
    if (st == I_TICK) b = nb;
    else if (st == I_PULL) b = until;
    else b = min(t_cmd, arr_head < arr_n ? D.arr_t[lb + arr_head] : kInf);
    if (b == kInf || b > t_end) break;
    t_cmd = kInf;
    const bool tick_end = (st == I_TICK);
    const bool pull_done = (st == I_PULL);
    // B1: pending interrupts leave without this step's token; KV released (A17, A18)
    if (!pull_done && intkind != INT_NONE) {
      if (intkind == INT_ALL) { run_n = 0; wn = 0; kv = 0; }
      else wn -= intk;                                  // wait tail (A7)
      intkind = INT_NONE;
    }
    if (tick_end) {
      // B2 + B3: credit one token to every running trajectory; completions leave in order
      const int n0 = run_n;
      int out = 0, ncomp = 0;
      long long release = 0;
      for (int base = 0; base < n0; base += 32) {
        const int k = base + (int)lane;
        const bool valid = k < n0;
        int rem = 1, id = 0;
        if (valid) { rem = D.run_rem[lb + k] - 1; id = D.run_id[lb + k]; }
        const bool done = valid && rem == 0;
        const bool keep = valid && !done;
        const unsigned mk = __ballot_sync(0xffffffffu, keep);
        const unsigned md = __ballot_sync(0xffffffffu, done);
        const int pos = out + __popc(mk & lanemask_lt());
        __syncwarp();
        if (keep) { D.run_rem[lb + pos] = rem; D.run_id[lb + pos] = id; }
        if (done) {
          const long long j = C.traj_off + id;
          const int Tj = D.T[j];
          release += k5 * (long long)(D.prompt[C.grp_off + id / G] + Tj);
          D.gen[j] = Tj;
          D.loc[j] = L_DONE;
          D.t_complete[j] = b;                          // reward due at b + R
          const int e = atomicAdd(&SS.ev_n, 1);
          D.ev_id[C.ev_off + e] = id;
        }
        out += __popc(mk);
        ncomp += __popc(md);
      }
      release = warp_sum(release);
      kv += k5 * n0 - release;
      tokens += n0;
      run_n = out;
      cc += ncomp;
      comps += ncomp;
      st = I_IDLE;
      __syncwarp();
    }
    if (pull_done) { v = pullv; cc = 0; st = I_IDLE; }
    // B4: preemption while KV exceeds M: newest admitted -> wait front (A21)
    while (kv > P.M && run_n > 0) {
      const int k = run_n - 1;
      const int id = D.run_id[lb + k];
      const long long j = C.traj_off + id;
      const int g_ = D.T[j] - D.run_rem[lb + k];
      kv -= k5 * (long long)(D.prompt[C.grp_off + id / G] + g_);
      whead = whead == 0 ? cap - 1 : whead - 1;
      if (lane == 0) {
        D.gen[j] = g_;
        D.loc[j] = L_WAIT;
        D.n_preempt[j] += 1;
        D.wait_id[lb + whead] = id;
      }
      ++wn;
      --run_n;
      ++preempts;
    }
    // B5: a pending Pull blocks generation for q
    if (pullpend) {
      pullpend = 0;
      st = I_PULL;
      until = b + P.q;
      __syncwarp();
      continue;
    }
    // B6: arrivals with t_arr <= b join the wait tail in (t_arr, id) order
    while (arr_head < arr_n && D.arr_t[lb + arr_head] <= b) {
      const int id = D.arr_id[lb + arr_head];
      int pos = whead + wn;
      if (pos >= cap) pos -= cap;
      if (lane == 0) { D.wait_id[lb + pos] = id; D.loc[C.traj_off + id] = L_WAIT; }
      ++wn;
      ++arr_head;
    }
    __syncwarp();
    // B7: FIFO admission while the head fits the KV budget
    while (wn > 0) {
      const int id = D.wait_id[lb + whead];
      const long long j = C.traj_off + id;
      const int gj = D.gen[j];
      const long long ctx = D.prompt[C.grp_off + id / G] + gj;
      if (kv + k5 * ctx > P.M) break;
      if (lane == 0) {
        D.run_id[lb + run_n] = id;
        D.run_rem[lb + run_n] = D.T[j] - gj;
        D.loc[j] = L_RUN;
      }
      kv += k5 * ctx;
      prefill += ctx;
      ++run_n;
      whead = whead + 1 == cap ? 0 : whead + 1;
      --wn;
    }
    __syncwarp();
    // B8: next decode step, Eq 7 + prefill stall (A20)
    if (run_n > 0) {
      nb = b + tick_latency(P, kv, run_n, prefill);
      prefill = 0;
      st = I_TICK;
      iters += run_n;
      ++ticks;
    } else {
      st = I_IDLE;
    }
  }
  // keep undelivered arrivals (held while pulling / later than the window) at the list front
  const int remain = arr_n - arr_head;
  if (arr_head > 0 && remain > 0) {
    for (int k0 = 0; k0 < remain; k0 += 32) {
      const int k = k0 + (int)lane;
      long long ta = 0;
      int ia = 0;
      if (k < remain) { ta = D.arr_t[lb + arr_head + k]; ia = D.arr_id[lb + arr_head + k]; }
      __syncwarp();
      if (k < remain) { D.arr_t[lb + k] = ta; D.arr_id[lb + k] = ia; }
      __syncwarp();
    }
  }
  if (lane == 0) {
    D.ist[gi] = st; D.inb[gi] = nb; D.iuntil[gi] = until;
    D.ipullpend[gi] = pullpend; D.iintkind[gi] = intkind;
    D.ikv[gi] = kv; D.iprefill[gi] = prefill; D.ic[gi] = cc; D.iv[gi] = v;
    D.irun_n[gi] = run_n; D.iwhead[gi] = whead; D.iwn[gi] = wn; D.iarr_n[gi] = remain;
    metric_add(SS, M_TICKS, ticks);
    metric_add(SS, M_TRAJ_ITERS, iters);
    metric_add(SS, M_TOKENS, tokens);
    metric_add(SS, M_COMPLETIONS, comps);
    metric_add(SS, M_PREEMPTIONS, preempts);
  }
}

}  // namespace sf

void sf_launch_advance(const sf::GParams &P, const sf::Dev &D, int n_inst_total, cudaStream_t st) {
  const int warps_per_block = 8;
  const int blocks = (n_inst_total + warps_per_block - 1) / warps_per_block;
  sf::k_advance<<<blocks, 32 * warps_per_block, 0, st>>>(P, D, n_inst_total);
}
