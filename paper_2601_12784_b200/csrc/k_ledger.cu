// k_ledger.cu -- reward -> ledger kernel (DESIGN.md §3.1 W8-W9; procedure ledger_scenario() in
// ledger.cuh), external Consume, metric reduction, dump and pool-scatter kernels.
#include "ledger.cuh"

namespace sf {

__global__ void __launch_bounds__(32 * kLedgerWarps) k_ledger(GParams P, Dev D) {
  __shared__ EvStage stage_all[kLedgerWarps];
  pdl_trigger();                                   // the next window's coordinator may be scheduled
  const int s = blockIdx.x * kLedgerWarps + (threadIdx.x >> 5);
  if (s >= P.n_scen) return;
  const ScenConst C = D.sc[s];                     // constant: its load overlaps the wait
  if (P.pdl) warp_wait_geq(&D.f_adv[s], P.epoch * C.I);   // all its instances advanced
  SF_TRACE_AT(4LL * s + 2);
  ledger_scenario(P, D, s, stage_all[threadIdx.x >> 5], C);
  SF_TRACE_AT(4LL * s + 3);
  fence_release();                                 // this lane's writes, device-wide
  __syncwarp();
  if ((threadIdx.x & 31) == 0) st_release(&D.f_led[s], P.epoch);
}

// External-trainer Consume for one scenario; out[0] = status (0 ok, 1 not ready),
// out[1] = v_buf, then Br (group, version) pairs (surplus groups Aborted, consume_buffer).
__global__ void k_collect(GParams P, Dev D, int s, int *out) {
  const unsigned lane = lane_id();
  const ScenConst C = D.sc[s];
  ScenState &SS = D.ss[s];
  const int cu = SS.cu;
  const int ring = cu % (C.eta + 1);
  if (D.led_nocc[C.ring_off + ring] < P.Br) { if (lane == 0) out[0] = 1; return; }
  if (lane == 0) { out[0] = 0; out[1] = cu; }
  CmdLog cl{SS.cmd_hash, SS.cmd_n, SS.window, 0};
  int err = 0;
  const int retired = consume_buffer(P, D, C, SS, ring, cu, cl, err, out + 2);
  err = warp_max(err);
  if (lane == 0) {
    D.led_nocc[C.ring_off + ring] = 0;
    D.led_nres[C.ring_off + ring] = 0;
    SS.batch_n += 1;
    SS.cu = cu + 1;
    SS.live -= retired;
    SS.cmd_hash = cl.hash; SS.cmd_n = cl.cmd_n;
    SS.m[M_BATCHES] += 1;
    SS.m[M_ABORTS] += cl.aborts;
    if (err) SS.err = err;
  }
}

// Proactive filtering (P:413 (2)) of group g of scenario s between windows; out[0] = 0 done,
// 1 the group has no ledger entry (not tracked: never routed, consumed or already dropped).
__global__ void k_filter(GParams P, Dev D, int s, int g, int *out) {
  const unsigned lane = lane_id();
  const ScenConst C = D.sc[s];
  ScenState &SS = D.ss[s];
  bool tracked = g >= 0 && g < SS.n_ingested && D.cvbuf[C.grp_off + g] == -1 && D.led_b[C.grp_off + g] >= 0;
  if (tracked) {
    const long long at = ring_base(C, P.B, D.led_b[C.grp_off + g]) + D.led_s[C.grp_off + g];
    tracked = D.led_st[at] != E_EMPTY && D.led_g[at] == g;
  }
  if (!tracked) { if (lane == 0) out[0] = 1; return; }
  CmdLog cl{SS.cmd_hash, SS.cmd_n, SS.window, 0};
  long long m_reloc = 0;
  int err = 0;
  filter_group(P, D, C, SS, g, SS.cu, cl, m_reloc, err);
  if (lane == 0) {
    out[0] = 0;
    SS.cmd_hash = cl.hash; SS.cmd_n = cl.cmd_n;
    SS.m[M_ABORTS] += cl.aborts;
    SS.m[M_RELOCATIONS] += m_reloc;
    if (err) SS.err = err;
  }
}

// Sum of per-scenario metric vectors (integer, order independent; slot 30 is a maximum) ->
// out[kMetrics].  Grid-wide: lane k of every warp accumulates metric k of a strided set of
// scenarios in a register (one coalesced 256-byte row per scenario), the warps of a block are
// combined in shared memory, and the last block to finish adds the per-block partials.
constexpr int kRedWarps = 8;
__global__ void __launch_bounds__(32 * kRedWarps) k_reduce_metrics(Dev D, int n_scen, long long *out) {
  __shared__ unsigned long long acc[kRedWarps][kMetrics];
  __shared__ bool last;
  const int warp = threadIdx.x >> 5, k = threadIdx.x & 31;
  const bool is_max = k == M_MAX_T;
  unsigned long long v = 0;
  for (int s = blockIdx.x * kRedWarps + warp; s < n_scen; s += gridDim.x * kRedWarps) {
    const ScenState &SS = D.ss[s];
    unsigned long long x = SS.m[k];
    if (k == M_CMD_HASH) x = SS.cmd_hash;
    if (k == M_SIM_TIME || k == M_MAX_T) x = (unsigned long long)SS.t;
    if (k == M_ERR_SCEN) x = SS.err != 0;
    v = is_max ? max(v, x) : v + x;
  }
  acc[warp][k] = v;
  __syncthreads();
  if (warp == 0) {
    unsigned long long t = 0;
#pragma unroll
    for (int w = 0; w < kRedWarps; ++w) t = is_max ? max(t, acc[w][k]) : t + acc[w][k];
    D.red_part[blockIdx.x * kMetrics + k] = t;
    __threadfence();
  }
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(D.red_ctr, 1u) == gridDim.x - 1;
  __syncthreads();
  if (last && warp == 0) {
    __threadfence();
    unsigned long long t = 0;
    for (int b = 0; b < (int)gridDim.x; ++b) {
      const unsigned long long x = D.red_part[b * kMetrics + k];
      t = is_max ? max(t, x) : t + x;
    }
    out[k] = (long long)t;
    if (k == 0) *D.red_ctr = 0;                    // ready for the next reduction on the stream
  }
}

// 13 int64 per trajectory (include/staleflow.h sf_dump_lifecycles)
__global__ void k_dump_lifecycles(GParams P, Dev D, int s, long long n_traj, long long *out) {
  const ScenConst C = D.sc[s];
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n_traj; j += (long long)gridDim.x * blockDim.x) {
    const long long a = C.traj_off + j;
    const int g = (int)(j / P.G);
    long long *r = out + 13 * j;
    r[0] = j; r[1] = g; r[2] = D.prompt[C.grp_off + g]; r[3] = D.T[a]; r[4] = D.gen[a];
    r[5] = D.gv[C.grp_off + g]; r[6] = D.loc[a] == L_REWARDED ? L_DONE : D.loc[a]; r[7] = D.tinst[a]; r[8] = D.n_routes[a];
    r[9] = D.n_preempt[a]; r[10] = D.n_interrupt[a]; r[11] = max(D.cvbuf[C.grp_off + g], -1); r[12] = D.t_complete[a];
  }
}
// running trajectories: gen = T - rem from the run lists
__global__ void k_dump_running(GParams P, Dev D, int s, long long *out) {
  const ScenConst C = D.sc[s];
  const int i = blockIdx.x;
  if (i >= C.I) return;
  const long long gi = C.inst_off + i;
  const long long lb = C.list_off + (long long)i * C.cap;
  for (int k = threadIdx.x; k < D.irun_n[gi]; k += blockDim.x) {
    const int id = D.run_id[lb + k];
    out[13LL * id + 4] = D.T[C.traj_off + id] - (D.run_done[lb + k] - D.itick[C.inst_off + i]);
  }
}

__global__ void k_dump_instances(GParams P, Dev D, int s, long long *out) {
  const ScenConst C = D.sc[s];
  for (int i = threadIdx.x; i < C.I; i += blockDim.x) {
    const long long gi = C.inst_off + i;
    long long *r = out + 7 * i;
    r[0] = D.iv[gi]; r[1] = D.ikv[gi]; r[2] = D.irun_n[gi]; r[3] = D.iwn[gi]; r[4] = D.ic[gi];
    r[5] = D.ist[gi];
    r[6] = D.ist[gi] == I_TICK ? D.inb[gi] : (D.ist[gi] == I_PULL ? D.iuntil[gi] : -1);
  }
}

// desc[4k..4k+3] = (scenario, first group, n_groups, source group offset).  Copies the groups into
// the pools and validates them on the way (prompt >= 0, 1 <= T <= lim - prompt with lim = M / k5,
// reading A27): *bad != 0 afterwards if any entry is invalid.  The pool counts are committed
// separately (k_commit_pool), only for a valid submission.
__global__ void k_scatter_pool(Dev D, int G, const int *desc, int n_desc, const int *prompt, const int *target, int lim,
                               int *bad) {
  const int k = blockIdx.x;
  if (k >= n_desc) return;
  const int s = desc[4 * k], g0 = desc[4 * k + 1], ng = desc[4 * k + 2], src = desc[4 * k + 3];
  const ScenConst C = D.sc[s];
  int b = 0;
  for (int a = threadIdx.x; a < ng; a += blockDim.x) {
    const int p = prompt[src + a];
    b |= p < 0;
    D.prompt[C.grp_off + g0 + a] = p;
  }
  for (long long a = threadIdx.x; a < (long long)ng * G; a += blockDim.x) {
    const int T = target[(long long)src * G + a];
    const int p = prompt[src + a / G];
    b |= (T < 1) | (T > lim - p);
    D.T[C.traj_off + (long long)g0 * G + a] = T;
  }
  if (__syncthreads_or(b) && threadIdx.x == 0) atomicOr(bad, 1);
}

__global__ void k_commit_pool(Dev D, const int *desc, int n_desc) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n_desc; k += gridDim.x * blockDim.x)
    D.ss[desc[4 * k]].n_pool = desc[4 * k + 1] + desc[4 * k + 2];
}

}  // namespace sf

void sf_launch_ledger(const sf::GParams &P, const sf::Dev &D, int n_scen, cudaStream_t st) {
  sf_launch_pdl(sf::k_ledger, (n_scen + sf::kLedgerWarps - 1) / sf::kLedgerWarps, 32 * sf::kLedgerWarps, st, P.pdl, P, D);
}
void sf_launch_collect(const sf::GParams &P, const sf::Dev &D, int scen, int *out_dev, cudaStream_t st) {
  sf::k_collect<<<1, 32, 0, st>>>(P, D, scen, out_dev);
}
void sf_launch_filter(const sf::GParams &P, const sf::Dev &D, int scen, int group, int *out_dev, cudaStream_t st) {
  sf::k_filter<<<1, 32, 0, st>>>(P, D, scen, group, out_dev);
}
void sf_launch_reduce_metrics(const sf::Dev &D, int n_scen, long long *out_dev, cudaStream_t st) {
  int blocks = (n_scen + 4 * sf::kRedWarps - 1) / (4 * sf::kRedWarps);     // >= 4 scenarios per warp
  blocks = blocks < 1 ? 1 : (blocks > sf::kRedBlocksMax ? sf::kRedBlocksMax : blocks);
  sf::k_reduce_metrics<<<blocks, 32 * sf::kRedWarps, 0, st>>>(D, n_scen, out_dev);
}
void sf_launch_dump_lifecycles(const sf::GParams &P, const sf::Dev &D, int scen, long long n_traj,
                               long long *out_dev, cudaStream_t st) {
  int blocks = (int)((n_traj + 255) / 256);
  if (blocks < 1) blocks = 1;
  if (blocks > 4096) blocks = 4096;
  sf::k_dump_lifecycles<<<blocks, 256, 0, st>>>(P, D, scen, n_traj, out_dev);
  sf::k_dump_running<<<sf::kMaxInst, 128, 0, st>>>(P, D, scen, out_dev);
}
void sf_launch_dump_instances(const sf::GParams &P, const sf::Dev &D, int scen, long long *out_dev,
                              cudaStream_t st) {
  sf::k_dump_instances<<<1, 128, 0, st>>>(P, D, scen, out_dev);
}
void sf_launch_scatter_pool(const sf::Dev &D, int G, const int *desc_dev, int n_desc, const int *prompt_dev,
                            const int *target_dev, int lim, int *bad_dev, cudaStream_t st) {
  if (n_desc > 0) sf::k_scatter_pool<<<n_desc, 256, 0, st>>>(D, G, desc_dev, n_desc, prompt_dev, target_dev, lim, bad_dev);
}
void sf_launch_commit_pool(const sf::Dev &D, const int *desc_dev, int n_desc, cudaStream_t st) {
  if (n_desc > 0) sf::k_commit_pool<<<(n_desc + 255) / 256, 256, 0, st>>>(D, desc_dev, n_desc);
}
