// k_ledger.cu -- reward events -> staleness ledger (DESIGN.md §3.1 W8-W9, §3.3), external
// Consume, metric reduction and dump kernels.
//
// One warp per scenario.  Reward events of the window are put in (t_reward, trajectory id)
// order with a warp rank sort (keys t_complete + R, id), then applied in that order: mark the
// member; once the whole GRPO group is rewarded delete its Reserved entry and cascade
// earlier Reserved entries into the hole, then Occupy the earliest empty slot
// (P:366).  Slot searches are warp ballots over 32 slots at a time.
#include "sf_internal.cuh"

namespace sf {

constexpr int kWarps = 4;

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

__device__ void complete_group(const GParams &P, const Dev &D, const ScenConst &C, ScenState &SS, int g, int cu,
                               long long &m_reloc, long long &m_occ, int &err) {
  const unsigned lane = lane_id();
  const int B = P.B, eta = C.eta;
  int hb = D.led_b[C.grp_off + g], hs = D.led_s[C.grp_off + g];
  const int vg = D.gv[C.grp_off + g];
  {
    const long long base = ring_base(C, B, hb);
    if (D.led_st[base + hs] != E_RESERVED || D.led_g[base + hs] != g) { err = ERR_LEDGER; return; }
    __syncwarp();
    if (lane == 0) {
      D.led_st[base + hs] = E_EMPTY; D.led_g[base + hs] = -1; D.led_v[base + hs] = -1;
      D.led_nres[C.ring_off + hb % (eta + 1)] -= 1;
    }
    __syncwarp();
  }
  // delete-and-relocate cascade (reading A13)
  for (;;) {
    int fb = -1, fs = -1;
    for (int bb = cu; bb < hb; ++bb) {
      if (D.led_nres[C.ring_off + bb % (eta + 1)] == 0) continue;
      const long long base = ring_base(C, B, bb);
      const int hole = hb;
      const int sl = first_slot(B, [&](int x) {
        return D.led_st[base + x] == E_RESERVED && D.led_v[base + x] + eta >= hole;
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
  // Occupy: earliest buffer >= cu with an empty slot, lowest slot
  int ob = -1, os = -1;
  for (int b = cu; b <= cu + eta; ++b) {
    const int r = C.ring_off + b % (eta + 1);
    if (B - D.led_nres[r] - D.led_nocc[r] <= 0) continue;
    const long long base = ring_base(C, B, b);
    os = first_slot(B, [&](int x) { return D.led_st[base + x] == E_EMPTY; });
    if (os >= 0) { ob = b; break; }
  }
  if (ob < 0) { err = ERR_LEDGER; return; }
  if (ob < vg || ob > vg + eta) { err = ERR_STALENESS; atomicAdd(&SS.m[M_VIOLATIONS], lane == 0 ? 1ULL : 0ULL); }
  __syncwarp();
  if (lane == 0) {
    const long long dst = ring_base(C, B, ob) + os;
    D.led_st[dst] = E_OCCUPIED; D.led_g[dst] = g; D.led_v[dst] = vg;
    D.led_nocc[C.ring_off + ob % (eta + 1)] += 1;
    D.led_b[C.grp_off + g] = ob;
    D.led_s[C.grp_off + g] = os;
  }
  __syncwarp();
  ++m_occ;
}

constexpr int kEvStage = 256;     // reward events staged per warp in shared memory

struct EvStage {
  long long t[kEvStage];
  int id[kEvStage];
  int srt[kEvStage];
};

__global__ void __launch_bounds__(128) k_ledger(GParams P, Dev D) {
  __shared__ EvStage stage_all[kWarps];
  const int s = blockIdx.x * kWarps + (threadIdx.x >> 5);
  if (s >= P.n_scen) return;
  const unsigned lane = lane_id();
  const ScenConst C = D.sc[s];
  ScenState &SS = D.ss[s];
  if (SS.err) return;
  EvStage &es = stage_all[threadIdx.x >> 5];
  const long long t_end = SS.t + P.delta;
  const int n = SS.ev_n;
  const int cu = SS.cu;
  int err = 0;
  long long m_reloc = 0, m_occ = 0;
  int np = 0;
  if (n <= kEvStage) {
    // stage (t_complete, id), rank-sort by (t_reward, id) (W8) in shared memory
    for (int e = lane; e < n; e += 32) {
      const int id = D.ev_id[C.ev_off + e];
      es.id[e] = id;
      es.t[e] = D.t_complete[C.traj_off + id];
    }
    __syncwarp();
    for (int e = lane; e < n; e += 32) {
      const long long te = es.t[e];
      const int ie = es.id[e];
      int rank = 0;
      for (int f = 0; f < n; ++f) rank += es.t[f] < te || (es.t[f] == te && es.id[f] < ie);
      es.srt[rank] = e;
    }
    __syncwarp();
    // apply in order, 32 events per batch: the members' reward counters are loaded in parallel and
    // same-group events inside a batch are counted with __match_any_sync
    for (int k0 = 0; k0 < n; k0 += 32) {
      const int k = k0 + (int)lane;
      const bool valid = k < n;
      const int e = valid ? es.srt[k] : 0;
      const int id = es.id[e];
      const bool ok = valid && es.t[e] + P.R <= t_end;
      const int g = id / P.G;
      const unsigned okm = __ballot_sync(0xffffffffu, ok);
      const int nrw = ok ? D.n_rew[C.grp_off + g] : 0;
      const unsigned same = __match_any_sync(0xffffffffu, ok ? g : -1 - (int)lane);
      const int nr = nrw + 1 + __popc(same & lanemask_lt());
      if (ok && (same >> lane) == 1u) D.n_rew[C.grp_off + g] = nrw + __popc(same);   // last of its group
      unsigned cm = __ballot_sync(0xffffffffu, ok && nr == P.G);
      __syncwarp();
      while (cm) {
        const int l = __ffs(cm) - 1;
        cm &= cm - 1;
        complete_group(P, D, C, SS, __shfl_sync(0xffffffffu, g, l), cu, m_reloc, m_occ, err);
        if (err) break;
      }
      np += __popc(okm);
      if (err || okm != __ballot_sync(0xffffffffu, valid)) break;   // sorted: the rest are later
    }
    __syncwarp();
    for (int k = np + (int)lane; k < n; k += 32) D.ev_id[C.ev_off + k - np] = es.id[es.srt[k]];
  } else {
    int *tmp = D.mlq + C.mlq_off;                     // scratch (the MLQ is rebuilt per cycle)
    for (int e = lane; e < n; e += 32) {
      const int ie = D.ev_id[C.ev_off + e];
      const long long te = D.t_complete[C.traj_off + ie];
      int rank = 0;
      for (int f = 0; f < n; ++f) {
        const int jf = D.ev_id[C.ev_off + f];
        const long long tf = D.t_complete[C.traj_off + jf];
        rank += (tf < te) || (tf == te && jf < ie);
      }
      tmp[rank] = ie;
    }
    __syncwarp();
    for (; np < n; ++np) {
      const int id = tmp[np];
      if (D.t_complete[C.traj_off + id] + P.R > t_end) break;
      const int g = id / P.G;
      const int nr = D.n_rew[C.grp_off + g] + 1;
      __syncwarp();
      if (lane == 0) D.n_rew[C.grp_off + g] = nr;
      __syncwarp();
      if (nr == P.G) {
        complete_group(P, D, C, SS, g, cu, m_reloc, m_occ, err);
        if (err) break;
      }
    }
    for (int e = np + (int)lane; e < n; e += 32) D.ev_id[C.ev_off + e - np] = tmp[e];
  }
  __syncwarp();
  if (lane == 0) {
    SS.ev_n = n - np;
    SS.t = t_end;                                       // W9
    SS.window += 1;
    if (err) SS.err = err;
    metric_add(SS, M_WINDOWS, 1);
    metric_add(SS, M_RELOCATIONS, m_reloc);
    metric_add(SS, M_OCCUPIED, m_occ);
  }
}

// External-trainer Consume for one scenario; out[0] = status (0 ok, 1 not ready),
// out[1] = v_buf, then B (group, version) pairs.
__global__ void k_collect(GParams P, Dev D, int s, int *out) {
  const unsigned lane = lane_id();
  const ScenConst C = D.sc[s];
  ScenState &SS = D.ss[s];
  const int cu = SS.cu;
  const int ring = cu % (C.eta + 1);
  if (D.led_nocc[C.ring_off + ring] != P.B) { if (lane == 0) out[0] = 1; return; }
  const long long base = C.led_off + (long long)ring * P.B;
  const long long bl = C.batch_off + (long long)SS.batch_n * (1 + 2 * P.B);
  if (lane == 0) { out[0] = 0; out[1] = cu; D.batches[bl] = cu; }
  for (int k = lane; k < P.B; k += 32) {
    const int g = D.led_g[base + k], v = D.led_v[base + k];
    out[2 + 2 * k] = g; out[3 + 2 * k] = v;
    D.batches[bl + 1 + 2 * k] = g; D.batches[bl + 2 + 2 * k] = v;
    const int stal = cu - v;
    if (stal < 0 || stal > C.eta) { atomicAdd(&SS.m[M_VIOLATIONS], 1ULL); SS.err = ERR_STALENESS; }
    atomicAdd(&SS.m[M_HIST0 + min(max(stal, 0), 8)], 1ULL);
    D.cvbuf[C.grp_off + g] = cu;
    for (int m = 0; m < P.G; ++m) D.loc[C.traj_off + (long long)g * P.G + m] = L_CONSUMED;
    D.led_st[base + k] = E_EMPTY; D.led_g[base + k] = -1; D.led_v[base + k] = -1;
  }
  __syncwarp();
  if (lane == 0) {
    D.led_nocc[C.ring_off + ring] = 0;
    D.led_nres[C.ring_off + ring] = 0;
    SS.batch_n += 1;
    SS.cu = cu + 1;
    SS.live -= P.B;
    SS.m[M_BATCHES] += 1;
  }
}

// Sum of per-scenario metric vectors (integer, order independent) -> out[kMetrics].
__global__ void k_reduce_metrics(Dev D, int n_scen, long long *out) {
  __shared__ unsigned long long acc[kMetrics];
  if (threadIdx.x < kMetrics) acc[threadIdx.x] = 0;
  __syncthreads();
  for (int s = threadIdx.x >> 5; s < n_scen; s += blockDim.x >> 5) {
    const ScenState &SS = D.ss[s];
    const int k = threadIdx.x & 31;
    unsigned long long v = SS.m[k];
    if (k == M_CMD_HASH) v = SS.cmd_hash;
    if (k == M_SIM_TIME) v = (unsigned long long)SS.t;
    if (k == M_ERR_SCEN) v = SS.err != 0;
    if (k == M_MAX_T) atomicMax(&acc[k], (unsigned long long)SS.t);
    else atomicAdd(&acc[k], v);
  }
  __syncthreads();
  if (threadIdx.x < kMetrics) out[threadIdx.x] = (long long)acc[threadIdx.x];
}

// 13 int64 per trajectory (include/staleflow.h sf_dump_lifecycles)
__global__ void k_dump_lifecycles(GParams P, Dev D, int s, long long n_traj, long long *out) {
  const ScenConst C = D.sc[s];
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n_traj; j += (long long)gridDim.x * blockDim.x) {
    const long long a = C.traj_off + j;
    const int g = (int)(j / P.G);
    long long *r = out + 13 * j;
    r[0] = j; r[1] = g; r[2] = D.prompt[C.grp_off + g]; r[3] = D.T[a]; r[4] = D.gen[a];
    r[5] = D.gv[C.grp_off + g]; r[6] = D.loc[a]; r[7] = D.tinst[a]; r[8] = D.n_routes[a];
    r[9] = D.n_preempt[a]; r[10] = D.n_interrupt[a]; r[11] = D.cvbuf[C.grp_off + g]; r[12] = D.t_complete[a];
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
    out[13LL * id + 4] = D.T[C.traj_off + id] - D.run_rem[lb + k];
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

// desc[4k..4k+3] = (scenario, first group, n_groups, source group offset)
__global__ void k_scatter_pool(Dev D, int G, const int *desc, int n_desc, const int *prompt, const int *target) {
  const int k = blockIdx.x;
  if (k >= n_desc) return;
  const int s = desc[4 * k], g0 = desc[4 * k + 1], ng = desc[4 * k + 2], src = desc[4 * k + 3];
  const ScenConst C = D.sc[s];
  for (int a = threadIdx.x; a < ng; a += blockDim.x) D.prompt[C.grp_off + g0 + a] = prompt[src + a];
  for (long long a = threadIdx.x; a < (long long)ng * G; a += blockDim.x)
    D.T[C.traj_off + (long long)g0 * G + a] = target[(long long)src * G + a];
  if (threadIdx.x == 0) D.ss[s].n_pool = g0 + ng;
}

}  // namespace sf

void sf_launch_ledger(const sf::GParams &P, const sf::Dev &D, int n_scen, cudaStream_t st) {
  sf::k_ledger<<<(n_scen + sf::kWarps - 1) / sf::kWarps, 128, 0, st>>>(P, D);
}
void sf_launch_collect(const sf::GParams &P, const sf::Dev &D, int scen, int *out_dev, cudaStream_t st) {
  sf::k_collect<<<1, 32, 0, st>>>(P, D, scen, out_dev);
}
void sf_launch_reduce_metrics(const sf::Dev &D, int n_scen, long long *out_dev, cudaStream_t st) {
  sf::k_reduce_metrics<<<1, 1024, 0, st>>>(D, n_scen, out_dev);
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
                            const int *target_dev, cudaStream_t st) {
  if (n_desc > 0) sf::k_scatter_pool<<<n_desc, 256, 0, st>>>(D, G, desc_dev, n_desc, prompt_dev, target_dev);
}
