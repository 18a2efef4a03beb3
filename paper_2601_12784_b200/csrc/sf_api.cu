// sf_api.cu -- host implementation of include/staleflow.h: context, device memory layout,
// window launch sequence, transfers and dumps.  No simulation arithmetic runs on the host.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/staleflow.h"
#include "sf_internal.cuh"

using sf::Dev;
using sf::GParams;
using sf::ScenConst;
using sf::ScenState;

struct sf_ctx {
  GParams P{};
  Dev D{};
  std::vector<ScenConst> hsc;
  std::vector<int> hn_pool;
  int n_inst_total = 0;
  int max_inst = 1;
  int fused = 0;                      // launch mode: 1 = one fused window kernel (k_window)
  int block = 0;                      // launch mode: one block (or cluster) per scenario for the whole call
  struct BlockClass {                 // block mode: scenarios of one instance-count class (k_window_cluster)
    int ks = 1, cl = 1, n = 0, off = 0;
    cudaStream_t st = nullptr;        // classes after the first run on their own stream (fork / join)
    cudaEvent_t ev = nullptr;
  } bc[3];
  std::vector<int> hblist;            // scenario indices, class by class (device copy d_blist)
  int *d_blist = nullptr;
  cudaEvent_t ev_fork = nullptr;
  int pdl = 1;                        // programmatic dependent launch between window kernels
  int lanes = 0;                      // split mode: one-lane-per-instance advance kernel (SF_ADVANCE=lanes)
  int pdl_mask = 0;                   // debugging (SF_PDL_MASK): bit 0 serializes the advance, bit 1 the ledger
  int dyn = 1;                        // dataflow window kernel (k_dyn.cu)
  int dyn_blocks = 0;
  long long epoch = 0;                // split-mode windows launched (PDL flag targets)
  int n_scen = 0;
  int device = 0;
  cudaStream_t stream = nullptr;
  std::vector<void *> allocs;
  std::string err;
  int poisoned = 0;
  long long launches = 0;
  long long *d_metrics = nullptr;
  int *d_collect = nullptr;
  int *d_stage = nullptr;
  size_t stage_cap = 0;
  int *h_desc = nullptr;              // pinned staging of submit descriptors
  size_t h_desc_cap = 0;
  std::vector<int> pool_tmp;
  long long *d_dump = nullptr;
  size_t dump_cap = 0;
  // live per-kernel timing (sf_profile): CUDA events recorded around every window kernel
  int prof_on = 0;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<int> ev_kind;
  size_t ev_used = 0;
  double prof_ms[4] = {0, 0, 0, 0};
  long long prof_n[4] = {0, 0, 0, 0};
};

namespace {

sf_status fail(sf_ctx *c, sf_status st, const std::string &msg) {
  if (c) {
    c->err = msg;
    if (st == SF_E_STATE || st == SF_E_CUDA) c->poisoned = 1;
  }
  return st;
}

bool cuda_ok(sf_ctx *c, cudaError_t e, const char *what) {
  if (e == cudaSuccess) return true;
  if (c) {
    c->err = std::string(what) + ": " + cudaGetErrorString(e);
    c->poisoned = 1;
  }
  return false;
}

template <typename T>
bool dalloc(sf_ctx *c, T **p, long long count, int fill_byte) {
  size_t bytes = (size_t)std::max<long long>(count, 1) * sizeof(T);
  void *q = nullptr;
  if (cudaMalloc(&q, bytes) != cudaSuccess) return false;
  c->allocs.push_back(q);
  if (cudaMemsetAsync(q, fill_byte, bytes, c->stream) != cudaSuccess) return false;
  *p = (T *)q;
  return true;
}

sf_status check_ctx(sf_ctx *c) {
  if (!c) return SF_E_INVALID;
  if (c->poisoned) return SF_E_STATE;
  return SF_OK;
}

// Every call runs on the context's device and restores the caller's current device on return.
struct DevGuard {
  int prev = -1, dev = -1;
  explicit DevGuard(int d) : dev(d) {
    cudaGetDevice(&prev);
    if (prev != d) cudaSetDevice(d);
  }
  ~DevGuard() {
    if (prev >= 0 && prev != dev) cudaSetDevice(prev);
  }
};

sf_status read_state(sf_ctx *c, int s, ScenState *out) {
  if (!cuda_ok(c, cudaMemcpyAsync(out, c->D.ss + s, sizeof(ScenState), cudaMemcpyDeviceToHost, c->stream), "D2H state") ||
      !cuda_ok(c, cudaStreamSynchronize(c->stream), "sync"))
    return SF_E_CUDA;
  return SF_OK;
}

sf_status reduce_metrics_host(sf_ctx *c, long long *out) {
  sf_launch_reduce_metrics(c->D, c->n_scen, c->d_metrics, c->stream);
  c->launches++;
  if (!cuda_ok(c, cudaGetLastError(), "reduce launch") ||
      !cuda_ok(c, cudaMemcpyAsync(out, c->d_metrics, sizeof(long long) * sf::kMetrics, cudaMemcpyDeviceToHost, c->stream),
               "D2H metrics") ||
      !cuda_ok(c, cudaStreamSynchronize(c->stream), "sync"))
    return SF_E_CUDA;
  return SF_OK;
}

// metric slot 29 of the reduction counts poisoned scenarios
sf_status check_errors(sf_ctx *c, const long long *m) {
  if (m[sf::M_ERR_SCEN] == 0) return SF_OK;
  std::vector<ScenState> ss(c->n_scen);
  if (!cuda_ok(c, cudaMemcpyAsync(ss.data(), c->D.ss, sizeof(ScenState) * c->n_scen, cudaMemcpyDeviceToHost, c->stream),
               "D2H states") ||
      !cuda_ok(c, cudaStreamSynchronize(c->stream), "sync"))
    return SF_E_CUDA;
  for (int s = 0; s < c->n_scen; ++s) {
    if (ss[s].err) {
      char buf[160];
      if (ss[s].err == sf::ERR_DEADLOCK)
        snprintf(buf, sizeof buf, "scenario %d: deadlock (no progress, nothing pending, work left) at window %lld", s,
                 ss[s].window);
      else
        snprintf(buf, sizeof buf, "scenario %d: invariant violated (code %d) at window %lld", s, ss[s].err, ss[s].window);
      return fail(c, SF_E_STATE, buf);
    }
  }
  return fail(c, SF_E_STATE, "invariant violated");
}

void prof_mark(sf_ctx *c, int kind) {
  if (!c->prof_on) return;
  if (c->ev_used == c->ev_pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    c->ev_pool.push_back(e);
    c->ev_kind.push_back(0);
  }
  c->ev_kind[c->ev_used] = kind;
  cudaEventRecord(c->ev_pool[c->ev_used++], c->stream);
}

}  // namespace

extern "C" {

sf_status sf_create(int32_t instances, int32_t eta, int32_t group_size, const sf_config *cfg, sf_ctx **out) {
  if (!cfg || !out || group_size < 1 || group_size > 4096 || cfg->batch_size < 1 || cfg->n_scenarios < 1 || cfg->k5_tok < 1 ||
      cfg->snap_period_ps <= 0 || cfg->pool_capacity_groups < 1 || cfg->kv_budget_tok < 1 ||
      cfg->command_log_capacity < 0 || cfg->route_lat_ps < 0 || cfg->pull_lat_ps < 0 || cfg->reward_lat_ps < 0 ||
      cfg->auto_train_windows < 0 || cfg->extra_groups < 0 || cfg->extra_members < 0 ||
      group_size + cfg->extra_members > 4096 || cfg->extra_groups > (1 << 20))
    return SF_E_INVALID;
  // 32-bit products on the hot path (sf_internal.cuh tick_latency): k1, k3, kp, k5 < 2^31, M < 2^30
  if (cfg->k1_ps_per_tok < 0 || cfg->k1_ps_per_tok >= (1LL << 31) || cfg->k3_ps < 0 || cfg->k3_ps >= (1LL << 31) ||
      cfg->kprefill_ps_per_tok < 0 || cfg->kprefill_ps_per_tok >= (1LL << 31) || cfg->kv_budget_tok >= (1LL << 30) ||
      cfg->k2_ps < 0 || cfg->k4_ps < 0 || cfg->k2_ps + cfg->k4_ps < 1)   // Eq 7 denominator >= 1
    return SF_E_INVALID;
  sf_ctx *c = new (std::nothrow) sf_ctx();
  if (!c) return SF_E_NOMEM;
  c->device = cfg->device;
  int prev_dev = 0;
  cudaGetDevice(&prev_dev);
  if (cudaSetDevice(cfg->device) != cudaSuccess) { delete c; return SF_E_CUDA; }
  struct Restore { int d; ~Restore() { cudaSetDevice(d); } } restore{prev_dev};
  c->stream = (cudaStream_t)cfg->cuda_stream;
  // redundant rollout (App C): B buffer slots and G members per group include the extra ones;
  // Br groups form a batch and Gr rewarded members complete a group
  const int ns = cfg->n_scenarios, B = cfg->batch_size + cfg->extra_groups, G = group_size + cfg->extra_members;
  GParams &P = c->P;
  P.B = B; P.G = G;
  P.Br = cfg->batch_size; P.Gr = group_size;
  P.red = P.Br < B || P.Gr < G;
  P.abortable = P.red;
  P.filt = 0;
  P.k1 = cfg->k1_ps_per_tok; P.k2 = cfg->k2_ps; P.k3 = cfg->k3_ps; P.k4 = cfg->k4_ps;
  P.k5 = cfg->k5_tok; P.kp = cfg->kprefill_ps_per_tok; P.M = cfg->kv_budget_tok;
  P.k1i = (int)P.k1; P.k3i = (int)P.k3; P.kpi = (int)P.kp;
  P.gmag = ((1ULL << 40) + G - 1) / G;           // grp_of() multiply-shift (sf_internal.cuh)
  P.mu = cfg->mu; P.phi_tp = cfg->phi_throughput; P.phi_wait = cfg->phi_wait;
  P.delta = cfg->snap_period_ps; P.r = cfg->route_lat_ps; P.q = cfg->pull_lat_ps; P.R = cfg->reward_lat_ps;
  P.atw = cfg->auto_train_windows; P.pool_cap = cfg->pool_capacity_groups;
  P.wd = cfg->watchdog_windows > 0 ? cfg->watchdog_windows : 0;
  P.cmdlog_cap = cfg->command_log_capacity; P.n_scen = ns;
  c->n_scen = ns;
  c->hsc.resize(ns);
  c->hn_pool.assign(ns, 0);
  long long inst = 0, led = 0, ring = 0, list = 0, bits = 0, mlq = 0, ev = 0, batch = 0, cmd = 0;
  const long long pool_traj = (long long)P.pool_cap * G;
  // TS bitmap words per scenario, padded to whole 32-word chunks (build_mlq reads whole chunks), and
  // the chunk-summary words (one bit per chunk)
  const long long bwords = ((pool_traj + 31) / 32 + 31) / 32 * 32;
  const long long swords = (bwords / 32 + 31) / 32;
  const long long batch_rec = (long long)(P.pool_cap / P.Br + 1) * (1 + 2 * P.Br);
  for (int s = 0; s < ns; ++s) {
    ScenConst &S = c->hsc[s];
    S.I = cfg->scenario_instances ? cfg->scenario_instances[s] : instances;
    S.eta = cfg->scenario_eta ? cfg->scenario_eta[s] : eta;
    S.strategy = (int)(cfg->scenario_strategy ? cfg->scenario_strategy[s] : cfg->strategy);
    // grp_of() (sf_internal.cuh): id * gmag must fit in 64 bits for every id < pool_traj, and the
    // multiply-shift is exact for id < 2^40 / G (both follow from this check for G <= 4096)
    const bool grp_ok = pool_traj < (1LL << 27) &&
                        ((unsigned __int128)(unsigned long long)(pool_traj - 1) * P.gmag >> 64) == 0 &&
                        (pool_traj - 1) < (long long)((1ULL << 40) / (unsigned long long)G);
    if (S.I < 1 || S.I > sf::kMaxInst || S.eta < 0 || S.eta > sf::kMaxEta || !grp_ok) {
      delete c;
      return SF_E_INVALID;
    }
    const long long cap64 = (long long)(S.eta + 1) * B * G;
    // every per-scenario offset below is narrowed to int (or indexes int-sized lists): reject any
    // configuration whose offsets reach 2^31 before narrowing
    if (cap64 * S.I >= (1LL << 31) || (long long)(s + 1) * P.pool_cap >= (1LL << 31) ||
        inst + S.I >= (1LL << 31) || led + (long long)(S.eta + 1) * B >= (1LL << 31) || ring + S.eta + 1 >= (1LL << 31)) {
      delete c;
      return SF_E_INVALID;
    }
    S.cap = (int)cap64;
    S.inst_off = (int)inst; S.grp_off = s * P.pool_cap; S.led_off = (int)led; S.ring_off = (int)ring;
    S.traj_off = (long long)s * pool_traj; S.list_off = list; S.bits_off = bits; S.mlq_off = mlq;
    S.ev_off = ev; S.batch_off = batch; S.cmd_off = cmd;
    S.sum_off = (int)(s * swords);
    c->max_inst = std::max(c->max_inst, S.I);
    inst += S.I; led += (long long)(S.eta + 1) * B; ring += S.eta + 1; list += (long long)S.I * S.cap;
    bits += bwords; mlq += 3LL * S.cap + 2; ev += S.cap; batch += batch_rec; cmd += 4LL * P.cmdlog_cap;
  }
  c->n_inst_total = (int)inst;
  // launch mode: three kernels per window with programmatic dependent launch by
  // default (SF_PDL=0: serialized); SF_LAUNCH=dyn the dataflow window kernel, SF_LAUNCH=fused the
  // fused per-scenario window kernel (tests run every mode)
  c->fused = 0;
  c->dyn = 0;
  // decode-step mode: closed-form skipping of quiet steps by default;
  // SF_ADVANCE=step processes every decode step individually (tests run both)
  c->P.skip = 1;
  // programmatic dependent launch between the window kernels; SF_PDL=0 disables
  c->pdl = 1;
  if (const char *m = getenv("SF_PDL")) c->pdl = strcmp(m, "0") != 0;
  if (const char *m = getenv("SF_PDL_MASK")) c->pdl_mask = atoi(m);
  c->P.pdl = 0;
  c->P.epoch = 0;
  // decode-advance kernel: one warp per instance with closed-form quiet steps by
  // default; SF_ADVANCE=step the same one step at a time; SF_ADVANCE=lanes one lane per instance
  // (advance_lanes.cuh; bit-exact, measured slower on C5)
  c->lanes = 0;
  if (const char *m = getenv("SF_ADVANCE")) {
    c->P.skip = strcmp(m, "step") != 0;
    c->lanes = strcmp(m, "lanes") == 0;
  }
  // few scenarios: one block per scenario for the whole call (k_window_cluster, the window's phases
  // separated by barriers instead of kernel launches) -- a 16-warp block for I <= 32, a cluster of 2
  // blocks for 32 < I <= 64, of 4 (8 when the GPU holds them all at once) for I > 64, so that a
  // large scenario's advance spreads over several SMs; used when every block has an SM of its own.
  // Many scenarios: the three-kernel split with programmatic dependent launch.
  // SF_CLUSTER=1 runs every class without clusters, SF_CLUSTER=4 / 8 fixes the I > 64 cluster.
  {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cfg->device);
    std::vector<int> cls[3];
    for (int s = 0; s < ns; ++s) cls[c->hsc[s].I <= 32 ? 0 : c->hsc[s].I <= 64 ? 1 : 2].push_back(s);
    int clB = 2, clC = 4;
    const char *ce = getenv("SF_CLUSTER");
    if (ce && atoi(ce) == 1) clB = clC = 1;
    if (ce && (atoi(ce) == 4 || atoi(ce) == 8)) clC = atoi(ce);
    const long long nA = (long long)cls[0].size(), nB = (long long)cls[1].size(), nC = (long long)cls[2].size();
    if (!ce && nC > 0 && nA + clB * nB + 8 * nC <= sms && sf_max_active_clusters(4, 8) >= nC) clC = 8;
    c->block = nA + clB * nB + clC * nC <= sms;
    const int ks[3] = {1, 2, 4}, cl[3] = {1, clB, clC};
    for (int k = 0; k < 3; ++k) {
      c->bc[k].ks = ks[k];
      c->bc[k].cl = cl[k];
      c->bc[k].n = (int)cls[k].size();
      c->bc[k].off = (int)c->hblist.size();
      c->hblist.insert(c->hblist.end(), cls[k].begin(), cls[k].end());
    }
  }
  if (const char *m = getenv("SF_LAUNCH")) {
    if (!strcmp(m, "split")) { c->fused = 0; c->dyn = 0; c->block = 0; }
    if (!strcmp(m, "fused")) { c->fused = c->max_inst <= 32; c->dyn = 0; c->block = 0; }
    if (!strcmp(m, "dyn")) { c->fused = 0; c->dyn = 1; c->block = 0; }
    if (!strcmp(m, "block")) { c->fused = 0; c->dyn = 0; c->block = 1; }
  }
  const long long ntraj = (long long)ns * pool_traj, ngrp = (long long)ns * P.pool_cap;
  Dev &D = c->D;
  bool ok = true;
  ScenConst *dsc = nullptr;
  ScenState *dss = nullptr;
  int *dinst_scen = nullptr;
  ok = ok && dalloc(c, &dsc, ns, 0) && dalloc(c, &dss, ns, 0) && dalloc(c, &dinst_scen, inst, 0) &&
       dalloc(c, &c->d_blist, ns, 0);
  ok = ok && dalloc(c, &D.T, ntraj, 0) && dalloc(c, &D.gen, ntraj, 0) && dalloc(c, &D.loc, ntraj, 0) &&
       dalloc(c, &D.tinst, ntraj, 0xFF) && dalloc(c, &D.n_routes, ntraj, 0) && dalloc(c, &D.n_preempt, ntraj, 0) &&
       dalloc(c, &D.n_interrupt, ntraj, 0) && dalloc(c, &D.t_complete, ntraj, 0xFF) && dalloc(c, &D.ready, ntraj, 0);
  ok = ok && dalloc(c, &D.prompt, ngrp, 0) && dalloc(c, &D.gv, ngrp, 0xFF) && dalloc(c, &D.n_rew, ngrp, 0) &&
       dalloc(c, &D.led_b, ngrp, 0xFF) && dalloc(c, &D.led_s, ngrp, 0xFF) && dalloc(c, &D.cvbuf, ngrp, 0xFF) &&
       dalloc(c, &D.gfilt, ngrp, 0);
  ok = ok && dalloc(c, &D.iv, inst, 0) && dalloc(c, &D.ic, inst, 0) && dalloc(c, &D.ist, inst, 0) &&
       dalloc(c, &D.ipullv, inst, 0) && dalloc(c, &D.ipullpend, inst, 0) && dalloc(c, &D.iintkind, inst, 0) &&
       dalloc(c, &D.iintk, inst, 0) && dalloc(c, &D.irun_n, inst, 0) && dalloc(c, &D.iwhead, inst, 0) &&
       dalloc(c, &D.iwn, inst, 0) && dalloc(c, &D.iarr_n, inst, 0) && dalloc(c, &D.ipv, inst, 0) &&
       dalloc(c, &D.iacc, inst, 0) && dalloc(c, &D.ikv, inst, 0) && dalloc(c, &D.inb, inst, 0) &&
       dalloc(c, &D.iuntil, inst, 0) && dalloc(c, &D.iprefill, inst, 0) && dalloc(c, &D.iabort, inst, 0) &&
       dalloc(c, &D.iabort_arr, inst, 0) &&
       dalloc(c, &D.f_coord, ns, 0) && dalloc(c, &D.f_adv, ns, 0) && dalloc(c, &D.f_led, ns, 0) &&
       dalloc(c, &D.q_ctr, 4 + (long long)ns + inst + ns, 0) &&
       dalloc(c, &D.red_part, (long long)sf::kRedBlocksMax * sf::kMetrics, 0) && dalloc(c, &D.red_ctr, 1, 0);
  if (ok) {
    D.q_done = D.q_ctr + 4;
    D.q_tasks = D.q_done + ns;
    D.q_total = (int)(inst + ns);
  }
  ok = ok && dalloc(c, &D.run_T, list, 0) && dalloc(c, &D.run_fin, list, 0) && dalloc(c, &D.iev, list, 0) &&
       dalloc(c, &D.iev_n, inst, 0);
  ok = ok && dalloc(c, &D.run_id, list, 0) && dalloc(c, &D.run_done, list, 0) && dalloc(c, &D.itick, inst, 0) && dalloc(c, &D.wait_id, list, 0) &&
       dalloc(c, &D.arr_id, list, 0) && dalloc(c, &D.arr_t, list, 0);
  ok = ok && dalloc(c, &D.led_st, led, 0) && dalloc(c, &D.led_g, led, 0xFF) && dalloc(c, &D.led_v, led, 0xFF) &&
       dalloc(c, &D.led_nres, ring, 0) && dalloc(c, &D.led_nocc, ring, 0);
  ok = ok && dalloc(c, &D.ev_t, 1, 0) && dalloc(c, &D.ev_id, ev, 0) && dalloc(c, &D.tsv_bits, bits, 0) &&
       dalloc(c, &D.tsv_sum, (long long)ns * swords, 0) && dalloc(c, &D.led_emp, ring * ((B + 31) / 32), 0xFF) &&
       dalloc(c, &D.mlq, mlq, 0) && dalloc(c, &D.batches, batch, 0) && dalloc(c, &D.cmdlog, cmd, 0);
  ok = ok && dalloc(c, &c->d_metrics, 2 * sf::kMetrics, 0) && dalloc(c, &c->d_collect, 2 + 2 * P.Br, 0);
  if (!ok) {
    sf_destroy(c);
    return SF_E_NOMEM;
  }
#ifdef SF_TIMING
  ok = dalloc(c, &D.dbg, 8LL * ns, 0) && dalloc(c, &D.dbg2, 8LL * inst, 0);
#else
  D.dbg = nullptr;
  D.dbg2 = nullptr;
#endif
#ifdef SF_TRACE
  ok = ok && dalloc(c, &D.trace, 4LL * ns + 2LL * inst, 0);
#else
  D.trace = nullptr;
#endif
  D.sc = dsc;
  D.ss = dss;
  D.inst_scen = dinst_scen;
  std::vector<int> hinst_scen(inst);
  for (int s = 0; s < ns; ++s)
    for (int i = 0; i < c->hsc[s].I; ++i) hinst_scen[c->hsc[s].inst_off + i] = s;
  std::vector<ScenState> hss(ns);
  std::memset(hss.data(), 0, sizeof(ScenState) * ns);
  bool cp = cudaMemcpyAsync(dsc, c->hsc.data(), sizeof(ScenConst) * ns, cudaMemcpyHostToDevice, c->stream) == cudaSuccess &&
            cudaMemcpyAsync(dss, hss.data(), sizeof(ScenState) * ns, cudaMemcpyHostToDevice, c->stream) == cudaSuccess &&
            cudaMemcpyAsync(dinst_scen, hinst_scen.data(), sizeof(int) * inst, cudaMemcpyHostToDevice, c->stream) == cudaSuccess &&
            cudaMemcpyAsync(c->d_blist, c->hblist.data(), sizeof(int) * ns, cudaMemcpyHostToDevice, c->stream) == cudaSuccess &&
            cudaStreamSynchronize(c->stream) == cudaSuccess;
  // block mode with several classes: one stream and event per class after the first (fork / join)
  if (cp && c->block && (c->bc[0].n > 0) + (c->bc[1].n > 0) + (c->bc[2].n > 0) > 1) {
    cp = cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) == cudaSuccess;
    for (int k = 0; k < 3 && cp; ++k)
      cp = cudaStreamCreateWithFlags(&c->bc[k].st, cudaStreamNonBlocking) == cudaSuccess &&
           cudaEventCreateWithFlags(&c->bc[k].ev, cudaEventDisableTiming) == cudaSuccess;
  }
  if (!cp) {
    sf_destroy(c);
    return SF_E_CUDA;
  }
  *out = c;
  return SF_OK;
}

void sf_destroy(sf_ctx *c) {
  if (!c) return;
  DevGuard dg(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  else cudaDeviceSynchronize();
  for (void *p : c->allocs) cudaFree(p);
  if (c->d_stage) cudaFree(c->d_stage);
  if (c->d_dump) cudaFree(c->d_dump);
  if (c->h_desc) cudaFreeHost(c->h_desc);
  for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
  for (auto &b : c->bc) {
    if (b.st) { cudaStreamSynchronize(b.st); cudaStreamDestroy(b.st); }
    if (b.ev) cudaEventDestroy(b.ev);
  }
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  delete c;
}

sf_status sf_submit_prompts_many(sf_ctx *c, int32_t n, const int32_t *scen_ids, const int32_t *n_groups,
                                 const int32_t *prompt, const int32_t *target) {
  sf_status st = check_ctx(c);
  if (st != SF_OK) return st;
  DevGuard dg(c->device);
  if (n < 0 || (n > 0 && (!scen_ids || !n_groups || !prompt || !target))) return fail(c, SF_E_INVALID, "null argument");
  const int G = c->P.G;
  // descriptors and capacity checks on the host; the per-element validation (A27) runs inside the
  // scatter kernel, and the pool counts are committed only if it found nothing invalid
  if ((size_t)4 * n > c->h_desc_cap) {
    if (c->h_desc) cudaFreeHost(c->h_desc);
    c->h_desc = nullptr;
    c->h_desc_cap = 0;
    if (cudaMallocHost(&c->h_desc, sizeof(int) * 4 * (size_t)n + sizeof(int)) != cudaSuccess)
      return fail(c, SF_E_NOMEM, "pinned staging alloc");
    c->h_desc_cap = 4 * (size_t)n;
  }
  int *desc = c->h_desc;
  std::vector<int> &pool = c->pool_tmp;
  pool = c->hn_pool;
  long long tot = 0;
  for (int k = 0; k < n; ++k) {
    const int s = scen_ids[k], ng = n_groups[k];
    if (s < 0 || s >= c->n_scen) return fail(c, SF_E_RANGE, "scenario index out of range");
    if (ng < 0 || pool[s] + ng > c->P.pool_cap) return fail(c, SF_E_RANGE, "pool capacity exceeded");
    desc[4 * k] = s; desc[4 * k + 1] = pool[s]; desc[4 * k + 2] = ng; desc[4 * k + 3] = (int)tot;
    pool[s] += ng;
    tot += ng;
  }
  if (tot == 0) return SF_OK;
  const size_t nd = 4 * (size_t)n;
  const size_t need = 1 + nd + (size_t)tot + (size_t)tot * G;
  if (need > c->stage_cap) {
    if (c->d_stage) cudaFree(c->d_stage);
    c->d_stage = nullptr;
    if (cudaMalloc(&c->d_stage, need * sizeof(int)) != cudaSuccess) return fail(c, SF_E_NOMEM, "staging alloc");
    c->stage_cap = need;
  }
  int *dbad = c->d_stage, *ddesc = c->d_stage + 1, *dp = ddesc + nd, *dt = dp + tot;
  const int lim = (int)(c->P.M / c->P.k5);         // k5 (p + T) <= M  <=>  p + T <= M / k5
  int bad = 0;
  if (!cuda_ok(c, cudaMemsetAsync(dbad, 0, sizeof(int), c->stream), "reset") ||
      !cuda_ok(c, cudaMemcpyAsync(ddesc, desc, nd * sizeof(int), cudaMemcpyHostToDevice, c->stream), "H2D desc") ||
      !cuda_ok(c, cudaMemcpyAsync(dp, prompt, tot * sizeof(int), cudaMemcpyHostToDevice, c->stream), "H2D prompts") ||
      !cuda_ok(c, cudaMemcpyAsync(dt, target, tot * G * sizeof(int), cudaMemcpyHostToDevice, c->stream), "H2D targets"))
    return SF_E_CUDA;
  sf_launch_scatter_pool(c->D, G, ddesc, n, dp, dt, lim, dbad, c->stream);
  c->launches++;
  if (!cuda_ok(c, cudaGetLastError(), "scatter launch") ||
      !cuda_ok(c, cudaMemcpyAsync(&bad, dbad, sizeof(int), cudaMemcpyDeviceToHost, c->stream), "D2H flag") ||
      !cuda_ok(c, cudaStreamSynchronize(c->stream), "sync"))        // the inputs are copied before return
    return SF_E_CUDA;
  if (bad) {                                        // name the first invalid entry; nothing committed
    long long off = 0;
    for (int k = 0; k < n; ++k) {
      for (long long a = 0; a < n_groups[k]; ++a) {
        const long long p = prompt[off + a];
        if (p < 0) return fail(c, SF_E_INVALID, "negative prompt length");
        for (int m = 0; m < G; ++m) {
          const long long T = target[(off + a) * G + m];
          if (T < 1 || (long long)c->P.k5 * (p + T) > c->P.M) return fail(c, SF_E_INVALID, "target < 1 or k5*(p+T) > M (A27)");
        }
      }
      off += n_groups[k];
    }
    return fail(c, SF_E_INVALID, "invalid prompt or target length");
  }
  sf_launch_commit_pool(c->D, ddesc, n, c->stream);
  c->launches++;
  if (!cuda_ok(c, cudaGetLastError(), "commit launch")) return SF_E_CUDA;
  c->hn_pool.swap(pool);
  return SF_OK;
}

sf_status sf_submit_prompts(sf_ctx *c, int32_t scenario, int32_t n_groups, const int32_t *prompt_len,
                            const int32_t *target_len) {
  return sf_submit_prompts_many(c, 1, &scenario, &n_groups, prompt_len, target_len);
}

// Block mode: one launch per non-empty scenario class; the first on the context stream, the others
// forked onto the class streams after the stream's prior work and joined back before what follows.
static cudaError_t launch_block_classes(sf_ctx *c, int n_windows) {
  cudaError_t e = cudaSuccess;
  const bool fork = c->ev_fork != nullptr;
  if (fork && (e = cudaEventRecord(c->ev_fork, c->stream)) != cudaSuccess) return e;
  bool main_used = false;
  for (auto &b : c->bc) {
    if (b.n == 0) continue;
    cudaStream_t st = c->stream;
    if (main_used) {
      st = b.st;
      if ((e = cudaStreamWaitEvent(st, c->ev_fork, 0)) != cudaSuccess) return e;
    }
    if ((e = sf_launch_window_cluster(c->P, c->D, c->d_blist + b.off, b.n, b.ks, b.cl, n_windows, st)) != cudaSuccess)
      return e;
    c->launches += 1;
    if (main_used) {
      if ((e = cudaEventRecord(b.ev, st)) != cudaSuccess) return e;
      if ((e = cudaStreamWaitEvent(c->stream, b.ev, 0)) != cudaSuccess) return e;
    }
    main_used = true;
  }
  return e;
}

sf_status sf_step(sf_ctx *c, int32_t n_windows, sf_step_stats *out) {
  sf_status st = check_ctx(c);
  if (st != SF_OK) return st;
  DevGuard dg(c->device);
  if (n_windows < 0) return fail(c, SF_E_INVALID, "n_windows < 0");
  long long before[sf::kMetrics] = {0}, after[sf::kMetrics] = {0};
  if (out) {                                           // cumulative metrics before the call, on the device
    sf_launch_reduce_metrics(c->D, c->n_scen, c->d_metrics + sf::kMetrics, c->stream);
    c->launches++;
  }
  if (c->fused && n_windows > 0) {
    prof_mark(c, 3);
    sf_launch_window_fused(c->P, c->D, c->n_scen, c->max_inst, n_windows, c->stream);
    prof_mark(c, 3);
    c->launches += 1;
  }
  if (c->block && !c->fused && n_windows > 0) {
    prof_mark(c, 3);
    if (!cuda_ok(c, launch_block_classes(c, n_windows), "block launch")) return SF_E_CUDA;
    prof_mark(c, 3);
  }
  // Split mode: three kernels per window.  With PDL each kernel may start while its predecessor
  // runs and waits per scenario on the progress flags (epoch = split windows so far), so a
  // scenario's advance starts when ITS coordinator is done instead of after the slowest one.
  // Profiling (events between kernels) serializes the launches.
  const int pdl = c->pdl && !c->prof_on;
  const bool dyn = c->dyn && !c->fused && !c->block && !c->prof_on;   // profiling attributes time per kernel: split
  if (dyn && n_windows > 0) {
    if (c->dyn_blocks == 0) c->dyn_blocks = sf_dyn_blocks(c->max_inst);
    const size_t qbytes = sizeof(int) * (4 + (size_t)c->n_scen + (size_t)c->D.q_total);
    for (int w = 0; w < n_windows; ++w) {
      GParams P = c->P;
      P.epoch = ++c->epoch;
      P.pdl = 0;
      if (!cuda_ok(c, cudaMemsetAsync(c->D.q_ctr, 0, qbytes, c->stream), "queue reset")) return SF_E_CUDA;
      sf_launch_window_dyn(P, c->D, c->n_scen, c->max_inst, c->dyn_blocks, c->stream);
      c->launches += 1;
    }
  }
  for (int w = 0; w < (c->fused || c->block || dyn ? 0 : n_windows); ++w) {
    GParams P = c->P;
    P.epoch = ++c->epoch;
    P.pdl = pdl && w > 0;                 // the first coordinator follows arbitrary stream work
    prof_mark(c, 0);
    sf_launch_begin_coord(P, c->D, c->n_scen, c->max_inst, c->stream);
    prof_mark(c, 0);
    P.pdl = pdl && !(c->pdl_mask & 1);
    prof_mark(c, 1);
    if (c->lanes) sf_launch_advance_lanes(P, c->D, c->n_inst_total, c->stream);
    else sf_launch_advance(P, c->D, c->n_inst_total, c->stream);
    prof_mark(c, 1);
    P.pdl = pdl && !(c->pdl_mask & 2);
    prof_mark(c, 2);
    sf_launch_ledger(P, c->D, c->n_scen, c->stream);
    prof_mark(c, 2);
    c->launches += 3;
  }
  if (!cuda_ok(c, cudaGetLastError(), "window launch")) return SF_E_CUDA;
  if (out) {
    sf_launch_reduce_metrics(c->D, c->n_scen, c->d_metrics, c->stream);
    c->launches++;
    long long both[2 * sf::kMetrics];
    if (!cuda_ok(c, cudaGetLastError(), "reduce launch") ||
        !cuda_ok(c, cudaMemcpyAsync(both, c->d_metrics, sizeof(both), cudaMemcpyDeviceToHost, c->stream), "D2H metrics") ||
        !cuda_ok(c, cudaStreamSynchronize(c->stream), "sync"))
      return SF_E_CUDA;
    std::memcpy(after, both, sizeof(after));
    std::memcpy(before, both + sf::kMetrics, sizeof(before));
    if ((st = check_errors(c, after)) != SF_OK) return st;
    out->windows = after[sf::M_WINDOWS] - before[sf::M_WINDOWS];
    out->ticks = after[sf::M_TICKS] - before[sf::M_TICKS];
    out->traj_iters = after[sf::M_TRAJ_ITERS] - before[sf::M_TRAJ_ITERS];
    out->tokens = after[sf::M_TOKENS] - before[sf::M_TOKENS];
    out->completions = after[sf::M_COMPLETIONS] - before[sf::M_COMPLETIONS];
    out->routes = after[sf::M_ROUTES] - before[sf::M_ROUTES];
    out->interrupts = after[sf::M_INTERRUPTS] - before[sf::M_INTERRUPTS];
    out->pulls = after[sf::M_PULLS] - before[sf::M_PULLS];
    out->preemptions = after[sf::M_PREEMPTIONS] - before[sf::M_PREEMPTIONS];
    out->batches = after[sf::M_BATCHES] - before[sf::M_BATCHES];
    out->invalid_snapshots = after[sf::M_INVALID_SNAP] - before[sf::M_INVALID_SNAP];
    out->violations = after[sf::M_VIOLATIONS] - before[sf::M_VIOLATIONS];
    out->sim_time_ps = after[sf::M_MAX_T];
  }
  return SF_OK;
}

sf_status sf_publish_params(sf_ctx *c, int32_t scenario, int32_t v) {
  sf_status st = check_ctx(c);
  if (st != SF_OK) return st;
  DevGuard dg(c->device);
  if (scenario < 0 || scenario >= c->n_scen) return fail(c, SF_E_RANGE, "scenario index out of range");
  ScenState s;
  if ((st = read_state(c, scenario, &s)) != SF_OK) return st;
  if (v != s.ps + 1 || v > s.cu) return fail(c, SF_E_VERSION, "publish: version must be ps+1 and <= consumed batches");
  s.ps = v;
  s.m[sf::M_PUBLISHES] += 1;
  if (!cuda_ok(c, cudaMemcpyAsync(&c->D.ss[scenario].ps, &s.ps, sizeof(int), cudaMemcpyHostToDevice, c->stream), "H2D ps") ||
      !cuda_ok(c, cudaMemcpyAsync(&c->D.ss[scenario].m[sf::M_PUBLISHES], &s.m[sf::M_PUBLISHES], sizeof(unsigned long long),
                                  cudaMemcpyHostToDevice, c->stream), "H2D m") ||
      !cuda_ok(c, cudaStreamSynchronize(c->stream), "sync"))
    return SF_E_CUDA;
  return SF_OK;
}

sf_status sf_mark_filtered(sf_ctx *c, int32_t scenario, int32_t first_group, int32_t n_groups, const uint8_t *flags) {
  sf_status st = check_ctx(c);
  if (st != SF_OK) return st;
  DevGuard dg(c->device);
  if (scenario < 0 || scenario >= c->n_scen) return fail(c, SF_E_RANGE, "scenario index out of range");
  if (first_group < 0 || n_groups < 0 || (long long)first_group + n_groups > c->P.pool_cap)
    return fail(c, SF_E_RANGE, "group range outside the pool");
  if (n_groups == 0) return SF_OK;
  if (!flags) return fail(c, SF_E_INVALID, "null argument");
  bool any = false;
  for (int a = 0; a < n_groups; ++a) any |= flags[a] != 0;
  if (!cuda_ok(c, cudaMemcpyAsync(c->D.gfilt + (long long)c->hsc[scenario].grp_off + first_group, flags, n_groups,
                                  cudaMemcpyHostToDevice, c->stream), "H2D filter flags") ||
      !cuda_ok(c, cudaStreamSynchronize(c->stream), "sync"))
    return SF_E_CUDA;
  if (any) { c->P.filt = 1; c->P.abortable = 1; }
  return SF_OK;
}

sf_status sf_filter_group(sf_ctx *c, int32_t scenario, int32_t group) {
  sf_status st = check_ctx(c);
  if (st != SF_OK) return st;
  DevGuard dg(c->device);
  if (scenario < 0 || scenario >= c->n_scen) return fail(c, SF_E_RANGE, "scenario index out of range");
  c->P.abortable = 1;                                  // later rewards of its members are ignored
  sf_launch_filter(c->P, c->D, scenario, group, c->d_collect, c->stream);
  c->launches++;
  int h = 0;
  if (!cuda_ok(c, cudaGetLastError(), "filter launch") ||
      !cuda_ok(c, cudaMemcpyAsync(&h, c->d_collect, sizeof(int), cudaMemcpyDeviceToHost, c->stream), "D2H") ||
      !cuda_ok(c, cudaStreamSynchronize(c->stream), "sync"))
    return SF_E_CUDA;
  if (h != 0) return fail(c, SF_E_INVALID, "filter: group has no ledger entry (UnknownKey)");
  long long m[sf::kMetrics];
  if ((st = reduce_metrics_host(c, m)) != SF_OK) return st;
  return check_errors(c, m);
}

sf_status sf_collect_batch(sf_ctx *c, int32_t scenario, int32_t cap, int32_t *v_buf, int32_t *group_ids,
                           int32_t *group_versions, int32_t *n_out) {
  sf_status st = check_ctx(c);
  if (st != SF_OK) return st;
  DevGuard dg(c->device);
  if (scenario < 0 || scenario >= c->n_scen) return fail(c, SF_E_RANGE, "scenario index out of range");
  const int B = c->P.Br;
  if (n_out) *n_out = B;
  if (cap < B) return fail(c, SF_E_RANGE, "collect: cap < batch_size");
  sf_launch_collect(c->P, c->D, scenario, c->d_collect, c->stream);
  c->launches++;
  std::vector<int> h(2 + 2 * B);
  if (!cuda_ok(c, cudaGetLastError(), "collect launch") ||
      !cuda_ok(c, cudaMemcpyAsync(h.data(), c->d_collect, h.size() * sizeof(int), cudaMemcpyDeviceToHost, c->stream), "D2H") ||
      !cuda_ok(c, cudaStreamSynchronize(c->stream), "sync"))
    return SF_E_CUDA;
  if (h[0] != 0) return SF_NOT_READY;
  if (v_buf) *v_buf = h[1];
  for (int k = 0; k < B; ++k) {
    if (group_ids) group_ids[k] = h[2 + 2 * k];
    if (group_versions) group_versions[k] = h[3 + 2 * k];
  }
  long long m[sf::kMetrics];
  if ((st = reduce_metrics_host(c, m)) != SF_OK) return st;
  return check_errors(c, m);
}

sf_status sf_read_metrics(sf_ctx *c, int64_t *out, int32_t len) {
  sf_status st = check_ctx(c);
  if (st != SF_OK) return st;
  DevGuard dg(c->device);
  if (!out || len < 0) return fail(c, SF_E_INVALID, "bad output");
  long long m[sf::kMetrics];
  if ((st = reduce_metrics_host(c, m)) != SF_OK) return st;
  for (int k = 0; k < len; ++k) out[k] = k < sf::kMetrics ? m[k] : 0;
  return SF_OK;
}

sf_status sf_read_metrics_device(sf_ctx *c, int64_t *out_dev) {
  sf_status st = check_ctx(c);
  if (st != SF_OK) return st;
  DevGuard dg(c->device);
  if (!out_dev) return fail(c, SF_E_INVALID, "null output");
  sf_launch_reduce_metrics(c->D, c->n_scen, (long long *)out_dev, c->stream);
  c->launches++;
  return cuda_ok(c, cudaGetLastError(), "reduce launch") ? SF_OK : SF_E_CUDA;
}

sf_status sf_read_scenario_metrics(sf_ctx *c, int32_t scenario, int64_t *out, int32_t len) {
  sf_status st = check_ctx(c);
  if (st != SF_OK) return st;
  DevGuard dg(c->device);
  if (scenario < 0 || scenario >= c->n_scen) return fail(c, SF_E_RANGE, "scenario index out of range");
  ScenState s;
  if ((st = read_state(c, scenario, &s)) != SF_OK) return st;
  for (int k = 0; k < len; ++k) {
    long long v = k < sf::kMetrics ? (long long)s.m[k] : 0;
    if (k == sf::M_CMD_HASH) v = (long long)s.cmd_hash;
    if (k == sf::M_SIM_TIME || k == sf::M_MAX_T) v = s.t;
    if (k == sf::M_ERR_SCEN) v = s.err != 0;
    out[k] = v;
  }
  return SF_OK;
}

sf_status sf_read_all_scenario_metrics(sf_ctx *c, int64_t *out, int64_t cap) {
  sf_status st = check_ctx(c);
  if (st != SF_OK) return st;
  DevGuard dg(c->device);
  if (!out || cap < (int64_t)c->n_scen * sf::kMetrics) return fail(c, SF_E_RANGE, "output too small");
  std::vector<ScenState> ss(c->n_scen);
  if (!cuda_ok(c, cudaMemcpyAsync(ss.data(), c->D.ss, sizeof(ScenState) * c->n_scen, cudaMemcpyDeviceToHost, c->stream),
               "D2H states") ||
      !cuda_ok(c, cudaStreamSynchronize(c->stream), "sync"))
    return SF_E_CUDA;
  for (int s = 0; s < c->n_scen; ++s) {
    for (int k = 0; k < sf::kMetrics; ++k) {
      long long v = (long long)ss[s].m[k];
      if (k == sf::M_CMD_HASH) v = (long long)ss[s].cmd_hash;
      if (k == sf::M_SIM_TIME || k == sf::M_MAX_T) v = ss[s].t;
      if (k == sf::M_ERR_SCEN) v = ss[s].err != 0;
      out[(long long)s * sf::kMetrics + k] = v;
    }
  }
  return SF_OK;
}

static sf_status ensure_dump(sf_ctx *c, size_t n) {
  if (n <= c->dump_cap) return SF_OK;
  if (c->d_dump) cudaFree(c->d_dump);
  c->d_dump = nullptr;
  if (cudaMalloc(&c->d_dump, n * sizeof(long long)) != cudaSuccess) return fail(c, SF_E_NOMEM, "dump alloc");
  c->dump_cap = n;
  return SF_OK;
}

sf_status sf_dump_lifecycles(sf_ctx *c, int32_t scenario, int64_t *rec, int64_t cap, int64_t *n) {
  sf_status st = check_ctx(c);
  if (st != SF_OK) return st;
  DevGuard dg(c->device);
  if (scenario < 0 || scenario >= c->n_scen) return fail(c, SF_E_RANGE, "scenario index out of range");
  const long long cnt = (long long)c->hn_pool[scenario] * c->P.G;
  if (n) *n = cnt;
  if (cap < cnt || (cnt > 0 && !rec)) return SF_E_RANGE;
  if (cnt == 0) return SF_OK;
  if ((st = ensure_dump(c, 13 * cnt)) != SF_OK) return st;
  sf_launch_dump_lifecycles(c->P, c->D, scenario, cnt, c->d_dump, c->stream);
  c->launches += 2;
  if (!cuda_ok(c, cudaGetLastError(), "dump launch") ||
      !cuda_ok(c, cudaMemcpyAsync(rec, c->d_dump, 13 * cnt * sizeof(long long), cudaMemcpyDeviceToHost, c->stream), "D2H") ||
      !cuda_ok(c, cudaStreamSynchronize(c->stream), "sync"))
    return SF_E_CUDA;
  return SF_OK;
}

sf_status sf_dump_batches(sf_ctx *c, int32_t scenario, int32_t *out, int64_t cap, int64_t *n) {
  sf_status st = check_ctx(c);
  if (st != SF_OK) return st;
  DevGuard dg(c->device);
  if (scenario < 0 || scenario >= c->n_scen) return fail(c, SF_E_RANGE, "scenario index out of range");
  ScenState s;
  if ((st = read_state(c, scenario, &s)) != SF_OK) return st;
  const long long cnt = (long long)s.batch_n * (1 + 2 * c->P.Br);
  if (n) *n = cnt;
  if (cap < cnt || (cnt > 0 && !out)) return SF_E_RANGE;
  if (cnt == 0) return SF_OK;
  if (!cuda_ok(c, cudaMemcpyAsync(out, c->D.batches + c->hsc[scenario].batch_off, cnt * sizeof(int), cudaMemcpyDeviceToHost,
                                  c->stream), "D2H") ||
      !cuda_ok(c, cudaStreamSynchronize(c->stream), "sync"))
    return SF_E_CUDA;
  return SF_OK;
}

sf_status sf_dump_commands(sf_ctx *c, int32_t scenario, int64_t *rec, int64_t cap, int64_t *n) {
  sf_status st = check_ctx(c);
  if (st != SF_OK) return st;
  DevGuard dg(c->device);
  if (scenario < 0 || scenario >= c->n_scen) return fail(c, SF_E_RANGE, "scenario index out of range");
  ScenState s;
  if ((st = read_state(c, scenario, &s)) != SF_OK) return st;
  const long long cnt = std::min<long long>(s.cmd_n, c->P.cmdlog_cap);
  if (n) *n = cnt;
  if (cap < cnt || (cnt > 0 && !rec)) return SF_E_RANGE;
  if (cnt == 0) return SF_OK;
  if (!cuda_ok(c, cudaMemcpyAsync(rec, c->D.cmdlog + c->hsc[scenario].cmd_off, 4 * cnt * sizeof(long long),
                                  cudaMemcpyDeviceToHost, c->stream), "D2H") ||
      !cuda_ok(c, cudaStreamSynchronize(c->stream), "sync"))
    return SF_E_CUDA;
  return SF_OK;
}

sf_status sf_dump_instances(sf_ctx *c, int32_t scenario, int64_t *out, int64_t cap, int64_t *n) {
  sf_status st = check_ctx(c);
  if (st != SF_OK) return st;
  DevGuard dg(c->device);
  if (scenario < 0 || scenario >= c->n_scen) return fail(c, SF_E_RANGE, "scenario index out of range");
  const int I = c->hsc[scenario].I;
  if (n) *n = I;
  if (cap < I || !out) return SF_E_RANGE;
  if ((st = ensure_dump(c, 7 * (size_t)I)) != SF_OK) return st;
  sf_launch_dump_instances(c->P, c->D, scenario, c->d_dump, c->stream);
  c->launches++;
  if (!cuda_ok(c, cudaGetLastError(), "dump launch") ||
      !cuda_ok(c, cudaMemcpyAsync(out, c->d_dump, 7 * I * sizeof(long long), cudaMemcpyDeviceToHost, c->stream), "D2H") ||
      !cuda_ok(c, cudaStreamSynchronize(c->stream), "sync"))
    return SF_E_CUDA;
  return SF_OK;
}

int64_t sf_kernel_launches(const sf_ctx *c) { return c ? c->launches : 0; }

#ifdef SF_TIMING
// debug builds only (-DSF_TIMING): per-scenario coordinator cycles of the last window
sf_status sf_debug_coord_cycles(sf_ctx *c, int64_t *out) {
  if (!c || !c->D.dbg) return SF_E_INVALID;
  cudaMemcpy(out, c->D.dbg, 8 * sizeof(long long) * c->n_scen, cudaMemcpyDeviceToHost);
  return SF_OK;
}
sf_status sf_debug_adv_cycles(sf_ctx *c, int64_t *out) {
  if (!c || !c->D.dbg2) return SF_E_INVALID;
  cudaMemcpy(out, c->D.dbg2, 8 * sizeof(long long) * c->n_inst_total, cudaMemcpyDeviceToHost);
  return SF_OK;
}
#endif

#ifdef SF_CHECK
// SF_CHECK builds: raw ledger ring of one scenario as (state, group, version) triples, then the
// per-buffer reserved / occupied counts, then ScenState.cu.
sf_status sf_debug_ledger(sf_ctx *c, int32_t scen, int64_t *out) {
  if (!c || scen < 0 || scen >= c->n_scen) return SF_E_INVALID;
  const ScenConst &S = c->hsc[scen];
  const int nslot = (S.eta + 1) * c->P.B;
  std::vector<uint8_t> st(nslot);
  std::vector<int> g(nslot), v(nslot), nres(S.eta + 1), nocc(S.eta + 1);
  ScenState ss;
  cudaMemcpy(st.data(), c->D.led_st + S.led_off, nslot, cudaMemcpyDeviceToHost);
  cudaMemcpy(g.data(), c->D.led_g + S.led_off, 4 * nslot, cudaMemcpyDeviceToHost);
  cudaMemcpy(v.data(), c->D.led_v + S.led_off, 4 * nslot, cudaMemcpyDeviceToHost);
  cudaMemcpy(nres.data(), c->D.led_nres + S.ring_off, 4 * (S.eta + 1), cudaMemcpyDeviceToHost);
  cudaMemcpy(nocc.data(), c->D.led_nocc + S.ring_off, 4 * (S.eta + 1), cudaMemcpyDeviceToHost);
  cudaMemcpy(&ss, c->D.ss + scen, sizeof(ScenState), cudaMemcpyDeviceToHost);
  long long k = 0;
  for (int i = 0; i < nslot; ++i) { out[k++] = st[i]; out[k++] = g[i]; out[k++] = v[i]; }
  for (int i = 0; i <= S.eta; ++i) { out[k++] = nres[i]; out[k++] = nocc[i]; }
  out[k++] = ss.cu;
  return SF_OK;
}
#endif

#ifdef SF_TRACE
sf_status sf_debug_trace(sf_ctx *c, int64_t *out) {
  if (!c || !c->D.trace) return SF_E_INVALID;
  cudaMemcpy(out, c->D.trace, sizeof(long long) * (4LL * c->n_scen + 2LL * c->n_inst_total), cudaMemcpyDeviceToHost);
  return SF_OK;
}
#endif

sf_status sf_profile(sf_ctx *c, int32_t enable) {
  sf_status st = check_ctx(c);
  if (st != SF_OK) return st;
  DevGuard dg(c->device);
  c->prof_on = enable ? 1 : 0;
  return SF_OK;
}

sf_status sf_profile_read(sf_ctx *c, double *ms, int64_t *launches, int32_t len) {
  sf_status st = check_ctx(c);
  if (st != SF_OK) return st;
  DevGuard dg(c->device);
  if (!cuda_ok(c, cudaStreamSynchronize(c->stream), "sync")) return SF_E_CUDA;
  for (size_t k = 0; k + 1 < c->ev_used; k += 2) {
    float e = 0.f;
    if (!cuda_ok(c, cudaEventElapsedTime(&e, c->ev_pool[k], c->ev_pool[k + 1]), "event elapsed")) return SF_E_CUDA;
    c->prof_ms[c->ev_kind[k]] += e;
    c->prof_n[c->ev_kind[k]] += 1;
  }
  c->ev_used = 0;
  for (int k = 0; k < len && k < 4; ++k) {
    if (ms) ms[k] = c->prof_ms[k];
    if (launches) launches[k] = c->prof_n[k];
    c->prof_ms[k] = 0;
    c->prof_n[k] = 0;
  }
  return SF_OK;
}

const char *sf_last_error(const sf_ctx *c) { return c ? c->err.c_str() : "null context"; }

}  // extern "C"
