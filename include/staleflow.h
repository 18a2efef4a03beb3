/* staleflow.h -- C99 ABI of the B200-native StaleFlow coordination-step library.
 *
 * Implements the staleness-constrained rollout-coordination step of StaleFlow
 * (arXiv 2601.12784, PAPER.md; DESIGN.md §3 "SF-SIM-1") on sm_100a CUDA.
 * Plain pointers and sizes only; no torch types.  Built into
 * paper_2601_12784_b200/libstaleflow.so.
 *
 * Units: time int64 picoseconds; lengths int32 tokens; KV in tokens (k5 per token).
 * Threading: a context is single-writer; different contexts are independent.
 * Streams: every call is ordered on cfg->cuda_stream (NULL = legacy default stream);
 *   calls that return host data synchronize that stream.
 * Ownership: the caller owns every input array (copied before return) and every output
 *   array (caller-allocated, capacity given).  The library owns all device memory and
 *   frees it in sf_destroy.  No exceptions cross the ABI.
 * Errors: every call returns an sf_status.  SF_E_STATE and SF_E_CUDA poison the context:
 *   every later call returns SF_E_STATE.  sf_last_error() describes the last failure.
 */
#ifndef STALEFLOW_H
#define STALEFLOW_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct sf_ctx sf_ctx;

typedef enum {
  SF_OK = 0,
  SF_NOT_READY = 1,   /* collect: earliest buffer is Waiting or Stuck            */
  SF_E_INVALID = -1,  /* bad argument / invalid config                          */
  SF_E_VERSION = -2,  /* publish: version != ps_version+1 or > #consumed batches */
  SF_E_STATE = -3,    /* invariant violated (staleness > eta, Eq 1 on a quiescent snapshot,     */
                      /*   ledger overflow); poisons the context                               */
  SF_E_NOMEM = -4,    /* device allocation failed                                              */
  SF_E_CUDA = -5,     /* CUDA error; poisons the context                                       */
  SF_E_RANGE = -6     /* bad scenario index, pool capacity exceeded, or output too small       */
                      /*   (then *n = the size needed)                                         */
} sf_status;

/* Strategy bits: 1 = StaleFlow strategy, 0 = its vanilla counterpart. */
#define SF_STRATEGY_ROUTING 1u     /* Alg 2 waterfall  vs fewest-trajectories routing */
#define SF_STRATEGY_SYNC 2u        /* Alg 3 selective sync vs greedy sync                  */
#define SF_STRATEGY_MIGRATION 4u   /* Alg 4 migration  vs none                         */

#define SF_METRICS_LEN 32          /* layout: DESIGN.md §6 */

typedef struct {
  int32_t batch_size;                 /* B: groups per training step = buffer capacity  */
  int32_t n_scenarios;                /* independent scenarios in this context (>= 1)           */
  const int32_t *scenario_eta;        /* [n_scenarios] or NULL (= eta argument)                 */
  const int32_t *scenario_instances;  /* [n_scenarios] or NULL (= instances argument), <= 128   */
  const uint32_t *scenario_strategy;  /* [n_scenarios] or NULL (= strategy)                     */
  int64_t k1_ps_per_tok, k2_ps, k3_ps, k4_ps;   /* Eq 7 coefficients (Table 6) in ps; */
                                      /*   k1, k3 < 2^31 (SF_E_INVALID otherwise)               */
  int32_t k5_tok;                     /* KV tokens per token, >= 1                       */
  int64_t kprefill_ps_per_tok;        /* prefill stall per admitted token (A20), < 2^31 */
  int64_t kv_budget_tok;              /* M, < 2^30                                       */
  double mu, phi_throughput;          /* waterfall threshold, migration gap              */
  int32_t phi_wait;                   /* migration wait threshold                        */
  int64_t snap_period_ps;             /* Delta: one sf_step window                               */
  int64_t route_lat_ps, pull_lat_ps, reward_lat_ps;  /* r, q, R                  */
  uint32_t strategy;                  /* SF_STRATEGY_* bits                                      */
  int32_t auto_train_windows;         /* > 0: library consumes Ready buffers and publishes this  */
                                      /*   many windows later; 0: caller drives collect/publish  */
  int32_t pool_capacity_groups;       /* max groups ever submitted per scenario (device pool)    */
  int32_t command_log_capacity;       /* per-scenario command records kept for sf_dump_commands  */
                                      /*   (0 = keep only the command hash)                      */
  int32_t extra_groups;               /* batch-level redundant rollout (App C):    */
                                      /*   buffers hold batch_size + extra_groups slots, are     */
                                      /*   Ready at >= batch_size Occupied; Consume returns the  */
                                      /*   first batch_size Occupied (slot order) and Aborts the */
                                      /*   surplus groups.  0 = off                  */
  int32_t extra_members;              /* group-level redundancy: group_size + extra_members      */
                                      /*   members are rolled out per group; a group completes   */
                                      /*   at group_size rewarded members and its other members  */
                                      /*   are Aborted at once (P:473 footnote)      */
  int32_t watchdog_windows;           /* > 0, auto trainer only: a scenario that makes no progress */
                                      /*   for this many consecutive windows with nothing pending */
                                      /*   (instances idle, no reward in flight, trainer idle)    */
                                      /*   while groups remain unconsumed is deadlocked (SPEC     */
                                      /*   S:494): it is poisoned and sf_step returns SF_E_STATE. */
                                      /*   0 = off (a streaming caller may still submit prompts)  */
  int32_t device;                     /* CUDA device ordinal                                     */
  void *cuda_stream;                  /* cudaStream_t (e.g. torch.cuda.Stream().cuda_stream)     */
} sf_config;

typedef struct {                      /* summed over all scenarios for one sf_step call          */
  int64_t windows, ticks, traj_iters, tokens, completions, routes, interrupts, pulls,
      preemptions, batches, invalid_snapshots, violations;
  int64_t sim_time_ps;                /* simulated time after the call (max over scenarios)      */
} sf_step_stats;

/* Create a context of cfg->n_scenarios independent scenarios, each with `instances` rollout
 * instances, staleness bound `eta` and GRPO group size `group_size`.
 * *out is written only on SF_OK.  Errors: SF_E_INVALID, SF_E_NOMEM, SF_E_CUDA. */
sf_status sf_create(int32_t instances, int32_t eta, int32_t group_size, const sf_config *cfg, sf_ctx **out);

/* Free all device memory of the context.  NULL-safe. */
void sf_destroy(sf_ctx *ctx);

/* Append n_groups prompts to a scenario's dataset pool: prompt_len[n_groups] and
 * target_len[n_groups*(group_size+extra_members)] (the simulated response length of each
 * member, the redundant ones included).  Host pointers, copied.  Ingestion into the TS happens inside sf_step under the (eta+1)*B
 * live-group cap.  Errors: SF_E_RANGE (scenario, pool capacity), SF_E_INVALID (target < 1 or
 * k5*(prompt+target) > M, reading A27). */
sf_status sf_submit_prompts(sf_ctx *ctx, int32_t scenario, int32_t n_groups, const int32_t *prompt_len,
                            const int32_t *target_len);

/* Batched submit for many scenarios with one host->device copy: scenario n_groups[k] groups go
 * to scenario scenario_ids[k]; prompts/targets concatenated in that order.  Host pointers. */
sf_status sf_submit_prompts_many(sf_ctx *ctx, int32_t n, const int32_t *scenario_ids, const int32_t *n_groups,
                                 const int32_t *prompt_len, const int32_t *target_len);

/* Advance every scenario by n_windows snapshot periods (DESIGN.md §3.1 W0-W9: trainer, ingest,
 * snapshot + Eq 1, Alg 3 sync, Alg 4 migration, Alg 2 routing, command application, decode
 * advance, reward -> ledger).  If out != NULL the stream is synchronized and out receives the
 * summed metric deltas of this call; with out == NULL the call only enqueues work. */
sf_status sf_step(sf_ctx *ctx, int32_t n_windows, sf_step_stats *out);

/* External-trainer Push: new_version must equal ps_version+1 and be <= the number of
 * consumed batches.  Errors: SF_E_VERSION, SF_E_RANGE. */
sf_status sf_publish_params(sf_ctx *ctx, int32_t scenario, int32_t new_version);

/* External-trainer Consume: if the earliest unconsumed buffer is Ready, write its
 * v_buf, the B group ids in slot order and their versions, set *n_out = B and retire it
 * (with extra_groups > 0: the first B Occupied entries; the surplus groups are Aborted).
 * SF_NOT_READY if Waiting/Stuck; SF_E_RANGE if cap < B (*n_out = B). */
sf_status sf_collect_batch(sf_ctx *ctx, int32_t scenario, int32_t cap, int32_t *v_buf, int32_t *group_ids,
                           int32_t *group_versions, int32_t *n_out);

/* Filtering (P:413 (2)).  flags[a] != 0 marks group first_group + a of the scenario's pool as
 * carrying no learning signal (e.g. identical rewards within the group, DAPO): when it completes
 * its entry is aborted instead of Occupied -- a later Occupied entry moves forward into the hole
 * (reading R-FILTER) -- and its members are dropped.  Host pointer, copied; may be
 * called before or after the groups are submitted.  Errors: SF_E_RANGE. */
sf_status sf_mark_filtered(sf_ctx *ctx, int32_t scenario, int32_t first_group, int32_t n_groups,
                           const uint8_t *flags);
/* Proactive filtering between windows of a tracked (Reserved or Occupied) group, e.g. one whose
 * stragglers stall training (P:413 (2); SPEC abort S:96-103): its ledger entry is aborted as above
 * and every member not yet consumed is Aborted (Abort commands for the in-flight ones).
 * Errors: SF_E_INVALID if the group has no ledger entry (UnknownKey), SF_E_RANGE. */
sf_status sf_filter_group(sf_ctx *ctx, int32_t scenario, int32_t group);

/* Cumulative int64 metrics summed over scenarios into host out[len]; slot 29
 * counts poisoned scenarios and slot 30 is the maximum simulated time. */
sf_status sf_read_metrics(sf_ctx *ctx, int64_t *out, int32_t len);
/* Same, written to DEVICE memory out_dev[SF_METRICS_LEN] on the context stream (no sync);
 * this is the NCCL all-reduce payload. */
sf_status sf_read_metrics_device(sf_ctx *ctx, int64_t *out_dev);
/* One scenario's cumulative metrics (host out[len]). */
sf_status sf_read_scenario_metrics(sf_ctx *ctx, int32_t scenario, int64_t *out, int32_t len);
/* Every scenario's cumulative metrics in one transfer: out[n_scenarios * SF_METRICS_LEN]
 * (host), scenario-major; slots 25/26/29/30 as in sf_read_scenario_metrics. */
sf_status sf_read_all_scenario_metrics(sf_ctx *ctx, int64_t *out, int64_t cap);

/* Per-trajectory lifecycle records, 13 int64 each: id, group, prompt, target, gen, v_group,
 * state (0 pool,1 TS,2 transit,3 wait,4 run,5 done,6 consumed,7 aborted), inst, n_routes, n_preempt,
 * n_interrupt, consumed_vbuf, t_complete.  *n = records available. */
sf_status sf_dump_lifecycles(sf_ctx *ctx, int32_t scenario, int64_t *records, int64_t cap, int64_t *n);
/* Consumed batches: per batch v_buf then B (group id, group version) pairs (int32). */
sf_status sf_dump_batches(sf_ctx *ctx, int32_t scenario, int32_t *out, int64_t cap, int64_t *n);
/* Command log (4 int64 per record: window, kind 1 Route/2 Interrupt/3 Pull/4 Abort, inst, traj);
 * records beyond command_log_capacity are dropped (the hash in the metrics covers all). */
sf_status sf_dump_commands(sf_ctx *ctx, int32_t scenario, int64_t *records, int64_t cap, int64_t *n);
/* Per-instance view, 7 int64 each: v, kv, n_run, n_wait, complete, state(0 idle,1 tick,2 pull),
 * next boundary (or -1). */
sf_status sf_dump_instances(sf_ctx *ctx, int32_t scenario, int64_t *out, int64_t cap, int64_t *n);

/* Number of kernels this context has launched so far. */
int64_t sf_kernel_launches(const sf_ctx *ctx);

/* Live per-kernel timing: while enabled, sf_step records CUDA events on the context stream
 * around each window kernel (0 coordinate, 1 advance, 2 ledger, 3 fused window kernel).  sf_profile_read synchronizes
 * the stream and returns (then resets) the accumulated milliseconds and launch counts in
 * ms[len] / launches[len] (len <= 4). */
sf_status sf_profile(sf_ctx *ctx, int32_t enable);
sf_status sf_profile_read(sf_ctx *ctx, double *ms, int64_t *launches, int32_t len);

/* ---- host-side tools adjacent to the step; no context needed ---- */

/* Least-squares fit of Eq 7 ("offline profiling and linear regression", P:636,
 * 1071): latency = k1*kv + max(k2, k3*n) + k4 from n_samples (kv, n_run, latency) samples, the
 * max() handled by iterated regime segmentation (<= 50 rounds).  k_out[4] = k1, k2, k3, k4 in the
 * samples' units.  SF_E_INVALID if n_samples < 4; SF_E_STATE if degenerate (rank deficient, e.g.
 * every sample in one regime). */
sf_status sf_fit_cost_model(int32_t n_samples, const double *kv, const double *n_run, const double *latency,
                            double *k_out);

/* Load-balancing communication plan for Push (App A.2; fig:comm): for each
 * requirement r (slice req_slice[r] needed by receiver req_receiver[r], input order), choose the
 * sender holding the slice with the smallest accumulated latency estimate (ties: lowest id) and
 * add slice_bytes / bandwidth + latency of that (sender, receiver) pair.  holds[n_senders *
 * n_slices] (0/1), bandwidth / latency [n_senders * n_receivers].  Writes out_sender[n_req] and
 * acc[n_senders].  SF_E_INVALID if a required slice has no holder. */
sf_status sf_plan_comm(int32_t n_slices, const double *slice_bytes, int32_t n_senders, int32_t n_receivers,
                       const uint8_t *holds, const double *bandwidth, const double *latency, int32_t n_req,
                       const int32_t *req_slice, const int32_t *req_receiver, int32_t *out_sender, double *acc);

/* Parameter server: Push / Pull requests under a read-write lock with
 * writer preference (a waiting Push blocks new Pulls), simulated over int64 ps.  Request k:
 * kind[k] (0 Pull, 1 Push), issue time, duration, and for a Push the version it writes.  Outputs
 * per request: t_start / t_end of its lock hold, version (a Pull: the version committed when its
 * read starts; a Push: its own, committed at t_end), status (0, or -2 VersionSkip for a Push whose
 * version is not the last accepted + 1; nothing else happens for it).  Host arrays, caller-owned.
 * Errors: SF_E_INVALID (null pointer, bad kind, negative duration). */
sf_status sf_ps_lock_sim(int32_t n, const int32_t *kind, const int64_t *t_issue, const int64_t *duration,
                         const int32_t *push_version, int32_t v0, int64_t *t_start, int64_t *t_end,
                         int32_t *version, int32_t *status);

/* Message for the last failing call; owned by the context, valid until the next call. */
const char *sf_last_error(const sf_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* STALEFLOW_H */
