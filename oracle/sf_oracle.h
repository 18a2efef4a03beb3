/* sf_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow CPU discrete-event oracle of StaleFlow's staleness-constrained
 * rollout-coordination step (arXiv 2601.12784), semantics SF-SIM-1 in
 * DESIGN.md §3.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no
 * code (and no header) with the CUDA product in paper_2601_12784_b200/.
 *
 * Units: time int64 picoseconds, lengths int32 tokens, KV in tokens (k5 per token).
 * Every function returns 0 on success, a negative code on error.
 */
#ifndef SF_ORACLE_H
#define SF_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define SFO_OK 0
#define SFO_NOT_READY 1
#define SFO_E_INVALID (-1)
#define SFO_E_VERSION (-2)
#define SFO_E_STATE (-3)
#define SFO_E_RANGE (-6)

#define SFO_METRICS_LEN 32

typedef struct {
  int32_t batch_size;                 /* B */
  int32_t n_scenarios;
  const int32_t *scenario_eta;        /* [n_scenarios] or NULL */
  const int32_t *scenario_instances;  /* [n_scenarios] or NULL */
  const uint32_t *scenario_strategy;  /* [n_scenarios] or NULL */
  int64_t k1, k2, k3, k4;             /* Table 6 in ps */
  int32_t k5;                         /* KV tokens per token */
  int64_t kp;                         /* prefill stall ps per token (reading A20) */
  int64_t M;                          /* KV budget, tokens */
  double mu, phi_tp;
  int32_t phi_wait;
  int64_t delta, r, q, R;             /* snapshot period, route, pull, reward latencies */
  uint32_t strategy;                  /* bit0 R, bit1 S, bit2 M (1 = StaleFlow) */
  int32_t atw;                        /* auto-train windows; 0 = external trainer */
  int32_t pool_capacity_groups;       /* max groups submitted per scenario */
  int32_t extra_groups;               /* batch-level redundancy: buffer slots = B + extra_groups (App C) */
  int32_t extra_members;              /* group-level redundancy: members per group = G + extra_members  */
  int32_t watchdog_windows;           /* > 0 (auto trainer only): deadlock after this many consecutive windows
                                         with no progress, nothing pending and work left */
} sfo_config;

typedef struct sfo_sim sfo_sim;

int sfo_create(int32_t instances, int32_t eta, int32_t group_size, const sfo_config *cfg, sfo_sim **out);
void sfo_destroy(sfo_sim *);
int sfo_submit_prompts(sfo_sim *, int32_t scenario, int32_t n_groups, const int32_t *prompt_len,
                       const int32_t *target_len);
/* Advance every scenario by n_windows snapshot periods; scenarios run on n_threads host threads. */
int sfo_step(sfo_sim *, int32_t n_windows, int32_t n_threads);
int sfo_publish_params(sfo_sim *, int32_t scenario, int32_t new_version);
/* Filtering (P:413 (2)): flags[a] != 0 marks group first_group + a as carrying no learning signal
 * (e.g. identical rewards, DAPO); such a group is dropped when it completes (reading R-FILTER). */
int sfo_mark_filtered(sfo_sim *, int32_t scenario, int32_t first_group, int32_t n, const uint8_t *flags);
/* Proactive filtering of a tracked (Reserved or Occupied) group between windows: its entry is
 * aborted (ledger abort) and its members leave.  SFO_E_INVALID if the group has no entry. */
int sfo_filter_group(sfo_sim *, int32_t scenario, int32_t group);
int sfo_collect_batch(sfo_sim *, int32_t scenario, int32_t cap, int32_t *v_buf, int32_t *group_ids,
                      int32_t *group_versions, int32_t *n_out);
/* metrics summed over scenarios (layout: DESIGN.md §6) */
int sfo_read_metrics(sfo_sim *, int64_t *out, int32_t len);
int sfo_read_scenario_metrics(sfo_sim *, int32_t scenario, int64_t *out, int32_t len);
/* 13 int64 per trajectory: id, group, prompt, target, gen, v, state, inst, n_routes,
 * n_preempt, n_interrupt, consumed_vbuf, t_complete */
int sfo_dump_lifecycles(sfo_sim *, int32_t scenario, int64_t *records, int64_t cap, int64_t *n);
/* per consumed batch: v_buf, then B (group id, group version) pairs */
int sfo_dump_batches(sfo_sim *, int32_t scenario, int32_t *out, int64_t cap, int64_t *n);
/* 4 int64 per command: window, kind (1 Route, 2 Interrupt, 3 Pull, 4 Abort), inst, traj (-1 for Pull) */
int sfo_dump_commands(sfo_sim *, int32_t scenario, int64_t *out, int64_t cap, int64_t *n);
/* per-instance snapshot view: v, kv, n_run, n_wait, complete, state(0 idle,1 tick,2 pull), nb */
int sfo_dump_instances(sfo_sim *, int32_t scenario, int64_t *out, int64_t cap, int64_t *n);

/* ---------------- unit-level entry points (used by the oracle's own pins) ---------------- */
typedef struct sfo_ledger sfo_ledger;
sfo_ledger *sfo_ledger_new(int32_t eta, int32_t batch_size);
/* batch-level redundancy: `capacity` slots per buffer, Ready at >= batch_size Occupied */
sfo_ledger *sfo_ledger_new2(int32_t eta, int32_t capacity, int32_t batch_size);
void sfo_ledger_free(sfo_ledger *);
int sfo_ledger_verify(const sfo_ledger *, int32_t v);                           /* 1/0 */
int sfo_ledger_reserve(sfo_ledger *, int32_t g, int32_t v, int32_t *b, int32_t *s);
int sfo_ledger_delete_relocate(sfo_ledger *, int32_t g);
/* abort a tracked entry: Reserved -> delete_and_relocate, Occupied -> emptied;
 * then later Occupied entries move forward into the hole (reading R-FILTER); *moves = moves */
int sfo_ledger_abort(sfo_ledger *, int32_t g, int32_t *moves);
int sfo_ledger_occupy(sfo_ledger *, int32_t g, int32_t v, int32_t *b, int32_t *s);
int sfo_ledger_state(const sfo_ledger *, int32_t b);  /* 0 Waiting, 1 Ready, 2 Stuck */
/* first batch_size Occupied entries in slot order; returns the surplus (aborted) groups through
 * surplus[capacity] / *n_surplus when non-NULL */
int sfo_ledger_consume(sfo_ledger *, int32_t *groups, int32_t *versions);
int sfo_ledger_consume2(sfo_ledger *, int32_t *groups, int32_t *versions, int32_t *surplus, int32_t *n_surplus);
int sfo_ledger_get(const sfo_ledger *, int32_t b, int32_t s, int32_t *st, int32_t *g, int32_t *v);
int32_t sfo_ledger_cu(const sfo_ledger *);
sfo_ledger *sfo_ledger_clone(const sfo_ledger *);

typedef struct {
  int64_t k1, k2, k3, k4; int32_t k5; int64_t kp, M;
  double mu, phi_tp; int32_t phi_wait; int32_t eta;
} sfo_params;

typedef struct { int32_t v; int64_t kv; int32_t n_run; int32_t n_wait; } sfo_inst_view;
typedef struct { int32_t id; int32_t g; int32_t v; int32_t l; } sfo_ts_item;  /* v = -1: versionless */

int64_t sfo_tick_latency(const sfo_params *, int64_t kv, int32_t n, int64_t prefill_tokens);
double sfo_throughput(const sfo_params *, int32_t n, int64_t kv);
double sfo_marginal_gain(const sfo_params *, const sfo_inst_view *, int32_t l);
double sfo_ideal_gain(const sfo_params *, int32_t l);
int sfo_check_routable(const sfo_params *, const sfo_inst_view *, int32_t tau_v, const sfo_ledger *);
/* Sorts items into MLQ order (Alg 2 line 2); writes the permutation. */
int sfo_mlq_order(const sfo_ts_item *items, int32_t n, int32_t *order);
/* Alg 2 over an already MLQ-ordered list; mutates S and L; out_inst[k] = instance of the k-th
 * routed item (items are routed as a prefix). vanilla = 1 selects §6.5 vanilla routing. */
int sfo_route(const sfo_params *, sfo_inst_view *S, int32_t I, const sfo_ts_item *mlq, int32_t n,
              sfo_ledger *L, int32_t vanilla, int32_t *out_inst);
/* Alg 3 (vanilla = 1: §6.5 greedy) -> selected instances ascending; returns count. */
int sfo_sync_select(const sfo_params *, const sfo_inst_view *S, int32_t I, const sfo_ts_item *mlq,
                    int32_t n, const sfo_ledger *L, int32_t ps_version, int32_t vanilla_sync,
                    int32_t vanilla_route, int32_t *out);
/* Alg 4 case counts: case1_k[i] = wait entries interrupted from the tail; *case2 = drained instance or -1 */
int sfo_migrate(const sfo_params *, const sfo_inst_view *S, int32_t I, int32_t *case1_k, int32_t *case2);

#ifdef __cplusplus
}
#endif
#endif
