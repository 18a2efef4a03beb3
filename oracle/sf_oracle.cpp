// sf_oracle.cpp -- TEST INFRASTRUCTURE ONLY (see sf_oracle.h).
//
// A plain, slow, obviously-correct discrete-event implementation of the
// StaleFlow coordination step (arXiv 2601.12784), written from PAPER.md in the
// paper's order and notation.  "P:n" = PAPER.md line n, "S:n" = SPEC.md line n,
// "A<n>" / "R-..." = readings listed in DESIGN.md §3-4.  Nothing here is
// blocked, fused or reordered for speed: every list is a std::vector/std::deque,
// every search is a linear scan in the order the paper states.
//
// Build: g++ -std=c++17 -O2 -ffp-contract=off -fno-fast-math -fPIC -shared
// (no FMA contraction so fp64 cost-model values are the correctly-rounded
// results of the written expression trees, reading A3).
#include "sf_oracle.h"

#include <algorithm>
#include <atomic>
#include <cstring>
#include <deque>
#include <limits>
#include <map>
#include <new>
#include <thread>
#include <vector>

// ============================================================== staleness ledger (§4.2)
namespace {
enum { E_EMPTY = 0, E_RESERVED = 1, E_OCCUPIED = 2 };
struct Entry { int st = E_EMPTY; int g = -1; int v = -1; };
}  // namespace

struct sfo_ledger {
  int eta = 0, B = 1;
  int Br = 1;                                  // batch size: Ready at >= Br Occupied (App C redundancy)
  int cu = 0;                                  // consumed_upto: earliest unconsumed V_buf
  std::vector<std::vector<Entry>> buf;         // buf[V_buf], all Empty until touched

  void ensure(int b) { while ((int)buf.size() <= b) buf.emplace_back(B); }
  bool has_empty(int b) const {
    if (b >= (int)buf.size()) return true;
    for (int s = 0; s < B; ++s) if (buf[b][s].st == E_EMPTY) return true;
    return false;
  }
  // Discriminator: "simulate a Reserve": true iff an empty entry can be claimed in
  // buffers V_traj+eta down to V_traj (never below consumed_upto).
  bool verify(int v) const {
    for (int b = v + eta; b >= std::max(v, cu); --b)
      if (has_empty(b)) return true;
    return false;
  }
  // Reserve: "backward scan across buffers from V_buf = V_traj + eta ... down to
  // V_buf = V_traj, reserving the latest available empty entry"; latest slot = highest index.
  bool reserve(int g, int v, int *ob, int *os) {
    for (int b = v + eta; b >= std::max(v, cu); --b) {
      ensure(b);
      for (int s = B - 1; s >= 0; --s) {
        if (buf[b][s].st == E_EMPTY) {
          buf[b][s].st = E_RESERVED; buf[b][s].g = g; buf[b][s].v = v;
          *ob = b; *os = s;
          return true;
        }
      }
    }
    return false;
  }
  bool find(int g, int *ob, int *os) const {
    for (int b = cu; b < (int)buf.size(); ++b)
      for (int s = 0; s < B; ++s)
        if (buf[b][s].st != E_EMPTY && buf[b][s].g == g) { *ob = b; *os = s; return true; }
    return false;
  }
  // Entry deletion and movement: delete the reserved entry at (b, s); then
  // repeatedly "scan buffers from smallest up to V_buf to find the earliest reserved entry B
  // satisfying V_B + eta >= V_buf, and move B to A's position" (A13: iterate to a fixpoint;
  // earliest buffer first, then lowest slot).  Returns the number of moves.
  int delete_and_relocate(int b, int s, int *fhb = nullptr, int *fhs = nullptr) {
    buf[b][s] = Entry();
    int hb = b, hs = s, moves = 0;
    for (;;) {
      bool found = false;
      for (int bb = cu; bb < hb && !found; ++bb) {
        for (int ss = 0; ss < B; ++ss) {
          const Entry &e = buf[bb][ss];
          if (e.st == E_RESERVED && e.v + eta >= hb) {
            buf[hb][hs] = e;
            buf[bb][ss] = Entry();
            hb = bb; hs = ss; ++moves;
            found = true;
            break;
          }
        }
      }
      if (!found) break;
    }
    if (fhb) { *fhb = hb; *fhs = hs; }
    return moves;
  }
  // Filtering (P:413 (2): "after abortion, occupied entries from later buffers can be moved
  // forward to fill the empty slot"; SPEC abort op S:96-103), reading R-FILTER: the hole at
  // (hb, hs) takes the Occupied entry of the earliest later buffer (lowest slot) whose version
  // admits buffer hb (v <= hb; v + eta >= hb holds since it sat in a later buffer); repeated with
  // the hole that move leaves.  Returns the number of moves.
  int fill_forward(int hb, int hs) {
    int moves = 0;
    for (;;) {
      bool found = false;
      for (int bb = hb + 1; bb < (int)buf.size() && !found; ++bb) {
        for (int ss = 0; ss < B; ++ss) {
          const Entry &e = buf[bb][ss];
          if (e.st == E_OCCUPIED && e.v <= hb) {
            buf[hb][hs] = e;
            buf[bb][ss] = Entry();
            hb = bb; hs = ss; ++moves;
            found = true;
            break;
          }
        }
      }
      if (!found) break;
    }
    return moves;
  }
  // Abort a tracked entry: a Reserved one through delete_and_relocate, an Occupied
  // one by emptying its slot; then fill_forward.  false if g has no entry (UnknownKey).
  bool abort_entry(int g, int *moves) {
    int b = -1, sl = -1;
    if (!find(g, &b, &sl)) return false;
    int hb = b, hs = sl, m = 0;
    if (buf[b][sl].st == E_RESERVED) m = delete_and_relocate(b, sl, &hb, &hs);
    else buf[b][sl] = Entry();
    m += fill_forward(hb, hs);
    if (moves) *moves = m;
    return true;
  }
  // Occupy: "scans forward and greedily occupies the earliest available empty entry"
  // (from consumed_upto, lowest slot first).
  bool occupy(int g, int v, int *ob, int *os) {
    for (int b = cu; b <= cu + eta + 1; ++b) {
      ensure(b);
      for (int s = 0; s < B; ++s) {
        if (buf[b][s].st == E_EMPTY) {
          buf[b][s].st = E_OCCUPIED; buf[b][s].g = g; buf[b][s].v = v;
          *ob = b; *os = s;
          return true;
        }
      }
    }
    return false;
  }
  // Buffer states: Ready (all occupied; under batch-level redundancy >= Br occupied,
  // S:41), Waiting (>= 1 empty), Stuck (full with >= 1 reserved).
  int state(int b) const {
    int occ = 0;
    if (b < (int)buf.size())
      for (int s = 0; s < B; ++s) occ += buf[b][s].st == E_OCCUPIED;
    if (occ >= Br) return 1;
    return has_empty(b) ? 0 : 2;
  }
};

// ============================================================== cost model (§5.3, App B)
namespace {
struct Params {
  int64_t k1, k2, k3, k4; int k5; int64_t kp, M;
  double mu, phi_tp; int phi_wait; int eta;
};
Params from_sfo(const sfo_params *p) {
  Params q;
  q.k1 = p->k1; q.k2 = p->k2; q.k3 = p->k3; q.k4 = p->k4; q.k5 = p->k5; q.kp = p->kp; q.M = p->M;
  q.mu = p->mu; q.phi_tp = p->phi_tp; q.phi_wait = p->phi_wait; q.eta = p->eta;
  return q;
}
struct View { int v; int64_t kv; int n_run; int n_wait; };
struct Item { int id; int g; int v; int l; };

// Eq 7 plus the prefill stall of reading A20, exact int64 picoseconds.
int64_t tick_latency(const Params &P, int64_t kv, int64_t n, int64_t prefill) {
  return P.k1 * kv + std::max(P.k2, P.k3 * n) + P.k4 + P.kp * prefill;
}
// Eq 2: T_i(S) = |run| / (k1 kv + max(k2, k3 |run|) + k4); 0 for an empty instance.
double throughput(const Params &P, int64_t n, int64_t kv) {
  if (n == 0) return 0.0;
  int64_t den = P.k1 * kv + std::max(P.k2, P.k3 * n) + P.k4;
  return (double)n / (double)den;
}
// Eq 3: gamma = (kv + k5 l <= M) and |wait| = 0; dT = T(S') - T(S); 0 when gamma = 0.
double marginal_gain(const Params &P, const View &s, int l) {
  bool gamma = (s.kv + (int64_t)P.k5 * l <= P.M) && (s.n_wait == 0);
  if (!gamma) return 0.0;
  return throughput(P, s.n_run + 1, s.kv + (int64_t)P.k5 * l) - throughput(P, s.n_run, s.kv);
}
// Eq 4 (Alg 2 line P:1175): 1 / (k1 k5 l + max(k2, k3) + k4).
double ideal_gain(const Params &P, int l) {
  int64_t den = P.k1 * (int64_t)P.k5 * l + std::max(P.k2, P.k3) + P.k4;
  return 1.0 / (double)den;
}
// check_routable (Alg P:1111-1129, reading A10: the tentative V_traj is a local).
bool check_routable(const View &s, int tau_v, const sfo_ledger &L) {
  if (tau_v < 0) return L.verify(s.v);
  return s.v >= tau_v;
}

// MLQ (Alg 2 line P:1148): queues by V_traj ascending, versionless last, by id within.
std::vector<Item> mlq_sort(std::vector<Item> items) {
  std::stable_sort(items.begin(), items.end(), [](const Item &a, const Item &b) {
    bool av = a.v >= 0, bv = b.v >= 0;
    if (av != bv) return av;            // versioned queues before the versionless queue
    if (a.v != b.v) return a.v < b.v;
    return a.id < b.id;
  });
  return items;
}

struct RouteDecision { int k; int inst; int vg_assigned; int b; int s; };

// Routing strategy, Alg 2, or vanilla routing (§6.5).  Items are routed
// strictly in the given MLQ order and the pass stops at the first trajectory that has no
// candidate or clears no threshold.  Reading A11: the first routed
// member of a versionless group fixes v_g = S[i].v and Reserves; later members use the
// partially-generated rule S[i].v >= v_g.
std::vector<RouteDecision> route(const Params &P, std::vector<View> &S, const std::vector<Item> &mlq,
                                 sfo_ledger &L, bool vanilla) {
  std::vector<RouteDecision> out;
  std::map<int, int> pass_vg;           // group -> V_traj assigned in this pass
  const int I = (int)S.size();
  for (int k = 0; k < (int)mlq.size(); ++k) {
    const Item &tau = mlq[k];
    int vg = tau.v;
    if (vg < 0 && pass_vg.count(tau.g)) vg = pass_vg[tau.g];
    // Step 1: candidate instances.
    std::vector<int> cand;
    for (int i = 0; i < I; ++i)
      if (check_routable(S[i], vg, L)) cand.push_back(i);
    if (cand.empty()) break;
    int sel = -1;
    if (vanilla) {
      // "Each trajectory in TS is routed to the instance with the fewest trajectories".
      for (int i : cand)
        if (sel < 0 || S[i].n_run + S[i].n_wait < S[sel].n_run + S[sel].n_wait) sel = i;
    } else {
      // Step 2: group by ascending inst_version.  Step 3: ideal gain.  Step 4: waterfall.
      double ideal = ideal_gain(P, tau.l);
      double thr = P.mu * ideal;
      std::vector<int> versions;
      for (int i : cand) versions.push_back(S[i].v);
      std::sort(versions.begin(), versions.end());
      versions.erase(std::unique(versions.begin(), versions.end()), versions.end());
      for (int ver : versions) {
        double best = -std::numeric_limits<double>::infinity();
        int bi = -1;
        for (int i : cand) {
          if (S[i].v != ver) continue;
          double dT = marginal_gain(P, S[i], tau.l);
          if (dT > best) { best = dT; bi = i; }
        }
        if (best >= thr) { sel = bi; break; }   // accept (Alg 2 line P:1191, A4)
      }
    }
    if (sel < 0) break;
    // Step 5: route, update the working snapshot (Eq 3's S'), Reserve for a new version.
    RouteDecision d{k, sel, -1, -1, -1};
    if (vg < 0) {
      vg = S[sel].v;
      pass_vg[tau.g] = vg;
      d.vg_assigned = vg;
      if (!L.reserve(tau.g, vg, &d.b, &d.s)) { d.inst = -2; out.push_back(d); return out; }
    }
    bool gamma = (S[sel].kv + (int64_t)P.k5 * tau.l <= P.M) && (S[sel].n_wait == 0);
    if (gamma) { S[sel].n_run += 1; S[sel].kv += (int64_t)P.k5 * tau.l; }
    else { S[sel].n_wait += 1; }
    out.push_back(d);
  }
  return out;
}

// Synchronization strategy, Alg 3; vanilla: every stale instance.
// Reading A16: each candidate is tried against the original S with only its version changed;
// the ledger used by the tentative routing is a scratch copy.
std::vector<int> sync_select(const Params &P, const std::vector<View> &S, const std::vector<Item> &mlq,
                             const sfo_ledger &L, int ps, bool vanilla_sync, bool vanilla_route) {
  std::vector<int> sel;
  const int I = (int)S.size();
  if (vanilla_sync) {
    for (int i = 0; i < I; ++i) if (S[i].v < ps) sel.push_back(i);
    return sel;
  }
  std::vector<int> cand;
  for (int i = 0; i < I; ++i) {
    if (ps > S[i].v) {
      bool can_route = false;
      for (const Item &tau : mlq)
        if (check_routable(S[i], tau.v, L)) { can_route = true; break; }
      if (!can_route) cand.push_back(i);
    }
  }
  for (int i : cand) {
    std::vector<View> tmp = S;
    tmp[i].v = ps;
    sfo_ledger Ltmp = L;
    std::vector<RouteDecision> r = route(P, tmp, mlq, Ltmp, vanilla_route);
    bool routed_to_i = false;
    for (const RouteDecision &d : r) if (d.inst == i) { routed_to_i = true; break; }
    if (routed_to_i) sel.push_back(i);
  }
  return sel;
}

// Migration strategy, Alg 4.  case1_k[i]: excess waiting trajectories (A7: the
// tail of the wait queue); case2: the highest-throughput instance when max/min > phi (A5, A6, A8).
void migrate(const Params &P, const std::vector<View> &S0, std::vector<int> &case1_k, int &case2) {
  std::vector<View> S = S0;
  const int I = (int)S.size();
  case1_k.assign(I, 0);
  for (int i = 0; i < I; ++i) {
    int wait_cnt = S[i].n_wait;
    if (wait_cnt > P.phi_wait) {
      case1_k[i] = wait_cnt - P.phi_wait;
      S[i].n_wait -= case1_k[i];
    }
  }
  std::vector<double> T(I);
  for (int i = 0; i < I; ++i) T[i] = throughput(P, S[i].n_run, S[i].kv);
  int imax = 0, imin = 0;
  for (int i = 1; i < I; ++i) {
    if (T[i] > T[imax]) imax = i;
    if (T[i] < T[imin]) imin = i;
  }
  case2 = -1;
  if (T[imin] > 0.0) {
    double gap = T[imax] / T[imin];
    if (gap > P.phi_tp) {
      int remaining = S0[imax].n_run + S0[imax].n_wait - case1_k[imax];
      if (remaining > 0) case2 = imax;
    }
  }
}
}  // namespace

// ============================================================== discrete-event simulation
namespace {
enum { L_POOL = 0, L_TS = 1, L_TRANSIT = 2, L_WAIT = 3, L_RUN = 4, L_DONE = 5, L_CONSUMED = 6, L_ABORTED = 7 };
enum { I_IDLE = 0, I_TICK = 1, I_PULL = 2 };
enum { CMD_ROUTE = 1, CMD_INTERRUPT = 2, CMD_PULL = 3, CMD_ABORT = 4 };
enum {
  M_WINDOWS = 0, M_TICKS, M_TRAJ_ITERS, M_TOKENS, M_COMPLETIONS, M_ROUTES, M_INTERRUPTS, M_PULLS,
  M_PREEMPTIONS, M_BATCHES, M_VALID_SNAP, M_INVALID_SNAP, M_VIOLATIONS, M_PUBLISHES, M_INGESTED,
  M_OCCUPIED, M_HIST0 /* ..M_HIST0+8 */, M_CMD_HASH = 25, M_SIM_TIME = 26, M_RESERVES = 27,
  M_RELOCATIONS = 28, M_ABORTS = 31
};
const int64_t INF = std::numeric_limits<int64_t>::max();

struct Traj {
  int g = 0, T = 0, gen = 0, st = L_POOL, inst = -1;
  bool rewarded = false;
  int n_routes = 0, n_preempt = 0, n_interrupt = 0;
  int64_t t_complete = -1, ready = 0;
};
struct Group { int p = 0, v = -1, n_rewarded = 0, consumed_vbuf = -1; bool filter = false, retired = false; };
struct Arrival { int64_t t; int id; };
struct Inst {
  int v = 0; int64_t kv = 0; std::vector<int> run; std::deque<int> wait; int c = 0;
  int st = I_IDLE; int64_t nb = 0, pull_until = 0; int pull_version = 0;
  bool pull_pending = false, cmd_at_t = false;
  std::vector<std::pair<int, int64_t>> interrupt_set;   // (trajectory, context held here at issue)
  std::vector<int> abort_set;                           // pending Abort commands (run / wait members)
  std::vector<Arrival> arrivals;
  int64_t prefill = 0;
  int pv = 0, acc = 0;                   // speculative state P[i], initialised to 0
};
struct Ev { int64_t t; int id; };

struct Scen {
  Params P;
  int I = 0, eta = 0, B = 0, G = 0; uint32_t strategy = 0;
  int Br = 0, Gr = 0;              // batch size and required members; B, G include redundancy (App C)
  int64_t delta = 0, r = 0, q = 0, R = 0; int atw = 0; int pool_cap = 0;
  int wd = 0, wd_idle = 0; int64_t wd_sig = 0;     // deadlock watchdog
  std::vector<Traj> traj; std::vector<Group> grp;
  int n_pool = 0, n_ingested = 0, live = 0;
  int settled = 0;                 // groups [0, settled) have every member DONE / CONSUMED / ABORTED
  std::vector<Inst> inst;
  sfo_ledger L;
  int ps = 0; int64_t t = 0, window = 0;
  bool trainer_busy = false; int64_t publish_at = 0;
  std::vector<Ev> rewards;
  std::vector<int> batches;
  std::vector<int64_t> cmds;
  uint64_t cmd_hash = 0;
  int64_t m[SFO_METRICS_LEN];
  int err = 0;
};

// Command checksum: the sum mod 2^64 of one mixed word per record, keyed by the
// record's index in the scenario's command stream (so reordering changes it).
uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
uint64_t record_hash(uint64_t index, int64_t window, int kind, int inst, int traj) {
  const uint64_t a = (uint64_t)window * 0x9E3779B97F4A7C15ULL + index;
  const uint64_t b = ((uint64_t)(uint32_t)traj << 32) | ((uint64_t)(uint32_t)kind << 24) | ((uint64_t)(uint32_t)inst & 0xffffffULL);
  return mix64(mix64(a) ^ b);
}
void log_cmd(Scen &s, int kind, int inst, int traj) {
  const uint64_t index = s.cmds.size() / 4;
  s.cmd_hash += record_hash(index, s.window, kind, inst, traj);
  int64_t w[4] = {s.window, kind, inst, traj};
  for (int k = 0; k < 4; ++k) s.cmds.push_back(w[k]);
}
int ctx_len(const Scen &s, int j) { return s.grp[s.traj[j].g].p + s.traj[j].gen; }

// Abort (P:473 footnote; Table 1 row P:577): trajectory j leaves for good.  On an instance it is
// removed at that instance's next boundary; an arrival in transit is dropped at delivery; a
// TS-resident one is dropped from the TS; a completed one's pending reward is ignored.
void abort_member(Scen &s, int j, bool force = false) {
  Traj &tr = s.traj[j];
  const int st = tr.st;
  // a rewarded member is kept unless its whole group is dropped (filtering, reading R-FILTER)
  if (st == L_ABORTED || st == L_CONSUMED || (tr.rewarded && !force)) return;
  if (st == L_TRANSIT || st == L_WAIT || st == L_RUN) {
    log_cmd(s, CMD_ABORT, tr.inst, j);
    s.inst[tr.inst].acc -= 1;
    if (s.inst[tr.inst].acc < 0) s.err = SFO_E_STATE;
    if (st != L_TRANSIT) s.inst[tr.inst].abort_set.push_back(j);
  }
  tr.st = L_ABORTED;
  s.m[M_ABORTS]++;
}

void abort_group(Scen &s, int g) {
  for (int m = 0; m < s.G; ++m) abort_member(s, g * s.G + m);
}

// Filtering (P:413 (2), reading R-FILTER): group g's ledger entry is aborted (abort_entry) and
// every member not yet consumed leaves (Abort commands for the in-flight ones); the group stops
// counting toward the live-group cap.
void filter_group(Scen &s, int g) {
  int moves = 0;
  if (!s.L.abort_entry(g, &moves)) { s.err = SFO_E_STATE; return; }
  s.m[M_RELOCATIONS] += moves;
  for (int m = 0; m < s.G; ++m) abort_member(s, g * s.G + m, true);
  s.grp[g].retired = true;
  s.live -= 1;
}

// Consume: retire the earliest Ready buffer as one batch -- its first Br Occupied entries in
// slot order; surplus entries (Occupied beyond Br, and Reserved) are aborted (App C).
// Staleness check (A30).
void consume(Scen &s, int *vbuf, int *gids, int *gv) {
  int cu = s.L.cu;
  if (vbuf) *vbuf = cu;
  s.batches.push_back(cu);
  int taken = 0, nonempty = 0;
  std::vector<int> surplus;
  for (int k = 0; k < s.B; ++k) {
    const Entry &e = s.L.buf[cu][k];
    if (e.st == E_EMPTY) continue;
    ++nonempty;
    if (e.st != E_OCCUPIED || taken == s.Br) { surplus.push_back(e.g); continue; }
    int stal = cu - e.v;
    if (stal < 0 || stal > s.eta) { s.m[M_VIOLATIONS]++; s.err = SFO_E_STATE; }
    s.m[M_HIST0 + std::min(std::max(stal, 0), 8)]++;
    s.grp[e.g].consumed_vbuf = cu;
    for (int m = 0; m < s.G; ++m)
      if (s.traj[e.g * s.G + m].rewarded) s.traj[e.g * s.G + m].st = L_CONSUMED;
    s.batches.push_back(e.g);
    s.batches.push_back(e.v);
    if (gids) gids[taken] = e.g;
    if (gv) gv[taken] = e.v;
    ++taken;
  }
  for (int g : surplus) abort_group(s, g);
  s.L.cu = cu + 1;
  s.live -= nonempty;
  s.m[M_BATCHES]++;
}

// Alg 1 on a validated snapshot: sync -> migration -> routing, issuing commands.
void coordinate(Scen &s) {
  const Params &P = s.P;
  const int64_t t = s.t;
  // Those three states are final (a trajectory never leaves them for the TS), so the TS scans below
  // can start after the leading run of groups whose members are all in them (a scan bound only).
  auto final_state = [&](int j) { return s.traj[j].st == L_DONE || s.traj[j].st == L_CONSUMED || s.traj[j].st == L_ABORTED; };
  while (s.settled < s.n_ingested) {
    bool all = true;
    for (int m = 0; m < s.G; ++m) all = all && final_state(s.settled * s.G + m);
    if (!all) break;
    s.settled++;
  }
  const int j0 = s.settled * s.G;
  // get_ts_trajs(): trajectories resident in the TS, MLQ-ordered.
  auto ts_items = [&]() {
    std::vector<Item> it;
    for (int j = j0; j < s.n_ingested * s.G; ++j)
      if (s.traj[j].st == L_TS) it.push_back(Item{j, s.traj[j].g, s.grp[s.traj[j].g].v, ctx_len(s, j)});
    return mlq_sort(it);
  };
  for (int j = j0; j < s.n_ingested * s.G; ++j)
    if (s.traj[j].st == L_TS) s.traj[j].ready = t;          // TS-resident: ready now (A18)
  std::vector<Item> mlq = ts_items();
  const int ps = s.ps;                                   // get_ps_version()
  std::vector<View> S(s.I);
  for (int i = 0; i < s.I; ++i)
    S[i] = View{s.inst[i].v, s.inst[i].kv, (int)s.inst[i].run.size(), (int)s.inst[i].wait.size()};
  auto apply_time = [&](int i) { return s.inst[i].st == I_TICK ? s.inst[i].nb : t; };
  auto interrupt = [&](int i, const std::vector<int> &victims) {
    for (int j : victims) {
      log_cmd(s, CMD_INTERRUPT, i, j);
      s.inst[i].interrupt_set.push_back({j, (int64_t)ctx_len(s, j)});
      s.traj[j].st = L_TS;
      s.traj[j].ready = apply_time(i);
      s.traj[j].n_interrupt++;
    }
    s.m[M_INTERRUPTS] += (int64_t)victims.size();
    s.inst[i].acc -= (int)victims.size();                  // Table 1, Interrupt row
    if (s.inst[i].acc < 0) s.err = SFO_E_STATE;            // NegativeCount
  };
  // Lines 3-8: synchronization.
  bool vanilla_route = !(s.strategy & 1u), vanilla_sync = !(s.strategy & 2u);
  std::vector<int> sel = sync_select(P, S, mlq, s.L, ps, vanilla_sync, vanilla_route);
  for (int i : sel) {
    std::vector<int> victims(s.inst[i].run.begin(), s.inst[i].run.end());
    victims.insert(victims.end(), s.inst[i].wait.begin(), s.inst[i].wait.end());
    if (!victims.empty()) interrupt(i, victims);           // only if non-empty
    log_cmd(s, CMD_PULL, i, -1);
    s.inst[i].pull_pending = true;
    s.inst[i].pull_version = ps;                           // delivered version captured at issue (A19)
    s.m[M_PULLS]++;
    s.inst[i].pv = ps; s.inst[i].acc = 0;                  // Table 1, Pull row
    S[i] = View{ps, 0, 0, 0};                              // discard + inst_version <- ps
  }
  // Lines 9-12: migration (StaleFlow only; vanilla migration is "no proactive migration").
  if (s.strategy & 4u) {
    std::vector<int> case1_k; int case2 = -1;
    migrate(P, S, case1_k, case2);
    std::vector<std::vector<int>> case1_victims(s.I);
    for (int i = 0; i < s.I; ++i) {
      if (case1_k[i] == 0) continue;
      const std::deque<int> &w = s.inst[i].wait;
      std::vector<int> victims(w.end() - case1_k[i], w.end());
      case1_victims[i] = victims;
      interrupt(i, victims);
      S[i].n_wait -= (int)victims.size();
    }
    if (case2 >= 0) {
      int i = case2;
      std::vector<int> victims;
      for (int j : s.inst[i].run) victims.push_back(j);
      for (int j : s.inst[i].wait)
        if (std::find(case1_victims[i].begin(), case1_victims[i].end(), j) == case1_victims[i].end())
          victims.push_back(j);
      interrupt(i, victims);
      S[i].kv = 0; S[i].n_run = 0; S[i].n_wait = 0;        // discard (A17)
    }
  }
  // Lines 11-13: routing over the TS (now including the interrupted trajectories).
  std::vector<Item> mlq2 = ts_items();
  std::vector<RouteDecision> routes = route(P, S, mlq2, s.L, vanilla_route);
  for (const RouteDecision &d : routes) {
    if (d.inst < 0) { s.err = SFO_E_STATE; return; }
    const Item &tau = mlq2[d.k];
    int j = tau.id;
    if (d.vg_assigned >= 0) { s.grp[tau.g].v = d.vg_assigned; s.m[M_RESERVES]++; }
    log_cmd(s, CMD_ROUTE, d.inst, j);
    s.traj[j].st = L_TRANSIT;
    s.traj[j].inst = d.inst;
    s.traj[j].n_routes++;
    s.inst[d.inst].arrivals.push_back(Arrival{s.traj[j].ready + s.r, j});  // t_arr = t_ready + r (A18)
    s.inst[d.inst].acc += 1;                                              // Table 1, Route row
    s.m[M_ROUTES]++;
  }
}

// Boundary procedure B1-B8 at instance i, time b.
void boundary(Scen &s, int i, int64_t b) {
  Inst &n = s.inst[i];
  const Params &P = s.P;
  const bool tick_end = (n.st == I_TICK && b == n.nb);
  const bool pull_done = (n.st == I_PULL && b == n.pull_until);
  n.cmd_at_t = false;
  // B1: pending interrupts leave run/wait without this tick's token; their KV is released.
  if (n.st != I_PULL && !n.interrupt_set.empty()) {
    // The KV released is the context this instance holds (A17): the trajectory's progress is
    // frozen here since issue, while it may already be running elsewhere after re-routing.
    for (const auto &jc : n.interrupt_set) {
      const int j = jc.first;
      auto it = std::find(n.run.begin(), n.run.end(), j);
      if (it != n.run.end()) { n.kv -= (int64_t)P.k5 * jc.second; n.run.erase(it); continue; }
      auto jt = std::find(n.wait.begin(), n.wait.end(), j);
      if (jt != n.wait.end()) { n.wait.erase(jt); continue; }
      s.err = SFO_E_STATE;
    }
    n.interrupt_set.clear();
  }
  // B1 (Abort): removed like an interrupt, but the trajectory does not return to the TS.  Unlike
  // interrupts (issued only on a valid snapshot, never to a pulling instance), aborts come from
  // Consume and reward processing at any time, so they apply at every boundary, the end of a
  // pull included (reading R-ABORT; a pulling instance was drained by Alg 3, so there only held
  // arrivals can be aborted, and those are dropped at B6).
  if (!n.abort_set.empty()) {
    for (int j : n.abort_set) {
      auto it = std::find(n.run.begin(), n.run.end(), j);
      if (it != n.run.end()) { n.kv -= (int64_t)P.k5 * ctx_len(s, j); n.run.erase(it); continue; }
      auto jt = std::find(n.wait.begin(), n.wait.end(), j);
      if (jt != n.wait.end()) { n.wait.erase(jt); continue; }
      s.err = SFO_E_STATE;
    }
    n.abort_set.clear();
  }
  if (tick_end) {
    // B2: one token for every remaining tick member (batched decode).
    for (int j : n.run) { s.traj[j].gen += 1; n.kv += P.k5; s.m[M_TOKENS]++; }
    // B3: completions leave run in order; reward event at b + R.
    std::vector<int> keep;
    for (int j : n.run) {
      Traj &tr = s.traj[j];
      if (tr.gen == tr.T) {
        n.kv -= (int64_t)P.k5 * ctx_len(s, j);
        n.c += 1;
        tr.st = L_DONE; tr.t_complete = b;
        s.rewards.push_back(Ev{b + s.R, j});
        s.m[M_COMPLETIONS]++;
      } else {
        keep.push_back(j);
      }
    }
    n.run = keep;
    n.st = I_IDLE;
  }
  if (pull_done) { n.v = n.pull_version; n.c = 0; n.st = I_IDLE; }
  // B4: preemption while the KV cache exceeds the budget: newest admitted -> wait front.
  while (n.kv > P.M) {
    int j = n.run.back();
    n.run.pop_back();
    n.kv -= (int64_t)P.k5 * ctx_len(s, j);
    n.wait.push_front(j);
    s.traj[j].st = L_WAIT; s.traj[j].n_preempt++;
    s.m[M_PREEMPTIONS]++;
  }
  // B5: a pending Pull blocks generation for q.
  if (n.pull_pending) {
    n.pull_pending = false;
    n.st = I_PULL;
    n.pull_until = b + s.q;
    return;
  }
  // B6: arrivals with t_arr <= b join the wait tail in (t_arr, id) order (held while pulling).
  std::sort(n.arrivals.begin(), n.arrivals.end(), [](const Arrival &a, const Arrival &c) {
    return a.t != c.t ? a.t < c.t : a.id < c.id;
  });
  std::vector<Arrival> later;
  for (const Arrival &a : n.arrivals) {
    if (a.t > b) later.push_back(a);
    else if (s.traj[a.id].st != L_ABORTED) { n.wait.push_back(a.id); s.traj[a.id].st = L_WAIT; }
  }
  n.arrivals = later;
  // B7: FIFO admission while the head fits in the KV budget (Eq 3's gamma rule).
  while (!n.wait.empty()) {
    int j = n.wait.front();
    int64_t ctx = ctx_len(s, j);
    if (n.kv + (int64_t)P.k5 * ctx > P.M) break;
    n.wait.pop_front();
    n.run.push_back(j);
    n.kv += (int64_t)P.k5 * ctx;
    n.prefill += ctx;
    s.traj[j].st = L_RUN;
  }
  // Invariant: kv = k5 x sum of the contexts of the running trajectories.
  {
    int64_t sum = 0;
    for (int j : n.run) sum += (int64_t)P.k5 * ctx_len(s, j);
    if (sum != n.kv || n.kv > P.M) s.err = SFO_E_STATE;
  }
  // B8: start the next decode step (Eq 7 + prefill stall, A20).
  if (!n.run.empty()) {
    int64_t Lat = tick_latency(P, n.kv, (int64_t)n.run.size(), n.prefill);
    n.prefill = 0;
    n.nb = b + Lat;
    n.st = I_TICK;
    s.m[M_TRAJ_ITERS] += (int64_t)n.run.size();
    s.m[M_TICKS]++;
  } else {
    n.st = I_IDLE;
  }
}

int64_t next_boundary(const Scen &s, const Inst &n) {
  if (n.st == I_TICK) return n.nb;
  if (n.st == I_PULL) return n.pull_until;
  int64_t b = INF;
  if (n.cmd_at_t) b = s.t;
  for (const Arrival &a : n.arrivals) b = std::min(b, a.t);
  return b;
}

// Staleness-manager side of a completed reward.
void apply_reward(Scen &s, int j) {
  if (s.traj[j].st == L_ABORTED) return;    // aborted after completing: the reward is ignored
  int g = s.traj[j].g;
  Group &gr = s.grp[g];
  s.traj[j].rewarded = true;
  gr.n_rewarded += 1;
  if (gr.n_rewarded < s.Gr) return;         // group sampling: occupy when Gr members complete
  // group-level redundancy: the surplus members are aborted the moment the group completes
  for (int m = 0; m < s.G; ++m) abort_member(s, g * s.G + m);
  int b = -1, sl = -1;
  if (!s.L.find(g, &b, &sl) || s.L.buf[b][sl].st != E_RESERVED) { s.err = SFO_E_STATE; return; }
  if (gr.filter) { filter_group(s, g); return; }   // no learning signal (P:413 (2), DAPO): dropped
  s.m[M_RELOCATIONS] += s.L.delete_and_relocate(b, sl);
  int ob = -1, os = -1;
  if (!s.L.occupy(g, gr.v, &ob, &os)) { s.err = SFO_E_STATE; return; }
  if (ob < gr.v || ob > gr.v + s.eta) { s.m[M_VIOLATIONS]++; s.err = SFO_E_STATE; }
  s.m[M_OCCUPIED]++;
}

void run_window(Scen &s) {
  if (s.err) return;
  const int64_t t = s.t, t_end = s.t + s.delta;
  // W10 (auto trainer) at the window boundary: publish if due, then consume if Ready (A24).
  if (s.atw > 0) {
    if (s.trainer_busy && s.publish_at <= t) { s.ps += 1; s.trainer_busy = false; s.m[M_PUBLISHES]++; }
    if (!s.trainer_busy && s.L.state(s.L.cu) == 1) {
      consume(s, nullptr, nullptr, nullptr);
      s.trainer_busy = true;
      s.publish_at = t + (int64_t)s.atw * s.delta;
    }
  }
  // W1: TS ingest up to (eta+1) x batch_size live groups (A23).
  while (s.live < (s.eta + 1) * s.B && s.n_ingested < s.n_pool) {   // B includes extra groups
    int g = s.n_ingested++;
    s.live++;
    s.m[M_INGESTED]++;
    for (int m = 0; m < s.G; ++m) s.traj[g * s.G + m].st = L_TS;
  }
  // W2: snapshot + Eq 1 validation (reading R-EQ1).
  bool valid = true;
  for (int i = 0; i < s.I; ++i) {
    const Inst &n = s.inst[i];
    bool quiescent = n.interrupt_set.empty() && n.abort_set.empty() && !n.pull_pending && n.arrivals.empty() &&
                     n.st != I_PULL;
    bool eq1 = n.pv == n.v && n.acc == (int)n.run.size() + (int)n.wait.size() + n.c;
    if (quiescent && !eq1) { s.m[M_VIOLATIONS]++; s.err = SFO_E_STATE; }
    if (!(quiescent && eq1)) valid = false;
  }
  if (valid) { s.m[M_VALID_SNAP]++; coordinate(s); }
  else s.m[M_INVALID_SNAP]++;
  if (s.err) return;
  // W6: commands to an idle instance apply now, as a boundary at t.
  for (int i = 0; i < s.I; ++i) {
    Inst &n = s.inst[i];
    if (n.st == I_IDLE && (n.pull_pending || !n.interrupt_set.empty() || !n.abort_set.empty())) n.cmd_at_t = true;
  }
  // W7: every instance advances through its boundaries <= t + Delta.
  for (int i = 0; i < s.I; ++i) {
    for (;;) {
      int64_t b = next_boundary(s, s.inst[i]);
      if (b == INF || b > t_end) break;
      boundary(s, i, b);
      if (s.err) return;
    }
  }
  // W8: reward events <= t + Delta in (time, id) order -> ledger.
  std::sort(s.rewards.begin(), s.rewards.end(), [](const Ev &a, const Ev &c) {
    return a.t != c.t ? a.t < c.t : a.id < c.id;
  });
  std::vector<Ev> later;
  for (const Ev &e : s.rewards) {
    if (e.t <= t_end) apply_reward(s, e.id);
    else later.push_back(e);
  }
  s.rewards = later;
  // Deadlock watchdog ("no events pending but steps unfinished", auto trainer only): a
  // window that made no progress (no decode step, command, completion, Occupy, Consume, publish or
  // ingest) ending with nothing pending (every instance idle without pending commands or arrivals,
  // no reward in flight, trainer idle) while groups remain unconsumed is a fixed point; the
  // scenario fails after wd such windows in a row.
  if (s.wd > 0 && s.atw > 0) {
    const int64_t sig = s.m[M_TICKS] + s.m[M_ROUTES] + s.m[M_INTERRUPTS] + s.m[M_PULLS] + s.m[M_COMPLETIONS] +
                        s.m[M_OCCUPIED] + s.m[M_BATCHES] + s.m[M_PUBLISHES] + s.m[M_INGESTED] + s.m[M_ABORTS];
    bool pending = s.trainer_busy || !s.rewards.empty();
    for (const Inst &n : s.inst)
      pending = pending || n.st != I_IDLE || n.pull_pending || !n.interrupt_set.empty() || !n.abort_set.empty() ||
                !n.arrivals.empty();
    const bool work_left = s.live > 0 || s.n_ingested < s.n_pool;
    if (sig == s.wd_sig && !pending && work_left) {
      if (++s.wd_idle >= s.wd) s.err = SFO_E_STATE;
    } else {
      s.wd_idle = 0;
    }
    s.wd_sig = sig;
  }
  // W9.
  s.t = t_end;
  s.window += 1;
  s.m[M_WINDOWS]++;
}
}  // namespace

struct sfo_sim {
  std::vector<Scen> sc;
  int err = 0;
};

// ============================================================== C ABI
extern "C" {

int sfo_create(int32_t instances, int32_t eta, int32_t group_size, const sfo_config *cfg, sfo_sim **out) {
  if (!cfg || !out || group_size < 1 || cfg->batch_size < 1 || cfg->n_scenarios < 1 ||
      cfg->pool_capacity_groups < 1 || cfg->delta <= 0 || cfg->k5 < 1)
    return SFO_E_INVALID;
  sfo_sim *sim = new (std::nothrow) sfo_sim();
  if (!sim) return SFO_E_INVALID;
  sim->sc.resize(cfg->n_scenarios);
  for (int k = 0; k < cfg->n_scenarios; ++k) {
    Scen &s = sim->sc[k];
    s.I = cfg->scenario_instances ? cfg->scenario_instances[k] : instances;
    s.eta = cfg->scenario_eta ? cfg->scenario_eta[k] : eta;
    s.strategy = cfg->scenario_strategy ? cfg->scenario_strategy[k] : cfg->strategy;
    if (s.I < 1 || s.eta < 0) { delete sim; return SFO_E_INVALID; }
    if (cfg->extra_groups < 0 || cfg->extra_members < 0) { delete sim; return SFO_E_INVALID; }
    s.Br = cfg->batch_size; s.Gr = group_size;
    s.B = cfg->batch_size + cfg->extra_groups; s.G = group_size + cfg->extra_members;
    s.P = Params{cfg->k1, cfg->k2, cfg->k3, cfg->k4, cfg->k5, cfg->kp, cfg->M,
                 cfg->mu, cfg->phi_tp, cfg->phi_wait, s.eta};
    s.delta = cfg->delta; s.r = cfg->r; s.q = cfg->q; s.R = cfg->R; s.atw = cfg->atw;
    s.wd = cfg->watchdog_windows;
    s.pool_cap = cfg->pool_capacity_groups;
    s.traj.assign((size_t)s.pool_cap * s.G, Traj());
    s.grp.assign(s.pool_cap, Group());
    s.inst.assign(s.I, Inst());
    s.L.eta = s.eta; s.L.B = s.B; s.L.Br = s.Br;
    std::memset(s.m, 0, sizeof(s.m));
  }
  *out = sim;
  return SFO_OK;
}

void sfo_destroy(sfo_sim *sim) { delete sim; }

int sfo_submit_prompts(sfo_sim *sim, int32_t k, int32_t n_groups, const int32_t *prompt, const int32_t *target) {
  if (!sim || k < 0 || k >= (int)sim->sc.size() || n_groups < 0) return SFO_E_RANGE;
  Scen &s = sim->sc[k];
  if (s.err) return SFO_E_STATE;
  if (s.n_pool + n_groups > s.pool_cap) return SFO_E_RANGE;
  for (int a = 0; a < n_groups; ++a) {
    if (prompt[a] < 0) return SFO_E_INVALID;
    for (int m = 0; m < s.G; ++m) {
      int T = target[a * s.G + m];
      if (T < 1 || (int64_t)s.P.k5 * (prompt[a] + T) > s.P.M) return SFO_E_INVALID;  // A27
    }
  }
  for (int a = 0; a < n_groups; ++a) {
    int g = s.n_pool + a;
    s.grp[g].p = prompt[a];
    for (int m = 0; m < s.G; ++m) { s.traj[g * s.G + m].g = g; s.traj[g * s.G + m].T = target[a * s.G + m]; }
  }
  s.n_pool += n_groups;
  return SFO_OK;
}

int sfo_step(sfo_sim *sim, int32_t n_windows, int32_t n_threads) {
  if (!sim || n_windows < 0) return SFO_E_INVALID;
  int ns = (int)sim->sc.size();
  for (int k = 0; k < ns; ++k) if (sim->sc[k].err) return SFO_E_STATE;
  if (n_threads < 1) n_threads = 1;
  if (n_threads > ns) n_threads = ns;
  std::atomic<int> next{0};                              // scenarios are independent: any order
  auto work = [&](int) {
    for (int k = next++; k < ns; k = next++)
      for (int w = 0; w < n_windows; ++w) run_window(sim->sc[k]);
  };
  if (n_threads == 1) work(0);
  else {
    std::vector<std::thread> th;
    for (int tid = 0; tid < n_threads; ++tid) th.emplace_back(work, tid);
    for (auto &x : th) x.join();
  }
  for (int k = 0; k < ns; ++k) if (sim->sc[k].err) return SFO_E_STATE;
  return SFO_OK;
}

int sfo_publish_params(sfo_sim *sim, int32_t k, int32_t v) {
  if (!sim || k < 0 || k >= (int)sim->sc.size()) return SFO_E_RANGE;
  Scen &s = sim->sc[k];
  if (s.err) return SFO_E_STATE;
  if (v != s.ps + 1 || v > s.L.cu) return SFO_E_VERSION;        // Push
  s.ps = v;
  s.m[M_PUBLISHES]++;
  return SFO_OK;
}

int sfo_collect_batch(sfo_sim *sim, int32_t k, int32_t cap, int32_t *v_buf, int32_t *gids, int32_t *gv,
                      int32_t *n_out) {
  if (!sim || k < 0 || k >= (int)sim->sc.size()) return SFO_E_RANGE;
  Scen &s = sim->sc[k];
  if (s.err) return SFO_E_STATE;
  if (n_out) *n_out = s.Br;
  if (cap < s.Br) return SFO_E_RANGE;
  if (s.L.state(s.L.cu) != 1) return SFO_NOT_READY;
  consume(s, v_buf, gids, gv);
  return s.err ? SFO_E_STATE : SFO_OK;
}

int sfo_mark_filtered(sfo_sim *sim, int32_t k, int32_t g0, int32_t n, const uint8_t *flags) {
  if (!sim || k < 0 || k >= (int)sim->sc.size() || g0 < 0 || n < 0) return SFO_E_RANGE;
  Scen &s = sim->sc[k];
  if (s.err) return SFO_E_STATE;
  if (g0 + n > s.pool_cap || (n > 0 && !flags)) return SFO_E_RANGE;
  for (int a = 0; a < n; ++a) s.grp[g0 + a].filter = flags[a] != 0;
  return SFO_OK;
}

int sfo_filter_group(sfo_sim *sim, int32_t k, int32_t g) {
  if (!sim || k < 0 || k >= (int)sim->sc.size()) return SFO_E_RANGE;
  Scen &s = sim->sc[k];
  if (s.err) return SFO_E_STATE;
  int b = -1, sl = -1;
  if (g < 0 || g >= s.n_ingested || !s.L.find(g, &b, &sl)) return SFO_E_INVALID;   // UnknownKey
  filter_group(s, g);
  return s.err ? SFO_E_STATE : SFO_OK;
}

int sfo_read_scenario_metrics(sfo_sim *sim, int32_t k, int64_t *out, int32_t len) {
  if (!sim || k < 0 || k >= (int)sim->sc.size() || len < 0) return SFO_E_RANGE;
  const Scen &s = sim->sc[k];
  for (int a = 0; a < len && a < SFO_METRICS_LEN; ++a) {
    int64_t v = s.m[a];
    if (a == M_CMD_HASH) v = (int64_t)s.cmd_hash;
    if (a == M_SIM_TIME || a == 30) v = s.t;       // slot 30: max simulated time (per scenario: t)
    if (a == 29) v = s.err != 0;                   // slot 29: poisoned scenarios
    out[a] = v;
  }
  return SFO_OK;
}

int sfo_read_metrics(sfo_sim *sim, int64_t *out, int32_t len) {
  if (!sim || len < 0) return SFO_E_RANGE;
  for (int a = 0; a < len; ++a) out[a] = 0;
  int64_t tmp[SFO_METRICS_LEN];
  for (int k = 0; k < (int)sim->sc.size(); ++k) {
    sfo_read_scenario_metrics(sim, k, tmp, SFO_METRICS_LEN);
    for (int a = 0; a < len && a < SFO_METRICS_LEN; ++a)
      out[a] = a == 30 ? std::max(out[a], tmp[a]) : (int64_t)((uint64_t)out[a] + (uint64_t)tmp[a]);
  }
  return SFO_OK;
}

int sfo_dump_lifecycles(sfo_sim *sim, int32_t k, int64_t *rec, int64_t cap, int64_t *n) {
  if (!sim || k < 0 || k >= (int)sim->sc.size()) return SFO_E_RANGE;
  const Scen &s = sim->sc[k];
  int64_t cnt = (int64_t)s.n_pool * s.G;
  if (n) *n = cnt;
  if (cap < cnt) return SFO_E_RANGE;
  for (int64_t j = 0; j < cnt; ++j) {
    const Traj &tr = s.traj[j];
    const Group &gr = s.grp[tr.g];
    int64_t *r = rec + 13 * j;
    r[0] = j; r[1] = tr.g; r[2] = gr.p; r[3] = tr.T; r[4] = tr.gen; r[5] = gr.v; r[6] = tr.st;
    r[7] = tr.inst; r[8] = tr.n_routes; r[9] = tr.n_preempt; r[10] = tr.n_interrupt;
    r[11] = gr.consumed_vbuf; r[12] = tr.t_complete;
  }
  return SFO_OK;
}

int sfo_dump_batches(sfo_sim *sim, int32_t k, int32_t *out, int64_t cap, int64_t *n) {
  if (!sim || k < 0 || k >= (int)sim->sc.size()) return SFO_E_RANGE;
  const Scen &s = sim->sc[k];
  if (n) *n = (int64_t)s.batches.size();
  if (cap < (int64_t)s.batches.size()) return SFO_E_RANGE;
  for (size_t a = 0; a < s.batches.size(); ++a) out[a] = s.batches[a];
  return SFO_OK;
}

int sfo_dump_commands(sfo_sim *sim, int32_t k, int64_t *out, int64_t cap, int64_t *n) {
  if (!sim || k < 0 || k >= (int)sim->sc.size()) return SFO_E_RANGE;
  const Scen &s = sim->sc[k];
  if (n) *n = (int64_t)s.cmds.size() / 4;
  if (cap < (int64_t)s.cmds.size() / 4) return SFO_E_RANGE;
  for (size_t a = 0; a < s.cmds.size(); ++a) out[a] = s.cmds[a];
  return SFO_OK;
}

int sfo_dump_instances(sfo_sim *sim, int32_t k, int64_t *out, int64_t cap, int64_t *n) {
  if (!sim || k < 0 || k >= (int)sim->sc.size()) return SFO_E_RANGE;
  const Scen &s = sim->sc[k];
  if (n) *n = s.I;
  if (cap < s.I) return SFO_E_RANGE;
  for (int i = 0; i < s.I; ++i) {
    const Inst &x = s.inst[i];
    int64_t *r = out + 7 * i;
    r[0] = x.v; r[1] = x.kv; r[2] = (int64_t)x.run.size(); r[3] = (int64_t)x.wait.size(); r[4] = x.c;
    r[5] = x.st; r[6] = x.st == I_TICK ? x.nb : (x.st == I_PULL ? x.pull_until : -1);
  }
  return SFO_OK;
}

// ---------------------------------------------------------------- unit-level
sfo_ledger *sfo_ledger_new(int32_t eta, int32_t B) { return sfo_ledger_new2(eta, B, B); }
sfo_ledger *sfo_ledger_new2(int32_t eta, int32_t cap, int32_t B) {
  if (eta < 0 || B < 1 || cap < B) return nullptr;
  sfo_ledger *L = new (std::nothrow) sfo_ledger();
  if (L) { L->eta = eta; L->B = cap; L->Br = B; }
  return L;
}
void sfo_ledger_free(sfo_ledger *L) { delete L; }
sfo_ledger *sfo_ledger_clone(const sfo_ledger *L) { return L ? new (std::nothrow) sfo_ledger(*L) : nullptr; }
int sfo_ledger_verify(const sfo_ledger *L, int32_t v) { return L->verify(v) ? 1 : 0; }
int sfo_ledger_reserve(sfo_ledger *L, int32_t g, int32_t v, int32_t *b, int32_t *s) {
  int ob, os, xb, xs;
  if (L->find(g, &xb, &xs)) return SFO_E_INVALID;            // DuplicateKey
  if (!L->reserve(g, v, &ob, &os)) return SFO_E_STATE;       // NoCapacity
  *b = ob; *s = os;
  return SFO_OK;
}
int sfo_ledger_delete_relocate(sfo_ledger *L, int32_t g) {
  int b, s;
  if (!L->find(g, &b, &s) || L->buf[b][s].st != E_RESERVED) return SFO_E_INVALID;
  return L->delete_and_relocate(b, s);
}
int sfo_ledger_abort(sfo_ledger *L, int32_t g, int32_t *moves) {
  return L->abort_entry(g, moves) ? SFO_OK : SFO_E_INVALID;
}
int sfo_ledger_occupy(sfo_ledger *L, int32_t g, int32_t v, int32_t *b, int32_t *s) {
  int ob, os;
  if (!L->occupy(g, v, &ob, &os)) return SFO_E_STATE;
  *b = ob; *s = os;
  return SFO_OK;
}
int sfo_ledger_state(const sfo_ledger *L, int32_t b) { return L->state(b); }
int sfo_ledger_consume(sfo_ledger *L, int32_t *groups, int32_t *versions) {
  return sfo_ledger_consume2(L, groups, versions, nullptr, nullptr);
}
int sfo_ledger_consume2(sfo_ledger *L, int32_t *groups, int32_t *versions, int32_t *surplus, int32_t *n_surplus) {
  if (L->state(L->cu) != 1) return SFO_NOT_READY;
  int taken = 0, ns = 0;
  for (int s = 0; s < L->B; ++s) {
    const Entry &e = L->buf[L->cu][s];
    if (e.st == E_EMPTY) continue;
    if (e.st == E_OCCUPIED && taken < L->Br) { groups[taken] = e.g; versions[taken] = e.v; ++taken; }
    else if (surplus) surplus[ns++] = e.g;
  }
  if (n_surplus) *n_surplus = ns;
  L->cu += 1;
  return SFO_OK;
}
int sfo_ledger_get(const sfo_ledger *L, int32_t b, int32_t s, int32_t *st, int32_t *g, int32_t *v) {
  if (b < 0 || s < 0 || s >= L->B) return SFO_E_RANGE;
  if (b >= (int)L->buf.size()) { *st = E_EMPTY; *g = -1; *v = -1; return SFO_OK; }
  *st = L->buf[b][s].st; *g = L->buf[b][s].g; *v = L->buf[b][s].v;
  return SFO_OK;
}
int32_t sfo_ledger_cu(const sfo_ledger *L) { return L->cu; }

int64_t sfo_tick_latency(const sfo_params *p, int64_t kv, int32_t n, int64_t prefill) {
  return tick_latency(from_sfo(p), kv, n, prefill);
}
double sfo_throughput(const sfo_params *p, int32_t n, int64_t kv) { return throughput(from_sfo(p), n, kv); }
double sfo_marginal_gain(const sfo_params *p, const sfo_inst_view *v, int32_t l) {
  return marginal_gain(from_sfo(p), View{v->v, v->kv, v->n_run, v->n_wait}, l);
}
double sfo_ideal_gain(const sfo_params *p, int32_t l) { return ideal_gain(from_sfo(p), l); }
int sfo_check_routable(const sfo_params *, const sfo_inst_view *v, int32_t tau_v, const sfo_ledger *L) {
  return check_routable(View{v->v, v->kv, v->n_run, v->n_wait}, tau_v, *L) ? 1 : 0;
}
int sfo_mlq_order(const sfo_ts_item *items, int32_t n, int32_t *order) {
  std::vector<Item> it(n);
  for (int k = 0; k < n; ++k) it[k] = Item{items[k].id, items[k].g, items[k].v, items[k].l};
  std::vector<Item> srt = mlq_sort(it);
  for (int k = 0; k < n; ++k) {
    for (int a = 0; a < n; ++a)
      if (items[a].id == srt[k].id) { order[k] = a; break; }
  }
  return SFO_OK;
}
static std::vector<View> views(const sfo_inst_view *S, int I) {
  std::vector<View> v(I);
  for (int i = 0; i < I; ++i) v[i] = View{S[i].v, S[i].kv, S[i].n_run, S[i].n_wait};
  return v;
}
static std::vector<Item> items_of(const sfo_ts_item *mlq, int n) {
  std::vector<Item> it(n);
  for (int k = 0; k < n; ++k) it[k] = Item{mlq[k].id, mlq[k].g, mlq[k].v, mlq[k].l};
  return it;
}
int sfo_route(const sfo_params *p, sfo_inst_view *S, int32_t I, const sfo_ts_item *mlq, int32_t n,
              sfo_ledger *L, int32_t vanilla, int32_t *out_inst) {
  std::vector<View> v = views(S, I);
  std::vector<RouteDecision> r = route(from_sfo(p), v, items_of(mlq, n), *L, vanilla != 0);
  for (size_t k = 0; k < r.size(); ++k) out_inst[k] = r[k].inst;
  for (int i = 0; i < I; ++i) { S[i].v = v[i].v; S[i].kv = v[i].kv; S[i].n_run = v[i].n_run; S[i].n_wait = v[i].n_wait; }
  return (int)r.size();
}
int sfo_sync_select(const sfo_params *p, const sfo_inst_view *S, int32_t I, const sfo_ts_item *mlq, int32_t n,
                    const sfo_ledger *L, int32_t ps, int32_t vanilla_sync, int32_t vanilla_route, int32_t *out) {
  std::vector<int> sel = sync_select(from_sfo(p), views(S, I), items_of(mlq, n), *L, ps, vanilla_sync != 0,
                                     vanilla_route != 0);
  for (size_t k = 0; k < sel.size(); ++k) out[k] = sel[k];
  return (int)sel.size();
}
int sfo_migrate(const sfo_params *p, const sfo_inst_view *S, int32_t I, int32_t *case1_k, int32_t *case2) {
  std::vector<int> k1; int c2 = -1;
  migrate(from_sfo(p), views(S, I), k1, c2);
  for (int i = 0; i < I; ++i) case1_k[i] = k1[i];
  *case2 = c2;
  return SFO_OK;
}

}  // extern "C"
