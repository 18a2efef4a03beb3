// sf_tools.cu -- host-side pieces of the method adjacent to the coordination step (SURVEY §8(f)
// row f4): cost-coefficient fitting and the load-balancing communication plan of
// App A.2.  Plain host C++ (tiny inputs); exported through include/staleflow.h.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <deque>
#include <functional>
#include <numeric>
#include <queue>
#include <vector>

#include "../../include/staleflow.h"

namespace {

// Least squares min |A x - y| for an m x 4 design matrix (column-major in `cols`) by modified
// Gram-Schmidt QR on unit-scaled columns (the columns span ~1 .. 1e6, so the normal equations
// would square a ~1e13 condition number).  false if a column is (numerically) dependent.
bool lstsq4(std::vector<double> cols[4], std::vector<double> y, double x[4]) {
  const size_t m = y.size();
  double scale[4], R[4][4] = {{0}};
  for (int c = 0; c < 4; ++c) {
    double mx = 0.0;
    for (size_t i = 0; i < m; ++i) mx = std::fmax(mx, std::fabs(cols[c][i]));
    if (mx == 0.0) return false;
    scale[c] = mx;
    for (size_t i = 0; i < m; ++i) cols[c][i] /= mx;
  }
  for (int c = 0; c < 4; ++c) {
    for (int k = 0; k < c; ++k) {
      double d = 0.0;
      for (size_t i = 0; i < m; ++i) d += cols[k][i] * cols[c][i];
      R[k][c] = d;
      for (size_t i = 0; i < m; ++i) cols[c][i] -= d * cols[k][i];
    }
    double nrm = 0.0;
    for (size_t i = 0; i < m; ++i) nrm += cols[c][i] * cols[c][i];
    nrm = std::sqrt(nrm);
    if (nrm < 1e-10) return false;                                // rank deficient
    R[c][c] = nrm;
    for (size_t i = 0; i < m; ++i) cols[c][i] /= nrm;
  }
  double qy[4];
  for (int c = 0; c < 4; ++c) {
    double d = 0.0;
    for (size_t i = 0; i < m; ++i) d += cols[c][i] * y[i];
    qy[c] = d;
    for (size_t i = 0; i < m; ++i) y[i] -= d * cols[c][i];
  }
  for (int c = 3; c >= 0; --c) {
    double v = qy[c];
    for (int k = c + 1; k < 4; ++k) v -= R[c][k] * x[k];
    x[c] = v / R[c][c];
  }
  for (int c = 0; c < 4; ++c) x[c] /= scale[c];
  return true;
}

}  // namespace

extern "C" {

// Least-squares fit of Eq 7: latency = k1 kv + max(k2, k3 n) + k4.  The max() is
// handled by regime segmentation iterated to a fixpoint (<= 50 rounds): samples with
// k3 n > k2 use the row [kv, 0, n, 1], the others [kv, 1, 0, 1]; the initial split puts the
// samples with n above the median in the compute regime.
sf_status sf_fit_cost_model(int32_t n_samples, const double *kv, const double *n_run, const double *latency,
                            double *k_out /* [4]: k1, k2, k3, k4 */) {
  if (n_samples < 4 || !kv || !n_run || !latency || !k_out) return SF_E_INVALID;
  std::vector<int> compute(n_samples);
  std::vector<double> ns(n_run, n_run + n_samples);
  std::vector<double> sorted = ns;
  std::sort(sorted.begin(), sorted.end());
  // the sample median (DESIGN.md §11 reading R-FIT): the middle order statistic, or the mean of
  // the two middle ones for an even count
  const double med = (n_samples & 1) ? sorted[n_samples / 2]
                                     : 0.5 * (sorted[n_samples / 2 - 1] + sorted[n_samples / 2]);
  for (int i = 0; i < n_samples; ++i) compute[i] = ns[i] > med;
  double x[4] = {0, 0, 0, 0};
  for (int round = 0; round < 50; ++round) {
    std::vector<double> cols[4];
    for (int c = 0; c < 4; ++c) cols[c].resize(n_samples);
    for (int i = 0; i < n_samples; ++i) {
      cols[0][i] = kv[i];
      cols[1][i] = compute[i] ? 0.0 : 1.0;
      cols[2][i] = compute[i] ? n_run[i] : 0.0;
      cols[3][i] = 1.0;
    }
    if (!lstsq4(cols, std::vector<double>(latency, latency + n_samples), x)) return SF_E_STATE;   // Degenerate
    bool changed = false;
    for (int i = 0; i < n_samples; ++i) {
      const int c = x[2] * n_run[i] > x[1];
      if (c != compute[i]) { compute[i] = c; changed = true; }
    }
    if (!changed) break;
  }
  for (int k = 0; k < 4; ++k) k_out[k] = x[k];
  return SF_OK;
}

// Load-balancing communication plan (App A.2): requirements (slice, receiver) in input
// order; estimate = slice bytes / bandwidth(sender -> receiver) + constant latency (fig:comm);
// assign the holding sender with the smallest accumulated estimate (ties: lowest sender id) and
// add the estimate to it.  holds[s * n_slices + k] != 0 if sender s holds slice k; bandwidth and
// latency are [n_senders * n_receivers].  out_sender[r] = the sender of requirement r;
// acc[n_senders] = accumulated estimates.  SF_E_INVALID if a slice has no holder.
sf_status sf_plan_comm(int32_t n_slices, const double *slice_bytes, int32_t n_senders, int32_t n_receivers,
                       const uint8_t *holds, const double *bandwidth, const double *latency, int32_t n_req,
                       const int32_t *req_slice, const int32_t *req_receiver, int32_t *out_sender, double *acc) {
  if (n_slices < 1 || n_senders < 1 || n_receivers < 1 || n_req < 0 || !slice_bytes || !holds || !bandwidth ||
      !latency || (n_req > 0 && (!req_slice || !req_receiver || !out_sender)) || !acc)
    return SF_E_INVALID;
  for (int s = 0; s < n_senders; ++s) acc[s] = 0.0;
  for (int r = 0; r < n_req; ++r) {
    const int k = req_slice[r], rv = req_receiver[r];
    if (k < 0 || k >= n_slices || rv < 0 || rv >= n_receivers) return SF_E_RANGE;
    int best = -1;
    for (int s = 0; s < n_senders; ++s)
      if (holds[(size_t)s * n_slices + k] && (best < 0 || acc[s] < acc[best])) best = s;
    if (best < 0) return SF_E_INVALID;                         // Uncoverable
    const size_t e = (size_t)best * n_receivers + rv;
    acc[best] += slice_bytes[k] / bandwidth[e] + latency[e];
    out_sender[r] = best;
  }
  return SF_OK;
}

// Parameter-server Push / Pull under a read-write lock with writer
// preference, as a discrete-event simulation over int64 ps.  Requests are taken in
// (t_issue, index) order; at equal times lock releases precede arrivals.  Grant rules: a Pull
// iff no Push is active or waiting; a Push iff no Pull or Push is active and no earlier Push
// waits; on a release a waiting Push goes first (once the readers drain), else all waiting
// Pulls at once.  A Pull delivers the version committed at its start; a Push commits at its
// end.  status[k] = -2 (VersionSkip) for a Push whose version is not the last accepted + 1.
sf_status sf_ps_lock_sim(int32_t n, const int32_t *kind, const int64_t *t_issue, const int64_t *duration,
                         const int32_t *push_version, int32_t v0, int64_t *t_start, int64_t *t_end,
                         int32_t *version, int32_t *status) {
  if (n < 0 || (n > 0 && (!kind || !t_issue || !duration || !push_version || !t_start || !t_end || !version ||
                          !status)))
    return SF_E_INVALID;
  for (int k = 0; k < n; ++k)
    if ((kind[k] != 0 && kind[k] != 1) || duration[k] < 0) return SF_E_INVALID;
  std::vector<int> order(n);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return t_issue[a] < t_issue[b]; });
  // release events (time, request) in time order; ties by request index
  using Rel = std::pair<int64_t, int>;
  std::priority_queue<Rel, std::vector<Rel>, std::greater<Rel>> rel;
  std::deque<int> wait_w, wait_r;                  // waiting Pushes / Pulls, arrival order
  int active_r = 0, active_w = -1;
  int32_t accepted = v0, committed = v0;
  for (int k = 0; k < n; ++k) { t_start[k] = -1; t_end[k] = -1; version[k] = -1; status[k] = 0; }
  auto grant = [&](int k, int64_t now) {
    t_start[k] = now;
    t_end[k] = now + duration[k];
    if (kind[k] == 1) { active_w = k; version[k] = push_version[k]; }
    else { ++active_r; version[k] = committed; }
    rel.push({t_end[k], k});
  };
  auto schedule = [&](int64_t now) {
    if (active_w >= 0) return;
    if (!wait_w.empty()) {
      if (active_r == 0) { const int k = wait_w.front(); wait_w.pop_front(); grant(k, now); }
      return;
    }
    while (!wait_r.empty()) { const int k = wait_r.front(); wait_r.pop_front(); grant(k, now); }
  };
  auto release_until = [&](int64_t t, bool all) {
    while (!rel.empty() && (all || rel.top().first <= t)) {
      const Rel r = rel.top();
      rel.pop();
      if (r.second == active_w) { committed = push_version[r.second]; active_w = -1; }
      else --active_r;
      schedule(r.first);
    }
  };
  for (int k : order) {
    const int64_t now = t_issue[k];
    release_until(now, false);
    if (kind[k] == 1) {
      if (push_version[k] != accepted + 1) { status[k] = -2; continue; }   // VersionSkip
      accepted = push_version[k];
      if (active_w < 0 && active_r == 0 && wait_w.empty()) grant(k, now);
      else wait_w.push_back(k);
    } else {
      if (active_w < 0 && wait_w.empty()) grant(k, now);
      else wait_r.push_back(k);
    }
  }
  release_until(0, true);
  return SF_OK;
}

}  // extern "C"
