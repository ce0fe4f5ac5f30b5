// Stateless decision kernels of the DARIS scheduler. Every scheduling decision
// reduces to one of these pure functions over plain arrays; the stateful
// Dispatcher (dispatcher.cpp: engine / executor path) and the object-level
// drop-in API (paper_2504_08795_b200/scheduler.py, timing.py, model.py, gpu.py:
// Python-owned Job / TaskState / ready lists, as in the reference) both call
// them, so the two views cannot disagree on arithmetic or tie order.
// Reference: /root/reference/pkg/src/stagesim/{timing,scheduler,model,gpu}.py.
#include <sstream>

#include "core/dispatcher.hpp"

namespace daris {

double window_peak(const double* v, int n) {  // timing.py:52-56: max() keeps the first maximum
  double best = v[0];
  for (int k = 1; k < n; ++k)
    if (v[k] > best) best = v[k];
  return best;
}

double Window::peak() const {
  const int start = (count < cap) ? 0 : head;
  double lin[64];
  std::vector<double> big;
  double* v = lin;
  if (count > 64) {
    big.resize(count);
    v = big.data();
  }
  for (int k = 0; k < count; ++k) v[k] = buf[(start + k) % cap];
  return window_peak(v, count);
}

double stage_fallback(double full_load, double nominal, double nominal_total) {  // timing.py:84-86
  const double share = nominal / nominal_total;
  return full_load * share;
}

double utilization_of(long long completed, double full_load, double task_est, double period) {  // timing.py:102-107
  return completed == 0 ? full_load / period : task_est / period;
}

void deadline_split(const double* est, int n, double deadline, double* out, int task_id) {  // timing.py:116-132
  PySum tot;
  for (int j = 0; j < n; ++j) tot.add(est[j]);
  const double total = tot.value();
  if (total <= 0)
    throw Error(DARIS_E_ZERO_TOTAL_ESTIMATE, "task " + std::to_string(task_id) +
                                                 " has no positive execution estimate to split its deadline over");
  PySum rest;
  for (int j = 0; j + 1 < n; ++j) {
    out[j] = est[j] / total * deadline;
    rest.add(out[j]);
  }
  out[n - 1] = deadline - rest.value();
}

void virtual_deadlines(double release, double abs_deadline, const double* shares, int n, double* out) {
  // model.py:216-227: cumulative from release (naive +=), the last pinned to the job deadline
  double acc = release;
  for (int j = 0; j < n; ++j) {
    if (j == n - 1) {
      out[j] = abs_deadline;
    } else {
      acc += shares[j];
      out[j] = acc;
    }
  }
}

daris_ledger_t ledger_sum(const daris_ledger_entry* e, int n) {  // scheduler.py:157-171 (naive +=, list order)
  double hp_total = 0.0, lp_total = 0.0, lp_active = 0.0, hp_active = 0.0;
  for (int k = 0; k < n; ++k) {
    const double u = e[k].util;
    if (e[k].hp) {
      hp_total += u;
      if (e[k].active_jobs > 0) hp_active += u;
    } else {
      lp_total += u;
      if (e[k].active_jobs > 0) lp_active += u;
    }
  }
  return {hp_total, lp_total, lp_active, hp_active};
}

void admission_eval(const daris_ledger_t& l, double u, bool hp, int n_streams, double* active, double* limit,
                    bool* admitted) {  // scheduler.py:179-200 (strict inequality)
  if (!hp) {
    *active = l.lp_active;
    *limit = n_streams - l.hp_total;
  } else {
    *active = l.hp_active + l.lp_active;
    *limit = static_cast<double>(n_streams);
  }
  *admitted = *active + u < *limit;
}

void greedy_place(const double* util, const int32_t* hp, const int32_t* ids, int n, int n_ctx, bool insertion,
                  int32_t* out_ctx, double* totals, int32_t* out_order) {  // scheduler.py:131-153 (Algorithm 1)
  for (int c = 0; c < n_ctx; ++c) totals[c] = 0.0;
  int placed = 0;
  for (int cls = 0; cls < 2; ++cls) {
    std::vector<int> group;
    for (int i = 0; i < n; ++i)
      if ((hp[i] != 0) == (cls == 0)) group.push_back(i);
    if (!insertion)  // sorted by (-u, id); stable for equal keys like Python's sorted
      std::stable_sort(group.begin(), group.end(), [&](int a, int b) {
        if (-util[a] != -util[b]) return -util[a] < -util[b];
        return ids[a] < ids[b];
      });
    for (int i : group) {
      int target = 0;
      for (int c = 1; c < n_ctx; ++c)
        if (totals[c] < totals[target]) target = c;  // min over (total, ctx): ties -> lowest id
      out_ctx[i] = target + 1;
      totals[target] += util[i];
      if (out_order) out_order[placed] = i;
      ++placed;
    }
  }
}

double predicted_finish_eval(double t, const double* backlog, long long n, int n_streams,
                             double task_est) {  // scheduler.py:202-213
  double b = 0.0;
  for (long long k = 0; k < n; ++k) b += backlog[k];
  return t + b / n_streams + task_est;
}

int priority_level(bool hp, bool is_last, bool late_pred, const daris_options& o) {  // scheduler.py:278-284
  if (o.no_fixed) return 0;
  const bool last = is_last && !o.no_last;
  const bool late = late_pred && !o.no_prior;
  return 4 * (hp ? 0 : 1) + 2 * (last ? 0 : 1) + (late ? 0 : 1);
}

bool key_less(const daris_ready_key& a, const daris_ready_key& b) {  // PriorityKey tuple order
  if (a.level != b.level) return a.level < b.level;
  if (a.edf != b.edf) return a.edf < b.edf;
  if (a.task != b.task) return a.task < b.task;
  return a.job < b.job;
}

int pick_ready(const daris_ready_key* keys, int n) {  // scheduler.py:289-296: min() keeps the first minimum
  int best = 0;
  for (int k = 1; k < n; ++k)
    if (key_less(keys[k], keys[best])) best = k;
  return best;
}

int next_completion_eval(const double* rem, const double* rates, const long long* job, const long long* stage, int n,
                         double now, double* t_out) {  // gpu.py:208-226
  if (n <= 0) throw Error(DARIS_E_NO_ACTIVE_STAGES, "no active stages to complete");
  int best = -1;
  double bt = 0;
  for (int i = 0; i < n; ++i) {
    const double r = rates[i];
    if (r <= 0) throw Error(DARIS_E_VALUE, "active stage has a non-positive rate");
    const double t = now + rem[i] / r;
    bool less;
    if (best < 0) less = true;
    else if (t != bt) less = t < bt;
    else if (job[i] != job[best]) less = job[i] < job[best];
    else less = stage[i] < stage[best];
    if (less) {
      best = i;
      bt = t;
    }
  }
  *t_out = bt;
  return best;
}

void advance_eval(double* rem, const double* rates, const long long* job, const long long* stage, int n,
                  double dt) {  // gpu.py:229-240: in list order, stopping at the first overshoot
  if (dt < 0) throw Error(DARIS_E_VALUE, "dt must be >= 0");
  for (int i = 0; i < n; ++i) {
    const double left = rem[i] - rates[i] * dt;
    if (left < -kEps) {
      std::ostringstream m;
      m.precision(3);
      m << std::scientific << "stage (job " << job[i] << ", stage " << stage[i] << ") overshoots completion by "
        << -left << " s";
      throw Error(DARIS_E_OVERSHOOT, m.str());
    }
    rem[i] = std::max(0.0, left);
  }
}

}  // namespace daris
