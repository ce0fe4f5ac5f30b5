// C ABI of the DARIS dispatcher (include/daris.h). Exceptions never cross the
// boundary: every entry point returns a status code that the Python wrapper
// maps back onto the reference's exception classes.
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "core/dispatcher.hpp"

struct daris_handle {
  std::unique_ptr<daris::Dispatcher> d;
  std::string last_error;
};

namespace {
template <class F>
int guard(daris_handle* h, F&& f) {
  try {
    f();
    if (h) h->last_error.clear();
    return DARIS_OK;
  } catch (const daris::Error& e) {
    if (h) h->last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    if (h) h->last_error = e.what();
    return DARIS_E_INTERNAL;
  }
}
void copy_err(char* err, size_t errlen, const std::string& m) {
  if (err && errlen) {
    std::strncpy(err, m.c_str(), errlen - 1);
    err[errlen - 1] = '\0';
  }
}
}  // namespace

extern "C" {

int daris_create(const daris_gpu_config* gpu, const daris_task_spec* tasks, int32_t n_tasks,
                 const daris_stage_spec* stages, int32_t n_stages, const daris_options* opts, daris_handle** out,
                 char* err, size_t errlen) {
  if (!gpu || !opts || !out || (n_tasks > 0 && (!tasks || !stages))) {
    copy_err(err, errlen, "null argument");
    return DARIS_E_VALUE;
  }
  try {
    daris::validate_gpu(*gpu);
    auto defs = daris::build_task_defs(tasks, n_tasks, stages, n_stages, opts->no_staging != 0);
    auto* h = new daris_handle();
    h->d = std::make_unique<daris::Dispatcher>(*gpu, std::move(defs), *opts);
    *out = h;
    return DARIS_OK;
  } catch (const daris::Error& e) {
    copy_err(err, errlen, e.what());
    return e.code;
  } catch (const std::exception& e) {
    copy_err(err, errlen, e.what());
    return DARIS_E_INTERNAL;
  }
}

void daris_destroy(daris_handle* h) { delete h; }

const char* daris_last_error(const daris_handle* h) { return h ? h->last_error.c_str() : ""; }

int daris_sm_per_context(const daris_gpu_config* gpu, int32_t* out) {
  return guard(nullptr, [&] { *out = daris::sm_per_context(*gpu); });
}

int daris_n_tasks(const daris_handle* h, int32_t* out) {
  *out = h->d->n_tasks();
  return DARIS_OK;
}

int daris_task_ids(const daris_handle* h, int32_t* out) {
  for (int i = 0; i < h->d->n_tasks(); ++i) out[i] = h->d->tasks()[i].id;
  return DARIS_OK;
}

int daris_task_stage_count(const daris_handle* h, int32_t task_id, int32_t* out) {
  return guard(const_cast<daris_handle*>(h),
               [&] { *out = static_cast<int32_t>(h->d->task(task_id).nominal.size()); });
}

int daris_task_info(const daris_handle* h, int32_t task_id, double* period, int32_t* n_stages, int32_t* priority) {
  return guard(const_cast<daris_handle*>(h), [&] {
    const daris::TaskDef& t = h->d->task(task_id);
    *period = t.period;
    *n_stages = static_cast<int32_t>(t.nominal.size());
    *priority = t.hp ? DARIS_HP : DARIS_LP;
  });
}

int daris_task_batch(const daris_handle* h, int32_t task_id, int32_t* batch) {
  return guard(const_cast<daris_handle*>(h), [&] { *batch = h->d->task(task_id).batch; });
}

int daris_full_load_sim(daris_handle* h, int32_t task_id, int32_t repetitions, const int32_t* draws, double* out) {
  return guard(h, [&] { *out = daris::full_load_time(*h->d, task_id, repetitions, draws); });
}

int daris_set_full_load(daris_handle* h, const double* per_task) {
  return guard(h, [&] {
    for (int i = 0; i < h->d->n_tasks(); ++i) {
      auto& r = h->d->rt(h->d->tasks()[i].id);
      r.full_load = per_task[i];
      r.ucache_valid = false;
    }
  });
}

int daris_populate(daris_handle* h) {
  return guard(h, [&] { h->d->populate(); });
}

int daris_home_context(const daris_handle* h, int32_t task_id, int32_t* out) {
  return guard(const_cast<daris_handle*>(h), [&] { *out = h->d->rt(task_id).home; });
}

int daris_release(daris_handle* h, int32_t task_id, double t, int32_t job_id, const double* stage_work,
                  daris_placement* out) {
  return guard(h, [&] { h->d->release(task_id, t, job_id, stage_work, out); });
}

int daris_dispatch(daris_handle* h, int32_t context, int32_t stream, double t, daris_stage_ref* out, int32_t* found) {
  return guard(h, [&] {
    if (context < 1 || context > h->d->gpu().n_contexts) throw daris::Error(DARIS_E_VALUE, "bad context");
    daris::StageJob* st = h->d->dispatch(context, stream, t);
    *found = st ? 1 : 0;
    if (st && out) {
      out->task = st->job->task;
      out->job = st->job->id;
      out->stage = st->j;
      out->context = st->ctx;
      out->stream = st->stream;
      out->started_at = st->start;
      out->virtual_deadline = st->vdl;
    }
  });
}

int daris_complete(daris_handle* h, int32_t job_id, int32_t stage, double t, int32_t* job_done, int32_t* missed) {
  return guard(h, [&] {
    daris::StageJob* st = h->d->find_stage(job_id, stage);
    if (!st) throw daris::Error(DARIS_E_NOT_FOUND, "unknown stage reference");
    bool m = false;
    const bool done = h->d->complete(st, t, &m);
    *job_done = done ? 1 : 0;
    *missed = m ? 1 : 0;
  });
}

int daris_complete_ex(daris_handle* h, int32_t job_id, int32_t stage, double t, int32_t record_sample,
                      int32_t* job_done, int32_t* missed) {
  return guard(h, [&] {
    daris::StageJob* st = h->d->find_stage(job_id, stage);
    if (!st) throw daris::Error(DARIS_E_NOT_FOUND, "unknown stage reference");
    bool m = false;
    const bool done = h->d->complete(st, t, &m, record_sample != 0);
    *job_done = done ? 1 : 0;
    *missed = m ? 1 : 0;
  });
}

int daris_ready_count(const daris_handle* h, int32_t context, int32_t* out) {
  return guard(const_cast<daris_handle*>(h), [&] { *out = h->d->ready_count(context); });
}

int daris_ledger(daris_handle* h, int32_t context, daris_ledger_t* out) {
  return guard(h, [&] {
    if (context < 1 || context > h->d->gpu().n_contexts) throw daris::Error(DARIS_E_VALUE, "bad context");
    *out = h->d->ledger(context);
  });
}

int daris_admission_test(daris_handle* h, int32_t task_id, int32_t job_id, int32_t context, double t,
                         daris_audit* out) {
  return guard(h, [&] {
    daris::Job probe;
    probe.id = job_id;
    probe.task = task_id;
    const daris::Audit a = h->d->admission_test(probe, context, t);
    *out = daris_audit{a.time, a.active, a.u, a.limit, a.job, a.task, a.prio, a.ctx, a.admitted ? 1 : 0, 0};
  });
}

int daris_predicted_finish(daris_handle* h, int32_t task_id, int32_t context, double t, double* out) {
  return guard(h, [&] { *out = h->d->predicted_finish(task_id, context, t); });
}

int daris_stage_estimate(daris_handle* h, int32_t task_id, int32_t stage, double* out) {
  return guard(h, [&] { *out = h->d->stage_estimate(task_id, stage); });
}

int daris_task_estimate(daris_handle* h, int32_t task_id, double* out) {
  return guard(h, [&] { *out = h->d->task_estimate(task_id); });
}

int daris_utilization(daris_handle* h, int32_t task_id, double* out) {
  return guard(h, [&] { *out = h->d->utilization(task_id); });
}

int daris_deadline_shares(daris_handle* h, int32_t task_id, double* out) {
  return guard(h, [&] {
    auto s = h->d->deadline_shares(task_id);
    for (size_t i = 0; i < s.size(); ++i) out[i] = s[i];
  });
}

int daris_record_execution(daris_handle* h, int32_t task_id, int32_t stage, double observed) {
  return guard(h, [&] { h->d->record_execution(task_id, stage, observed); });
}

int daris_note_job_complete(daris_handle* h, int32_t task_id) {
  return guard(h, [&] { h->d->note_job_complete(task_id); });
}

int daris_sim_run(daris_handle* h, double duration, double warmup_frac, const double* phases, int32_t collect_log,
                  daris_report* out) {
  return guard(h, [&] {
    h->d->collect_log = collect_log != 0;
    daris::sim_run(*h->d, duration, warmup_frac, phases, out, nullptr);
  });
}

int daris_trace_run(daris_handle* h, double duration, double warmup_frac, const double* phases,
                    const daris_trace_entry* trace, int64_t n_trace, int32_t collect_log, daris_report* out) {
  return guard(h, [&] {
    std::unordered_map<long long, double> m;
    std::unordered_set<long long> unsampled;
    m.reserve(static_cast<size_t>(n_trace) * 2 + 1);
    for (int64_t i = 0; i < n_trace; ++i) {
      const long long key = (static_cast<long long>(trace[i].task) << 40) |
                            (static_cast<long long>(trace[i].job) << 8) | static_cast<long long>(trace[i].stage);
      m[key] = trace[i].duration;
      if (trace[i].flags & DARIS_TRACE_UNSAMPLED) unsampled.insert(key);
    }
    h->d->collect_log = collect_log != 0;
    daris::sim_run(*h->d, duration, warmup_frac, phases, out, &m, &unsampled);
  });
}

int64_t daris_log_count(const daris_handle* h) { return static_cast<int64_t>(h->d->log.size()); }

int64_t daris_log_copy(const daris_handle* h, daris_log_record* buf, int64_t cap) {
  const auto& L = h->d->log;
  int64_t n = static_cast<int64_t>(L.size());
  if (cap < n) n = cap;
  for (int64_t i = 0; i < n; ++i) {
    const daris::LogRec& r = L[static_cast<size_t>(i)];
    buf[i] = daris_log_record{r.time, r.kind, r.task, r.job, r.stage, r.ctx, r.stream, r.rate};
  }
  return n;
}

int64_t daris_audit_count(const daris_handle* h) { return static_cast<int64_t>(h->d->audits.size()); }

int64_t daris_audit_copy(const daris_handle* h, daris_audit* buf, int64_t cap) {
  const auto& A = h->d->audits;
  int64_t n = static_cast<int64_t>(A.size());
  if (cap < n) n = cap;
  for (int64_t i = 0; i < n; ++i) {
    const daris::Audit& a = A[static_cast<size_t>(i)];
    buf[i] = daris_audit{a.time, a.active, a.u, a.limit, a.job, a.task, a.prio, a.ctx, a.admitted ? 1 : 0, 0};
  }
  return n;
}

void daris_log_clear(daris_handle* h) {
  h->d->log.clear();
  h->d->audits.clear();
}

void daris_log_push(daris_handle* h, const daris_log_record* r) {
  if (h->d->collect_log) h->d->log.push_back({r->time, r->kind, r->task, r->job, r->stage, r->context, r->stream, r->rate});
}

void daris_log_reserve(daris_handle* h, int64_t records, int64_t audits) {
  auto& L = h->d->log;
  auto& A = h->d->audits;
  if (records > 0 && static_cast<size_t>(records) > L.capacity()) {
    const size_t keep = L.size();
    L.resize(static_cast<size_t>(records));  // touch every page now, not inside the timed loop
    L.resize(keep);
  }
  if (audits > 0 && static_cast<size_t>(audits) > A.capacity()) {
    const size_t keep = A.size();
    A.resize(static_cast<size_t>(audits));
    A.resize(keep);
  }
}

int daris_ready_total(const daris_handle* h, int32_t* out) {
  int n = 0;
  for (int c = 1; c <= h->d->gpu().n_contexts; ++c) n += h->d->ready_count(c);
  *out = n;
  return DARIS_OK;
}

int daris_water_fill(const int32_t* widths, int32_t n, double capacity, double* out_alloc, int32_t* out_is_int,
                     double* out_level, int32_t* has_level) {
  return guard(nullptr, [&] {
    std::vector<int> w(widths, widths + n);
    std::vector<daris::Alloc> a;
    const double level = daris::water_fill(w, capacity, a);
    for (int i = 0; i < n; ++i) {
      out_alloc[i] = a[i].v;
      out_is_int[i] = a[i].is_int ? 1 : 0;
    }
    *has_level = std::isnan(level) ? 0 : 1;
    *out_level = level;
  });
}

int daris_allocate_rates(const daris_gpu_config* gpu, const int32_t* widths, const int32_t* ctx_ids, int32_t n,
                         double* out_alloc, double* out_rates, double* out_scale) {
  return guard(nullptr, [&] {
    const int per = daris::sm_per_context(*gpu);
    std::vector<int> w(widths, widths + n), c(ctx_ids, ctx_ids + n);
    std::vector<daris::Alloc> a;
    std::vector<double> r;
    *out_scale = daris::allocate_rates(*gpu, per, w, c, a, r);
    for (int i = 0; i < n; ++i) {
      out_alloc[i] = a[i].v;
      out_rates[i] = r[i];
    }
  });
}

double daris_py_sum(const double* values, const int32_t* is_int, int64_t n) {
  daris::PySum s;
  for (int64_t i = 0; i < n; ++i) {
    if (is_int && is_int[i]) s.add_int(static_cast<long long>(values[i]));
    else s.add(values[i]);
  }
  return s.value();
}

}  // extern "C"

// ---------------------------------------------------------------- stateless kernels
namespace {
thread_local std::string eval_error;
template <class F>
int eval_guard(F&& f) {
  try {
    f();
    eval_error.clear();
    return DARIS_OK;
  } catch (const daris::Error& e) {
    eval_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    eval_error = e.what();
    return DARIS_E_INTERNAL;
  }
}
}  // namespace

extern "C" {

const char* daris_eval_last_error(void) { return eval_error.c_str(); }

int daris_eval_window_peak(const double* samples, int32_t n, double* out) {
  return eval_guard([&] {
    if (n < 1) throw daris::Error(DARIS_E_VALUE, "empty window has no peak");
    *out = daris::window_peak(samples, n);
  });
}

int daris_eval_stage_fallback(double full_load, double nominal, double nominal_total, double* out) {
  return eval_guard([&] { *out = daris::stage_fallback(full_load, nominal, nominal_total); });
}

int daris_eval_utilization(int64_t completed_jobs, double full_load, double task_estimate, double period,
                           double* out) {
  return eval_guard([&] { *out = daris::utilization_of(completed_jobs, full_load, task_estimate, period); });
}

int daris_eval_deadline_shares(const double* estimates, int32_t n, double deadline, int32_t task_id,
                               double* out_shares) {
  return eval_guard([&] {
    if (n < 1) throw daris::Error(DARIS_E_VALUE, "a task has at least one stage");
    daris::deadline_split(estimates, n, deadline, out_shares, task_id);
  });
}

int daris_eval_virtual_deadlines(double release, double deadline, const double* shares, int32_t n,
                                 double* out_abs_deadline, double* out) {
  return eval_guard([&] {
    if (n < 1) throw daris::Error(DARIS_E_VALUE, "a task has at least one stage");
    const double abs_dl = release + deadline;  // model.py:211
    *out_abs_deadline = abs_dl;
    daris::virtual_deadlines(release, abs_dl, shares, n, out);
  });
}

int daris_eval_ledger(const daris_ledger_entry* tasks, int32_t n, daris_ledger_t* out) {
  return eval_guard([&] { *out = daris::ledger_sum(tasks, n); });
}

int daris_eval_admission(const daris_ledger_t* ledger, double job_util, int32_t hp, int32_t n_streams,
                         double* out_active, double* out_limit, int32_t* out_admitted) {
  return eval_guard([&] {
    bool ok;
    daris::admission_eval(*ledger, job_util, hp != 0, n_streams, out_active, out_limit, &ok);
    *out_admitted = ok ? 1 : 0;
  });
}

int daris_eval_placement(const double* util, const int32_t* hp, const int32_t* ids, int32_t n, int32_t n_contexts,
                         int32_t insertion_order, int32_t* out_context, int32_t* out_order, double* out_totals) {
  return eval_guard([&] {
    if (n_contexts < 1) throw daris::Error(DARIS_E_VALUE, "n_contexts must be >= 1");
    daris::greedy_place(util, hp, ids, n, n_contexts, insertion_order != 0, out_context, out_totals, out_order);
  });
}

int daris_eval_predicted_finish(double t, const double* backlog_estimates, int64_t n, int32_t n_streams,
                                double task_estimate, double* out) {
  return eval_guard([&] { *out = daris::predicted_finish_eval(t, backlog_estimates, n, n_streams, task_estimate); });
}

int daris_eval_priority_level(int32_t hp, int32_t is_last, int32_t predecessor_missed, int32_t no_last,
                              int32_t no_prior, int32_t no_fixed, int32_t* out) {
  return eval_guard([&] {
    daris_options o{};
    o.no_last = no_last;
    o.no_prior = no_prior;
    o.no_fixed = no_fixed;
    *out = daris::priority_level(hp != 0, is_last != 0, predecessor_missed != 0, o);
  });
}

int daris_eval_pick(const daris_ready_key* keys, int32_t n, int32_t* out_index) {
  return eval_guard([&] {
    if (n < 1) throw daris::Error(DARIS_E_VALUE, "empty ready list");
    *out_index = daris::pick_ready(keys, n);
  });
}

int daris_eval_next_completion(const double* remaining, const double* rates, const int64_t* job_ids,
                               const int64_t* stage_indices, int32_t n, double now, int32_t* out_index,
                               double* out_time) {
  static_assert(sizeof(long long) == sizeof(int64_t), "int64 layout");
  return eval_guard([&] {
    *out_index = daris::next_completion_eval(remaining, rates, reinterpret_cast<const long long*>(job_ids),
                                             reinterpret_cast<const long long*>(stage_indices), n, now, out_time);
  });
}

int daris_eval_advance(double* remaining, const double* rates, const int64_t* job_ids,
                       const int64_t* stage_indices, int32_t n, double dt) {
  return eval_guard([&] {
    daris::advance_eval(remaining, rates, reinterpret_cast<const long long*>(job_ids),
                        reinterpret_cast<const long long*>(stage_indices), n, dt);
  });
}

}  // extern "C"

int daris_partition_layout(int32_t n_contexts, int32_t sm_per_context, const int32_t* unit_sms, int32_t n_units,
                           int32_t* first_unit, int32_t* n_taken, int32_t* sm_count) {
  if (n_contexts < 1 || sm_per_context < 1 || n_units < 1 || !unit_sms || !first_unit || !n_taken || !sm_count)
    return DARIS_E_VALUE;
  std::vector<int> start(static_cast<size_t>(n_units) + 1, 0);
  for (int u = 0; u < n_units; ++u) {
    if (unit_sms[u] < 1) return DARIS_E_VALUE;
    start[u + 1] = start[u] + unit_sms[u];
  }
  const int covered = start[n_units];
  // nearest unit start to x (modulo the device), ties to the lower
  auto boundary = [&](double x) {
    x = std::fmod(x, static_cast<double>(covered));
    int best = 0;
    double dist = x;
    for (int u = 1; u <= n_units; ++u) {
      if (std::fabs(start[u] - x) < dist) {
        dist = std::fabs(start[u] - x);
        best = u;
      }
    }
    return best % n_units;
  };
  for (int k = 0; k < n_contexts; ++k) {
    const double x0 = static_cast<double>(k) * covered / n_contexts;
    const int u0 = boundary(x0);
    int taken = (boundary(x0 + sm_per_context) - u0 + n_units) % n_units;
    if (taken == 0) taken = sm_per_context * 2 >= covered ? n_units : 1;
    int cov = 0;
    for (int q = 0; q < taken; ++q) cov += unit_sms[(u0 + q) % n_units];
    first_unit[k] = u0;
    n_taken[k] = taken;
    sm_count[k] = cov;
  }
  return DARIS_OK;
}

