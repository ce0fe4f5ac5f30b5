// DARIS dispatcher: task model, execution-time tracking and the scheduling
// core. Reference semantics: /root/reference/pkg/src/stagesim/{model,timing,
// scheduler}.py (cited per function). Arithmetic mirrors CPython 3.12.
#include "core/dispatcher.hpp"

#include <algorithm>
#include <set>
#include <sstream>

namespace daris {

// ---------------------------------------------------------------- gpu.py helpers
int ceil_even(double x) {  // gpu.py:76-78
  return 2 * static_cast<int>(std::ceil(x / 2.0 - kEps));
}

int sm_per_context(const daris_gpu_config& g) {  // gpu.py:81-86
  const double os = g.oversubscription;
  if (!(1.0 <= os && os <= g.n_contexts + kEps)) {
    std::ostringstream m;
    m << "oversubscription " << os << " outside [1, " << g.n_contexts << "]";
    throw Error(DARIS_E_INVALID_OVERSUB, m.str());
  }
  return ceil_even(os * g.total_sms / g.n_contexts);
}

double batching_gain(int ref_b, double ref_g, int b) {  // gpu.py:262-268
  if (b < 1) throw Error(DARIS_E_INVALID_BATCH, "batch size must be an integer >= 1");
  if (ref_b == 0) return 1.0;  // no curve (UNIT_BATCHING)
  if (b == 1 || ref_b == 1) return 1.0;
  const double exponent = std::log(static_cast<double>(b)) / std::log(static_cast<double>(ref_b));
  const double g = std::pow(ref_g, exponent);
  return std::max(1.0, g);  // Python max(1.0, g): first arg kept on ties
}

double effective_stage_time(double nominal, int b, int ref_b, double ref_g) {  // gpu.py:273-284
  if (b < 1) throw Error(DARIS_E_INVALID_BATCH, "batch size must be an integer >= 1");
  return nominal * b / batching_gain(ref_b, ref_g, b);
}

void validate_gpu(const daris_gpu_config& g) {  // gpu.py:53-68
  if (g.total_sms < 1) throw Error(DARIS_E_VALUE, "total_sms must be >= 1");
  if (g.n_contexts < 1 || g.n_streams < 1) throw Error(DARIS_E_VALUE, "n_contexts and n_streams must be >= 1");
  if (!(1.0 <= g.oversubscription && g.oversubscription <= g.n_contexts + kEps)) {
    std::ostringstream m;
    m << "oversubscription must lie in [1, n_contexts], got " << g.oversubscription << " with " << g.n_contexts
      << " contexts";
    throw Error(DARIS_E_INVALID_OVERSUB, m.str());
  }
  if (g.policy == DARIS_POLICY_STR && g.n_contexts != 1)
    throw Error(DARIS_E_VALUE, "the stream-only policy uses a single context");
  if (g.policy == DARIS_POLICY_MPS && g.n_streams != 1)
    throw Error(DARIS_E_VALUE, "the context-only policy uses a single stream per context");
  if (g.kappa < 0) throw Error(DARIS_E_VALUE, "interference_kappa must be >= 0");
}

// ---------------------------------------------------------------- model.py:72-112
std::vector<TaskDef> build_task_defs(const daris_task_spec* tasks, int n, const daris_stage_spec* stages,
                                     int n_stages, bool no_staging) {
  if (n <= 0) throw Error(DARIS_E_EMPTY_TASK_SET, "a task set needs at least one task");
  std::set<int> seen, dups;
  for (int i = 0; i < n; ++i) {
    if (!seen.insert(tasks[i].id).second) dups.insert(tasks[i].id);
  }
  if (!dups.empty()) {
    std::ostringstream m;
    m << "duplicate task ids: [";
    bool first = true;
    for (int d : dups) { m << (first ? "" : ", ") << d; first = false; }
    m << "]";
    throw Error(DARIS_E_DUPLICATE_ID, m.str());
  }
  if (*seen.begin() != 1 || *seen.rbegin() != n)
    throw Error(DARIS_E_INVALID_TASK_IDS, "task ids must be dense 1.." + std::to_string(n));
  std::vector<TaskDef> out;
  out.reserve(n);
  for (int i = 0; i < n; ++i) {
    const daris_task_spec& s = tasks[i];
    if (s.n_stages < 1) throw Error(DARIS_E_INVALID_STAGE, "task " + std::to_string(s.id) + " has no stages");
    if (!(s.period > 0))
      throw Error(DARIS_E_INVALID_STAGE, "task " + std::to_string(s.id) + " has a non-positive period");
    if (s.deadline != s.period)
      throw Error(DARIS_E_VALUE, "task " + std::to_string(s.id) + ": deadline must equal period");
    if (s.first_stage < 0 || s.first_stage + s.n_stages > n_stages)
      throw Error(DARIS_E_VALUE, "stage slice out of range");
    TaskDef t;
    t.id = s.id;
    t.hp = (s.priority == DARIS_HP);
    t.period = s.period;
    t.deadline = s.deadline;
    t.batch = s.batch_size < 1 ? 1 : s.batch_size;
    if (s.batch_size < 1) throw Error(DARIS_E_INVALID_BATCH, "batch size must be an integer >= 1");
    t.ref_b = s.curve_ref_batch;
    t.ref_g = s.curve_ref_gain;
    if (t.ref_b < 0) throw Error(DARIS_E_INVALID_BATCH, "reference batch must be >= 1");
    if (t.ref_b > 0 && !(t.ref_g > 0)) throw Error(DARIS_E_VALUE, "reference gain must be positive");
    for (int j = 0; j < s.n_stages; ++j) {
      const daris_stage_spec& p = stages[s.first_stage + j];
      if (!(p.nominal_time > 0))
        throw Error(DARIS_E_INVALID_STAGE, "task " + std::to_string(s.id) + " stage " + std::to_string(j) +
                                               ": nominal time must be positive");
      if (p.width < 1)
        throw Error(DARIS_E_INVALID_STAGE, "task " + std::to_string(s.id) + " stage " + std::to_string(j) +
                                               ": width must be >= 1 SM");
      t.nominal.push_back(p.nominal_time);
      t.width.push_back(p.width);
    }
    t.nominal_total = py_sum(t.nominal);
    out.push_back(std::move(t));
  }
  std::sort(out.begin(), out.end(), [](const TaskDef& a, const TaskDef& b) { return a.id < b.id; });
  if (no_staging) {  // collapse_stages (model.py:102-112)
    for (TaskDef& t : out) {
      const int w = *std::max_element(t.width.begin(), t.width.end());
      const double total = t.nominal_total;
      t.nominal.assign(1, total);
      t.width.assign(1, w);
      t.nominal_total = py_sum(t.nominal);
    }
  }
  for (TaskDef& t : out) {
    t.work.clear();
    for (double nom : t.nominal) t.work.push_back(effective_stage_time(nom, t.batch, t.ref_b, t.ref_g));
  }
  return out;
}

// ---------------------------------------------------------------- Dispatcher
Dispatcher::Dispatcher(const daris_gpu_config& gpu, std::vector<TaskDef> tasks, const daris_options& opts)
    : gpu_(gpu), opts_(opts), tasks_(std::move(tasks)) {
  validate_gpu(gpu_);
  if (opts_.window_size < 1) throw Error(DARIS_E_VALUE, "window capacity must be >= 1");
  rt_.resize(tasks_.size());
  for (size_t i = 0; i < tasks_.size(); ++i) {
    idx_[tasks_[i].id] = static_cast<int>(i);
    rt_[i].win.resize(tasks_[i].nominal.size());
    for (Window& w : rt_[i].win) w.cap = opts_.window_size;
  }
  ctx_tasks_.resize(gpu_.n_contexts);
  ready_.resize(gpu_.n_contexts);
  live_.resize(gpu_.n_contexts);
}

int Dispatcher::index_of(int id) const {
  auto it = idx_.find(id);
  if (it == idx_.end()) throw Error(DARIS_E_NOT_FOUND, "unknown task " + std::to_string(id));
  return it->second;
}

void Dispatcher::record_execution(int tid, int j, double observed) {  // timing.py:45-50,75-76
  if (!(observed > 0)) {
    std::ostringstream m;
    m << "observed time must be positive, got " << observed;
    throw Error(DARIS_E_NONPOSITIVE_SAMPLE, m.str());
  }
  rt(tid).win.at(j).record(observed);
}

double Dispatcher::stage_estimate(int tid, int j) const {  // timing.py:78-86
  const int i = index_of(tid);
  const Window& w = rt_[i].win.at(j);
  if (!w.empty()) return w.peak();
  const TaskDef& t = tasks_[i];
  return stage_fallback(rt_[i].full_load, t.nominal[j], t.nominal_total);
}

double Dispatcher::task_estimate(int tid) const {  // timing.py:88-90
  const TaskDef& t = task(tid);
  PySum s;
  for (size_t j = 0; j < t.nominal.size(); ++j) s.add(stage_estimate(tid, static_cast<int>(j)));
  return s.value();
}

double Dispatcher::utilization(int tid) {  // timing.py:92-108
  TaskRT& r = rt(tid);
  if (r.ucache_valid) return r.ucache;
  const TaskDef& t = task(tid);
  const double u = utilization_of(r.completed, r.full_load, r.completed == 0 ? 0.0 : task_estimate(tid), t.period);
  r.ucache = u;
  r.ucache_valid = true;
  return u;
}

void Dispatcher::note_job_complete(int tid) {  // timing.py:110-114
  TaskRT& r = rt(tid);
  r.completed += 1;
  r.ucache_valid = false;
}

std::vector<double> Dispatcher::deadline_shares(int tid) const {  // timing.py:116-132
  const TaskDef& t = task(tid);
  const size_t n = t.nominal.size();
  std::vector<double> est(n);
  for (size_t j = 0; j < n; ++j) est[j] = stage_estimate(tid, static_cast<int>(j));
  std::vector<double> shares(n);
  deadline_split(est.data(), static_cast<int>(n), t.deadline, shares.data(), tid);
  return shares;
}

void Dispatcher::populate() {  // scheduler.py:131-153
  const int n = static_cast<int>(tasks_.size());
  std::vector<double> util(n), totals(gpu_.n_contexts);
  std::vector<int32_t> hp(n), ids(n), home(n);
  for (int i = 0; i < n; ++i) {
    ids[i] = tasks_[i].id;
    hp[i] = tasks_[i].hp ? 1 : 0;
    util[i] = utilization(ids[i]);
  }
  std::vector<int32_t> order(n);
  greedy_place(util.data(), hp.data(), ids.data(), n, gpu_.n_contexts, opts_.placement_insertion != 0,
               home.data(), totals.data(), order.data());
  for (int i : order) {  // ctx_tasks order = placement order (feeds the += ledgers)
    rt_[i].home = home[i];
    ctx_tasks_[home[i] - 1].push_back(ids[i]);
  }
}

daris_ledger_t Dispatcher::ledger(int ctx) {  // scheduler.py:157-171
  const auto& ids = ctx_tasks_.at(ctx - 1);
  std::vector<daris_ledger_entry> e(ids.size());
  for (size_t k = 0; k < ids.size(); ++k) {
    e[k].util = utilization(ids[k]);
    e[k].hp = task(ids[k]).hp ? 1 : 0;
    e[k].active_jobs = static_cast<int32_t>(std::min<long long>(rt(ids[k]).active, 1 << 30));
  }
  return ledger_sum(e.data(), static_cast<int>(e.size()));
}

Audit Dispatcher::admission_test(const Job& job, int ctx, double t) {  // scheduler.py:179-200
  const daris_ledger_t l = ledger(ctx);
  const double u = utilization(job.task);
  const bool hp = task(job.task).hp;
  double active, limit;
  bool ok;
  admission_eval(l, u, hp, gpu_.n_streams, &active, &limit, &ok);
  return {t, active, u, limit, job.id, job.task, hp ? DARIS_HP : DARIS_LP, ctx, ok};
}

double Dispatcher::predicted_finish(int tid, int ctx, double t) const {  // scheduler.py:202-213
  std::vector<double> backlog;
  for (const Job* live : live_.at(ctx - 1))
    for (const StageJob& st : live->stages)
      if (st.state != DONE) backlog.push_back(stage_estimate(live->task, st.j));
  return predicted_finish_eval(t, backlog.data(), static_cast<long long>(backlog.size()), gpu_.n_streams,
                               task_estimate(tid));
}

void Dispatcher::place(Job* job, int ctx) {  // scheduler.py:268-274
  job->place = ctx;
  rt(job->task).active += 1;
  live_[ctx - 1].push_back(job);
  StageJob& first = job->stages[0];
  if (first.state != PENDING) throw Error(DARIS_E_VALUE, "illegal stage transition");
  first.state = READY;
  ready_[ctx - 1].push_back(&first);
}

void Dispatcher::migrate_task(int tid, int old_ctx, int new_ctx) {  // scheduler.py:261-266
  if (task(tid).hp) throw Error(DARIS_E_INTERNAL, "high-priority tasks never migrate");
  auto& from = ctx_tasks_[old_ctx - 1];
  from.erase(std::find(from.begin(), from.end(), tid));
  ctx_tasks_[new_ctx - 1].push_back(tid);
  rt(tid).home = new_ctx;
}

Job* Dispatcher::release(int tid, double t, int job_id, const double* stage_work, daris_placement* out) {
  // make_job (model.py:201-230)
  const TaskDef& spec = task(tid);
  const double abs_dl = t + spec.deadline;
  const std::vector<double> shares = deadline_shares(tid);
  auto job = std::make_unique<Job>();
  job->id = job_id;
  job->task = tid;
  job->release = t;
  job->dl = abs_dl;
  job->batch = spec.batch;
  const int n = static_cast<int>(spec.nominal.size());
  job->stages.resize(n);
  std::vector<double> vdls(n);
  virtual_deadlines(t, abs_dl, shares.data(), n, vdls.data());
  for (int j = 0; j < n; ++j) {
    const double vdl = vdls[j];
    StageJob& s = job->stages[j];
    s.job = job.get();
    s.j = j;
    s.width = spec.width[j];
    s.rem = stage_work ? stage_work[j] : spec.work[j];
    s.vdl = vdl;
  }
  Job* jp = job.get();
  if (jobs_.count(job_id)) throw Error(DARIS_E_VALUE, "duplicate job id " + std::to_string(job_id));

  // admit_or_migrate (scheduler.py:215-259)
  const int home = rt(tid).home;
  daris_placement pl{0, 0, 0, 0};
  auto audit = [&](int ctx) {
    Audit a = admission_test(*jp, ctx, t);
    audits.push_back(a);
    pl.n_audits += 1;
    return a.admitted;
  };
  int target = 0;
  if (spec.hp) {
    if (!opts_.hpa || audit(home)) target = home;
  } else if (audit(home)) {
    target = home;
  } else {
    std::vector<int> ok;
    for (int c = 1; c <= gpu_.n_contexts; ++c) {
      if (c == home) continue;
      if (audit(c)) ok.push_back(c);
    }
    if (!ok.empty()) {
      target = ok[0];
      double best = predicted_finish(tid, ok[0], t);
      for (size_t k = 1; k < ok.size(); ++k) {
        const double f = predicted_finish(tid, ok[k], t);
        if (f < best) {  // ties keep the lower context id
          best = f;
          target = ok[k];
        }
      }
      migrate_task(tid, home, target);
      pl.migrated_from = home;
    }
  }
  pl.context = target;
  if (out) *out = pl;
  if (target == 0) return nullptr;  // rejected: the job never runs
  jobs_[job_id] = std::move(job);
  place(jp, target);
  return jp;
}

int Dispatcher::level_key(const StageJob* st) const {  // scheduler.py:278-287
  const Job* job = st->job;
  const bool is_last = st->j == static_cast<int>(job->stages.size()) - 1;
  return priority_level(task(job->task).hp, is_last, st->late_pred, opts_);
}

StageJob* Dispatcher::dispatch(int ctx, int stream, double t) {  // scheduler.py:289-296
  auto& q = ready_.at(ctx - 1);
  if (q.empty()) return nullptr;
  thread_local std::vector<daris_ready_key> keys;
  keys.resize(q.size());
  for (size_t k = 0; k < q.size(); ++k) {
    const StageJob* s = q[k];
    keys[k] = {opts_.edf_on_job_deadline ? s->job->dl : s->vdl, level_key(s), s->job->task, s->job->id, 0};
  }
  const size_t best = static_cast<size_t>(pick_ready(keys.data(), static_cast<int>(keys.size())));
  StageJob* st = q[best];
  q.erase(q.begin() + static_cast<long>(best));
  st->state = RUNNING;  // engine.py:445-449
  st->start = t;
  st->ctx = ctx;
  st->stream = stream;
  return st;
}

StageJob* Dispatcher::find_stage(int job_id, int j) {
  auto it = jobs_.find(job_id);
  if (it == jobs_.end()) return nullptr;
  if (j < 0 || j >= static_cast<int>(it->second->stages.size())) return nullptr;
  return &it->second->stages[j];
}

bool Dispatcher::complete(StageJob* st, double t, bool* missed, bool record_sample) {  // scheduler.py:300-324
  if (st->state != RUNNING) throw Error(DARIS_E_VALUE, "illegal stage transition");
  const double observed = t - st->start;
  // record_sample = false: the real-time executor's stage was in flight across a
  // GPU-wide pause, so its time is not an execution-time sample (real mode only)
  if (record_sample) record_execution(st->job->task, st->j, observed);
  st->state = DONE;
  Job* job = st->job;
  if (st->j != static_cast<int>(job->stages.size()) - 1) {
    StageJob& next = job->stages[st->j + 1];
    next.late_pred = t > st->vdl;
    next.state = READY;
    int ctx = job->place;
    if (opts_.stage_migration) {
      // extension (north star): the next stage follows the task's current home,
      // so an LP task migrated at release moves its in-flight job too.
      const int home = rt(job->task).home;
      if (home != ctx) {
        auto& from = live_[ctx - 1];
        from.erase(std::find(from.begin(), from.end(), job));
        live_[home - 1].push_back(job);
        job->place = home;
        ctx = home;
      }
    }
    ready_[ctx - 1].push_back(&next);
    *missed = false;
    return false;
  }
  job->done_at = t;
  TaskRT& r = rt(job->task);
  r.active -= 1;
  note_job_complete(job->task);
  auto& lv = live_[job->place - 1];
  lv.erase(std::find(lv.begin(), lv.end(), job));
  *missed = t > job->dl;
  jobs_.erase(job->id);  // frees the job (and st); caller must not touch st afterwards
  return true;
}

void Dispatcher::verify_invariants(const std::vector<std::vector<StageJob*>>& streams) {  // engine.py:535-551
  for (int c = 1; c <= gpu_.n_contexts; ++c) {
    const daris_ledger_t l = ledger(c);
    if (!(l.lp_active <= l.lp_total + 1e-9) || !(l.hp_active <= l.hp_total + 1e-9))
      throw Error(DARIS_E_INTERNAL, "ledger invariant violated");
    bool free_stream = false;
    for (StageJob* s : streams[c - 1])
      if (!s) free_stream = true;
    if (free_stream && !ready_[c - 1].empty())
      throw Error(DARIS_E_INTERNAL, "context " + std::to_string(c) + " idles a stream while stages are ready");
  }
  for (const TaskDef& t : tasks_) {
    const TaskRT& r = rt(t.id);
    const double expected = r.completed == 0 ? r.full_load / t.period : task_estimate(t.id) / t.period;
    if (std::fabs(utilization(t.id) - expected) >= 1e-12) throw Error(DARIS_E_INTERNAL, "stale utilization cache");
  }
}

}  // namespace daris
