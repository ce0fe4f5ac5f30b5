// Parity backends of the DARIS engine: the SM water-filling rate model
// (gpu.py:118-240), the offline full-load measurement (timing.py:147-218) and
// the deterministic event loop (engine.py:379-531), plus a trace-replay mode
// where every stage runs for a recorded duration.
#include <algorithm>
#include <limits>
#include <queue>
#include <sstream>

#include "core/dispatcher.hpp"

namespace daris {

double water_fill(const std::vector<int>& widths, double capacity, std::vector<Alloc>& out) {  // gpu.py:118-152
  if (capacity <= 0) throw Error(DARIS_E_VALUE, "capacity must be positive");
  const size_t n = widths.size();
  out.assign(n, Alloc{0.0, false});
  if (n == 0) return NAN;
  long long total = 0;
  for (int w : widths) total += w;
  if (static_cast<double>(total) <= capacity + kEps) {
    for (size_t i = 0; i < n; ++i) out[i] = Alloc{static_cast<double>(widths[i]), true};
    return NAN;
  }
  std::vector<int> order(n);
  for (size_t i = 0; i < n; ++i) order[i] = static_cast<int>(i);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
    if (widths[a] != widths[b]) return widths[a] < widths[b];
    return a < b;
  });
  double remaining = capacity;
  long long active = static_cast<long long>(n);
  for (size_t pos = 0; pos < n; ++pos) {
    const int idx = order[pos];
    const double level = remaining / static_cast<double>(active);
    if (static_cast<double>(widths[idx]) <= level) {
      out[idx] = Alloc{static_cast<double>(widths[idx]), false};
      remaining -= widths[idx];
      active -= 1;
    } else {
      for (size_t q = pos; q < n; ++q) out[order[q]] = Alloc{level, false};
      return level;
    }
  }
  throw Error(DARIS_E_INTERNAL, "water_fill failed to settle on a level");
}

double allocate_rates(const daris_gpu_config& g, int per_ctx_sms, const std::vector<int>& widths,
                      const std::vector<int>& ctx, std::vector<Alloc>& alloc,
                      std::vector<double>& rates) {  // gpu.py:167-205
  const size_t n = widths.size();
  alloc.assign(n, Alloc{0.0, false});
  // group members per context in first-appearance order (dict insertion order)
  std::vector<int> ctx_order;
  std::vector<std::vector<int>> members;
  for (size_t i = 0; i < n; ++i) {
    size_t k = 0;
    while (k < ctx_order.size() && ctx_order[k] != ctx[i]) ++k;
    if (k == ctx_order.size()) {
      ctx_order.push_back(ctx[i]);
      members.emplace_back();
    }
    members[k].push_back(static_cast<int>(i));
  }
  std::vector<int> w;
  std::vector<Alloc> fills;
  for (size_t k = 0; k < ctx_order.size(); ++k) {
    if (static_cast<int>(members[k].size()) > g.n_streams) {
      std::ostringstream m;
      m << "context " << ctx_order[k] << " holds " << members[k].size() << " stages but has " << g.n_streams
        << " streams";
      throw Error(DARIS_E_VALUE, m.str());
    }
    w.clear();
    for (int i : members[k]) w.push_back(widths[i]);
    water_fill(w, static_cast<double>(per_ctx_sms), fills);
    for (size_t q = 0; q < members[k].size(); ++q) alloc[members[k][q]] = fills[q];
  }
  PySum total;
  for (const Alloc& a : alloc) {
    if (a.is_int) total.add_int(static_cast<long long>(a.v));
    else total.add(a.v);
  }
  double scale = 1.0;
  const double tot = total.value();
  if (tot > g.total_sms + kEps) {
    scale = g.total_sms / tot;
    for (Alloc& a : alloc) a = Alloc{a.v * scale, false};
  }
  rates.assign(n, 0.0);
  const double kappa = g.kappa;
  for (size_t k = 0; k < ctx_order.size(); ++k) {
    const long long crowd = static_cast<long long>(members[k].size());
    const double slowdown = kappa > 0 ? 1.0 + kappa * static_cast<double>(crowd - 1) : 1.0;
    for (int i : members[k]) rates[i] = alloc[i].v / widths[i] / slowdown;
  }
  return scale;
}

// earliest finisher; ties on (job, stage) keys (gpu.py:208-226) — decide.cpp
static int next_completion(const std::vector<double>& rem, const std::vector<long long>& k1,
                           const std::vector<long long>& k2, const std::vector<double>& rates, double now,
                           double* t_out) {
  return next_completion_eval(rem.data(), rates.data(), k1.data(), k2.data(), static_cast<int>(rem.size()), now,
                              t_out);
}

static void advance_progress(std::vector<double>& rem, const std::vector<double>& rates, double dt,
                             const std::vector<long long>& k1, const std::vector<long long>& k2) {  // gpu.py:229-240
  advance_eval(rem.data(), rates.data(), k1.data(), k2.data(), static_cast<int>(rem.size()), dt);
}

// One repetition of the busy-system measurement (timing.py:184-218).
static double busy_system_run(const Dispatcher& d, int target_idx, const int32_t* draws) {
  const daris_gpu_config& g = d.gpu();
  const int per = sm_per_context(g);
  const int n_slots = g.n_contexts * g.n_streams;
  const auto& tasks = d.tasks();
  std::vector<int> slot_task(n_slots);
  slot_task[0] = target_idx;
  for (int s = 1; s < n_slots; ++s) {
    const int pick = draws[s - 1];
    if (pick < 0 || pick >= static_cast<int>(tasks.size())) throw Error(DARIS_E_VALUE, "competitor draw out of range");
    slot_task[s] = pick;
  }
  std::vector<int> width(n_slots), ctx(n_slots), lap(n_slots, 0);
  std::vector<double> rem(n_slots);
  std::vector<long long> k1(n_slots), k2(n_slots, 0);
  for (int s = 0; s < n_slots; ++s) {
    const TaskDef& t = tasks[slot_task[s]];
    width[s] = t.width[0];
    rem[s] = t.work[0];
    ctx[s] = s / g.n_streams + 1;
    k1[s] = s;
  }
  std::vector<Alloc> alloc;
  std::vector<double> rates;
  double now = 0.0;
  for (;;) {
    allocate_rates(g, per, width, ctx, alloc, rates);
    double t;
    const int i = next_completion(rem, k1, k2, rates, now, &t);
    advance_progress(rem, rates, t - now, k1, k2);
    now = t;
    const TaskDef& spec = tasks[slot_task[i]];
    const int following = lap[i] + 1;
    const int n_st = static_cast<int>(spec.work.size());
    if (i == 0 && following == n_st) return now;
    const int pos = following % n_st;
    lap[i] = pos;
    k2[i] += 1;
    width[i] = spec.width[pos];
    rem[i] = spec.work[pos];
  }
}

double full_load_time(const Dispatcher& d, int task_id, int reps, const int32_t* draws) {  // timing.py:147-181
  if (reps < 1) throw Error(DARIS_E_VALUE, "repetitions must be >= 1");
  const int idx = d.index_of(task_id);
  const int per_rep = d.gpu().n_contexts * d.gpu().n_streams - 1;
  PySum s;
  for (int r = 0; r < reps; ++r) s.add(busy_system_run(d, idx, draws + static_cast<size_t>(r) * per_rep));
  return s.value() / reps;
}

// ------------------------------------------------------------------ event loop
namespace {
struct Acc {  // engine.py:153-220 (+ p99)
  double warmup_end;
  long long rel[2] = {0, 0}, acc[2] = {0, 0}, rej[2] = {0, 0}, cmp[2] = {0, 0}, miss[2] = {0, 0};
  std::vector<double> resp[2];
  long long inputs = 0;
};

daris_response_stats stats(std::vector<double> v) {  // engine.py:97-116
  daris_response_stats s{0, 0, 0, 0, 0, 0};
  if (v.empty()) return s;
  std::sort(v.begin(), v.end());
  const size_t n = v.size();
  s.mean = py_sum(v) / static_cast<double>(n);
  s.min = v.front();
  s.max = v.back();
  s.p95 = v[static_cast<size_t>(std::ceil(0.95 * static_cast<double>(n))) - 1];
  s.p99 = v[static_cast<size_t>(std::ceil(0.99 * static_cast<double>(n))) - 1];
  s.count = static_cast<int64_t>(n);
  return s;
}
}  // namespace

void sim_run(Dispatcher& d, double duration, double warmup_frac, const double* phases, daris_report* out,
             const std::unordered_map<long long, double>* trace, const std::unordered_set<long long>* unsampled) {
  if (!(duration > 0)) throw Error(DARIS_E_INVALID_SCENARIO, "duration must be positive");
  if (!(0.0 <= warmup_frac && warmup_frac < 1.0))
    throw Error(DARIS_E_INVALID_SCENARIO, "warmup fraction must lie in [0, 1)");
  const daris_gpu_config& g = d.gpu();
  for (const TaskDef& t : d.tasks())
    for (int w : t.width)
      if (w > g.total_sms) throw Error(DARIS_E_INVALID_SCENARIO, "stage width exceeds the device");
  const int per = sm_per_context(g);
  Acc acc;
  acc.warmup_end = duration * warmup_frac;

  // release heap (time, task id) — heapq order
  using Rel = std::pair<double, int>;
  std::priority_queue<Rel, std::vector<Rel>, std::greater<Rel>> heap;
  std::vector<long long> rel_index(d.n_tasks(), 0);
  std::vector<double> phase(d.n_tasks());
  for (int i = 0; i < d.n_tasks(); ++i) {
    phase[i] = phases[i];
    if (phase[i] < duration) heap.push({phase[i], d.tasks()[i].id});
  }

  std::vector<std::vector<StageJob*>> streams(g.n_contexts, std::vector<StageJob*>(g.n_streams, nullptr));
  std::vector<StageJob*> active;
  std::vector<double> rem, rates;
  std::vector<long long> k1, k2;
  std::vector<int> widths, ctxs;
  std::vector<Alloc> alloc;
  int job_counter = 0;
  double now = 0.0;
  const bool check = d.opts().check_invariants != 0;
  std::vector<double> work_buf;

  auto refill = [&]() {  // engine.py:434-469
    std::vector<StageJob*> started;
    for (int c = 1; c <= g.n_contexts; ++c) {
      for (;;) {
        int slot = -1;
        for (int s = 0; s < g.n_streams; ++s)
          if (!streams[c - 1][s]) {
            slot = s;
            break;
          }
        if (slot < 0) break;
        StageJob* st = d.dispatch(c, slot, now);
        if (!st) break;
        streams[c - 1][slot] = st;
        started.push_back(st);
      }
    }
    active.clear();
    for (int c = 0; c < g.n_contexts; ++c)
      for (StageJob* s : streams[c])
        if (s) active.push_back(s);
    const size_t n = active.size();
    rem.resize(n);
    k1.resize(n);
    k2.resize(n);
    widths.resize(n);
    ctxs.resize(n);
    for (size_t i = 0; i < n; ++i) {
      rem[i] = active[i]->rem;
      k1[i] = active[i]->job->id;
      k2[i] = active[i]->j;
      widths[i] = active[i]->width;
      ctxs[i] = active[i]->ctx;
    }
    if (n) {
      if (trace) {
        rates.assign(n, 1.0);
      } else {
        allocate_rates(g, per, widths, ctxs, alloc, rates);
        PySum tot;
        for (const Alloc& a : alloc) {
          if (a.is_int) tot.add_int(static_cast<long long>(a.v));
          else tot.add(a.v);
        }
        if (!(tot.value() <= g.total_sms + kEps)) throw Error(DARIS_E_INTERNAL, "allocation exceeds the device");
      }
    } else {
      rates.clear();
    }
    for (StageJob* st : started) {
      size_t i = 0;
      while (active[i] != st) ++i;
      d.logrec(now, DARIS_LOG_STAGE_START, st->job->task, st->job->id, st->j, st->ctx, st->stream, rates[i]);
    }
    if (check) d.verify_invariants(streams);
  };

  for (;;) {
    double t_event = duration;
    int kind = 2;
    if (!heap.empty() && (heap.top().first < t_event || (heap.top().first == t_event && 0 < kind))) {
      t_event = heap.top().first;
      kind = 0;
    }
    int pend = -1;
    if (!active.empty()) {
      double tc;
      pend = next_completion(rem, k1, k2, rates, now, &tc);
      if (tc < t_event || (tc == t_event && 1 < kind)) {
        t_event = tc;
        kind = 1;
      }
    }
    if (!active.empty()) {
      advance_progress(rem, rates, t_event - now, k1, k2);
      for (size_t i = 0; i < active.size(); ++i) active[i]->rem = rem[i];
    }
    now = t_event;
    if (kind == 0) {  // RELEASE (engine.py:485-507)
      const int tid = heap.top().second;
      heap.pop();
      job_counter += 1;
      const TaskDef& spec = d.task(tid);
      const double* work = nullptr;
      if (trace) {
        work_buf.resize(spec.work.size());
        for (size_t j = 0; j < spec.work.size(); ++j) {
          // keyed (task, job, stage) like the recorded trace and the reference shim
          const long long key = (static_cast<long long>(tid) << 40) | (static_cast<long long>(job_counter) << 8) |
                                static_cast<long long>(j);
          auto it = trace->find(key);
          // jobs the recorded run rejected never execute: any placeholder works
          work_buf[j] = it == trace->end() ? spec.work[j] : it->second;
        }
        work = work_buf.data();
      }
      // make_job + admission (audits go to their own list), then the release
      // record followed by the admission outcome, as engine.py:487-502 emits them
      daris_placement pl;
      d.release(tid, now, job_counter, work, &pl);
      d.logrec(now, DARIS_LOG_RELEASE, tid, job_counter);
      const int hp = spec.hp ? 0 : 1;
      if (now >= acc.warmup_end) {
        acc.rel[hp] += 1;
        if (pl.context) acc.acc[hp] += 1;
        else acc.rej[hp] += 1;
      }
      if (pl.context == 0) d.logrec(now, DARIS_LOG_REJECT, tid, job_counter);
      else d.logrec(now, DARIS_LOG_ADMIT, tid, job_counter, -1, pl.context);
      const int ti = d.index_of(tid);
      rel_index[ti] += 1;
      const double next_release = phase[ti] + static_cast<double>(rel_index[ti]) * spec.period;
      if (next_release < duration) heap.push({next_release, tid});
      refill();
    } else if (kind == 1) {  // STAGE_COMPLETE (engine.py:509-523)
      StageJob* st = active[pend];
      const double rate = rates[pend];
      streams[st->ctx - 1][st->stream] = nullptr;
      const int task_id = st->job->task, job_id = st->job->id, j = st->j, ctx = st->ctx, stream = st->stream;
      const double release = st->job->release;
      const int batch = st->job->batch;
      bool missed = false;
      const bool sample = !unsampled || !unsampled->count((static_cast<long long>(task_id) << 40) |
                                                          (static_cast<long long>(job_id) << 8) | j);
      const bool done = d.complete(st, now, &missed, sample);  // may free the job
      d.logrec(now, DARIS_LOG_STAGE_COMPLETE, task_id, job_id, j, ctx, stream, rate);
      if (done) {
        d.logrec(now, DARIS_LOG_JOB_COMPLETE, task_id, job_id, -1, ctx);
        if (release >= acc.warmup_end) {
          const int hp = d.task(task_id).hp ? 0 : 1;
          acc.cmp[hp] += 1;
          acc.inputs += batch;
          acc.resp[hp].push_back(now - release);
          if (missed) acc.miss[hp] += 1;
        }
      }
      active[pend] = nullptr;
      refill();
    } else {
      d.logrec(duration, DARIS_LOG_SIM_END);
      break;
    }
  }

  daris_report r{};
  r.duration = duration;
  r.warmup = acc.warmup_end;
  const double window = duration - acc.warmup_end;
  r.jps = window > 0 ? static_cast<double>(acc.inputs) / window : 0.0;
  r.dmr_hp = acc.acc[0] ? static_cast<double>(acc.miss[0]) / static_cast<double>(acc.acc[0]) : 0.0;
  r.dmr_lp = acc.acc[1] ? static_cast<double>(acc.miss[1]) / static_cast<double>(acc.acc[1]) : 0.0;
  r.response_hp = stats(acc.resp[0]);
  r.response_lp = stats(acc.resp[1]);
  r.released_hp = acc.rel[0];
  r.released_lp = acc.rel[1];
  r.accepted_hp = acc.acc[0];
  r.accepted_lp = acc.acc[1];
  r.rejected_hp = acc.rej[0];
  r.rejected_lp = acc.rej[1];
  r.completed_hp = acc.cmp[0];
  r.completed_lp = acc.cmp[1];
  r.missed_hp = acc.miss[0];
  r.missed_lp = acc.miss[1];
  *out = r;
}

}  // namespace daris
