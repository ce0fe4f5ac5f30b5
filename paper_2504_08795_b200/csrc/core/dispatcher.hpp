// DARIS dispatcher core (C++). Owns tasks, per-task timing state, context
// placement, per-context ready queues and live jobs. Semantics follow the
// reference's model.py / timing.py / scheduler.py; float arithmetic replicates
// CPython 3.12 exactly (see PySum) so decisions are bit-identical.
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <deque>
#include <memory>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "daris.h"

namespace daris {

constexpr double kEps = 1e-9;  // gpu.py:33, engine.py:58

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

// CPython 3.12 builtin sum() over a mix of ints and floats (bltinmodule.c):
// an exact int prefix, then Neumaier-compensated float accumulation where int
// items are added without compensation.
struct PySum {
  bool in_int = true;
  long long i = 0;
  double f = 0.0, c = 0.0;
  void add_int(long long v) {
    if (in_int) i += v;
    else f += static_cast<double>(v);
  }
  void add(double x) {
    if (in_int) {
      in_int = false;
      f = static_cast<double>(i) + x;
      c = 0.0;
      return;
    }
    const double t = f + x;
    if (std::fabs(f) >= std::fabs(x)) c += (f - t) + x;
    else c += (x - t) + f;
    f = t;
  }
  double value() const {
    if (in_int) return static_cast<double>(i);
    if (c != 0.0 && std::isfinite(c)) return f + c;
    return f;
  }
};

inline double py_sum(const std::vector<double>& v) {
  PySum s;
  for (double x : v) s.add(x);
  return s.value();
}

int ceil_even(double x);                           // gpu.py:76-78
int sm_per_context(const daris_gpu_config& g);     // gpu.py:81-86
double batching_gain(int ref_b, double ref_g, int b);            // gpu.py:262-268
double effective_stage_time(double nominal, int b, int ref_b, double ref_g);  // gpu.py:273-284

struct TaskDef {
  int id = 0;
  bool hp = true;
  double period = 0, deadline = 0;
  std::vector<double> nominal;
  std::vector<int> width;
  int batch = 1, ref_b = 0;
  double ref_g = 1.0;
  double nominal_total = 0;  // py sum of nominal (model.py:47-49)
  std::vector<double> work;  // effective stage time per stage
};

// Ring of the last `cap` samples (timing.py:33-62).
struct Window {
  std::vector<double> buf;
  int cap = 5, count = 0, head = 0;
  void record(double v) {
    if (static_cast<int>(buf.size()) < cap) buf.push_back(v);
    else buf[head] = v;
    head = (head + 1) % cap;
    if (count < cap) ++count;
  }
  bool empty() const { return count == 0; }
  // max() over the samples oldest->newest (decide.cpp window_peak)
  double peak() const;
};

enum StageSt : uint8_t { PENDING = 0, READY = 1, RUNNING = 2, DONE = 3 };

struct Job;
struct StageJob {
  Job* job = nullptr;
  int j = 0;
  int width = 0;
  double rem = 0;        // remaining full-width seconds (sim backend)
  double vdl = 0;        // virtual absolute deadline
  bool late_pred = false;
  StageSt state = PENDING;
  double start = 0;
  int ctx = -1, stream = -1;
};

struct Job {
  int id = 0, task = 0, batch = 1, place = 0;
  double release = 0, dl = 0, done_at = -1;
  std::vector<StageJob> stages;
};

struct TaskRT {
  int home = 0;
  double full_load = 0;
  std::vector<Window> win;
  long long completed = 0;
  long long active = 0;
  bool ucache_valid = false;
  double ucache = 0;
};

struct Audit {
  double time, active, u, limit;
  int job, task, prio, ctx;
  bool admitted;
};

struct LogRec {
  double time;
  int kind, task, job, stage, ctx, stream;
  double rate;
};

class Dispatcher {
 public:
  Dispatcher(const daris_gpu_config& gpu, std::vector<TaskDef> tasks, const daris_options& opts);

  // --- tasks / timing (timing.py) ---
  int n_tasks() const { return static_cast<int>(tasks_.size()); }
  const TaskDef& task(int id) const { return tasks_.at(index_of(id)); }
  const std::vector<TaskDef>& tasks() const { return tasks_; }
  int index_of(int id) const;
  TaskRT& rt(int id) { return rt_.at(index_of(id)); }
  void record_execution(int tid, int j, double observed);
  double stage_estimate(int tid, int j) const;
  double task_estimate(int tid) const;
  double utilization(int tid);
  void note_job_complete(int tid);
  std::vector<double> deadline_shares(int tid) const;

  // --- scheduler (scheduler.py) ---
  void populate();
  daris_ledger_t ledger(int ctx);
  Audit admission_test(const Job& job, int ctx, double t);
  double predicted_finish(int tid, int ctx, double t) const;
  // make_job + admit_or_migrate. Returns the job (owned by the dispatcher while live).
  Job* release(int tid, double t, int job_id, const double* stage_work, daris_placement* out);
  StageJob* dispatch(int ctx, int stream, double t);
  bool complete(StageJob* st, double t, bool* missed, bool record_sample = true);
  StageJob* find_stage(int job_id, int j);
  int ready_count(int ctx) const { return static_cast<int>(ready_.at(ctx - 1).size()); }

  const daris_gpu_config& gpu() const { return gpu_; }
  const daris_options& opts() const { return opts_; }
  std::vector<Audit> audits;
  std::vector<LogRec> log;
  bool collect_log = true;
  void logrec(double t, int kind, int task = -1, int job = -1, int stage = -1, int ctx = -1, int stream = -1,
              double rate = NAN) {
    if (collect_log) log.push_back({t, kind, task, job, stage, ctx, stream, rate});
  }
  void verify_invariants(const std::vector<std::vector<StageJob*>>& streams);

 private:
  int level_key(const StageJob* st) const;
  void place(Job* job, int ctx);
  void migrate_task(int tid, int old_ctx, int new_ctx);

  daris_gpu_config gpu_;
  daris_options opts_;
  std::vector<TaskDef> tasks_;
  std::vector<TaskRT> rt_;
  std::unordered_map<int, int> idx_;
  std::vector<std::vector<int>> ctx_tasks_;     // per context, insertion order
  std::vector<std::vector<StageJob*>> ready_;   // per context, insertion order
  std::vector<std::vector<Job*>> live_;         // per context, insertion order
  std::unordered_map<int, std::unique_ptr<Job>> jobs_;
};

// Validation + construction helper shared by the C ABI (model.py:72-112).
std::vector<TaskDef> build_task_defs(const daris_task_spec* tasks, int n, const daris_stage_spec* stages,
                                     int n_stages, bool no_staging);
void validate_gpu(const daris_gpu_config& g);

// --- rate model (gpu.py:118-240) -------------------------------------------
struct Alloc {
  double v;
  bool is_int;
};
// returns level or NaN when everything fits
double water_fill(const std::vector<int>& widths, double capacity, std::vector<Alloc>& out);
// rates for (width, ctx) pairs; returns scale
double allocate_rates(const daris_gpu_config& g, int per_ctx_sms, const std::vector<int>& widths,
                      const std::vector<int>& ctx, std::vector<Alloc>& alloc, std::vector<double>& rates);

double full_load_time(const Dispatcher& d, int task_id, int reps, const int32_t* draws);

// --- stateless decision kernels (decide.cpp), shared by the Dispatcher and the
// object-level drop-in API (daris_eval_* in the C ABI) ------------------------
double window_peak(const double* v, int n);                                       // timing.py:52-56
double stage_fallback(double full_load, double nominal, double nominal_total);     // timing.py:84-86
double utilization_of(long long completed, double full_load, double task_est, double period);  // timing.py:102-107
void deadline_split(const double* est, int n, double deadline, double* out, int task_id);      // timing.py:116-132
void virtual_deadlines(double release, double abs_deadline, const double* shares, int n, double* out);  // model.py:216-227
daris_ledger_t ledger_sum(const daris_ledger_entry* e, int n);                     // scheduler.py:157-171
void admission_eval(const daris_ledger_t& l, double u, bool hp, int n_streams, double* active, double* limit,
                    bool* admitted);                                               // scheduler.py:179-200
void greedy_place(const double* util, const int32_t* hp, const int32_t* ids, int n, int n_ctx, bool insertion,
                  int32_t* out_ctx, double* totals, int32_t* out_order);           // scheduler.py:131-153
double predicted_finish_eval(double t, const double* backlog, long long n, int n_streams, double task_est);
int priority_level(bool hp, bool is_last, bool late_pred, const daris_options& o);  // scheduler.py:278-284
bool key_less(const daris_ready_key& a, const daris_ready_key& b);
int pick_ready(const daris_ready_key* keys, int n);                                // scheduler.py:289-296
int next_completion_eval(const double* rem, const double* rates, const long long* job, const long long* stage, int n,
                         double now, double* t_out);                              // gpu.py:208-226
void advance_eval(double* rem, const double* rates, const long long* job, const long long* stage, int n,
                  double dt);                                                      // gpu.py:229-240

struct RunResult {
  daris_report report;
};
void sim_run(Dispatcher& d, double duration, double warmup_frac, const double* phases, daris_report* out,
             const std::unordered_map<long long, double>* trace,
             const std::unordered_set<long long>* unsampled = nullptr);

}  // namespace daris
