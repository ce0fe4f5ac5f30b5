/* DARIS dispatcher — C ABI (drop-in core for the reference's execution path).
 *
 * The reference (stagesim, pure Python) keeps all scheduling state in Python
 * objects mutated in place. Here one opaque handle owns it in C++; callers hold
 * only the handle and copy out POD results. Every entry point below replaces a
 * reference interface (paths relative to /root/reference/pkg/src/stagesim):
 *
 *   daris_create            build_task_set + collapse_stages + TaskState.fresh +
 *                           TimingTracker + build_contexts + Scheduler.__init__
 *                           (model.py:72-112,181-198; timing.py:64-73;
 *                            gpu.py:44-115; scheduler.py:102-127)
 *   daris_full_load_sim     measure_full_load_time / _busy_system_run (timing.py:147-218)
 *   daris_set_full_load     Simulation.run offline baseline install (engine.py:400-403)
 *   daris_populate          Scheduler.populate_contexts (scheduler.py:131-153)
 *   daris_release           make_job + Scheduler.admit_or_migrate (model.py:201-230;
 *                           scheduler.py:215-274)
 *   daris_dispatch          Scheduler.dispatch + the RUNNING transition done by the
 *                           engine (scheduler.py:289-296; engine.py:444-449)
 *   daris_complete          Scheduler.complete_stage (scheduler.py:300-324)
 *   daris_ledger            Scheduler.context_utilization (scheduler.py:157-171)
 *   daris_admission_test    Scheduler.admission_test (scheduler.py:179-200)
 *   daris_predicted_finish  Scheduler.predicted_finish (scheduler.py:202-213)
 *   daris_stage_estimate /
 *   daris_task_estimate /
 *   daris_utilization /
 *   daris_deadline_shares   TimingTracker (timing.py:78-132)
 *   daris_record_execution  TimingTracker.record_execution (timing.py:75-76)
 *   daris_sim_run           Simulation.run event loop with the rate model
 *                           (engine.py:379-531; gpu.py:118-240)
 *   daris_trace_run         the same loop in trace-replay mode: each stage runs for
 *                           its recorded duration
 *   daris_log_* / daris_audit_*   SimResult.records / SimResult.admissions
 *
 * Floating point follows CPython 3.12 bit for bit (builtin sum = Neumaier
 * compensation for floats, naive for ints; no FMA contraction). The handle
 * is NOT thread-safe: one dispatcher thread per GPU instance.
 */
#ifndef DARIS_H
#define DARIS_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* status codes; nonzero maps 1:1 onto stagesim's exception classes (errors.py:4-73) */
enum daris_status {
  DARIS_OK = 0,
  DARIS_E_EMPTY_TASK_SET = 1,        /* EmptyTaskSet */
  DARIS_E_DUPLICATE_ID = 2,          /* DuplicateId */
  DARIS_E_INVALID_TASK_IDS = 3,      /* InvalidTaskIds */
  DARIS_E_INVALID_STAGE = 4,         /* InvalidStage */
  DARIS_E_NONPOSITIVE_SAMPLE = 5,    /* NonpositiveSample */
  DARIS_E_ZERO_TOTAL_ESTIMATE = 6,   /* ZeroTotalEstimate */
  DARIS_E_INVALID_OVERSUB = 7,       /* InvalidOversubscription */
  DARIS_E_NO_ACTIVE_STAGES = 8,      /* NoActiveStages */
  DARIS_E_OVERSHOOT = 9,             /* OvershootBeyondCompletion */
  DARIS_E_INVALID_BATCH = 10,        /* InvalidBatch */
  DARIS_E_INVALID_SCENARIO = 11,     /* InvalidScenario */
  DARIS_E_VALUE = 12,                /* ValueError */
  DARIS_E_INTERNAL = 13,             /* AssertionError / internal invariant */
  DARIS_E_NOT_FOUND = 14             /* unknown task / job / stage reference */
};

enum daris_priority { DARIS_HP = 0, DARIS_LP = 1 };
enum daris_policy { DARIS_POLICY_STR = 0, DARIS_POLICY_MPS = 1, DARIS_POLICY_MPS_STR = 2 };
enum daris_log_kind {
  DARIS_LOG_RELEASE = 0, DARIS_LOG_ADMIT = 1, DARIS_LOG_REJECT = 2, DARIS_LOG_STAGE_START = 3,
  DARIS_LOG_STAGE_COMPLETE = 4, DARIS_LOG_JOB_COMPLETE = 5, DARIS_LOG_SIM_END = 6
};

typedef struct daris_gpu_config {
  int32_t total_sms, n_contexts, n_streams, policy;
  double oversubscription, kappa;
} daris_gpu_config;

typedef struct daris_stage_spec {
  double nominal_time; /* seconds at full width, batch 1 */
  int32_t width;       /* max SMs the stage can use */
  int32_t _pad;
} daris_stage_spec;

typedef struct daris_task_spec {
  int32_t id, priority;
  double period, deadline;
  int32_t first_stage, n_stages; /* slice of the stage array */
  int32_t batch_size, curve_ref_batch; /* curve_ref_batch 0 = no batching curve */
  double curve_ref_gain;
} daris_task_spec;

typedef struct daris_options {
  int32_t window_size;          /* MRET window ws (timing.py:29) */
  int32_t no_staging, no_last, no_prior, no_fixed; /* AblationFlags (scheduler.py:44-58) */
  int32_t hpa;                  /* SchedulerMode.hpa_enabled */
  int32_t placement_insertion;  /* placement_order == "insertion" */
  int32_t edf_on_job_deadline;
  int32_t check_invariants;     /* Simulation._verify_invariants (engine.py:535-551) */
  int32_t stage_migration;      /* extension, off in parity runs: successor stages may
                                   follow their task to a new home context */
} daris_options;

typedef struct daris_stage_ref {
  int32_t task, job, stage, context, stream;
  double started_at, virtual_deadline;
} daris_stage_ref;

typedef struct daris_placement {
  int32_t context;        /* 0 = rejected */
  int32_t migrated_from;  /* 0 = stayed home */
  int32_t n_audits;       /* admission tests run for this job */
  int32_t _pad;
} daris_placement;

typedef struct daris_ledger_t {
  double hp_total, lp_total, lp_active, hp_active;
} daris_ledger_t;

typedef struct daris_audit {
  double time, active_util, job_util, limit;
  int32_t job, task, priority, context, admitted, _pad;
} daris_audit;

/* int fields use -1 for "None"; rate is NaN when absent */
typedef struct daris_log_record {
  double time;
  int32_t kind, task, job, stage, context, stream;
  double rate;
} daris_log_record;

typedef struct daris_response_stats {
  double mean, min, max, p95, p99;
  int64_t count;
} daris_response_stats;

typedef struct daris_report {
  double duration, warmup, jps, dmr_hp, dmr_lp;
  daris_response_stats response_hp, response_lp;
  int64_t released_hp, released_lp, accepted_hp, accepted_lp, rejected_hp, rejected_lp;
  int64_t completed_hp, completed_lp, missed_hp, missed_lp;
} daris_report;

typedef struct daris_trace_entry {
  int32_t task, job, stage;
  int32_t flags;            /* DARIS_TRACE_UNSAMPLED: the stage completes without recording its
                               time into the MRET window (the recorded run had it in flight
                               across a GPU-wide pause); 0 in every reference-parity trace */
  double duration;
} daris_trace_entry;

enum { DARIS_TRACE_UNSAMPLED = 1 };

/* one task of a context's ctx_tasks list, for daris_eval_ledger */
typedef struct daris_ledger_entry {
  double util;           /* TimingTracker.utilization(task) */
  int32_t hp;            /* task priority is HP */
  int32_t active_jobs;   /* TaskState.active_jobs */
} daris_ledger_entry;

/* PriorityKey (scheduler.py:66-73) of one ready stage */
typedef struct daris_ready_key {
  double edf;
  int32_t level, task, job, _pad;
} daris_ready_key;

typedef struct daris_handle daris_handle;

int daris_create(const daris_gpu_config* gpu, const daris_task_spec* tasks, int32_t n_tasks,
                 const daris_stage_spec* stages, int32_t n_stages, const daris_options* opts,
                 daris_handle** out, char* err, size_t errlen);
void daris_destroy(daris_handle* h);
const char* daris_last_error(const daris_handle* h);

int daris_sm_per_context(const daris_gpu_config* gpu, int32_t* out);
int daris_n_tasks(const daris_handle* h, int32_t* out);
int daris_task_ids(const daris_handle* h, int32_t* out);               /* sorted, n_tasks entries */
int daris_task_stage_count(const daris_handle* h, int32_t task_id, int32_t* out);
int daris_task_info(const daris_handle* h, int32_t task_id, double* period, int32_t* n_stages,
                    int32_t* priority);
/* Images per job of a task (TaskSpec batch_size; the JPS accounting unit). */
int daris_task_batch(const daris_handle* h, int32_t task_id, int32_t* batch);

int daris_full_load_sim(daris_handle* h, int32_t task_id, int32_t repetitions, const int32_t* draws,
                        double* out);
int daris_set_full_load(daris_handle* h, const double* per_task);      /* task-id order */
int daris_populate(daris_handle* h);
int daris_home_context(const daris_handle* h, int32_t task_id, int32_t* out);

int daris_release(daris_handle* h, int32_t task_id, double t, int32_t job_id, const double* stage_work,
                  daris_placement* out);
int daris_dispatch(daris_handle* h, int32_t context, int32_t stream, double t, daris_stage_ref* out,
                   int32_t* found);
int daris_complete(daris_handle* h, int32_t job_id, int32_t stage, double t, int32_t* job_done,
                   int32_t* missed);
/* daris_complete with record_sample = 0: the stage completes as in
 * Scheduler.complete_stage but its observed time does not enter the MRET
 * window (timing.py:45-50 not applied). Used by the real-time executor for
 * stages that were in flight across a detected GPU-wide pause, which would
 * otherwise freeze an inflated utilisation until the task's next completion
 * (timing.py:92-114). record_sample = 1 is exactly daris_complete. */
int daris_complete_ex(daris_handle* h, int32_t job_id, int32_t stage, double t, int32_t record_sample,
                      int32_t* job_done, int32_t* missed);
int daris_ready_count(const daris_handle* h, int32_t context, int32_t* out);

/* SM partition layout of the real executor (gpu.py:76-86's ceil_even(OS*SMs/N_c)
 * made physical): the device is a cyclic sequence of `n_units` SM units (on B200:
 * the 28-SM split remainder, then fifteen co-scheduled 8-SM groups); partition k
 * is the run of units between the unit boundaries nearest to k/N_c of the device
 * and `sm_per_context` SMs further (ties to the lower boundary). OS > 1 gives
 * overlapping partitions (each SM in about OS of them), OS = 1 tiles the device.
 * Outputs per context: first unit, number of units, SMs. Pure arithmetic (CPU). */
int daris_partition_layout(int32_t n_contexts, int32_t sm_per_context, const int32_t* unit_sms, int32_t n_units,
                           int32_t* first_unit, int32_t* n_taken, int32_t* sm_count);

int daris_ledger(daris_handle* h, int32_t context, daris_ledger_t* out);
int daris_admission_test(daris_handle* h, int32_t task_id, int32_t job_id, int32_t context, double t,
                         daris_audit* out);
int daris_predicted_finish(daris_handle* h, int32_t task_id, int32_t context, double t, double* out);
int daris_stage_estimate(daris_handle* h, int32_t task_id, int32_t stage, double* out);
int daris_task_estimate(daris_handle* h, int32_t task_id, double* out);
int daris_utilization(daris_handle* h, int32_t task_id, double* out);
int daris_deadline_shares(daris_handle* h, int32_t task_id, double* out);
int daris_record_execution(daris_handle* h, int32_t task_id, int32_t stage, double observed);
int daris_note_job_complete(daris_handle* h, int32_t task_id);

int daris_sim_run(daris_handle* h, double duration, double warmup_frac, const double* phases,
                  int32_t collect_log, daris_report* out);
int daris_trace_run(daris_handle* h, double duration, double warmup_frac, const double* phases,
                    const daris_trace_entry* trace, int64_t n_trace, int32_t collect_log, daris_report* out);

int64_t daris_log_count(const daris_handle* h);
int64_t daris_log_copy(const daris_handle* h, daris_log_record* buf, int64_t cap);
int64_t daris_audit_count(const daris_handle* h);
int64_t daris_audit_copy(const daris_handle* h, daris_audit* buf, int64_t cap);
void daris_log_clear(daris_handle* h);
/* append one record (used by the GPU executor so real runs log like the sim) */
void daris_log_push(daris_handle* h, const daris_log_record* rec);
/* pre-size (and pre-fault) the log and audit buffers so a real-time run never
   reallocates them mid-flight (a multi-MB realloc stalls the dispatch loop) */
void daris_log_reserve(daris_handle* h, int64_t records, int64_t audits);
/* pending admitted work: ready stages summed over contexts */
int daris_ready_total(const daris_handle* h, int32_t* out);

/* Rate model kernels exposed for the unit tests (gpu.py:118-205). widths are
 * ints; out_is_int marks allocations that stayed Python ints (the "fits" branch). */
int daris_water_fill(const int32_t* widths, int32_t n, double capacity, double* out_alloc,
                     int32_t* out_is_int, double* out_level, int32_t* has_level);
int daris_allocate_rates(const daris_gpu_config* gpu, const int32_t* widths, const int32_t* ctx_ids,
                         int32_t n, double* out_alloc, double* out_rates, double* out_scale);
double daris_py_sum(const double* values, const int32_t* is_int, int64_t n);

/* Stateless decision kernels. The stateful handle above runs every decision
 * through these same functions (csrc/core/decide.cpp); the object-level drop-in
 * API (Scheduler / TimingTracker / make_job / next_completion / advance_progress
 * over Python-owned TaskState, Job and ready lists, exactly as the reference's
 * tests drive them) calls them directly. Each replaces one reference expression:
 *   daris_eval_window_peak        ExecutionWindow.peak (timing.py:52-56)
 *   daris_eval_stage_fallback     TimingTracker.stage_estimate, empty window (timing.py:84-86)
 *   daris_eval_utilization        TimingTracker.utilization, uncached value (timing.py:102-107)
 *   daris_eval_deadline_shares    TimingTracker.deadline_shares (timing.py:116-132)
 *   daris_eval_virtual_deadlines  make_job's cumulative stage deadlines (model.py:211-227)
 *   daris_eval_ledger             Scheduler.context_utilization (scheduler.py:157-171)
 *   daris_eval_admission          Scheduler.admission_test (scheduler.py:179-200)
 *   daris_eval_placement          Scheduler.populate_contexts (scheduler.py:131-153)
 *   daris_eval_predicted_finish   Scheduler.predicted_finish (scheduler.py:202-213)
 *   daris_eval_priority_level     Scheduler.priority_key level (scheduler.py:278-284)
 *   daris_eval_pick               Scheduler.dispatch's min() (scheduler.py:289-296)
 *   daris_eval_next_completion    gpu.next_completion (gpu.py:208-226)
 *   daris_eval_advance            gpu.advance_progress, remaining[] updated in place (gpu.py:229-240)
 * Messages of failing calls are readable with daris_eval_last_error (thread-local). */
const char* daris_eval_last_error(void);
int daris_eval_window_peak(const double* samples, int32_t n, double* out);
int daris_eval_stage_fallback(double full_load, double nominal, double nominal_total, double* out);
int daris_eval_utilization(int64_t completed_jobs, double full_load, double task_estimate, double period,
                           double* out);
int daris_eval_deadline_shares(const double* estimates, int32_t n, double deadline, int32_t task_id,
                               double* out_shares);
int daris_eval_virtual_deadlines(double release, double deadline, const double* shares, int32_t n,
                                 double* out_abs_deadline, double* out);
int daris_eval_ledger(const daris_ledger_entry* tasks, int32_t n, daris_ledger_t* out);
int daris_eval_admission(const daris_ledger_t* ledger, double job_util, int32_t hp, int32_t n_streams,
                         double* out_active, double* out_limit, int32_t* out_admitted);
int daris_eval_placement(const double* util, const int32_t* hp, const int32_t* ids, int32_t n, int32_t n_contexts,
                         int32_t insertion_order, int32_t* out_context, int32_t* out_order, double* out_totals);
int daris_eval_predicted_finish(double t, const double* backlog_estimates, int64_t n, int32_t n_streams,
                                double task_estimate, double* out);
int daris_eval_priority_level(int32_t hp, int32_t is_last, int32_t predecessor_missed, int32_t no_last,
                              int32_t no_prior, int32_t no_fixed, int32_t* out);
int daris_eval_pick(const daris_ready_key* keys, int32_t n, int32_t* out_index);
int daris_eval_next_completion(const double* remaining, const double* rates, const int64_t* job_ids,
                               const int64_t* stage_indices, int32_t n, double now, int32_t* out_index,
                               double* out_time);
int daris_eval_advance(double* remaining, const double* rates, const int64_t* job_ids,
                       const int64_t* stage_indices, int32_t n, double dt);

#ifdef __cplusplus
}
#endif
#endif
