/* DARIS real-time GPU executor — C ABI.
 *
 * Replaces the reference engine's device side: the simulated SM partitions
 * (`build_contexts`, `sm_per_context`, gpu.py:81-115) become CUDA green
 * contexts carved out of the B200's 148 SMs (overlapping windows when the
 * oversubscription OS > 1), each with `n_streams` streams; the rate model
 * (`allocate_rates/next_completion/advance_progress`, gpu.py:167-240) becomes
 * real execution of per-stage CUDA graphs, with completions observed through
 * CUDA events; and the DES loop (engine.py:379-531) becomes a wall-clock loop
 * that releases periodic jobs, calls the native dispatcher (daris.h) for
 * admission / migration / dispatch / completion, and launches the stage graph
 * of the dispatched (task, stage) on the (context, stream) slot it got.
 *
 * Times handed to the dispatcher are quantised to multiples of 2^-20 s, so
 * every sum/difference the scheduler forms is exact and a recorded trace
 * replays bit-exactly through the reference.
 */
#ifndef DARIS_EXEC_H
#define DARIS_EXEC_H
#include <stddef.h>
#include <stdint.h>
#include "daris.h"
#ifdef __cplusplus
extern "C" {
#endif

enum daris_partition_mode {
  DARIS_PART_GREEN = 0, /* CUDA green contexts (hard SM partitions) */
  DARIS_PART_SOFT = 1   /* plain streams; partitions only via kernel grid sizing */
};

typedef struct daris_exec_config {
  int32_t device;
  int32_t n_contexts, n_streams;
  int32_t sm_per_context;   /* from daris_sm_per_context() */
  int32_t partition_mode;   /* daris_partition_mode */
  int32_t slots_per_task;   /* buffer sets per task (jobs of one task in flight) */
  int32_t max_tasks, max_stages;
} daris_exec_config;

typedef struct daris_exec_partition {
  int32_t context;          /* 1-based */
  int32_t sm_count;         /* SMs the partition actually owns */
  int32_t first_group, n_groups; /* cyclic window of layout units: unit 0 = the SMs the group split
                                    leaves over (28 on B200), then the co-scheduled groups */
  int32_t green;            /* 1 if a green context backs it */
  int32_t group_size;       /* SMs per co-scheduling group: the largest thread-block cluster
                               a kernel in this partition can launch (8; 2 with DARIS_PART_GROUP=2;
                               1 for a partition of only the split remainder) */
} daris_exec_partition;

/* per-stage execution record (one per completed stage) */
typedef struct daris_stage_trace {
  int32_t task, job, stage, context, stream, slot;
  double start, end;        /* quantised executor time (s) */
  double gpu_start, gpu_end; /* device time (s) of the stage's first / last work on its stream, from
                                timing events (only when DARIS_GPU_TIMING is set; NaN otherwise) */
  int32_t sampled;          /* 1: its time entered the MRET window; 0: it was in flight across a
                               detected GPU-wide pause and completed via daris_complete_ex(.., 0, ..)
                               (replay it with DARIS_TRACE_UNSAMPLED) */
  int32_t _pad;
} daris_stage_trace;

typedef struct daris_exec_stats {
  int64_t graph_launches;   /* stage graphs launched in the run */
  int64_t copies_h2d, copies_d2h, copies_d2d;
  int64_t h2d_bytes, d2h_bytes;
  int64_t slot_waits;       /* jobs that took over a buffer set whose previous job was still on
                               the GPU (ordered behind its last stage by an event wait) */
  int64_t polls;
  double wall_seconds;      /* host wall time of the run incl. drain */
  double release_lag_max;   /* worst delay between a nominal release and its processing */
  double loop_gap_max;      /* longest host gap between two polling passes (host stalls) */
  double progress_gap_max;  /* longest time with stages in flight and no completion observed */
  int64_t stalls;           /* GPU-wide stalls: progress gaps above the stall threshold */
  double first_stall_at;    /* executor time of the first stall (-1 if none) */
  int64_t slot_deferred;    /* stage-0 launches held (stream kept) until a buffer set freed up:
                               more live jobs of one task than it has buffer sets */
  int64_t slot_backlog_max; /* most admitted jobs of one task waiting for a buffer set */
  int64_t unsampled;        /* stages completed without an MRET sample (in flight across a stall) */
} daris_exec_stats;

typedef struct daris_exec daris_exec;

int daris_exec_create(const daris_exec_config* cfg, daris_exec** out, char* err, size_t errlen);
void daris_exec_destroy(daris_exec* ex);
int daris_exec_partition_info(const daris_exec* ex, int32_t context, daris_exec_partition* out);

/* stream of (context, stream) — pass to the kernel launchers while capturing */
int daris_exec_stream(daris_exec* ex, int32_t context, int32_t stream, void** out);

/* graph capture of one stage body on a context's capture stream */
int daris_exec_capture_begin(daris_exec* ex, int32_t context, void** stream_out);
int daris_exec_capture_end(daris_exec* ex, int32_t task, int32_t stage, int32_t context, int32_t slot);
int daris_exec_graph_count(const daris_exec* ex, int64_t* out);
/* Isolated time of one captured stage graph: `reps` back-to-back launches on
 * the partition's stream 0 between CUDA events (after 3 warm launches); the
 * stage's nominal_time (model.py:24-27 StageProfile) on this partition. */
int daris_exec_time_graph(daris_exec* ex, int32_t task, int32_t stage, int32_t context, int32_t slot, int32_t reps,
                          double* out_seconds);

/* per (task, slot) I/O buffers. input: device buffer the first stage reads;
 * output: device buffer the last stage writes. Pools: n_inputs images of
 * in_bytes each, either in pinned host memory (end-to-end mode, H2D each job)
 * or in device memory (resident mode, D2D each job); NULL skips the copy. */
int daris_exec_set_io(daris_exec* ex, int32_t task, int32_t slot, void* dev_input, void* dev_output);
int daris_exec_set_pool(daris_exec* ex, int32_t task, const void* pool, int32_t pool_on_host, int32_t n_inputs,
                        int64_t in_bytes, void* host_out, int64_t out_bytes);

/* Run the periodic workload for `duration` seconds of wall clock on a
 * populated dispatcher. phases[i] = release offset of the i-th task (id
 * order); periods come from the dispatcher's tasks. Metrics cover jobs
 * released in [warmup, duration); in-flight jobs are drained and counted. */
int daris_exec_run(daris_exec* ex, daris_handle* h, double duration, double warmup, const double* phases,
                   int32_t collect_log, daris_report* report, daris_exec_stats* stats);

/* A progress gap (stages in flight, no completion) longer than `seconds`
 * counts as a GPU-wide stall in daris_exec_stats (default 1 ms). An idle B200
 * shows ~1.7 ms whole-GPU pauses every few seconds (tools/freeze_probe.cu), so
 * runs can tell an environmental pause from a scheduling failure. */
int daris_exec_set_stall_threshold(daris_exec* ex, double seconds);
/* (start, length) in executor seconds of every stall of the last run that ended
 * in a completion; returns the number of pairs (copies min(n, cap_pairs)) */
int64_t daris_exec_stall_copy(const daris_exec* ex, double* buf, int64_t cap_pairs);

int64_t daris_exec_trace_count(const daris_exec* ex);
int64_t daris_exec_trace_copy(const daris_exec* ex, daris_stage_trace* buf, int64_t cap);

/* Full-load (AFET) calibration on the real GPU: every (context, stream) slot
 * loops jobs of the tasks in `slot_tasks` (n_contexts*n_streams entries, slot 0
 * is the target) for `seconds`; returns the mean job time of each task id seen
 * in slot 0 position rotations (out[i] for task id i+1, 0 if unseen).
 * task_hp (nullable, indexed by task id - 1): nonzero launches that task's
 * stages on the high-priority streams, as daris_exec_run does for HP tasks, so
 * the baseline is measured under the contention HP stages really see. */
int daris_exec_busy_calibrate(daris_exec* ex, const int32_t* task_stage_counts, int32_t n_tasks,
                              const int32_t* slot_tasks, double seconds, double* out_mean_job_time,
                              const int32_t* task_hp);

const char* daris_exec_last_error(const daris_exec* ex);

/* time quantum used for every executor timestamp (2^-20 s) */
double daris_exec_quantum(void);

#ifdef __cplusplus
}
#endif
#endif
