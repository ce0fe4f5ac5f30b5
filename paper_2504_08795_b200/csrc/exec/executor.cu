// DARIS real-time executor on B200: green-context SM partitions, per-partition
// stream slots, per-(task, stage, partition, buffer-slot) CUDA graphs, and the
// wall-clock release / dispatch / completion loop driving the native
// dispatcher through its C ABI (include/daris.h, include/daris_exec.h).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <sched.h>
#include <sys/resource.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <cerrno>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <queue>
#include <string>
#include <unordered_map>
#include <vector>
#include <deque>
#include <functional>

#include "../../../include/daris_exec.h"

namespace {

constexpr double kQuantum = 1.0 / 1048576.0;  // 2^-20 s
inline double quant(double s) { return std::floor(s / kQuantum + 0.5) * kQuantum; }

struct Driver {
  PFN_cuDeviceGetDevResource_v12040 getDevResource = nullptr;
  PFN_cuDevSmResourceSplitByCount_v12040 split = nullptr;
  PFN_cuDevResourceGenerateDesc_v12040 genDesc = nullptr;
  PFN_cuGreenCtxCreate_v12040 greenCreate = nullptr;
  PFN_cuGreenCtxDestroy_v12040 greenDestroy = nullptr;
  PFN_cuGreenCtxStreamCreate_v12050 greenStream = nullptr;
  PFN_cuDeviceGet_v2000 deviceGet = nullptr;
  PFN_cuStreamWriteValue32_v11070 writeValue32 = nullptr;  // optional: completion flags
  bool ok = false;
};

template <class T>
bool entry(const char* name, T& fn) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    return false;
  fn = reinterpret_cast<T>(p);
  return true;
}

Driver& driver() {
  static Driver d;
  static bool init = false;
  if (!init) {
    init = true;
    d.ok = entry("cuDeviceGetDevResource", d.getDevResource) && entry("cuDevSmResourceSplitByCount", d.split) &&
           entry("cuDevResourceGenerateDesc", d.genDesc) && entry("cuGreenCtxCreate", d.greenCreate) &&
           entry("cuGreenCtxDestroy", d.greenDestroy) && entry("cuGreenCtxStreamCreate", d.greenStream) &&
           entry("cuDeviceGet", d.deviceGet);
    if (!entry("cuStreamWriteValue32", d.writeValue32)) d.writeValue32 = nullptr;
  }
  return d;
}

struct Partition {
  int sm_count = 0, first_group = 0, n_groups = 0, group_size = 0;
  CUgreenCtx green = nullptr;
  std::vector<cudaStream_t> streams;     // low (default) priority: LP stages
  std::vector<cudaStream_t> streams_hi;  // highest priority: HP stages (CTA scheduling preference)
  std::vector<cudaEvent_t> done;
  cudaStream_t capture = nullptr;
};

struct Running {
  bool busy = false;
  bool held = false;  // stage 0 dispatched onto this stream, launch held until its job gets a buffer set
  int task = 0, job = 0, stage = 0, slot = 0;
  double start = 0;
  int ev = -1;  // index of the stage's timing-event pair (DARIS_GPU_TIMING)
  int epoch = 0;  // stall epoch when dispatched: a different one at completion = in flight across a pause
};

struct TaskInfo {
  int id = 0, n_stages = 0, prio = 0, batch = 1;
  double period = 0;
};

}  // namespace

struct daris_exec {
  daris_exec_config cfg{};
  std::vector<Partition> parts;
  // graphs[((task*max_stages + stage)*n_ctx + ctx)*slots + slot]
  std::vector<cudaGraphExec_t> graphs;
  // per (task, slot) I/O
  std::vector<void*> dev_in, dev_out;
  // per task pools
  struct Pool {
    const char* src = nullptr;
    bool on_host = false;
    int n = 0;
    int64_t in_bytes = 0;
    char* host_out = nullptr;
    int64_t out_bytes = 0;
  };
  std::vector<Pool> pools;
  std::vector<cudaEvent_t> slot_free;  // per (task, slot)
  std::vector<cudaEvent_t> in_ready;   // per (task, slot): the job's input copy is done
  std::vector<int> slot_owner;          // job id holding the buffer set, 0 = free
  std::vector<char> slot_handoff;       // holder has launched its last stage: slot_free is recorded, the
                                        // set may pass to the next job behind a GPU event wait
  std::vector<daris_stage_trace> trace;
  std::string err;
  int64_t graph_count = 0;
  double stall_threshold = 1e-3;
  std::vector<double> stall_log;  // (start, length) pairs of the last run's GPU-wide stalls
  // DARIS_EXEC_FLAGS=1: stage completion as a stream memory write of a sequence
  // number into host-mapped memory (one word per (context, stream) slot), polled
  // with a plain load instead of cudaEventQuery
  uint32_t* flags = nullptr;
  CUdeviceptr flags_dev = 0;

  size_t gidx(int task, int stage, int ctx, int slot) const {
    return ((static_cast<size_t>(task - 1) * cfg.max_stages + stage) * cfg.n_contexts + (ctx - 1)) *
               cfg.slots_per_task + slot;
  }
  size_t sidx(int task, int slot) const { return static_cast<size_t>(task - 1) * cfg.slots_per_task + slot; }
};

namespace {

int fail(daris_exec* ex, const std::string& m, int code = DARIS_E_VALUE) {
  if (ex) ex->err = m;
  return code;
}

#define CUDA_TRY(ex, call)                                                                 \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess) return fail(ex, std::string(#call) + ": " + cudaGetErrorString(e_), DARIS_E_INTERNAL); \
  } while (0)

int build_partitions(daris_exec* ex) {
  const daris_exec_config& c = ex->cfg;
  int total_sms = 0;
  cudaDeviceGetAttribute(&total_sms, cudaDevAttrMultiProcessorCount, c.device);
  ex->parts.resize(c.n_contexts);
  bool green = c.partition_mode == DARIS_PART_GREEN;
  Driver& d = driver();
  std::vector<CUdevResource> groups;
  CUdevResource rem;
  std::memset(&rem, 0, sizeof(rem));
  CUdevice dev = 0;
  if (green) {
    if (!d.ok) green = false;
  }
  if (green) {
    d.deviceGet(&dev, c.device);
    CUdevResource all;
    if (d.getDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS) green = false;
    if (green) {
      // Co-scheduled 8-SM groups (the hardware granularity on cc >= 9.0): a kernel
      // in the partition can launch clusters of up to 8 CTAs (split-K through DSMEM).
      // DARIS_PART_GROUP=2 trades that for 2-SM granularity (IGNORE_SM_COSCHEDULING:
      // clusters of 2 only; tools/probe_cluster.cu).
      const char* ge = std::getenv("DARIS_PART_GROUP");
      const bool fine = ge && std::atoi(ge) == 2;
      unsigned n = static_cast<unsigned>(all.sm.smCount);
      groups.resize(n);
      if (d.split(groups.data(), &n, &all, &rem, fine ? CU_DEV_SM_RESOURCE_SPLIT_IGNORE_SM_COSCHEDULING : 0,
                  fine ? 2 : 8) != CUDA_SUCCESS ||
          n == 0)
        green = false;
      groups.resize(n);
    }
  }
  // Layout units: the co-scheduled groups plus, when the split leaves one, the
  // remainder (148 - 15 x 8 = 28 SMs on B200) as one more unit, first in the
  // cyclic order. A green context over groups + remainder exposes all of their
  // SMs to ordinary CTAs, and 8-CTA clusters still co-schedule on its 8-SM
  // groups (tools/probe_mixed_green.cu), so every SM of the device is used.
  struct Unit {
    int index;  // into groups, or -1 = the remainder
    int sms;
  };
  std::vector<Unit> units;
  if (green && rem.sm.smCount > 0) units.push_back({-1, static_cast<int>(rem.sm.smCount)});
  const int G = green ? static_cast<int>(groups.size()) : total_sms / 2;
  const int gsize = green ? static_cast<int>(groups[0].sm.smCount) : 2;
  for (int g = 0; g < G; ++g) units.push_back({g, gsize});
  const int U = static_cast<int>(units.size());
  std::vector<int32_t> unit_sms(U), lay_first(c.n_contexts), lay_taken(c.n_contexts), lay_sms(c.n_contexts);
  for (int u = 0; u < U; ++u) unit_sms[u] = units[u].sms;
  if (daris_partition_layout(c.n_contexts, c.sm_per_context, unit_sms.data(), U, lay_first.data(), lay_taken.data(),
                             lay_sms.data()) != DARIS_OK)
    return fail(ex, "partition layout failed", DARIS_E_INTERNAL);
  for (int k = 0; k < c.n_contexts; ++k) {
    Partition& p = ex->parts[k];
    // the layout rule: daris_partition_layout (include/daris.h, libdaris_core)
    const int u0 = lay_first[k], taken = lay_taken[k], cov = lay_sms[k];
    // the largest cluster its kernels may launch: a co-scheduled group's size if
    // the partition holds one, else 1 (the remainder's SMs are scattered over
    // GPCs, so an 8-CTA cluster may not fit: split-K then reduces through L2)
    bool has_group = false;
    for (int q = 0; q < taken; ++q) has_group |= units[(u0 + q) % U].index >= 0;
    p.group_size = green ? (has_group ? gsize : 1) : total_sms;
    p.n_groups = taken;
    p.first_group = u0;
    p.sm_count = cov;
    if (green) {
      std::vector<CUdevResource> res;
      for (int q = 0; q < taken; ++q) {
        const Unit& un = units[(u0 + q) % U];
        res.push_back(un.index < 0 ? rem : groups[un.index]);
      }
      CUdevResourceDesc desc;
      if (d.genDesc(&desc, res.data(), static_cast<unsigned>(res.size())) != CUDA_SUCCESS ||
          d.greenCreate(&p.green, desc, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS) {
        return fail(ex, "green context creation failed", DARIS_E_INTERNAL);
      }
    }
    int prio_low = 0, prio_high = 0;
    cudaDeviceGetStreamPriorityRange(&prio_low, &prio_high);
    // HP stages run on the highest-priority streams (their CTAs are scheduled first
    // when SMs free up). With grids planned for the per-job share this lifts the C2
    // knee (A/B on one box: 12.2k vs 11.5k inf/s, profiles/r01_bench_hpprio*.json);
    // with partition-sized grids it starved LP stages. DARIS_HP_STREAM_PRIORITY=0: off.
    const char* hp_env = std::getenv("DARIS_HP_STREAM_PRIORITY");
    if (hp_env && std::atoi(hp_env) == 0) prio_high = prio_low;
    const int n_streams = 2 * c.n_streams + 1;  // low + high priority per slot, + capture stream
    for (int s = 0; s < n_streams; ++s) {
      const int prio = (s >= c.n_streams && s < 2 * c.n_streams) ? prio_high : prio_low;
      cudaStream_t st;
      if (p.green) {
        CUstream cs;
        if (d.greenStream(&cs, p.green, CU_STREAM_NON_BLOCKING, prio) != CUDA_SUCCESS)
          return fail(ex, "green stream creation failed", DARIS_E_INTERNAL);
        st = reinterpret_cast<cudaStream_t>(cs);
      } else {
        CUDA_TRY(ex, cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, prio));
      }
      if (s < c.n_streams) p.streams.push_back(st);
      else if (s < 2 * c.n_streams) p.streams_hi.push_back(st);
      else p.capture = st;
    }
    for (int s = 0; s < c.n_streams; ++s) {
      cudaEvent_t e;
      CUDA_TRY(ex, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      p.done.push_back(e);
    }
  }
  if (!green) ex->cfg.partition_mode = DARIS_PART_SOFT;
  return DARIS_OK;
}

struct Acc {
  double warmup;
  long long rel[2] = {0, 0}, acc[2] = {0, 0}, rej[2] = {0, 0}, cmp[2] = {0, 0}, miss[2] = {0, 0};
  std::vector<double> resp[2];
  long long inputs = 0;
};

daris_response_stats stats_of(std::vector<double> v) {
  daris_response_stats s{0, 0, 0, 0, 0, 0};
  if (v.empty()) return s;
  std::sort(v.begin(), v.end());
  const size_t n = v.size();
  double sum = 0, c = 0;  // Neumaier, as CPython's sum
  for (double x : v) {
    const double t = sum + x;
    if (std::fabs(sum) >= std::fabs(x)) c += (sum - t) + x;
    else c += (x - t) + sum;
    sum = t;
  }
  s.mean = (sum + c) / static_cast<double>(n);
  s.min = v.front();
  s.max = v.back();
  s.p95 = v[static_cast<size_t>(std::ceil(0.95 * n)) - 1];
  s.p99 = v[static_cast<size_t>(std::ceil(0.99 * n)) - 1];
  s.count = static_cast<int64_t>(n);
  return s;
}

void push_log(daris_handle* h, double t, int kind, int task = -1, int job = -1, int stage = -1, int ctx = -1,
              int stream = -1, double rate = NAN) {
  daris_log_record r{t, kind, task, job, stage, ctx, stream, rate};
  daris_log_push(h, &r);
}

}  // namespace

extern "C" {

double daris_exec_quantum(void) { return kQuantum; }

int daris_exec_create(const daris_exec_config* cfg, daris_exec** out, char* err, size_t errlen) {
  auto ex = std::make_unique<daris_exec>();
  auto bail = [&](int code) {
    if (err && errlen) {
      std::strncpy(err, ex->err.c_str(), errlen - 1);
      err[errlen - 1] = 0;
    }
    return code;
  };
  if (!cfg || cfg->n_contexts < 1 || cfg->n_streams < 1 || cfg->slots_per_task < 1 || cfg->max_tasks < 1 ||
      cfg->max_stages < 1 || cfg->sm_per_context < 1) {
    ex->err = "invalid executor config";
    return bail(DARIS_E_VALUE);
  }
  ex->cfg = *cfg;
  if (cudaSetDevice(cfg->device) != cudaSuccess || cudaFree(nullptr) != cudaSuccess) {
    ex->err = "no CUDA device";
    return bail(DARIS_E_INTERNAL);
  }
  int rc = build_partitions(ex.get());
  if (rc != DARIS_OK) return bail(rc);
  const size_t ng = static_cast<size_t>(cfg->max_tasks) * cfg->max_stages * cfg->n_contexts * cfg->slots_per_task;
  ex->graphs.assign(ng, nullptr);
  const size_t ns = static_cast<size_t>(cfg->max_tasks) * cfg->slots_per_task;
  ex->dev_in.assign(ns, nullptr);
  ex->dev_out.assign(ns, nullptr);
  ex->slot_owner.assign(ns, 0);
  ex->slot_handoff.assign(ns, 0);
  ex->slot_free.resize(ns);
  ex->in_ready.resize(ns);
  for (auto* v : {&ex->slot_free, &ex->in_ready})
    for (auto& e : *v) {
      if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
        ex->err = "event creation failed";
        return bail(DARIS_E_INTERNAL);
      }
    }
  ex->pools.resize(cfg->max_tasks);
  *out = ex.release();
  return DARIS_OK;
}

void daris_exec_destroy(daris_exec* ex) {
  if (!ex) return;
  cudaDeviceSynchronize();
  for (auto g : ex->graphs)
    if (g) cudaGraphExecDestroy(g);
  for (auto e : ex->slot_free) cudaEventDestroy(e);
  for (auto e : ex->in_ready) cudaEventDestroy(e);
  if (ex->flags) cudaFreeHost(ex->flags);
  for (auto& p : ex->parts) {
    for (auto e : p.done) cudaEventDestroy(e);
    for (auto s : p.streams) cudaStreamDestroy(s);
    for (auto s : p.streams_hi) cudaStreamDestroy(s);
    if (p.capture) cudaStreamDestroy(p.capture);
    if (p.green && driver().greenDestroy) driver().greenDestroy(p.green);
  }
  delete ex;
}

const char* daris_exec_last_error(const daris_exec* ex) { return ex ? ex->err.c_str() : ""; }

int daris_exec_partition_info(const daris_exec* ex, int32_t context, daris_exec_partition* out) {
  if (context < 1 || context > ex->cfg.n_contexts) return DARIS_E_VALUE;
  const Partition& p = ex->parts[context - 1];
  *out = daris_exec_partition{context, p.sm_count, p.first_group, p.n_groups, p.green ? 1 : 0, p.group_size};
  return DARIS_OK;
}

int daris_exec_stream(daris_exec* ex, int32_t context, int32_t stream, void** out) {
  if (context < 1 || context > ex->cfg.n_contexts || stream < 0 || stream >= ex->cfg.n_streams) return DARIS_E_VALUE;
  *out = ex->parts[context - 1].streams[stream];
  return DARIS_OK;
}

int daris_exec_capture_begin(daris_exec* ex, int32_t context, void** stream_out) {
  if (context < 1 || context > ex->cfg.n_contexts) return fail(ex, "bad context");
  cudaStream_t s = ex->parts[context - 1].capture;
  CUDA_TRY(ex, cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  *stream_out = s;
  return DARIS_OK;
}

int daris_exec_capture_end(daris_exec* ex, int32_t task, int32_t stage, int32_t context, int32_t slot) {
  if (context < 1 || context > ex->cfg.n_contexts) return fail(ex, "bad context");
  cudaStream_t s = ex->parts[context - 1].capture;
  cudaGraph_t g = nullptr;
  CUDA_TRY(ex, cudaStreamEndCapture(s, &g));
  if (task < 1 || task > ex->cfg.max_tasks || stage < 0 || stage >= ex->cfg.max_stages || slot < 0 ||
      slot >= ex->cfg.slots_per_task) {
    cudaGraphDestroy(g);
    return fail(ex, "graph key out of range");
  }
  cudaGraphExec_t ge = nullptr;
  cudaError_t e = cudaGraphInstantiate(&ge, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) return fail(ex, std::string("graph instantiate: ") + cudaGetErrorString(e), DARIS_E_INTERNAL);
  cudaGraphExec_t& slotg = ex->graphs[ex->gidx(task, stage, context, slot)];
  if (slotg) cudaGraphExecDestroy(slotg);
  else ex->graph_count++;
  slotg = ge;
  return DARIS_OK;
}

int daris_exec_time_graph(daris_exec* ex, int32_t task, int32_t stage, int32_t context, int32_t slot, int32_t reps,
                          double* out_seconds) {
  if (context < 1 || context > ex->cfg.n_contexts || task < 1 || task > ex->cfg.max_tasks || stage < 0 ||
      stage >= ex->cfg.max_stages || slot < 0 || slot >= ex->cfg.slots_per_task || reps < 1 || !out_seconds)
    return fail(ex, "bad graph key");
  cudaGraphExec_t g = ex->graphs[ex->gidx(task, stage, context, slot)];
  if (!g) return fail(ex, "no graph captured for that key");
  cudaStream_t s = ex->parts[context - 1].streams[0];
  cudaEvent_t e0, e1;
  CUDA_TRY(ex, cudaEventCreate(&e0));
  CUDA_TRY(ex, cudaEventCreate(&e1));
  for (int i = 0; i < 3; ++i) CUDA_TRY(ex, cudaGraphLaunch(g, s));  // warm (L2, icache, TMA descriptors)
  CUDA_TRY(ex, cudaEventRecord(e0, s));
  for (int i = 0; i < reps; ++i) CUDA_TRY(ex, cudaGraphLaunch(g, s));
  CUDA_TRY(ex, cudaEventRecord(e1, s));
  CUDA_TRY(ex, cudaEventSynchronize(e1));
  float ms = 0.f;
  CUDA_TRY(ex, cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  *out_seconds = static_cast<double>(ms) * 1e-3 / reps;
  return DARIS_OK;
}

int daris_exec_graph_count(const daris_exec* ex, int64_t* out) {
  *out = ex->graph_count;
  return DARIS_OK;
}

int daris_exec_set_io(daris_exec* ex, int32_t task, int32_t slot, void* dev_input, void* dev_output) {
  if (task < 1 || task > ex->cfg.max_tasks || slot < 0 || slot >= ex->cfg.slots_per_task) return fail(ex, "bad key");
  ex->dev_in[ex->sidx(task, slot)] = dev_input;
  ex->dev_out[ex->sidx(task, slot)] = dev_output;
  return DARIS_OK;
}

int daris_exec_set_pool(daris_exec* ex, int32_t task, const void* pool, int32_t pool_on_host, int32_t n_inputs,
                        int64_t in_bytes, void* host_out, int64_t out_bytes) {
  if (task < 1 || task > ex->cfg.max_tasks) return fail(ex, "bad task");
  auto& p = ex->pools[task - 1];
  p.src = static_cast<const char*>(pool);
  p.on_host = pool_on_host != 0;
  p.n = n_inputs;
  p.in_bytes = in_bytes;
  p.host_out = static_cast<char*>(host_out);
  p.out_bytes = out_bytes;
  return DARIS_OK;
}

int64_t daris_exec_stall_copy(const daris_exec* ex, double* buf, int64_t cap_pairs) {
  const int64_t n = static_cast<int64_t>(ex->stall_log.size() / 2);
  if (buf) std::memcpy(buf, ex->stall_log.data(), sizeof(double) * 2 * static_cast<size_t>(std::min(n, cap_pairs)));
  return n;
}

int daris_exec_set_stall_threshold(daris_exec* ex, double seconds) {
  if (!(seconds > 0)) return fail(ex, "stall threshold must be positive");
  ex->stall_threshold = seconds;
  return DARIS_OK;
}

int64_t daris_exec_trace_count(const daris_exec* ex) { return static_cast<int64_t>(ex->trace.size()); }

int64_t daris_exec_trace_copy(const daris_exec* ex, daris_stage_trace* buf, int64_t cap) {
  const int64_t n = std::min<int64_t>(cap, static_cast<int64_t>(ex->trace.size()));
  std::memcpy(buf, ex->trace.data(), static_cast<size_t>(n) * sizeof(daris_stage_trace));
  return n;
}

// The dispatcher thread runs the wall-clock loop at the highest CFS priority
// (nice -20 for this thread when the process may, e.g. as root on the GPU box):
// a preempted poller shows up directly as stage-dispatch lag and HP deadline
// misses at sub-millisecond periods. Not SCHED_FIFO: a busy-polling real-time
// thread exhausts the kernel's RT budget (950 ms per 1 s) and is then throttled
// for 50 ms — measured as 50.4 ms whole-schedule stalls. Restored on exit;
// DARIS_EXEC_NICE=0 disables.
struct NiceGuard {
  int old = 0;
  bool set = false;
  pid_t tid = 0;
  NiceGuard() {
    const char* e = std::getenv("DARIS_EXEC_NICE");
    if (e && std::atoi(e) == 0) return;
    tid = static_cast<pid_t>(syscall(SYS_gettid));
    errno = 0;
    old = getpriority(PRIO_PROCESS, static_cast<id_t>(tid));
    if (errno != 0) return;
    set = setpriority(PRIO_PROCESS, static_cast<id_t>(tid), -20) == 0;
  }
  ~NiceGuard() {
    if (set) setpriority(PRIO_PROCESS, static_cast<id_t>(tid), old);
  }
};

int daris_exec_run(daris_exec* ex, daris_handle* h, double duration, double warmup, const double* phases,
                   int32_t collect_log, daris_report* report, daris_exec_stats* stats) {
  using clock = std::chrono::steady_clock;
  NiceGuard loop_priority;
  // Bumped when a GPU-wide stall is detected and again when it ends: a stage
  // whose dispatch and completion epochs differ was in flight across the pause,
  // and its time is not an execution-time sample (daris_complete_ex).
  int stall_epoch = 0;
  const daris_exec_config& c = ex->cfg;
  int32_t n_tasks = 0;
  daris_n_tasks(h, &n_tasks);
  if (n_tasks > c.max_tasks) return fail(ex, "more tasks than the executor was sized for");
  std::vector<int32_t> ids(n_tasks);
  daris_task_ids(h, ids.data());
  std::vector<TaskInfo> info(n_tasks + 1);
  for (int i = 0; i < n_tasks; ++i) {
    TaskInfo& t = info[ids[i]];
    t.id = ids[i];
    daris_task_info(h, t.id, &t.period, &t.n_stages, &t.prio);
    daris_task_batch(h, t.id, &t.batch);
    if (t.n_stages > c.max_stages) return fail(ex, "task has more stages than the executor supports");
  }
  (void)collect_log;
  // every graph the run may need must exist: HP tasks in their home context, LP anywhere
  for (int i = 0; i < n_tasks; ++i) {
    const TaskInfo& t = info[ids[i]];
    int32_t home = 0;
    daris_home_context(h, t.id, &home);
    for (int s = 0; s < t.n_stages; ++s)
      for (int k = 1; k <= c.n_contexts; ++k) {
        if (t.prio == DARIS_HP && k != home) continue;
        for (int q = 0; q < c.slots_per_task; ++q)
          if (!ex->graphs[ex->gidx(t.id, s, k, q)])
            return fail(ex, "missing stage graph for task " + std::to_string(t.id) + " stage " + std::to_string(s) +
                                " context " + std::to_string(k));
      }
  }
  ex->trace.clear();
  ex->stall_log.clear();
  // every buffer set is idle between runs (each run ends with a device sync)
  std::fill(ex->slot_owner.begin(), ex->slot_owner.end(), 0);
  std::fill(ex->slot_handoff.begin(), ex->slot_handoff.end(), 0);
  daris_exec_stats st{};
  Acc acc;
  acc.warmup = warmup;

  using Rel = std::pair<double, int>;
  std::priority_queue<Rel, std::vector<Rel>, std::greater<Rel>> heap;
  std::vector<double> phase(n_tasks + 1), period(n_tasks + 1);
  std::vector<long long> rel_idx(n_tasks + 1, 0), seq(n_tasks + 1, 0);
  for (int i = 0; i < n_tasks; ++i) {
    const int id = ids[i];
    phase[id] = quant(phases[i]);
    period[id] = info[id].period;  // Python quantises periods before creating the handle
    if (phase[id] < duration) heap.push({phase[id], id});
  }
  // Size every growing buffer for the whole run up front (and fault its pages
  // in now): a multi-MB vector reallocation inside the loop stalls dispatch
  // for ~1 ms and shows up as a burst of deadline misses.
  long long expect_jobs = 0;
  int max_st = 1;
  for (int i = 0; i < n_tasks; ++i) {
    const TaskInfo& t = info[ids[i]];
    if (t.period > 0) expect_jobs += static_cast<long long>(std::ceil(duration / t.period)) + 1;
    max_st = std::max(max_st, t.n_stages);
  }
  expect_jobs = expect_jobs + expect_jobs / 4 + 64;
  daris_log_reserve(h, expect_jobs * (3 + 2 * max_st) + 16, expect_jobs * (c.n_contexts + 1));
  {
    const size_t keep = ex->trace.size();
    ex->trace.resize(static_cast<size_t>(expect_jobs * max_st));
    ex->trace.resize(keep);
  }
  for (int k = 0; k < 2; ++k) {
    acc.resp[k].resize(static_cast<size_t>(expect_jobs));
    acc.resp[k].clear();
  }
  // optional device-side stage timing: a (begin, end) timing-event pair per launch
  const bool gpu_timing = std::getenv("DARIS_GPU_TIMING") != nullptr;
  std::vector<cudaEvent_t> tev;
  cudaEvent_t tref = nullptr;
  int tev_next = 0;
  if (gpu_timing) {
    tev.resize(static_cast<size_t>(2 * expect_jobs * max_st));
    for (auto& e : tev) CUDA_TRY(ex, cudaEventCreate(&e));
    CUDA_TRY(ex, cudaEventCreate(&tref));
  }
  std::unordered_map<int, int> job_slot;     // job -> buffer slot
  std::unordered_map<int, double> job_rel;   // job -> release time
  std::unordered_map<int, int> job_seq;      // job -> per-task sequence number
  job_slot.reserve(1024);
  job_rel.reserve(1024);
  job_seq.reserve(1024);
  std::vector<std::vector<Running>> run(c.n_contexts, std::vector<Running>(c.n_streams));
  int job_counter = 0;
  const char* fe = std::getenv("DARIS_EXEC_FLAGS");
  const bool use_flags = fe && fe[0] == '1' && driver().writeValue32;
  std::vector<uint32_t> flag_seq(static_cast<size_t>(c.n_contexts * c.n_streams), 0);
  if (use_flags) {
    if (!ex->flags) {
      void* hp = nullptr;
      CUDA_TRY(ex, cudaHostAlloc(&hp, flag_seq.size() * sizeof(uint32_t), cudaHostAllocMapped | cudaHostAllocPortable));
      ex->flags = static_cast<uint32_t*>(hp);
      void* dp = nullptr;
      CUDA_TRY(ex, cudaHostGetDevicePointer(&dp, hp, 0));
      ex->flags_dev = reinterpret_cast<CUdeviceptr>(dp);
    }
    for (size_t i = 0; i < flag_seq.size(); ++i) flag_seq[i] = ex->flags[i];
  }
  int in_flight = 0;

  // A job's input (one image or batch from the task's pool) is copied into its
  // buffer set when the job is admitted — the moment its data exists — on a
  // copy stream per context, so the transfer overlaps the job's wait for a
  // stream slot; stage 0 then waits on the copy's event on the GPU.
  std::vector<cudaStream_t> copy_streams(c.n_contexts, nullptr);
  {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    for (auto& cs : copy_streams) CUDA_TRY(ex, cudaStreamCreateWithPriority(&cs, cudaStreamNonBlocking, hi));
  }
  struct StreamsGuard {
    std::vector<cudaStream_t>& v;
    ~StreamsGuard() {
      cudaDeviceSynchronize();
      for (auto cs : v)
        if (cs) cudaStreamDestroy(cs);
    }
  } copy_guard{copy_streams};
  std::unordered_map<int, int> staged_in;  // admitted jobs whose input copy is issued (stage 0 not yet launched)
  staged_in.reserve(1024);
  const char* sie = std::getenv("DARIS_STAGE_INPUT");  // 0: copy at stage-0 dispatch on the stage's stream
  const bool input_at_admission = !(sie && sie[0] == '0');
  // Buffer sets (activations, split-K workspace and counters, input / output)
  // are owned by one job at a time, tracked here on the host. A set passes to
  // the next job of its task only once the holder has LAUNCHED its last stage
  // (slot_free recorded after it: the new job's first GPU work waits on that
  // event) or has completed. A job admitted while every set of its task is
  // held waits in a per-task FIFO with no input staged; if its stage 0 is
  // dispatched first, the launch is held on the stream it was given until a
  // set frees up (the stage's time includes the wait, as a busy stream would).
  std::vector<std::deque<int>> slot_queue(n_tasks + 1);
  std::unordered_map<int, int> job_ctx;       // job -> context it was admitted into (copy stream)
  std::unordered_map<int, char> job_waits;    // job took over a set still in use on the GPU
  std::deque<std::pair<int, int>> held;       // (context, stream) of held stage-0 launches, FIFO
  job_ctx.reserve(1024);
  job_waits.reserve(1024);
  int n_held = 0;
  auto acquire_slot = [&](int task) -> std::pair<int, bool> {  // (slot, needs GPU wait) or (-1, _)
    for (int q = 0; q < c.slots_per_task; ++q)
      if (ex->slot_owner[ex->sidx(task, q)] == 0) return {q, false};
    for (int q = 0; q < c.slots_per_task; ++q)
      if (ex->slot_handoff[ex->sidx(task, q)]) return {q, true};
    return {-1, false};
  };
  auto stage_input = [&](int task, int job) -> int {
    if (!input_at_admission) return DARIS_OK;
    const auto& pool = ex->pools[task - 1];
    const size_t si = ex->sidx(task, job_slot[job]);
    if (!(pool.src && pool.n > 0 && ex->dev_in[si])) return DARIS_OK;
    cudaStream_t cs = copy_streams[job_ctx[job] - 1];
    if (job_waits[job]) CUDA_TRY(ex, cudaStreamWaitEvent(cs, ex->slot_free[si], 0));
    const char* src = pool.src + static_cast<int64_t>(job_seq[job] % pool.n) * pool.in_bytes;
    CUDA_TRY(ex, cudaMemcpyAsync(ex->dev_in[si], src, static_cast<size_t>(pool.in_bytes),
                                 pool.on_host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, cs));
    CUDA_TRY(ex, cudaEventRecord(ex->in_ready[si], cs));
    staged_in[job] = 1;
    if (pool.on_host) {
      st.copies_h2d++;
      st.h2d_bytes += pool.in_bytes;
    } else {
      st.copies_d2d++;
    }
    return DARIS_OK;
  };
  // give `job` buffer set `q`: claim it and stage the job's input
  auto assign_slot = [&](int task, int job, std::pair<int, bool> got) -> int {
    const size_t si = ex->sidx(task, got.first);
    ex->slot_owner[si] = job;
    ex->slot_handoff[si] = 0;
    job_slot[job] = got.first;
    job_waits[job] = got.second ? 1 : 0;
    if (got.second) st.slot_waits++;
    return stage_input(task, job);
  };
  std::function<int(const daris_stage_ref&)> launch;
  std::vector<std::vector<daris_stage_ref>> held_ref(c.n_contexts, std::vector<daris_stage_ref>(c.n_streams));
  // a set of `task` may have freed up: serve its FIFO, then any held stage-0 launches
  auto serve_slot_queue = [&](int task) -> int {
    auto& qd = slot_queue[task];
    while (!qd.empty()) {
      const auto got = acquire_slot(task);
      if (got.first < 0) break;
      const int job = qd.front();
      qd.pop_front();
      const int rc = assign_slot(task, job, got);
      if (rc != DARIS_OK) return rc;
    }
    for (;;) {  // launch (FIFO) every held stage 0 whose job now has a set; launch may recurse
      auto it = std::find_if(held.begin(), held.end(), [&](const std::pair<int, int>& cs) {
        const daris_stage_ref& r = held_ref[cs.first - 1][cs.second];
        auto js = job_slot.find(r.job);
        return r.task == task && js != job_slot.end() && js->second >= 0;
      });
      if (it == held.end()) break;
      const daris_stage_ref r = held_ref[it->first - 1][it->second];
      run[it->first - 1][it->second].held = false;
      held.erase(it);
      n_held--;
      const int rc = launch(r);
      if (rc != DARIS_OK) return rc;
    }
    return DARIS_OK;
  };
  launch = [&](const daris_stage_ref& r) -> int {
    Partition& p = ex->parts[r.context - 1];
    const TaskInfo& t = info[r.task];
    cudaStream_t s = (t.prio == DARIS_HP ? p.streams_hi : p.streams)[r.stream];
    Running& rr = run[r.context - 1][r.stream];
    const bool was_held = rr.busy && rr.held;  // a held stage-0 launch released now: keeps its dispatch epoch
    if (r.stage == 0 && job_slot[r.job] < 0) {  // no buffer set yet: hold the launch on this stream
      rr.busy = true;
      rr.held = true;
      rr.task = r.task;
      rr.job = r.job;
      rr.stage = r.stage;
      rr.slot = -1;
      rr.start = r.started_at;
      rr.ev = -1;
      rr.epoch = stall_epoch;
      held_ref[r.context - 1][r.stream] = r;
      held.push_back({r.context, r.stream});
      n_held++;
      st.slot_deferred++;
      return DARIS_OK;
    }
    const int slot = job_slot[r.job];
    const size_t si = ex->sidx(r.task, slot);
    if (r.stage == 0) {
      if (staged_in.count(r.job)) {
        CUDA_TRY(ex, cudaStreamWaitEvent(s, ex->in_ready[si], 0));  // orders behind slot_free too
        staged_in.erase(r.job);
      } else {
        if (job_waits[r.job]) CUDA_TRY(ex, cudaStreamWaitEvent(s, ex->slot_free[si], 0));
        const auto& pool = ex->pools[r.task - 1];
        if (!input_at_admission && pool.src && pool.n > 0 && ex->dev_in[si]) {
          const char* src = pool.src + static_cast<int64_t>(job_seq[r.job] % pool.n) * pool.in_bytes;
          CUDA_TRY(ex, cudaMemcpyAsync(ex->dev_in[si], src, static_cast<size_t>(pool.in_bytes),
                                       pool.on_host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, s));
          if (pool.on_host) {
            st.copies_h2d++;
            st.h2d_bytes += pool.in_bytes;
          } else {
            st.copies_d2d++;
          }
        }
      }
    }
    cudaGraphExec_t g = ex->graphs[ex->gidx(r.task, r.stage, r.context, slot)];
    if (!g) return fail(ex, "no graph for dispatched stage", DARIS_E_INTERNAL);
    int ev = -1;
    if (gpu_timing && tev_next + 2 <= static_cast<int>(tev.size())) {
      ev = tev_next;
      tev_next += 2;
      CUDA_TRY(ex, cudaEventRecord(tev[ev], s));
    }
    CUDA_TRY(ex, cudaGraphLaunch(g, s));
    if (ev >= 0) CUDA_TRY(ex, cudaEventRecord(tev[ev + 1], s));
    st.graph_launches++;
    if (use_flags) {
      const size_t fi = static_cast<size_t>((r.context - 1) * c.n_streams + r.stream);
      if (driver().writeValue32(reinterpret_cast<CUstream>(s), ex->flags_dev + fi * sizeof(uint32_t), ++flag_seq[fi],
                                CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS)
        return fail(ex, "cuStreamWriteValue32 failed", DARIS_E_INTERNAL);
    } else {
      CUDA_TRY(ex, cudaEventRecord(p.done[r.stream], s));
    }
    rr.busy = true;
    rr.held = false;
    rr.task = r.task;
    rr.job = r.job;
    rr.stage = r.stage;
    rr.slot = slot;
    rr.start = r.started_at;
    rr.ev = ev;
    if (!was_held) rr.epoch = stall_epoch;
    in_flight++;
    if (r.stage == t.n_stages - 1) {
      const auto& pool = ex->pools[r.task - 1];
      if (pool.host_out && pool.out_bytes > 0 && ex->dev_out[si]) {
        CUDA_TRY(ex, cudaMemcpyAsync(pool.host_out, ex->dev_out[si], static_cast<size_t>(pool.out_bytes),
                                     cudaMemcpyDeviceToHost, s));
        st.copies_d2h++;
        st.d2h_bytes += pool.out_bytes;
      }
      CUDA_TRY(ex, cudaEventRecord(ex->slot_free[si], s));
      ex->slot_handoff[si] = 1;  // the set may now pass on behind slot_free
      if (!slot_queue[r.task].empty()) return serve_slot_queue(r.task);
    }
    return DARIS_OK;
  };

  int status = DARIS_OK;
  auto refill = [&](double t) -> int {
    for (int k = 1; k <= c.n_contexts; ++k) {
      for (int s = 0; s < c.n_streams; ++s) {
        if (run[k - 1][s].busy) continue;
        daris_stage_ref r;
        int32_t found = 0;
        int rc = daris_dispatch(h, k, s, t, &r, &found);
        if (rc != DARIS_OK) return fail(ex, std::string("dispatch: ") + daris_last_error(h), rc);
        if (!found) break;  // this context has nothing ready
        push_log(h, t, DARIS_LOG_STAGE_START, r.task, r.job, r.stage, k, s, 1.0);
        rc = launch(r);
        if (rc != DARIS_OK) return rc;
      }
    }
    return DARIS_OK;
  };

  const auto t0 = clock::now();
  if (gpu_timing) CUDA_TRY(ex, cudaEventRecord(tref, ex->parts[0].streams[0]));
  auto elapsed = [&]() { return std::chrono::duration<double>(clock::now() - t0).count(); };
  struct Done {
    int ctx, stream, job, stage;
  };
  std::vector<Done> done;
  double last_pass = 0.0;
  double last_progress = 0.0;  // last completion observed, or last moment nothing was in flight
  bool in_stall = false;
  st.first_stall_at = -1.0;
  for (;;) {
    const double raw_now = elapsed();
    if (raw_now - last_pass > st.loop_gap_max) st.loop_gap_max = raw_now - last_pass;
    last_pass = raw_now;
    if (in_flight == 0) {
      last_progress = raw_now;
      in_stall = false;
    } else {
      const double gap = raw_now - last_progress;
      if (gap > st.progress_gap_max) st.progress_gap_max = gap;
      if (gap > ex->stall_threshold && !in_stall) {
        in_stall = true;
        stall_epoch++;
        st.stalls++;
        if (st.first_stall_at < 0) st.first_stall_at = raw_now - gap;
      }
    }
    const double now = quant(raw_now);
    bool progressed = false;
    // 1) due releases, in (time, task) order, each at its nominal instant
    while (!heap.empty() && heap.top().first <= now) {
      const Rel rel = heap.top();
      heap.pop();
      const int tid = rel.second;
      const double tr = rel.first;
      st.release_lag_max = std::max(st.release_lag_max, now - tr);
      job_counter += 1;
      daris_placement pl;
      int rc = daris_release(h, tid, tr, job_counter, nullptr, &pl);
      if (rc != DARIS_OK) {
        status = fail(ex, std::string("release: ") + daris_last_error(h), rc);
        break;
      }
      push_log(h, tr, DARIS_LOG_RELEASE, tid, job_counter);
      const int hp = info[tid].prio == DARIS_HP ? 0 : 1;
      if (tr >= acc.warmup) {
        acc.rel[hp]++;
        if (pl.context) acc.acc[hp]++;
        else acc.rej[hp]++;
      }
      if (pl.context == 0) {
        push_log(h, tr, DARIS_LOG_REJECT, tid, job_counter);
      } else {
        push_log(h, tr, DARIS_LOG_ADMIT, tid, job_counter, -1, pl.context);
        job_seq[job_counter] = static_cast<int>(seq[tid]);
        job_rel[job_counter] = tr;
        job_ctx[job_counter] = pl.context;
        job_slot[job_counter] = -1;
        const auto got = slot_queue[tid].empty() ? acquire_slot(tid) : std::make_pair(-1, false);
        if (got.first >= 0) {
          status = assign_slot(tid, job_counter, got);
          if (status != DARIS_OK) break;
        } else {
          slot_queue[tid].push_back(job_counter);
          st.slot_backlog_max = std::max<int64_t>(st.slot_backlog_max, static_cast<int64_t>(slot_queue[tid].size()));
        }
      }
      seq[tid] += 1;
      rel_idx[tid] += 1;
      const double next = phase[tid] + static_cast<double>(rel_idx[tid]) * period[tid];
      if (next < duration) heap.push({next, tid});
      status = refill(tr);
      if (status != DARIS_OK) break;
      progressed = true;
    }
    if (status != DARIS_OK) break;
    // 2) completions observed now, in (job, stage) order
    done.clear();
    for (int k = 0; k < c.n_contexts; ++k)
      for (int s = 0; s < c.n_streams; ++s) {
        Running& rr = run[k][s];
        if (!rr.busy || rr.held) continue;
        st.polls++;
        cudaError_t q;
        if (use_flags) {
          const size_t fi = static_cast<size_t>(k * c.n_streams + s);
          q = *reinterpret_cast<volatile uint32_t*>(ex->flags + fi) == flag_seq[fi] ? cudaSuccess : cudaErrorNotReady;
          // a faulted stage never writes its flag: surface the error during a stall
          if (q != cudaSuccess && in_stall) {
            cudaError_t e = cudaStreamQuery(run[k][s].task && info[run[k][s].task].prio == DARIS_HP
                                                ? ex->parts[k].streams_hi[s] : ex->parts[k].streams[s]);
            if (e != cudaSuccess && e != cudaErrorNotReady) q = e;
          }
        } else {
          q = cudaEventQuery(ex->parts[k].done[s]);
        }
        if (q == cudaSuccess) {
          done.push_back({k + 1, s, rr.job, rr.stage});
          if (in_stall) {
            ex->stall_log.push_back(last_progress);
            ex->stall_log.push_back(raw_now - last_progress);
            stall_epoch++;
          }
          last_progress = raw_now;
          in_stall = false;
        }
        else if (q != cudaErrorNotReady) {
          status = fail(ex, std::string("stage failed on the GPU: ") + cudaGetErrorString(q), DARIS_E_INTERNAL);
          break;
        }
      }
    if (status != DARIS_OK) break;
    std::sort(done.begin(), done.end(), [](const Done& a, const Done& b) {
      return a.job != b.job ? a.job < b.job : a.stage < b.stage;
    });
    for (const Done& d : done) {
      Running& rr = run[d.ctx - 1][d.stream];
      double t = now;
      if (t <= rr.start) t = rr.start + kQuantum;  // a stage always takes at least one quantum
      if (t > duration) {
        // past the horizon the reference's event loop has ended (SIM_END at
        // `duration`, engine.py:508-531): the stage drains on the GPU but is
        // neither logged, counted nor followed by another dispatch; its
        // duration stays in the trace so a replay also finishes it late
        ex->trace.push_back(daris_stage_trace{rr.task, rr.job, rr.stage, d.ctx, d.stream, rr.slot, rr.start, t,
                                              static_cast<double>(rr.ev), NAN, rr.epoch == stall_epoch ? 1 : 0, 0});
        rr.busy = false;
        in_flight--;
        progressed = true;
        continue;
      }
      int32_t job_done = 0, missed = 0;
      const int32_t sampled = rr.epoch == stall_epoch ? 1 : 0;
      if (!sampled) st.unsampled++;
      int rc = daris_complete_ex(h, d.job, d.stage, t, sampled, &job_done, &missed);
      if (rc != DARIS_OK) {
        status = fail(ex, std::string("complete: ") + daris_last_error(h), rc);
        break;
      }
      ex->trace.push_back(daris_stage_trace{rr.task, rr.job, rr.stage, d.ctx, d.stream, rr.slot, rr.start, t,
                                            static_cast<double>(rr.ev), NAN, sampled, 0});
      push_log(h, t, DARIS_LOG_STAGE_COMPLETE, rr.task, rr.job, rr.stage, d.ctx, d.stream, 1.0);
      rr.busy = false;
      in_flight--;
      if (job_done) {
        push_log(h, t, DARIS_LOG_JOB_COMPLETE, rr.task, rr.job, -1, d.ctx);
        const size_t si_done = ex->sidx(rr.task, rr.slot);
        if (ex->slot_owner[si_done] == rr.job) {  // not yet handed to a later job
          ex->slot_owner[si_done] = 0;
          ex->slot_handoff[si_done] = 0;
        }
        const double released = job_rel[rr.job];
        if (released >= acc.warmup) {
          const int hp = info[rr.task].prio == DARIS_HP ? 0 : 1;
          acc.cmp[hp]++;
          acc.inputs += info[rr.task].batch;  // JPS counts images (engine.py:153-220)
          acc.resp[hp].push_back(t - released);
          if (missed) acc.miss[hp]++;
        }
        job_slot.erase(rr.job);
        job_rel.erase(rr.job);
        job_seq.erase(rr.job);
        job_ctx.erase(rr.job);
        job_waits.erase(rr.job);
        if (!slot_queue[rr.task].empty()) {
          status = serve_slot_queue(rr.task);
          if (status != DARIS_OK) break;
        }
      }
      status = refill(t);
      if (status != DARIS_OK) break;
      progressed = true;
    }
    if (status != DARIS_OK) break;
    if (in_flight == 0 && n_held > 0 && now <= duration) {
      // held stage-0 launches occupy streams while the jobs holding their task's
      // buffer sets have nothing on the GPU: none of them can ever progress
      status = fail(ex, "buffer sets exhausted: " + std::to_string(n_held) +
                            " stage-0 launches wait for a buffer set while no stage is in flight "
                            "(more live jobs of a task than its buffer slots; raise slots)", DARIS_E_INTERNAL);
      break;
    }
    if (heap.empty() && in_flight == 0) {
      if (now > duration) break;
      int32_t ready = 0;
      daris_ready_total(h, &ready);
      if (ready == 0) break;
      status = refill(now);  // (cannot happen with free streams, kept for safety)
      if (status != DARIS_OK) break;
    }
    (void)progressed;
  }
  if (status != DARIS_OK) {
    cudaDeviceSynchronize();
    return status;
  }
  cudaDeviceSynchronize();
  for (auto& tr : ex->trace) {
    const int ev = std::isnan(tr.gpu_start) ? -1 : static_cast<int>(tr.gpu_start);
    tr.gpu_start = tr.gpu_end = NAN;
    if (gpu_timing && ev >= 0) {
      float a = 0, b = 0;
      if (cudaEventElapsedTime(&a, tref, tev[ev]) == cudaSuccess &&
          cudaEventElapsedTime(&b, tref, tev[ev + 1]) == cudaSuccess) {
        tr.gpu_start = a * 1e-3;
        tr.gpu_end = b * 1e-3;
      }
    }
  }
  for (auto e : tev) cudaEventDestroy(e);
  if (tref) cudaEventDestroy(tref);
  push_log(h, duration, DARIS_LOG_SIM_END);
  st.wall_seconds = elapsed();

  daris_report r{};
  r.duration = duration;
  r.warmup = warmup;
  const double window = duration - warmup;
  r.jps = window > 0 ? static_cast<double>(acc.inputs) / window : 0.0;
  r.dmr_hp = acc.acc[0] ? static_cast<double>(acc.miss[0]) / acc.acc[0] : 0.0;
  r.dmr_lp = acc.acc[1] ? static_cast<double>(acc.miss[1]) / acc.acc[1] : 0.0;
  r.response_hp = stats_of(acc.resp[0]);
  r.response_lp = stats_of(acc.resp[1]);
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
  if (report) *report = r;
  if (stats) *stats = st;
  return DARIS_OK;
}

int daris_exec_busy_calibrate(daris_exec* ex, const int32_t* task_stage_counts, int32_t n_tasks,
                              const int32_t* slot_tasks, double seconds, double* out_mean_job_time,
                              const int32_t* task_hp) {
  using clock = std::chrono::steady_clock;
  const daris_exec_config& c = ex->cfg;
  const int n_slots = c.n_contexts * c.n_streams;
  struct Loop {
    int task, stage, ctx, stream, slot;
    double job_start;
  };
  std::vector<Loop> loops(n_slots);
  const auto t0 = clock::now();
  auto now = [&]() { return std::chrono::duration<double>(clock::now() - t0).count(); };
  // every concurrently looping copy of a task needs its own buffer set: the
  // k-th stream running task t uses buffer slot k (stage programs and split-K
  // scratch belong to a buffer set and must never run twice at once)
  std::vector<int> uses(static_cast<size_t>(n_tasks) + 1, 0);
  for (int s = 0; s < n_slots; ++s) {
    const int task = slot_tasks[s];
    if (task < 1 || task > n_tasks) return fail(ex, "bad calibration task");
    const int slot = uses[task]++;
    if (slot >= c.slots_per_task)
      return fail(ex, "calibration runs task " + std::to_string(task) + " on more streams than it has buffer slots");
    loops[s] = Loop{task, 0, s / c.n_streams + 1, s % c.n_streams, slot, 0.0};
  }
  auto go = [&](Loop& l) -> int {
    Partition& p = ex->parts[l.ctx - 1];
    cudaGraphExec_t g = ex->graphs[ex->gidx(l.task, l.stage, l.ctx, l.slot)];
    if (!g) return fail(ex, "calibration needs graphs for every task in every context");
    // the stream class daris_exec_run launches this task's stages on (HP: high priority)
    cudaStream_t strm = (task_hp && task_hp[l.task - 1] ? p.streams_hi : p.streams)[l.stream];
    CUDA_TRY(ex, cudaGraphLaunch(g, strm));
    CUDA_TRY(ex, cudaEventRecord(p.done[l.stream], strm));
    return DARIS_OK;
  };
  for (auto& l : loops) {
    l.job_start = now();
    int rc = go(l);
    if (rc) return rc;
  }
  double sum = 0;
  long long jobs = 0;
  while (now() < seconds || jobs == 0) {
    for (int s = 0; s < n_slots; ++s) {
      Loop& l = loops[s];
      cudaError_t q = cudaEventQuery(ex->parts[l.ctx - 1].done[l.stream]);
      if (q == cudaErrorNotReady) continue;
      if (q != cudaSuccess) return fail(ex, cudaGetErrorString(q), DARIS_E_INTERNAL);
      l.stage += 1;
      if (l.stage == task_stage_counts[l.task - 1]) {
        const double t = now();
        if (s == 0) {
          sum += t - l.job_start;
          jobs++;
        }
        l.stage = 0;
        l.job_start = t;
      }
      int rc = go(l);
      if (rc) return rc;
    }
    if (now() > seconds * 20 + 5) break;  // safety
  }
  cudaDeviceSynchronize();
  *out_mean_job_time = jobs ? sum / jobs : 0.0;
  return DARIS_OK;
}

}  // extern "C"
