// Stage-boundary latency: a stage (kernel A, ~50 us) finishes; the host sees it
// (event poll) and starts the next stage (kernel B) on the same stream.
//   (a) today:      poll A's event -> cudaGraphLaunch(graph of B)
//   (b) pre-launch: right after A, enqueue a gated graph [gate kernel -> IF node{B}];
//                   poll A's event -> write GO into a host-mapped flag; the gate
//                   (spinning on the flag) sets the IF condition and B runs
//   (c) like (b) but SKIP: B must not run, and a normally launched B follows
// Gap = B's first %globaltimer - A's last %globaltimer (device clock), over N reps.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/prelaunch_probe.bin tools/prelaunch_probe.cu
#include <cuda_runtime.h>
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <vector>

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__global__ void stage_a(unsigned long long* t_end, unsigned long long ns) {
  const unsigned long long t0 = gt();
  while (gt() - t0 < ns) {
  }
  if (threadIdx.x == 0) *t_end = gt();
}
__global__ void stage_b(unsigned long long* t_start, int* runs) {
  if (threadIdx.x == 0) {
    *t_start = gt();
    atomicAdd(runs, 1);
  }
}
__global__ void gate(cudaGraphConditionalHandle h, const volatile unsigned* flag, const unsigned* expect) {
  const unsigned e = *expect;
  unsigned v;
  const unsigned long long t0 = gt();
  while (((v = *flag) >> 1) != e) {
    __nanosleep(64);
    if (gt() - t0 > 1000000000ull) {  // 1 s: never hang the GPU, treat as SKIP
      v = 0;
      break;
    }
  }
  cudaGraphSetConditional(h, v & 1u);
}

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e_ = (x);                                                        \
    if (e_ != cudaSuccess) {                                                     \
      printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      return 1;                                                                  \
    }                                                                            \
  } while (0)

int main() {
  cudaStream_t s, cap;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
  unsigned long long *t_end, *t_start;
  int* runs;
  unsigned* expect;
  CK(cudaMalloc(&t_end, 8));
  CK(cudaMalloc(&t_start, 8));
  CK(cudaMalloc(&runs, 4));
  CK(cudaMalloc(&expect, 4));
  unsigned* hflag;
  CK(cudaHostAlloc(&hflag, 64, cudaHostAllocMapped));
  *hflag = 0;
  unsigned* dflag;
  CK(cudaHostGetDevicePointer(&dflag, hflag, 0));
  // plain graph of B
  cudaGraph_t gb;
  CK(cudaStreamBeginCapture(cap, cudaStreamCaptureModeRelaxed));
  stage_b<<<1, 32, 0, cap>>>(t_start, runs);
  CK(cudaStreamEndCapture(cap, &gb));
  cudaGraphExec_t eb;
  CK(cudaGraphInstantiate(&eb, gb, 0));
  // gated graph: gate -> IF{B}
  cudaGraph_t gg;
  CK(cudaGraphCreate(&gg, 0));
  cudaGraphConditionalHandle h;
  CK(cudaGraphConditionalHandleCreate(&h, gg, 0, cudaGraphCondAssignDefault));
  cudaGraphNode_t gn, cn;
  cudaKernelNodeParams kp = {};
  const unsigned* dflag_c = dflag;
  const unsigned* expect_c = expect;
  void* args[] = {&h, &dflag_c, &expect_c};
  kp.func = reinterpret_cast<void*>(gate);
  kp.gridDim = dim3(1);
  kp.blockDim = dim3(32);
  kp.kernelParams = args;
  CK(cudaGraphAddKernelNode(&gn, gg, nullptr, 0, &kp));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeIf;
  cp.conditional.size = 1;
  CK(cudaGraphAddNode(&cn, gg, &gn, 1, &cp));
  CK(cudaStreamBeginCaptureToGraph(cap, cp.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                   cudaStreamCaptureModeRelaxed));
  stage_b<<<1, 32, 0, cap>>>(t_start, runs);
  cudaGraph_t dummy;
  CK(cudaStreamEndCapture(cap, &dummy));
  cudaGraphExec_t eg;
  CK(cudaGraphInstantiate(&eg, gg, 0));
  cudaEvent_t ev;
  CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));

  const int N = 200;
  unsigned seq = 0;
  for (int mode = 0; mode < 3; ++mode) {
    std::vector<double> gaps;
    int skipped_ok = 0;
    for (int i = 0; i < N; ++i) {
      CK(cudaMemset(runs, 0, 4));
      CK(cudaStreamSynchronize(s));
      stage_a<<<1, 32, 0, s>>>(t_end, 50000);
      CK(cudaEventRecord(ev, s));
      if (mode >= 1) {
        ++seq;
        CK(cudaMemcpyAsync(expect, &seq, 4, cudaMemcpyHostToDevice, s));  // (stream-ordered seq)
        CK(cudaGraphLaunch(eg, s));
      }
      while (cudaEventQuery(ev) == cudaErrorNotReady) {
      }
      if (mode == 0) {
        CK(cudaGraphLaunch(eb, s));
      } else if (mode == 1) {
        reinterpret_cast<volatile unsigned*>(hflag)[0] = (seq << 1) | 1u;  // GO
      } else {
        reinterpret_cast<volatile unsigned*>(hflag)[0] = (seq << 1);  // SKIP, then the normal launch
        CK(cudaGraphLaunch(eb, s));
      }
      CK(cudaStreamSynchronize(s));
      unsigned long long a, b;
      int r;
      CK(cudaMemcpy(&a, t_end, 8, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(&b, t_start, 8, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(&r, runs, 4, cudaMemcpyDeviceToHost));
      if (i >= 10) gaps.push_back((double)(b - a) * 1e-3);
      if (r == 1) ++skipped_ok;
    }
    std::sort(gaps.begin(), gaps.end());
    printf("mode %d (%s): gap p50 %.2f us p90 %.2f us p99 %.2f us; B ran exactly once in %d/%d reps\n", mode,
           mode == 0 ? "poll + cudaGraphLaunch" : mode == 1 ? "pre-launched gate, GO" : "pre-launched gate, SKIP + launch",
           gaps[gaps.size() / 2], gaps[gaps.size() * 9 / 10], gaps[gaps.size() * 99 / 100], skipped_ok, N);
  }
  return 0;
}
