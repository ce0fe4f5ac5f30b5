// Probe: can B200 green contexts give DARIS its SM partitions?
//  - split granularity with/without IGNORE_SM_COSCHEDULING
//  - confinement: which SMs do blocks launched into a green-context stream hit
//  - overlap: two descriptors built from the same split sharing groups (OS > 1)
//  - memory allocated in the primary context usable from green streams
//  - CUDA graph capture + launch on a green stream, event timing, launch latency
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/probe_green.cu -lcuda -o /tmp/probe
#include <cuda.h>
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <set>
#include <vector>

#define CK(x)                                                                     \
  do {                                                                            \
    CUresult r_ = (x);                                                            \
    if (r_ != CUDA_SUCCESS) {                                                     \
      const char* s_ = nullptr;                                                   \
      cuGetErrorString(r_, &s_);                                                  \
      printf("FAIL %s -> %d %s (line %d)\n", #x, (int)r_, s_ ? s_ : "", __LINE__); \
    }                                                                             \
  } while (0)
#define RK(x)                                                                                  \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess) printf("FAIL %s -> %s (line %d)\n", #x, cudaGetErrorString(e_), __LINE__); \
  } while (0)

__global__ void smid_kernel(int* out, int spin) {
  unsigned s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  long long t0 = clock64();
  while (clock64() - t0 < spin) {
  }
  if (threadIdx.x == 0) out[blockIdx.x] = (int)s;
}

static std::set<int> run_on(CUstream st, int* dbuf, int blocks, int spin) {
  smid_kernel<<<blocks, 64, 0, (cudaStream_t)st>>>(dbuf, spin);
  RK(cudaGetLastError());
  RK(cudaStreamSynchronize((cudaStream_t)st));
  std::vector<int> h(blocks);
  RK(cudaMemcpy(h.data(), dbuf, blocks * sizeof(int), cudaMemcpyDeviceToHost));
  return std::set<int>(h.begin(), h.end());
}

static void print_set(const char* tag, const std::set<int>& s) {
  printf("%s: %zu SMs [", tag, s.size());
  int k = 0;
  for (int v : s) {
    if (k++ < 12) printf("%d ", v);
  }
  printf("%s]\n", s.size() > 12 ? "..." : "");
}

int main() {
  CK(cuInit(0));
  RK(cudaSetDevice(0));
  RK(cudaFree(0));
  CUdevice dev;
  CK(cuDeviceGet(&dev, 0));
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("device SMs = %d\n", sms);
  CUdevResource all;
  CK(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
  printf("SM resource count = %u\n", all.sm.smCount);

  for (unsigned flags : {0u, (unsigned)CU_DEV_SM_RESOURCE_SPLIT_IGNORE_SM_COSCHEDULING}) {
    for (unsigned mc : {1u, 2u, 4u, 8u, 16u, 20u, 36u, 37u, 38u, 40u, 72u, 74u, 76u}) {
      unsigned n = 64;
      CUdevResource groups[64], rem;
      CUresult r = cuDevSmResourceSplitByCount(groups, &n, &all, &rem, flags, mc);
      if (r != CUDA_SUCCESS) {
        printf("split flags=%u min=%u -> err %d\n", flags, mc, (int)r);
        continue;
      }
      printf("split flags=%u min=%u -> %u groups of %u, remainder %u\n", flags, mc, n, n ? groups[0].sm.smCount : 0,
             rem.sm.smCount);
    }
  }

  int* dbuf = nullptr;
  RK(cudaMalloc(&dbuf, 4096 * sizeof(int)));

  // baseline: primary context stream
  cudaStream_t ps;
  RK(cudaStreamCreateWithFlags(&ps, cudaStreamNonBlocking));
  print_set("primary", run_on((CUstream)ps, dbuf, 1024, 20000));

  // fine split into groups, then build two overlapping partitions
  const unsigned flags = CU_DEV_SM_RESOURCE_SPLIT_IGNORE_SM_COSCHEDULING;
  unsigned n = 148;
  CUdevResource groups[148], rem;
  CK(cuDevSmResourceSplitByCount(groups, &n, &all, &rem, flags, 2));
  printf("fine split: %u groups of %u, remainder %u\n", n, groups[0].sm.smCount, rem.sm.smCount);
  const unsigned half = n / 2;
  auto make_ctx = [&](unsigned first, unsigned count, CUgreenCtx* g) {
    std::vector<CUdevResource> res;
    for (unsigned k = 0; k < count; ++k) res.push_back(groups[(first + k) % n]);
    CUdevResourceDesc desc;
    CK(cuDevResourceGenerateDesc(&desc, res.data(), (unsigned)res.size()));
    CK(cuGreenCtxCreate(g, desc, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  };
  CUgreenCtx gA, gB, gC;
  make_ctx(0, half, &gA);          // first half
  make_ctx(half, n - half, &gB);   // second half
  make_ctx(half / 2, half, &gC);   // overlaps both (OS > 1)
  CUstream sA, sB, sC;
  CK(cuGreenCtxStreamCreate(&sA, gA, CU_STREAM_NON_BLOCKING, 0));
  CK(cuGreenCtxStreamCreate(&sB, gB, CU_STREAM_NON_BLOCKING, 0));
  CK(cuGreenCtxStreamCreate(&sC, gC, CU_STREAM_NON_BLOCKING, 0));
  CUdevResource ra;
  CK(cuGreenCtxGetDevResource(gA, &ra, CU_DEV_RESOURCE_TYPE_SM));
  printf("green A reports %u SMs\n", ra.sm.smCount);
  // runtime launch into a green stream while the primary context is current
  auto A = run_on(sA, dbuf, 1024, 20000);
  auto B = run_on(sB, dbuf + 1024, 1024, 20000);
  auto Cc = run_on(sC, dbuf + 2048, 1024, 20000);
  print_set("green A", A);
  print_set("green B", B);
  print_set("green C (overlap)", Cc);
  int ab = 0, ac = 0;
  for (int s : A) {
    ab += B.count(s);
    ac += Cc.count(s);
  }
  printf("|A∩B| = %d  |A∩C| = %d\n", ab, ac);

  // with the green context made current
  CUcontext cA;
  CK(cuCtxFromGreenCtx(&cA, gA));
  CK(cuCtxPushCurrent(cA));
  print_set("green A (current)", run_on(sA, dbuf, 1024, 20000));
  // graph capture on a green stream
  cudaGraph_t g;
  cudaGraphExec_t ge;
  RK(cudaStreamBeginCapture((cudaStream_t)sA, cudaStreamCaptureModeThreadLocal));
  for (int i = 0; i < 4; ++i) smid_kernel<<<256, 64, 0, (cudaStream_t)sA>>>(dbuf + 3072, 1000);
  RK(cudaStreamEndCapture((cudaStream_t)sA, &g));
  RK(cudaGraphInstantiate(&ge, g, 0));
  CUcontext popped;
  CK(cuCtxPopCurrent(&popped));
  // launch the graph from the primary context onto B's stream and A's stream
  RK(cudaGraphLaunch(ge, (cudaStream_t)sB));
  RK(cudaStreamSynchronize((cudaStream_t)sB));
  {
    std::vector<int> h(256);
    RK(cudaMemcpy(h.data(), dbuf + 3072, 256 * sizeof(int), cudaMemcpyDeviceToHost));
    std::set<int> s(h.begin(), h.end());
    int inA = 0;
    for (int v : s) inA += A.count(v);
    printf("graph captured on A, launched on B stream: %zu SMs, %d in A's set\n", s.size(), inA);
  }
  RK(cudaGraphLaunch(ge, (cudaStream_t)sA));
  RK(cudaStreamSynchronize((cudaStream_t)sA));
  {
    std::vector<int> h(256);
    RK(cudaMemcpy(h.data(), dbuf + 3072, 256 * sizeof(int), cudaMemcpyDeviceToHost));
    std::set<int> s(h.begin(), h.end());
    int inA = 0;
    for (int v : s) inA += A.count(v);
    printf("graph captured on A, launched on A stream: %zu SMs, %d in A's set\n", s.size(), inA);
  }
  // graph captured on primary stream, launched into green stream B
  cudaGraph_t g2;
  cudaGraphExec_t ge2;
  RK(cudaStreamBeginCapture(ps, cudaStreamCaptureModeThreadLocal));
  smid_kernel<<<512, 64, 0, ps>>>(dbuf + 3072, 20000);
  RK(cudaStreamEndCapture(ps, &g2));
  RK(cudaGraphInstantiate(&ge2, g2, 0));
  RK(cudaGraphLaunch(ge2, (cudaStream_t)sB));
  RK(cudaStreamSynchronize((cudaStream_t)sB));
  {
    std::vector<int> h(512);
    RK(cudaMemcpy(h.data(), dbuf + 3072, 512 * sizeof(int), cudaMemcpyDeviceToHost));
    std::set<int> s(h.begin(), h.end());
    int inB = 0;
    for (int v : s) inB += B.count(v);
    printf("graph captured on primary, launched on B stream: %zu SMs, %d in B's set\n", s.size(), inB);
  }

  // latency: empty-ish graph launch + event query loop
  cudaEvent_t ev;
  RK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  auto t0 = std::chrono::steady_clock::now();
  const int N = 2000;
  for (int i = 0; i < N; ++i) {
    RK(cudaGraphLaunch(ge2, ps));
  }
  auto t1 = std::chrono::steady_clock::now();
  RK(cudaStreamSynchronize(ps));
  printf("graph launch host cost: %.2f us\n", std::chrono::duration<double, std::micro>(t1 - t0).count() / N);
  int polls = 0;
  smid_kernel<<<1, 32, 0, ps>>>(dbuf, 2000000);
  RK(cudaEventRecord(ev, ps));
  t0 = std::chrono::steady_clock::now();
  while (cudaEventQuery(ev) == cudaErrorNotReady) ++polls;
  t1 = std::chrono::steady_clock::now();
  printf("event poll: %d polls over %.1f us (%.3f us/poll)\n", polls,
         std::chrono::duration<double, std::micro>(t1 - t0).count(),
         std::chrono::duration<double, std::micro>(t1 - t0).count() / (polls ? polls : 1));
  printf("done\n");
  return 0;
}
