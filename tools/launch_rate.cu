// Kernel-launch throughput of the GPU front end: S streams, each replaying a
// CUDA graph of K small kernels (G CTAs each, each CTA spinning `ns` ns), for
// a fixed number of rounds; prints kernels/s over all streams. With ns = 0 this
// is the launch/retire ceiling for graphs of short dependent kernels — the
// regime batch-1 DNN layers live in.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/launch_rate.bin tools/launch_rate.cu
// ./tools/launch_rate.bin
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

__global__ void spin(long long ns) {
  if (ns <= 0) return;
  long long t0;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
  long long t = t0;
  while (t - t0 < ns) asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
}

static double run(int S, int K, int G, long long ns, bool pdl, int rounds) {
  std::vector<cudaStream_t> st(S);
  std::vector<cudaGraphExec_t> ge(S);
  for (int s = 0; s < S; ++s) {
    cudaStreamCreateWithFlags(&st[s], cudaStreamNonBlocking);
    cudaGraph_t g;
    cudaStreamBeginCapture(st[s], cudaStreamCaptureModeThreadLocal);
    for (int k = 0; k < K; ++k) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(G);
      cfg.blockDim = dim3(128);
      cfg.stream = st[s];
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = pdl ? 1 : 0;
      cudaLaunchKernelEx(&cfg, spin, ns);
    }
    cudaStreamEndCapture(st[s], &g);
    cudaGraphInstantiate(&ge[s], g, 0);
    cudaGraphDestroy(g);
  }
  for (int s = 0; s < S; ++s) cudaGraphLaunch(ge[s], st[s]);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, 0);
  cudaDeviceSynchronize();
  for (int r = 0; r < rounds; ++r)
    for (int s = 0; s < S; ++s) cudaGraphLaunch(ge[s], st[s]);
  cudaDeviceSynchronize();
  cudaEventRecord(e1, 0);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  for (int s = 0; s < S; ++s) {
    cudaGraphExecDestroy(ge[s]);
    cudaStreamDestroy(st[s]);
  }
  const double kernels = double(S) * K * rounds;
  return kernels / (ms * 1e-3);
}

int main() {
  const int K = 57;  // one ResNet-50 forward's launches
  const int rounds = 400;
  printf("streams ctas spin_ns pdl kernels_per_s per_stream_us_per_kernel\n");
  for (long long ns : {0LL, 3000LL}) {
    for (int G : {16, 64}) {
      for (bool pdl : {false, true}) {
        for (int S : {1, 2, 4, 8, 16, 32}) {
          double r = run(S, K, G, ns, pdl, rounds);
          printf("%2d %3d %5lld %d %10.0f %8.2f\n", S, G, ns, pdl ? 1 : 0, r, 1e6 * S / r);
        }
      }
    }
  }
  return 0;
}
