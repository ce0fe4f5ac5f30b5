// Whole-GPU freeze detector: a few CTAs spin on %globaltimer for `seconds`
// and record every gap between consecutive reads above a threshold. Run it
// alone on an idle B200 to tell environmental stalls (driver / power / other
// contexts) from stalls caused by our own kernels.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/freeze_probe.cu -o tools/freeze_probe.bin
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void spin(unsigned long long ns, unsigned long long thresh, unsigned long long* out, int cap, int* n) {
  if (threadIdx.x != 0) return;
  const unsigned long long t0 = gt();
  unsigned long long prev = t0;
  for (;;) {
    const unsigned long long t = gt();
    if (t - prev > thresh) {
      const int i = atomicAdd(n, 1);
      if (i < cap) {
        out[2 * i] = prev - t0;
        out[2 * i + 1] = (t - prev) | (static_cast<unsigned long long>(blockIdx.x) << 48);
      }
    }
    prev = t;
    if (t - t0 > ns) break;
  }
}

int main(int argc, char** argv) {
  const double seconds = argc > 1 ? atof(argv[1]) : 5.0;
  const int blocks = argc > 2 ? atoi(argv[2]) : 8;
  const unsigned long long thresh = argc > 3 ? strtoull(argv[3], nullptr, 10) : 50000ull;  // 50 us
  const int cap = 4096;
  unsigned long long* out;
  int* n;
  cudaMalloc(&out, sizeof(unsigned long long) * 2 * cap);
  cudaMalloc(&n, sizeof(int));
  cudaMemset(n, 0, sizeof(int));
  spin<<<blocks, 32>>>(static_cast<unsigned long long>(seconds * 1e9), thresh, out, cap, n);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    return 1;
  }
  int hn = 0;
  cudaMemcpy(&hn, n, sizeof(int), cudaMemcpyDeviceToHost);
  static unsigned long long h[2 * 4096];
  cudaMemcpy(h, out, sizeof(unsigned long long) * 2 * cap, cudaMemcpyDeviceToHost);
  printf("freeze_probe: %.1f s, %d CTAs, threshold %llu ns: %d gaps\n", seconds, blocks, thresh, hn);
  unsigned long long big = 0;
  for (int i = 0; i < hn && i < cap; ++i) {
    const unsigned long long g = h[2 * i + 1] & ((1ull << 48) - 1);
    if (g > big) big = g;
    if (i < 60) printf("  cta %llu at %.6f s gap %.1f us\n", h[2 * i + 1] >> 48, h[2 * i] * 1e-9, g * 1e-3);
  }
  printf("max gap %.1f us\n", big * 1e-3);
  return 0;
}
