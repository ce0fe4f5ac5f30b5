// L2 -> SM latency probe for the activation gather pattern: each of 128
// threads issues 8 x 16-B cp.async.cg (or ld.global.cg) per round from an
// L2-resident buffer, waits, repeats. Reports ns per round (clock64-free:
// globaltimer) for 1 CTA and for many CTAs reading the same lines.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/l2_latency.cu -o tools/l2_latency.bin
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void probe(const char* buf, size_t span, int rounds, int mode, unsigned long long* out) {
  __shared__ __align__(128) char sm[128 * 128];
  const int t = threadIdx.x;
  const int row_sub = t >> 3, chunk = t & 7;
  unsigned long long t0 = gt();
  unsigned acc = 0;
  for (int r = 0; r < rounds; ++r) {
    const size_t base = (static_cast<size_t>(r) * 128 * 128 * 7) % (span - 128 * 128);
    if (mode == 0) {
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        const int row = p * 16 + row_sub;
        const char* src = buf + base + row * 128 + chunk * 16;
        unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(sm + row * 128 + ((chunk ^ (row & 7)) << 4)));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
      }
      asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
    } else {
      uint4 v[8];
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        const int row = p * 16 + row_sub;
        v[p] = __ldcg(reinterpret_cast<const uint4*>(buf + base + row * 128 + chunk * 16));
      }
#pragma unroll
      for (int p = 0; p < 8; ++p) acc += v[p].x ^ v[p].w;
    }
    __syncthreads();
  }
  unsigned long long t1 = gt();
  if (t == 0) out[blockIdx.x] = (t1 - t0) / rounds;
  if (acc == 0x12345678) out[0] = 0;
}

int main() {
  const size_t span = 8 << 20;  // 8 MB: L2-resident
  char* buf;
  cudaMalloc(&buf, span);
  cudaMemset(buf, 1, span);
  unsigned long long* out;
  cudaMalloc(&out, 1024 * sizeof(unsigned long long));
  unsigned long long h[1024];
  for (int mode = 0; mode < 2; ++mode) {
    for (int ctas : {1, 8, 74, 148}) {
      probe<<<ctas, 128>>>(buf, span, 200, mode, out);  // warm
      probe<<<ctas, 128>>>(buf, span, 2000, mode, out);
      cudaDeviceSynchronize();
      cudaMemcpy(h, out, ctas * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
      unsigned long long mn = ~0ull, mx = 0;
      for (int i = 0; i < ctas; ++i) { mn = h[i] < mn ? h[i] : mn; mx = h[i] > mx ? h[i] : mx; }
      printf("%s ctas=%3d: ns per 16 KB round min %llu max %llu\n", mode == 0 ? "cp.async.cg" : "ld.global.cg", ctas, mn, mx);
    }
  }
  return 0;
}
