// Floor of the persistent stage kernel's layer hand-off: CTA 0 writes a 16 KB
// tile with plain stores, fences and bumps a counter; every other CTA polls
// the counter (relaxed), fences, then cp.async-gathers the fresh tile and
// acks. Reports, per consumer SM, the publish->observe latency and the read
// latency of freshly written data, against the same read of stale data.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/dataflow_latency.cu -o tools/dataflow_latency.bin
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

__global__ void flow(char* buf, int* flag, int* ack, unsigned long long* pub_t, int rounds, unsigned long long* out) {
  __shared__ __align__(128) char sm[128 * 128];
  __shared__ unsigned long long t_seen, t_read;
  const int t = threadIdx.x;
  const int row_sub = t >> 3, chunk = t & 7;
  unsigned long long obs = 0, rd = 0, rd_stale = 0;
  for (int r = 1; r <= rounds; ++r) {
    if (blockIdx.x == 0) {
      if (t == 0) while (ld_relaxed(ack) < (r - 1) * (int)(gridDim.x - 1)) {}
      __syncthreads();
      uint4* b = reinterpret_cast<uint4*>(buf);
      for (int i = t; i < 1024; i += blockDim.x) b[i] = make_uint4(r, r, r, r);
      __syncthreads();
      if (t == 0) {
        __threadfence();
        *pub_t = gt();
        __threadfence();
        atomicAdd(flag, 1);
      }
    } else {
      if (t == 0) {
        while (ld_relaxed(flag) < r) {}
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        t_seen = gt();
      }
      __syncthreads();
      const unsigned long long a = gt();
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        const int row = p * 16 + row_sub;
        unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(sm + row * 128 + ((chunk ^ (row & 7)) << 4)));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(buf + row * 128 + chunk * 16) : "memory");
      }
      asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
      __syncthreads();
      const unsigned long long b = gt();
      // same read again: now the lines are no longer "fresh"
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        const int row = p * 16 + row_sub;
        unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(sm + row * 128 + ((chunk ^ (row & 7)) << 4)));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(buf + 16384 + row * 128 + chunk * 16) : "memory");
      }
      asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
      __syncthreads();
      const unsigned long long c = gt();
      if (t == 0) {
        obs += t_seen - *(volatile unsigned long long*)pub_t;
        rd += b - a;
        rd_stale += c - b;
        atomicAdd(ack, 1);
      }
    }
  }
  if (t == 0 && blockIdx.x > 0) {
    out[3 * blockIdx.x] = obs / rounds;
    out[3 * blockIdx.x + 1] = rd / rounds;
    out[3 * blockIdx.x + 2] = (rd_stale / rounds) | (static_cast<unsigned long long>(smid()) << 32);
  }
}

int main() {
  char* buf;
  int *flag, *ack;
  unsigned long long *pub, *out;
  cudaMalloc(&buf, 1 << 20);
  cudaMemset(buf, 0, 1 << 20);
  cudaMalloc(&flag, 4);
  cudaMalloc(&ack, 4);
  cudaMalloc(&pub, 8);
  cudaMalloc(&out, 3 * 8 * 256);
  for (int grid : {2, 9, 74, 148}) {
    cudaMemset(flag, 0, 4);
    cudaMemset(ack, 0, 4);
    flow<<<grid, 128>>>(buf, flag, ack, pub, 500, out);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    static unsigned long long h[3 * 256];
    cudaMemcpy(h, out, 3 * 8 * grid, cudaMemcpyDeviceToHost);
    double so = 0, sr = 0, ss = 0; unsigned long long mo = 0, mr = 0;
    for (int i = 1; i < grid; ++i) {
      so += h[3 * i]; sr += h[3 * i + 1]; ss += (h[3 * i + 2] & 0xffffffffull);
      mo = h[3 * i] > mo ? h[3 * i] : mo; mr = h[3 * i + 1] > mr ? h[3 * i + 1] : mr;
    }
    const int n = grid - 1;
    printf("grid %3d: publish->observe mean %.0f ns (max %llu), fresh 16KB read %.0f ns (max %llu), stale read %.0f ns\n",
           grid, so / n, mo, sr / n, mr, ss / n);
  }
  return 0;
}
