// DSMEM reduction micro-benchmark: the conv kernel's cluster split-K moves
// each CTA's fp32 partial rows (128 rows x 64 columns, rows owned round-robin
// in S contiguous blocks) to the owning CTA. Timed variants (cluster of S CTAs,
// 128 producer threads, %globaltimer around the exchange, median over CTAs):
//   0  push, row per thread: st.async 16 B x 16 per row, remote mbarrier tx (the kernel today)
//   1  push, contiguous per warp: rows staged in local smem, then st.async of
//      consecutive 16-B chunks (a warp writes 512 contiguous bytes)
//   2  push, contiguous plain stores (st.shared::cluster) + cluster barrier
//   3  pull: rows staged in local smem, cluster barrier, the owner reads its
//      rows from every peer with ld.shared::cluster (16 B per lane, contiguous)
// Also checks the reduced sums.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dsmem_probe.bin tools/dsmem_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>

constexpr int kRows = 128, kCols = 64;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint32_t rank_id() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ uint32_t map_rank(uint32_t a, uint32_t r) {
  uint32_t o; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r)); return o;
}
__device__ __forceinline__ void csync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__device__ __forceinline__ void st_async(uint32_t a, float4 v, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1,%2,%3,%4}, [%5];"
               ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(bar) : "memory");
}
__device__ __forceinline__ void st_cl(uint32_t a, float4 v) {
  asm volatile("st.shared::cluster.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
__device__ __forceinline__ float4 ld_cl(uint32_t a) {
  float4 v; asm volatile("ld.shared::cluster.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a)); return v;
}

template <int S>
__global__ void probe(int variant, float* out, unsigned long long* ns) {
  extern __shared__ __align__(1024) float sm[];
  float* stage = sm;                       // [128][64] this CTA's partial (variants 1, 3)
  float* recv = sm + kRows * kCols;        // [S][rpc][64] owner receive buffer
  __shared__ __align__(8) uint64_t bar;
  const int t = threadIdx.x;
  const uint32_t me = rank_id();
  constexpr int rpc = (kRows + S - 1) / S;
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  // this thread's row of the partial (as the epilogue holds it after tcgen05.ld)
  float v[kCols];
#pragma unroll
  for (int c = 0; c < kCols; ++c) v[c] = static_cast<float>((me + 1) * 1000 + t) + c * 0.25f;
  const int r_begin = (me * kRows) / S, r_end = ((me + 1) * kRows) / S;
  if (t == 0) {
    const uint32_t bytes = static_cast<uint32_t>(S * (r_end - r_begin) * kCols * 4);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(bytes) : "memory");
  }
  csync();
  const unsigned long long t0 = gt();
  const int row = t;
  const int owner = ((row + 1) * S - 1) / kRows;
  const int j = row - (owner * kRows) / S;
  if (variant == 0) {
    const uint32_t dst = map_rank(smem_u32(recv + (static_cast<size_t>(me) * rpc + j) * kCols), owner);
    const uint32_t rb = map_rank(smem_u32(&bar), owner);
#pragma unroll
    for (int q = 0; q < kCols / 4; ++q) st_async(dst + q * 16, make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]), rb);
  } else {
    // stage the row locally (16-B chunks, XOR-swizzled by row to spread banks)
#pragma unroll
    for (int q = 0; q < kCols / 4; ++q)
      *reinterpret_cast<float4*>(stage + row * kCols + ((q ^ (row & 15)) * 4)) =
          make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    __syncthreads();
    if (variant == 1 || variant == 2) {
      // 16-B chunks in (row, chunk) order: lanes of a warp cover 2 rows x 16 chunks = 512 contiguous bytes
      for (int k = t; k < kRows * (kCols / 4); k += 128) {
        const int r = k / (kCols / 4), q = k % (kCols / 4);
        const int own = ((r + 1) * S - 1) / kRows;
        const int jj = r - (own * kRows) / S;
        const float4 x = *reinterpret_cast<const float4*>(stage + r * kCols + ((q ^ (r & 15)) * 4));
        const uint32_t dst = map_rank(smem_u32(recv + (static_cast<size_t>(me) * rpc + jj) * kCols + q * 4), own);
        if (variant == 1) st_async(dst, x, map_rank(smem_u32(&bar), own));
        else st_cl(dst, x);
      }
    }
  }
  if (variant == 2 || variant == 3) csync();
  float sum[4] = {0, 0, 0, 0};
  const int items = (r_end - r_begin) * (kCols / 4);
  if (variant <= 1) {
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(smem_u32(&bar)) : "memory");
    for (int k = t; k < items; k += 128) {
      const int jj = k / (kCols / 4), q = k % (kCols / 4);
      for (int s = 0; s < S; ++s) {
        const float4 x = *reinterpret_cast<const float4*>(recv + (static_cast<size_t>(s) * rpc + jj) * kCols + q * 4);
        sum[0] += x.x; sum[1] += x.y; sum[2] += x.z; sum[3] += x.w;
      }
    }
  } else if (variant == 2) {
    for (int k = t; k < items; k += 128) {
      const int jj = k / (kCols / 4), q = k % (kCols / 4);
      for (int s = 0; s < S; ++s) {
        const float4 x = *reinterpret_cast<const float4*>(recv + (static_cast<size_t>(s) * rpc + jj) * kCols + q * 4);
        sum[0] += x.x; sum[1] += x.y; sum[2] += x.z; sum[3] += x.w;
      }
    }
  } else {
    for (int k = t; k < items; k += 128) {
      const int jj = k / (kCols / 4), q = k % (kCols / 4);
      const int r = r_begin + jj;
      float4 x[S];
#pragma unroll
      for (int s = 0; s < S; ++s) x[s] = ld_cl(map_rank(smem_u32(stage + r * kCols + ((q ^ (r & 15)) * 4)), s));
#pragma unroll
      for (int s = 0; s < S; ++s) { sum[0] += x[s].x; sum[1] += x[s].y; sum[2] += x[s].z; sum[3] += x[s].w; }
    }
  }
  const unsigned long long t1 = gt();
  out[blockIdx.x * 128 + t] = sum[0] + sum[1] + sum[2] + sum[3];
  if (t == 0) ns[blockIdx.x] = t1 - t0;
  csync();  // nobody leaves while peers may still read its smem
}

template <int S>
void run(int variant) {
  const int clusters = 8, blocks = clusters * S;
  float* out;
  unsigned long long* ns;
  cudaMalloc(&out, blocks * 128 * 4);
  cudaMalloc(&ns, blocks * 8);
  const int smem = kRows * kCols * 4 + S * ((kRows + S - 1) / S) * kCols * 4;
  cudaFuncSetAttribute(probe<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = S;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  std::vector<double> med;
  for (int rep = 0; rep < 20; ++rep) {
    cudaLaunchKernelEx(&cfg, probe<S>, variant, out, ns);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("S=%d variant %d: %s\n", S, variant, cudaGetErrorString(e)); return; }
    std::vector<unsigned long long> h(blocks);
    cudaMemcpy(h.data(), ns, blocks * 8, cudaMemcpyDeviceToHost);
    std::sort(h.begin(), h.end());
    if (rep >= 5) med.push_back(h[blocks / 2] * 1e-3);
  }
  std::sort(med.begin(), med.end());
  // check: owner rows' sums
  std::vector<float> ho(blocks * 128);
  cudaMemcpy(ho.data(), out, ho.size() * 4, cudaMemcpyDeviceToHost);
  double err = 0;
  for (int b = 0; b < blocks; ++b) {
    const int me = b % S;
    const int rb = (me * kRows) / S, re = ((me + 1) * kRows) / S, items = (re - rb) * (kCols / 4);
    for (int t = 0; t < 128; ++t) {
      double want = 0;
      for (int k = t; k < items; k += 128) {
        const int jj = k / (kCols / 4), q = k % (kCols / 4), r = rb + jj;
        for (int s = 0; s < S; ++s)
          for (int e = 0; e < 4; ++e) want += (s + 1) * 1000 + r + (q * 4 + e) * 0.25;
      }
      err = std::max(err, std::abs(want - ho[b * 128 + t]) / (std::abs(want) + 1));
    }
  }
  printf("S=%d variant %d: exchange+reduce median %.2f us (p10 %.2f, p90 %.2f), rel err %.2e\n", S, variant,
         med[med.size() / 2], med[med.size() / 10], med[med.size() * 9 / 10], err);
  cudaFree(out);
  cudaFree(ns);
}

int main() {
  for (int v = 0; v < 4; ++v) run<3>(v);
  for (int v = 0; v < 4; ++v) run<6>(v);
  for (int v = 0; v < 4; ++v) run<8>(v);
  return 0;
}
