// Per-SM streaming rate of bulk TMA copies (global -> shared) as a function of
// bytes in flight: G CTAs (one per SM), each streams `per_cta` bytes through a
// ring of S stages of B bytes (one elected thread issues cp.async.bulk, the
// consumer only waits and re-arms). L2-resident (8 MB buffer, re-read) vs
// HBM (1 GB buffer). Answers: is ~40 GB/s per CTA (the conv mainloops) a
// hardware limit or a pipeline-depth limit?
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_stream_probe.bin tools/tma_stream_probe.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void stream_kernel(const uint8_t* __restrict__ src, size_t span, size_t per_cta, int S, int B,
                              unsigned long long* cycles_out) {
  extern __shared__ __align__(1024) uint8_t ring[];
  __shared__ uint64_t full[16], empty[16];
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&empty[i])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const size_t n = per_cta / B;
  const size_t base = (static_cast<size_t>(blockIdx.x) * per_cta) % span;
  long long t0 = 0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  if (tid == 0) {  // producer
    for (size_t i = 0; i < n; ++i) {
      const int s = static_cast<int>(i % S);
      if (i >= static_cast<size_t>(S)) {
        const uint32_t par = static_cast<uint32_t>(((i / S) & 1) ^ 1);
        asm volatile(
            "{\n\t.reg .pred p;\nW1_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W1_%=;\n\t}" ::"r"(
                smem_u32(&empty[s])),
            "r"(par));
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(B));
      const uint8_t* g = src + (base + i * B) % span;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_u32(ring + s * B)),
                   "l"(g), "r"(B), "r"(smem_u32(&full[s]))
                   : "memory");
    }
  } else if (tid == 32) {  // consumer
    for (size_t i = 0; i < n; ++i) {
      const int s = static_cast<int>(i % S);
      const uint32_t par = static_cast<uint32_t>((i / S) & 1);
      asm volatile(
          "{\n\t.reg .pred p;\nW2_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W2_%=;\n\t}" ::"r"(
              smem_u32(&full[s])),
          "r"(par));
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])));
    }
    long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    cycles_out[blockIdx.x] = static_cast<unsigned long long>(t1 - t0);
  }
}


// same ring, tensor-map loads: box {64 bf16 (128 B), R rows}, 128B swizzle (the conv kernels' B operand)
__global__ void stream_tensor_kernel(const __grid_constant__ CUtensorMap map, int rows_total, size_t per_cta, int S,
                                     int R, unsigned long long* ns_out) {
  extern __shared__ __align__(1024) uint8_t ring[];
  __shared__ uint64_t full[16], empty[16];
  const int tid = threadIdx.x;
  const int B = R * 128;
  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&empty[i])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const size_t n = per_cta / B;
  long long t0 = 0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  if (tid == 0) {
    for (size_t i = 0; i < n; ++i) {
      const int s = static_cast<int>(i % S);
      if (i >= static_cast<size_t>(S)) {
        const uint32_t par = static_cast<uint32_t>(((i / S) & 1) ^ 1);
        asm volatile(
            "{\n\t.reg .pred p;\nW1_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W1_%=;\n\t}" ::"r"(
                smem_u32(&empty[s])),
            "r"(par));
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(B));
      const int row = static_cast<int>((static_cast<size_t>(blockIdx.x) * n + i) * R % rows_total);
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
              smem_u32(ring + s * B)),
          "l"(reinterpret_cast<uint64_t>(&map)), "r"(smem_u32(&full[s])), "r"(0), "r"(row)
          : "memory");
    }
  } else if (tid == 32) {
    for (size_t i = 0; i < n; ++i) {
      const int s = static_cast<int>(i % S);
      const uint32_t par = static_cast<uint32_t>((i / S) & 1);
      asm volatile(
          "{\n\t.reg .pred p;\nW2_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W2_%=;\n\t}" ::"r"(
              smem_u32(&full[s])),
          "r"(par));
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])));
    }
    long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    ns_out[blockIdx.x] = static_cast<unsigned long long>(t1 - t0);
  }
}


// tensor-map ring with P producer threads (one per warp) issuing interleaved loads:
// is the per-CTA serialisation per issuing thread?
__global__ void stream_tensor_multi(const __grid_constant__ CUtensorMap map, int rows_total, size_t per_cta, int S,
                                    int R, int P, unsigned long long* ns_out) {
  extern __shared__ __align__(1024) uint8_t ring[];
  __shared__ uint64_t full[16], empty[16];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int B = R * 128;
  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&empty[i])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const size_t n = per_cta / B;
  long long t0 = 0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  if (warp < P && lane == 0) {
    for (size_t i = warp; i < n; i += P) {
      const int s = static_cast<int>(i % S);
      if (i >= static_cast<size_t>(S)) {
        const uint32_t par = static_cast<uint32_t>(((i / S) & 1) ^ 1);
        asm volatile(
            "{\n\t.reg .pred p;\nW1_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W1_%=;\n\t}" ::"r"(
                smem_u32(&empty[s])),
            "r"(par));
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(B));
      const int row = static_cast<int>((static_cast<size_t>(blockIdx.x) * n + i) * R % rows_total);
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
              smem_u32(ring + s * B)),
          "l"(reinterpret_cast<uint64_t>(&map)), "r"(smem_u32(&full[s])), "r"(0), "r"(row)
          : "memory");
    }
  } else if (warp == P && lane == 0) {
    for (size_t i = 0; i < n; ++i) {
      const int s = static_cast<int>(i % S);
      const uint32_t par = static_cast<uint32_t>((i / S) & 1);
      asm volatile(
          "{\n\t.reg .pred p;\nW2_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W2_%=;\n\t}" ::"r"(
              smem_u32(&full[s])),
          "r"(par));
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])));
    }
    long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    ns_out[blockIdx.x] = static_cast<unsigned long long>(t1 - t0);
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t big = size_t(1) << 30, small = size_t(8) << 20;
  uint8_t* buf;
  cudaMalloc(&buf, big);
  cudaMemset(buf, 1, big);
  unsigned long long* ns;
  cudaMalloc(&ns, 1024 * sizeof(unsigned long long));
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  printf("span  ctas stages stage_KB inflight_KB  per_cta_GBps  total_GBps\n");
  for (size_t span : {small, big}) {
    for (int G : {1, 24, sms}) {
      for (int B : {8192, 16384, 32768}) {
        for (int S : {2, 4, 8}) {
          if (S * B > 192 * 1024) continue;
          const size_t per_cta = (span == small) ? (size_t(4) << 20) : (size_t(6) << 20);
          stream_kernel<<<G, 64, S * B>>>(buf, span, per_cta, S, B, ns);  // warm
          stream_kernel<<<G, 64, S * B>>>(buf, span, per_cta, S, B, ns);
          cudaDeviceSynchronize();
          unsigned long long h[1024];
          cudaMemcpy(h, ns, G * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
          double mx = 0, sum = 0;
          for (int i = 0; i < G; ++i) {
            mx = h[i] > mx ? h[i] : mx;
            sum += per_cta / (h[i] * 1e-9) / 1e9;
          }
          printf("%s %4d %6d %8d %11d %13.1f %11.1f\n", span == small ? "L2 " : "HBM", G, S, B / 1024, S * B / 1024,
                 sum / G, G * per_cta / (mx * 1e-9) / 1e9);
        }
      }
    }
  }
  // tensor-map loads (L2-resident 8 MB matrix of 128-B rows)
  PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&encode), cudaEnableDefault, &q);
  cudaFuncSetAttribute(stream_tensor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  printf("tensor TMA (box 64 x R bf16, SW128), L2-resident\n");
  printf("ctas/SM ctas stages box_KB  per_cta_GBps  total_GBps\n");
  const int rows_total = static_cast<int>(small / 128);
  for (int R : {64, 128, 256}) {
    CUtensorMap map;
    cuuint64_t dims[2] = {64, static_cast<cuuint64_t>(rows_total)};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {64, static_cast<cuuint32_t>(R)};
    cuuint32_t estr[2] = {1, 1};
    encode(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int per_sm : {1, 3}) {
      for (int S : {2, 4, 8}) {
        const int B = R * 128;
        if (S * B * per_sm > 200 * 1024) continue;
        const int G = sms * per_sm;
        const size_t per_cta = size_t(4) << 20;
        stream_tensor_kernel<<<G, 64, S * B>>>(map, rows_total, per_cta, S, R, ns);
        stream_tensor_kernel<<<G, 64, S * B>>>(map, rows_total, per_cta, S, R, ns);
        cudaDeviceSynchronize();
        unsigned long long h[1024];
        cudaMemcpy(h, ns, G * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
        double mx = 0, sum = 0;
        for (int i = 0; i < G; ++i) {
          mx = h[i] > mx ? h[i] : mx;
          sum += per_cta / (h[i] * 1e-9) / 1e9;
        }
        printf("%7d %4d %6d %6d %13.1f %11.1f\n", per_sm, G, S, B / 1024, sum / G, G * per_cta / (mx * 1e-9) / 1e9);
      }
    }
  }
  printf("tensor TMA, P producer threads per CTA, 1 CTA/SM, 8 stages\n");
  printf("P box_KB per_cta_GBps\n");
  cudaFuncSetAttribute(stream_tensor_multi, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int R : {64, 128}) {
    CUtensorMap map;
    cuuint64_t dims[2] = {64, static_cast<cuuint64_t>(rows_total)};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {64, static_cast<cuuint32_t>(R)};
    cuuint32_t estr[2] = {1, 1};
    encode(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int P : {1, 2, 4, 8}) {
      const int B = R * 128, S = 8, G = sms;
      const size_t per_cta = size_t(4) << 20;
      stream_tensor_multi<<<G, 32 * (P + 1), S * B>>>(map, rows_total, per_cta, S, R, P, ns);
      stream_tensor_multi<<<G, 32 * (P + 1), S * B>>>(map, rows_total, per_cta, S, R, P, ns);
      cudaDeviceSynchronize();
      unsigned long long h[1024];
      cudaMemcpy(h, ns, G * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
      double sum = 0;
      for (int i = 0; i < G; ++i) sum += per_cta / (h[i] * 1e-9) / 1e9;
      printf("%d %6d %13.1f\n", P, B / 1024, sum / G);
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
