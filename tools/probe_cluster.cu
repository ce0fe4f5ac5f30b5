// Probe: thread-block clusters (DSMEM) inside green-context partitions built
// with IGNORE_SM_COSCHEDULING (2-SM groups): which cluster sizes launch, and
// does a DSMEM reduction across the cluster give the right answer?
#include <cuda.h>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
#include <cstdio>
#include <vector>
namespace cg = cooperative_groups;

__global__ void cluster_sum(const float* in, float* out, int* smids) {
  __shared__ float buf[256];
  cg::cluster_group cl = cg::this_cluster();
  unsigned r = cl.block_rank();
  buf[threadIdx.x] = in[blockIdx.x * 256 + threadIdx.x];
  unsigned s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  if (threadIdx.x == 0) smids[blockIdx.x] = (int)s;
  cl.sync();
  float acc = 0.f;
  for (unsigned k = 0; k < cl.num_blocks(); ++k) {
    float* remote = cl.map_shared_rank(buf, k);
    acc += remote[threadIdx.x];
  }
  cl.sync();
  if (r == 0) out[(blockIdx.x / cl.num_blocks()) * 256 + threadIdx.x] = acc;
}

int main() {
  cuInit(0);
  cudaSetDevice(0);
  cudaFree(0);
  CUdevice dev;
  cuDeviceGet(&dev, 0);
  CUdevResource all;
  cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM);
  for (unsigned flags : {0u, (unsigned)CU_DEV_SM_RESOURCE_SPLIT_IGNORE_SM_COSCHEDULING}) {
    unsigned n = 148;
    CUdevResource groups[148], rem;
    unsigned minc = flags ? 2 : 8;
    if (cuDevSmResourceSplitByCount(groups, &n, &all, &rem, flags, minc) != CUDA_SUCCESS) { printf("split fail\n"); continue; }
    unsigned want = flags ? 37 : 9;  // ~74 or 72 SMs
    std::vector<CUdevResource> res(groups, groups + want);
    CUdevResourceDesc desc;
    cuDevResourceGenerateDesc(&desc, res.data(), want);
    CUgreenCtx g;
    if (cuGreenCtxCreate(&g, desc, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS) { printf("green fail\n"); continue; }
    CUstream cs;
    cuGreenCtxStreamCreate(&cs, g, CU_STREAM_NON_BLOCKING, 0);
    cudaStream_t st = (cudaStream_t)cs;
    for (int csz : {2, 4, 8, 16}) {
      const int blocks = 64;
      float *in, *out; int* sm;
      cudaMalloc(&in, blocks * 256 * 4); cudaMalloc(&out, blocks * 256 * 4); cudaMalloc(&sm, blocks * 4);
      std::vector<float> h(blocks * 256);
      for (int i = 0; i < blocks * 256; ++i) h[i] = (float)(i % 7);
      cudaMemcpy(in, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
      if (csz == 16) cudaFuncSetAttribute(cluster_sum, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(blocks); cfg.blockDim = dim3(256); cfg.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = csz; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      int maxc = -1;
      cudaError_t oe = cudaOccupancyMaxActiveClusters(&maxc, (void*)cluster_sum, &cfg);
      cudaError_t e = cudaLaunchKernelEx(&cfg, cluster_sum, (const float*)in, out, sm);
      cudaError_t e2 = cudaStreamSynchronize(st);
      std::vector<float> o(blocks * 256);
      cudaMemcpy(o.data(), out, o.size() * 4, cudaMemcpyDeviceToHost);
      bool ok = (e == cudaSuccess && e2 == cudaSuccess);
      for (int c = 0; ok && c < blocks / csz; ++c)
        for (int t = 0; t < 256; ++t) {
          float ref = 0;
          for (int k = 0; k < csz; ++k) ref += h[(c * csz + k) * 256 + t];
          if (o[c * 256 + t] != ref) { ok = false; break; }
        }
      printf("flags=%u cluster=%d: occupancy(maxActiveClusters)=%d (%s) launch=%s sync=%s correct=%d\n", flags, csz, maxc,
             cudaGetErrorString(oe), cudaGetErrorString(e), cudaGetErrorString(e2), (int)ok);
      cudaGetLastError();
      cudaFree(in); cudaFree(out); cudaFree(sm);
    }
  }
  return 0;
}
