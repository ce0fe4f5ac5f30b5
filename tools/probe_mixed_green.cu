// Probe: a green context built from co-scheduled 8-SM groups PLUS 2-SM groups
// carved from the split remainder (the SMs an 8-SM split leaves out: 148 - 120).
// Does it expose all its SMs to ordinary kernels, and do 8-CTA clusters still
// launch (on the 8-SM groups) and reduce correctly through DSMEM?
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/probe_mixed_green.bin tools/probe_mixed_green.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
#include <cstdio>
#include <set>
#include <vector>
namespace cg = cooperative_groups;

__global__ void cluster_sum(const float* in, float* out) {
  __shared__ float buf[256];
  cg::cluster_group cl = cg::this_cluster();
  buf[threadIdx.x] = in[blockIdx.x * 256 + threadIdx.x];
  cl.sync();
  float acc = 0.f;
  for (unsigned k = 0; k < cl.num_blocks(); ++k) acc += cl.map_shared_rank(buf, k)[threadIdx.x];
  cl.sync();
  if (cl.block_rank() == 0) out[(blockIdx.x / cl.num_blocks()) * 256 + threadIdx.x] = acc;
}

__global__ void where(int* smids) {
  unsigned s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  long long t0 = clock64();
  while (clock64() - t0 < 200000) {
  }
  if (threadIdx.x == 0) smids[blockIdx.x] = (int)s;
}

int main() {
  cuInit(0);
  cudaSetDevice(0);
  cudaFree(0);
  CUdevice dev;
  cuDeviceGet(&dev, 0);
  CUdevResource all;
  cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM);
  unsigned n8 = 148;
  CUdevResource g8[148], rem, g2[148], rem2;
  if (cuDevSmResourceSplitByCount(g8, &n8, &all, &rem, 0, 8) != CUDA_SUCCESS) { printf("split8 fail\n"); return 1; }
  printf("8-SM groups: %u (%u SMs), remainder %u SMs\n", n8, n8 * g8[0].sm.smCount, rem.sm.smCount);
  unsigned n2 = 148;
  CUresult r2 = CUDA_ERROR_INVALID_VALUE;
  for (unsigned fl : {(unsigned)CU_DEV_SM_RESOURCE_SPLIT_IGNORE_SM_COSCHEDULING, 0u}) {
    for (unsigned mc : {2u, 4u, 8u}) {
      unsigned nn = 148;
      CUresult rr = cuDevSmResourceSplitByCount(g2, &nn, &rem, &rem2, fl, mc);
      printf("remainder split flags=%u min=%u: rc=%d n=%u group=%u left=%u\n", fl, mc, (int)rr, nn,
             rr == CUDA_SUCCESS ? g2[0].sm.smCount : 0, rr == CUDA_SUCCESS ? rem2.sm.smCount : 0);
      if (rr == CUDA_SUCCESS && r2 != CUDA_SUCCESS) { r2 = rr; n2 = nn; }
    }
  }
  // alternative: 2-SM groups of the whole device (IGNORE) — the remainder SMs are somewhere in there
  unsigned nall = 148;
  CUdevResource gall[148], remall;
  CUresult ra = cuDevSmResourceSplitByCount(gall, &nall, &all, &remall, CU_DEV_SM_RESOURCE_SPLIT_IGNORE_SM_COSCHEDULING, 2);
  printf("whole device into 2-SM groups: rc=%d n=%u\n", (int)ra, nall);
  if (r2 != CUDA_SUCCESS) n2 = 0;
  // and: the remainder as one resource next to 8-SM groups
  {
    std::vector<CUdevResource> res(g8, g8 + 7);
    res.push_back(rem);
    CUdevResourceDesc desc;
    CUresult e = cuDevResourceGenerateDesc(&desc, res.data(), (unsigned)res.size());
    CUgreenCtx g;
    CUresult e2 = e == CUDA_SUCCESS ? cuGreenCtxCreate(&g, desc, dev, CU_GREEN_CTX_DEFAULT_STREAM) : e;
    CUdevResource got{};
    if (e2 == CUDA_SUCCESS) cuGreenCtxGetDevResource(g, &got, CU_DEV_RESOURCE_TYPE_SM);
    printf("7 x8 + remainder(%u): desc rc=%d green rc=%d -> %u SMs\n", rem.sm.smCount, (int)e, (int)e2, got.sm.smCount);
  }
  for (int variant = 0; variant < 5; ++variant) {
    // 0: 7 eight-groups + 5 two-groups; 1: 9 eight-groups; 2: all 8-groups + all 2-groups;
    // 3: 6 eight-groups + the remainder; 4: all 8-groups + the remainder (148 SMs)
    std::vector<CUdevResource> res;
    int k8 = variant == 0 ? 7 : variant == 1 ? 9 : variant == 3 ? 6 : (int)n8;
    int k2 = variant == 0 ? 5 : variant == 1 ? 0 : variant >= 3 ? 0 : (int)n2;
    for (int i = 0; i < k8; ++i) res.push_back(g8[i]);
    for (int i = 0; i < k2 && r2 == CUDA_SUCCESS; ++i) res.push_back(g2[i]);
    if (variant >= 3) res.push_back(rem);
    CUdevResourceDesc desc;
    CUresult e = cuDevResourceGenerateDesc(&desc, res.data(), (unsigned)res.size());
    CUgreenCtx g;
    CUresult e2 = e == CUDA_SUCCESS ? cuGreenCtxCreate(&g, desc, dev, CU_GREEN_CTX_DEFAULT_STREAM) : e;
    if (e2 != CUDA_SUCCESS) { printf("variant %d: desc rc=%d green rc=%d\n", variant, (int)e, (int)e2); continue; }
    CUdevResource got;
    cuGreenCtxGetDevResource(g, &got, CU_DEV_RESOURCE_TYPE_SM);
    CUstream cs;
    cuGreenCtxStreamCreate(&cs, g, CU_STREAM_NON_BLOCKING, 0);
    cudaStream_t st = (cudaStream_t)cs;
    int* sm;
    cudaMalloc(&sm, 4096 * 4);
    where<<<1024, 32, 0, st>>>(sm);
    cudaError_t le = cudaStreamSynchronize(st);
    std::vector<int> h(1024);
    cudaMemcpy(h.data(), sm, 1024 * 4, cudaMemcpyDeviceToHost);
    std::set<int> distinct(h.begin(), h.end());
    printf("variant %d: %d x8 + %d x2 groups%s -> green ctx reports %u SMs; plain kernel ran on %zu distinct SMs (%s)\n",
           variant, k8, k2, variant >= 3 ? " + remainder" : "", got.sm.smCount, distinct.size(), cudaGetErrorString(le));
    for (int csz : {2, 8}) {
      const int blocks = 1024;
      float *in, *out;
      cudaMalloc(&in, blocks * 256 * 4);
      cudaMalloc(&out, blocks * 256 * 4);
      std::vector<float> hi(blocks * 256);
      for (int i = 0; i < blocks * 256; ++i) hi[i] = (float)(i % 7);
      cudaMemcpy(in, hi.data(), hi.size() * 4, cudaMemcpyHostToDevice);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(blocks);
      cfg.blockDim = dim3(256);
      cfg.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = csz;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int maxc = -1;
      cudaOccupancyMaxActiveClusters(&maxc, (void*)cluster_sum, &cfg);
      cudaError_t l = cudaLaunchKernelEx(&cfg, cluster_sum, (const float*)in, out);
      cudaError_t s2 = cudaStreamSynchronize(st);
      std::vector<float> o(blocks * 256);
      cudaMemcpy(o.data(), out, o.size() * 4, cudaMemcpyDeviceToHost);
      bool ok = l == cudaSuccess && s2 == cudaSuccess;
      for (int c = 0; ok && c < blocks / csz; ++c)
        for (int t = 0; t < 256; ++t) {
          float ref = 0;
          for (int k = 0; k < csz; ++k) ref += hi[(c * csz + k) * 256 + t];
          if (o[c * 256 + t] != ref) { ok = false; break; }
        }
      printf("   cluster %d: maxActiveClusters=%d launch=%s sync=%s correct=%d\n", csz, maxc, cudaGetErrorString(l),
             cudaGetErrorString(s2), (int)ok);
      cudaGetLastError();
      cudaFree(in);
      cudaFree(out);
    }
    cudaFree(sm);
  }
  return 0;
}
