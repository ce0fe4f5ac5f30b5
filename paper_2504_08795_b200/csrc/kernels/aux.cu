// Memory-bound stage kernels (CUDA cores): input pack / stem im2col, pooling,
// depthwise conv and the small-batch linear (weight-streaming GEMV).
// All use 16-byte vector accesses along the contiguous NHWC channel axis.
#include <cuda_runtime.h>
#include <cstdlib>
#include <cuda_bf16.h>
#include <cstdint>
#include "sm100.cuh"
#include "../../../include/daris_kernels.h"

namespace daris {

static inline int grid_for(long long work, int block) {
  long long g = (work + block - 1) / block;
  return static_cast<int>(g < 1 ? 1 : g);
}

// one thread per (output pixel, 8-wide K chunk)
__global__ void stem_im2col_kernel(const float* __restrict__ x, __nv_bfloat16* __restrict__ out, int n, int c, int h,
                                   int w, int kh, int kw, int stride, int pad, int ho, int wo, int kpad) {
  pdl_wait();
  pdl_trigger();
  const int chunks = kpad / 8;
  const long long total = static_cast<long long>(n) * ho * wo * chunks;
  const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= total) return;
  const int ch = static_cast<int>(idx % chunks);
  const long long m = idx / chunks;
  const int ow = static_cast<int>(m % wo);
  const int oh = static_cast<int>((m / wo) % ho);
  const int img = static_cast<int>(m / (static_cast<long long>(wo) * ho));
  const int ktot = c * kh * kw;
  float v[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int k = ch * 8 + e;
    float val = 0.f;
    if (k < ktot) {
      const int ci = k / (kh * kw);
      const int rs = k - ci * kh * kw;
      const int r = rs / kw, s = rs - (rs / kw) * kw;
      const int ih = oh * stride - pad + r, iw = ow * stride - pad + s;
      if (ih >= 0 && ih < h && iw >= 0 && iw < w) val = __ldg(x + ((static_cast<size_t>(img) * c + ci) * h + ih) * w + iw);
    }
    v[e] = val;
  }
  uint4 pk;
  pk.x = pack_bf16x2(v[0], v[1]);
  pk.y = pack_bf16x2(v[2], v[3]);
  pk.z = pack_bf16x2(v[4], v[5]);
  pk.w = pack_bf16x2(v[6], v[7]);
  reinterpret_cast<uint4*>(out)[idx] = pk;
}

// I: index type — 32-bit whenever every index fits (64-bit division is a long
// dependent instruction chain per thread: the batch-64 pack ran at 3.1 TB/s)
template <typename I>
__global__ void pack_nhwc_kernel(const float* __restrict__ x, __nv_bfloat16* __restrict__ out, int n, int c, int h,
                                 int w, int cpad, int border, int extra) {
  pdl_wait();
  pdl_trigger();
  const int chunks = cpad / 8;
  const I hw_size = static_cast<I>(h) * w;
  const I total = static_cast<I>(n) * hw_size * chunks;
  const I idx = static_cast<I>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= total) return;
  const int ch = static_cast<int>(idx % chunks);
  const I p = idx / chunks;
  const int img = static_cast<int>(p / hw_size);
  const I hw = p - static_cast<I>(img) * hw_size;
  float v[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int ci = ch * 8 + e;
    v[e] = ci < c ? __ldg(x + (static_cast<I>(img) * c + ci) * hw_size + hw) : 0.f;
  }
  uint4 pk;
  pk.x = pack_bf16x2(v[0], v[1]);
  pk.y = pack_bf16x2(v[2], v[3]);
  pk.z = pack_bf16x2(v[4], v[5]);
  pk.w = pack_bf16x2(v[6], v[7]);
  if (border == 0 && extra == 0) {
    reinterpret_cast<uint4*>(out)[idx] = pk;
  } else {  // interior of a zero-bordered [n][h + 2b][w + 2b + extra][cpad] buffer (borders stay zero)
    const int y = static_cast<int>(hw / w), xx = static_cast<int>(hw - static_cast<I>(y) * w);
    const I hp = h + 2 * border, wp = w + 2 * border + extra;
    const I o = ((static_cast<I>(img) * hp + y + border) * wp + xx + border) * chunks + ch;
    reinterpret_cast<uint4*>(out)[o] = pk;
  }
}

static bool fits_int32(long long n, long long c, long long h, long long w, long long cpad, long long border,
                       long long extra) {
  const long long lim = (1ll << 31) - 1;
  return n * c * h * w < lim && n * (h + 2 * border) * (w + 2 * border + extra) * (cpad / 8) < lim &&
         n * h * w * (cpad / 8) < lim;
}

// one thread per (output pixel, 8 channels)
__global__ void maxpool_kernel(const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ y, int n, int h,
                               int w, int c, int k, int stride, int pad, int ho, int wo) {
  pdl_wait();
  pdl_trigger();
  const int chunks = c / 8;
  const long long total = static_cast<long long>(n) * ho * wo * chunks;
  const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= total) return;
  const int ch = static_cast<int>(idx % chunks);
  const long long m = idx / chunks;
  const int ow = static_cast<int>(m % wo);
  const int oh = static_cast<int>((m / wo) % ho);
  const int img = static_cast<int>(m / (static_cast<long long>(wo) * ho));
  float best[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) best[e] = -INFINITY;
  for (int r = 0; r < k; ++r) {
    const int ih = oh * stride - pad + r;
    if (ih < 0 || ih >= h) continue;
    for (int s = 0; s < k; ++s) {
      const int iw = ow * stride - pad + s;
      if (iw < 0 || iw >= w) continue;
      uint4 v = __ldg(reinterpret_cast<const uint4*>(x + ((static_cast<size_t>(img) * h + ih) * w + iw) * c) + ch);
      uint32_t vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float2 f = unpack_bf16x2(vv[e]);
        best[2 * e] = fmaxf(best[2 * e], f.x);
        best[2 * e + 1] = fmaxf(best[2 * e + 1], f.y);
      }
    }
  }
  uint4 pk;
  pk.x = pack_bf16x2(best[0], best[1]);
  pk.y = pack_bf16x2(best[2], best[3]);
  pk.z = pack_bf16x2(best[4], best[5]);
  pk.w = pack_bf16x2(best[6], best[7]);
  reinterpret_cast<uint4*>(y)[idx] = pk;
}

// 3x3 pooling (the ResNet stem pool) with 32-bit index math and the maximum
// taken on packed bf16 pairs: no per-element unpack, all 9 window loads in
// flight at once (the generic kernel's 64-bit divisions and fp32 unpacking
// made it issue-bound: 39 us at batch 64, 3.3 TB/s)
__global__ void maxpool3_kernel(const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ y, int h, int w,
                                int chunks, int stride, int pad, int ho, int wo, int total) {
  pdl_wait();
  pdl_trigger();
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= total) return;
  const int ch = idx % chunks;
  const int m = idx / chunks;
  const int ow = m % wo;
  const int t = m / wo;
  const int oh = t % ho;
  const int img = t / ho;
  const uint4* base = reinterpret_cast<const uint4*>(x) + static_cast<size_t>(img) * h * w * chunks + ch;
  uint4 v[9];
  bool ok[9];
#pragma unroll
  for (int q = 0; q < 9; ++q) {
    const int ih = oh * stride - pad + q / 3, iw = ow * stride - pad + q % 3;
    ok[q] = ih >= 0 && ih < h && iw >= 0 && iw < w;
    v[q] = ok[q] ? __ldg(base + (ih * w + iw) * chunks) : make_uint4(0, 0, 0, 0);
  }
  __nv_bfloat162 best[4];
  const __nv_bfloat162 ninf = __halves2bfloat162(__ushort_as_bfloat16(0xff80), __ushort_as_bfloat16(0xff80));
#pragma unroll
  for (int e = 0; e < 4; ++e) best[e] = ninf;
#pragma unroll
  for (int q = 0; q < 9; ++q) {
    if (!ok[q]) continue;
    const __nv_bfloat162* p = reinterpret_cast<const __nv_bfloat162*>(&v[q]);
#pragma unroll
    for (int e = 0; e < 4; ++e) best[e] = __hmax2(best[e], p[e]);
  }
  reinterpret_cast<uint4*>(y)[idx] = *reinterpret_cast<const uint4*>(best);
}

// (image, 8 channels) per group of 8 lanes; the lanes split the pixels and
// reduce with shuffles, so each thread has only ~hw/8 loads in flight
template <typename OutT>
__global__ void avgpool_kernel(const __nv_bfloat16* __restrict__ x, OutT* __restrict__ y, int n, int hw, int c) {
  pdl_wait();
  pdl_trigger();
  const int chunks = c / 8;
  const int gidx = blockIdx.x * blockDim.x + threadIdx.x;
  const int part = gidx & 7;
  const int idx = gidx >> 3;
  const bool valid = idx < n * chunks;
  const int img = valid ? idx / chunks : 0, ch = valid ? idx - (idx / chunks) * chunks : 0;
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (valid) {
    const uint4* src = reinterpret_cast<const uint4*>(x + static_cast<size_t>(img) * hw * c) + ch;
#pragma unroll 4
    for (int p = part; p < hw; p += 8) {
      const uint4 v = __ldg(src + static_cast<size_t>(p) * chunks);
      const uint32_t vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = unpack_bf16x2(vv[e]);
        acc[2 * e] += f.x;
        acc[2 * e + 1] += f.y;
      }
    }
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], 1);
    acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], 2);
    acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], 4);
  }
  if (valid && part == 0) {
    const float inv = 1.f / static_cast<float>(hw);
    if constexpr (sizeof(OutT) == 4) {
      float4* dst = reinterpret_cast<float4*>(y + static_cast<size_t>(img) * c + ch * 8);
      dst[0] = make_float4(acc[0] * inv, acc[1] * inv, acc[2] * inv, acc[3] * inv);
      dst[1] = make_float4(acc[4] * inv, acc[5] * inv, acc[6] * inv, acc[7] * inv);
    } else {
      uint4 pk;
      pk.x = pack_bf16x2(acc[0] * inv, acc[1] * inv);
      pk.y = pack_bf16x2(acc[2] * inv, acc[3] * inv);
      pk.z = pack_bf16x2(acc[4] * inv, acc[5] * inv);
      pk.w = pack_bf16x2(acc[6] * inv, acc[7] * inv);
      *reinterpret_cast<uint4*>(y + static_cast<size_t>(img) * c + ch * 8) = pk;
    }
  }
}

// Weight-streaming linear: one warp per output feature, all batch rows at once
// (groups of 4), weights read with 16-B non-allocating loads.
constexpr int kLinB = 4;
__device__ __forceinline__ uint4 ld_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void load_x8(const void* x, int x_bf16, size_t off, float* out) {
  if (x_bf16) {
    uint4 v = __ldg(reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(x) + off));
    uint32_t vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float2 f = unpack_bf16x2(vv[e]);
      out[2 * e] = f.x;
      out[2 * e + 1] = f.y;
    }
  } else {
    const float4* p = reinterpret_cast<const float4*>(static_cast<const float*>(x) + off);
    float4 a = __ldg(p), b = __ldg(p + 1);
    out[0] = a.x; out[1] = a.y; out[2] = a.z; out[3] = a.w;
    out[4] = b.x; out[5] = b.y; out[6] = b.z; out[7] = b.w;
  }
}
__global__ void linear_kernel(const void* __restrict__ x, int x_bf16, const __nv_bfloat16* __restrict__ w,
                              const float* __restrict__ bias, void* __restrict__ y, int y_bf16, int batch, int k,
                              int o, int relu) {
  const int warps_per_block = blockDim.x >> 5;
  const int out_idx = blockIdx.x * warps_per_block + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  constexpr int kPre = 16;  // rows up to 16 x 256 = 4096 elements: held in registers
  if (k <= kPre * 256 && batch <= kLinB) {
    // Weights do not depend on the previous layer: issue the whole row slice of
    // this lane before griddepcontrol.wait, so the fetch overlaps the producer's tail.
    uint4 wv[kPre];
    const __nv_bfloat16* wrow = w + static_cast<size_t>(out_idx < o ? out_idx : 0) * k;
#pragma unroll
    for (int i = 0; i < kPre; ++i) {
      const int kk = lane * 8 + i * 256;
      wv[i] = (out_idx < o && kk < k) ? ld_stream(wrow + kk) : make_uint4(0, 0, 0, 0);
    }
    pdl_wait();
    pdl_trigger();
    if (out_idx >= o) return;
    float acc[kLinB] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int i = 0; i < kPre; ++i) {
      const int kk = lane * 8 + i * 256;
      if (kk < k) {
        const uint32_t ww[4] = {wv[i].x, wv[i].y, wv[i].z, wv[i].w};
        float wf[8];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = unpack_bf16x2(ww[e]);
          wf[2 * e] = f.x;
          wf[2 * e + 1] = f.y;
        }
#pragma unroll
        for (int bb = 0; bb < kLinB; ++bb) {
          if (bb < batch) {
            float xv[8];
            load_x8(x, x_bf16, static_cast<size_t>(bb) * k + kk, xv);
#pragma unroll
            for (int e = 0; e < 8; ++e) acc[bb] = fmaf(xv[e], wf[e], acc[bb]);
          }
        }
      }
    }
#pragma unroll
    for (int bb = 0; bb < kLinB; ++bb) {
      float v = acc[bb];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      if (lane == 0 && bb < batch) {
        v += bias ? bias[out_idx] : 0.f;
        if (relu) v = fmaxf(v, 0.f);
        const size_t oi = static_cast<size_t>(bb) * o + out_idx;
        if (y_bf16)
          static_cast<__nv_bfloat16*>(y)[oi] = __float2bfloat16_rn(v);
        else
          static_cast<float*>(y)[oi] = v;
      }
    }
    return;
  }
  pdl_wait();
  pdl_trigger();
  if (out_idx >= o) return;
  const __nv_bfloat16* wrow = w + static_cast<size_t>(out_idx) * k;
  for (int b0 = 0; b0 < batch; b0 += kLinB) {
    float acc[kLinB] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 8
    for (int kk = lane * 8; kk < k; kk += 32 * 8) {  // unrolled: 8 weight loads in flight per lane
      uint4 wv = ld_stream(wrow + kk);
      uint32_t ww[4] = {wv.x, wv.y, wv.z, wv.w};
      float wf[8];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float2 f = unpack_bf16x2(ww[e]);
        wf[2 * e] = f.x;
        wf[2 * e + 1] = f.y;
      }
#pragma unroll
      for (int bb = 0; bb < kLinB; ++bb) {
        if (b0 + bb < batch) {
          float xv[8];
          load_x8(x, x_bf16, static_cast<size_t>(b0 + bb) * k + kk, xv);
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[bb] = fmaf(xv[e], wf[e], acc[bb]);
        }
      }
    }
#pragma unroll
    for (int bb = 0; bb < kLinB; ++bb) {
      float v = acc[bb];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      if (lane == 0 && b0 + bb < batch) {
        v += bias ? bias[out_idx] : 0.f;
        if (relu) v = fmaxf(v, 0.f);
        const size_t oi = static_cast<size_t>(b0 + bb) * o + out_idx;
        if (y_bf16)
          static_cast<__nv_bfloat16*>(y)[oi] = __float2bfloat16_rn(v);
        else
          static_cast<float*>(y)[oi] = v;
      }
    }
  }
}

// depthwise conv: one thread per (output pixel, 8 channels)
__global__ void dwconv_kernel(const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ y,
                              const __nv_bfloat16* __restrict__ wt, const float* __restrict__ scale,
                              const float* __restrict__ bias, int n, int h, int w, int c, int k, int stride, int pad,
                              int ho, int wo, int relu) {
  pdl_wait();
  pdl_trigger();
  const int chunks = c / 8;
  const long long total = static_cast<long long>(n) * ho * wo * chunks;
  const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= total) return;
  const int ch = static_cast<int>(idx % chunks);
  const long long m = idx / chunks;
  const int ow = static_cast<int>(m % wo);
  const int oh = static_cast<int>((m / wo) % ho);
  const int img = static_cast<int>(m / (static_cast<long long>(wo) * ho));
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int r = 0; r < k; ++r) {
    const int ih = oh * stride - pad + r;
    if (ih < 0 || ih >= h) continue;
    for (int s = 0; s < k; ++s) {
      const int iw = ow * stride - pad + s;
      if (iw < 0 || iw >= w) continue;
      uint4 v = __ldg(reinterpret_cast<const uint4*>(x + ((static_cast<size_t>(img) * h + ih) * w + iw) * c) + ch);
      uint4 q = __ldg(reinterpret_cast<const uint4*>(wt + static_cast<size_t>(r * k + s) * c) + ch);
      uint32_t vv[4] = {v.x, v.y, v.z, v.w}, qq[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float2 a = unpack_bf16x2(vv[e]), b = unpack_bf16x2(qq[e]);
        acc[2 * e] = fmaf(a.x, b.x, acc[2 * e]);
        acc[2 * e + 1] = fmaf(a.y, b.y, acc[2 * e + 1]);
      }
    }
  }
  float o[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    float v = acc[e] * __ldg(scale + ch * 8 + e) + __ldg(bias + ch * 8 + e);
    if (relu == 1) v = fmaxf(v, 0.f);
    if (relu == 6) v = fminf(fmaxf(v, 0.f), 6.f);
    o[e] = v;
  }
  uint4 pk;
  pk.x = pack_bf16x2(o[0], o[1]);
  pk.y = pack_bf16x2(o[2], o[3]);
  pk.z = pack_bf16x2(o[4], o[5]);
  pk.w = pack_bf16x2(o[6], o[7]);
  reinterpret_cast<uint4*>(y)[idx] = pk;
}

}  // namespace daris

using namespace daris;

extern "C" int daris_stem_im2col(const float* x, void* out, int32_t n, int32_t c, int32_t h, int32_t w, int32_t kh,
                                 int32_t kw, int32_t stride, int32_t pad, int32_t ho, int32_t wo, int32_t kpad,
                                 void* stream) {
  if (!x || !out) return DARIS_K_BAD_ARG;
  if (kpad % 64 != 0 || kpad < c * kh * kw) return DARIS_K_BAD_SHAPE;
  const long long work = static_cast<long long>(n) * ho * wo * (kpad / 8);
  cudaError_t return_code = launch_pdl(stem_im2col_kernel, dim3(grid_for(work, 256)), dim3(256), 0, static_cast<cudaStream_t>(stream),
      x, static_cast<__nv_bfloat16*>(out), n, c, h, w, kh, kw, stride, pad, ho, wo, kpad);
  return static_cast<int>(return_code);
}

extern "C" int daris_pack_nhwc(const float* x, void* out, int32_t n, int32_t c, int32_t h, int32_t w, int32_t cpad,
                               void* stream) {
  if (!x || !out) return DARIS_K_BAD_ARG;
  if (cpad % 8 != 0 || cpad < c) return DARIS_K_BAD_SHAPE;
  const long long work = static_cast<long long>(n) * h * w * (cpad / 8);
  cudaError_t return_code = fits_int32(n, c, h, w, cpad, 0, 0)
      ? launch_pdl(pack_nhwc_kernel<int>, dim3(grid_for(work, 256)), dim3(256), 0, static_cast<cudaStream_t>(stream),
                   x, static_cast<__nv_bfloat16*>(out), n, c, h, w, cpad, 0, 0)
      : launch_pdl(pack_nhwc_kernel<long long>, dim3(grid_for(work, 256)), dim3(256), 0,
                   static_cast<cudaStream_t>(stream), x, static_cast<__nv_bfloat16*>(out), n, c, h, w, cpad, 0, 0);
  return static_cast<int>(return_code);
}

extern "C" int daris_pack_nhwc_bordered(const float* x, void* out, int32_t n, int32_t c, int32_t h, int32_t w,
                                        int32_t cpad, int32_t border, int32_t extra, void* stream) {
  if (!x || !out) return DARIS_K_BAD_ARG;
  if (cpad % 8 != 0 || cpad < c || border < 0 || extra < 0) return DARIS_K_BAD_SHAPE;
  const long long work = static_cast<long long>(n) * h * w * (cpad / 8);
  cudaError_t rc = fits_int32(n, c, h, w, cpad, border, extra)
      ? launch_pdl(pack_nhwc_kernel<int>, dim3(grid_for(work, 256)), dim3(256), 0, static_cast<cudaStream_t>(stream),
                   x, static_cast<__nv_bfloat16*>(out), n, c, h, w, cpad, border, extra)
      : launch_pdl(pack_nhwc_kernel<long long>, dim3(grid_for(work, 256)), dim3(256), 0,
                   static_cast<cudaStream_t>(stream), x, static_cast<__nv_bfloat16*>(out), n, c, h, w, cpad, border,
                   extra);
  return static_cast<int>(rc);
}

extern "C" int daris_maxpool(const void* x, void* y, int32_t n, int32_t h, int32_t w, int32_t c, int32_t k,
                             int32_t stride, int32_t pad, int32_t ho, int32_t wo, void* stream) {
  if (!x || !y) return DARIS_K_BAD_ARG;
  if (c % 8 != 0) return DARIS_K_BAD_SHAPE;
  const long long work = static_cast<long long>(n) * ho * wo * (c / 8);
  if (k == 3 && work < (1ll << 31) && static_cast<long long>(n) * h * w * (c / 8) < (1ll << 31))
    return static_cast<int>(launch_pdl(maxpool3_kernel, dim3(grid_for(work, 256)), dim3(256), 0,
                                       static_cast<cudaStream_t>(stream), static_cast<const __nv_bfloat16*>(x),
                                       static_cast<__nv_bfloat16*>(y), h, w, c / 8, stride, pad, ho, wo,
                                       static_cast<int>(work)));
  cudaError_t return_code = launch_pdl(maxpool_kernel, dim3(grid_for(work, 256)), dim3(256), 0, static_cast<cudaStream_t>(stream),
      static_cast<const __nv_bfloat16*>(x), static_cast<__nv_bfloat16*>(y), n, h, w, c, k, stride, pad, ho, wo);
  return static_cast<int>(return_code);
}

extern "C" int daris_avgpool(const void* x, float* y, int32_t n, int32_t hw, int32_t c, void* stream) {
  if (!x || !y) return DARIS_K_BAD_ARG;
  if (c % 8 != 0) return DARIS_K_BAD_SHAPE;
  const int work = n * (c / 8) * 8;  // 8 lanes per (image, 8 channels)
  cudaError_t return_code = launch_pdl(avgpool_kernel<float>, dim3(grid_for(work, 128)), dim3(128), 0, static_cast<cudaStream_t>(stream),
      static_cast<const __nv_bfloat16*>(x), y, n, hw, c);
  return static_cast<int>(return_code);
}

extern "C" int daris_avgpool_bf16(const void* x, void* y, int32_t n, int32_t hw, int32_t c, void* stream) {
  if (!x || !y) return DARIS_K_BAD_ARG;
  if (c % 8 != 0) return DARIS_K_BAD_SHAPE;
  const int work = n * (c / 8) * 8;
  cudaError_t return_code = launch_pdl(avgpool_kernel<__nv_bfloat16>, dim3(grid_for(work, 128)), dim3(128), 0,
      static_cast<cudaStream_t>(stream), static_cast<const __nv_bfloat16*>(x), static_cast<__nv_bfloat16*>(y), n, hw, c);
  return static_cast<int>(return_code);
}

extern "C" int daris_linear(const void* x, int32_t x_bf16, const void* w, const float* bias, void* y, int32_t y_bf16,
                            int32_t batch, int32_t k, int32_t o, int32_t relu, void* stream) {
  if (!x || !w || !y) return DARIS_K_BAD_ARG;
  if (k % 8 != 0 || batch < 1 || o < 1) return DARIS_K_BAD_SHAPE;
  const int warps = 8;
  cudaError_t return_code = launch_pdl(linear_kernel, dim3((o + warps - 1) / warps), dim3(warps * 32), 0, static_cast<cudaStream_t>(stream), 
      x, x_bf16, static_cast<const __nv_bfloat16*>(w), bias, y, y_bf16, batch, k, o, relu);
  return static_cast<int>(return_code);
}

extern "C" int daris_dwconv(const void* x, void* y, const void* weight, const float* scale, const float* bias,
                            int32_t n, int32_t h, int32_t w, int32_t c, int32_t k, int32_t stride, int32_t pad,
                            int32_t ho, int32_t wo, int32_t relu, void* stream) {
  if (!x || !y || !weight || !scale || !bias) return DARIS_K_BAD_ARG;
  if (c % 8 != 0) return DARIS_K_BAD_SHAPE;
  const long long work = static_cast<long long>(n) * ho * wo * (c / 8);
  cudaError_t return_code = launch_pdl(dwconv_kernel, dim3(grid_for(work, 256)), dim3(256), 0, static_cast<cudaStream_t>(stream),
      static_cast<const __nv_bfloat16*>(x), static_cast<__nv_bfloat16*>(y),
      static_cast<const __nv_bfloat16*>(weight), scale, bias, n, h, w, c, k, stride, pad, ho, wo, relu);
  return static_cast<int>(return_code);
}
